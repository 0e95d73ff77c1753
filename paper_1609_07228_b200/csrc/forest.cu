// forest.cu — randomized truncated KD-forest on B200, bit-identical to the
// reference TreeBuilder (proj/src/kd_forest.cpp:29-97, build_forest :245-264).
//
// Why DFS and not level-synchronous: the reference draws split dimensions
// from a per-tree std::mt19937_64(substream(seed, t)) in DFS PRE-ORDER of the
// internal nodes (kd_forest.cpp:53, recursion :87-88).  A right child's draw
// index depends on the internal-node count of its left sibling's subtree, so
// no level-synchronous schedule can reproduce the reference's trees.  Each
// tree is therefore built by one CTA walking the tree in pre-order with an
// explicit stack:
//   * nodes larger than kWarpSubtree points: the whole CTA (512 threads)
//     computes the mean (exact double sum, see below) and the stable
//     partition with block-wide ballot scans;
//   * subtrees of <= kWarpSubtree points: warp 0 finishes the entire subtree
//     with warp-synchronous ops (no block barriers), after prefetching the
//     subtree's rows into L2 so the per-node gathers hit L2, not HBM.
//   * the MT19937-64 state lives in shared memory; warp 0 regenerates 312
//     words at a time with a 3-phase parallel twist.
// Trees run concurrently (one CTA per tree).
//
// Exact mean: the reference sums x[p][d] sequentially in double.  A parallel
// double sum equals it bit-for-bit whenever every partial sum is exactly
// representable, which holds when (top bit of the largest |x|) +
// ceil(log2(size)) - (lowest set bit over all x) <= 53.  That is checked per
// node (always true for integer-valued data and for gen_synthetic data); when
// it fails the node's sum is done serially in point_index order.
#include <climits>
#include <cstdio>
#include <cstdlib>

#include "../../include/annkit_b200.h"
#include "internal.cuh"

#include <cooperative_groups.h>
#include <cub/cub.cuh>

namespace annk {
namespace {

constexpr uint32_t kBlock = 256;
constexpr uint32_t kWarps = kBlock / 32;
constexpr uint32_t kWarpSubtree = 4096;
constexpr uint32_t kSortSmem = 2048;
constexpr uint32_t kTileMax = 1024;      // staged-tile path: points per tile
constexpr uint32_t kStageBytes = 147456;  // staged rows (u8 path), row stride ld8 + 4
constexpr uint32_t kStack = 160;
constexpr uint32_t kTileStack = 128;
constexpr uint32_t kMaxCluster = 8;      // CTAs per tree (thread-block cluster)
constexpr uint32_t kClusterMin = 8192;  // nodes above this many points use the whole cluster
constexpr size_t kPrefetchBytes = 4u << 20;
constexpr uint32_t kDrawWin = 256;
// staged tiles: warp 0 only decides the splits; it hands every node to warp kWarps-1 through
// a ring of 32-byte events, and that warp writes the records (node, leaf children, depth,
// even, parent links) and does the split's float division -- off the tree's dependent chain
constexpr uint32_t kEvRing = 128;              // events (power of two)
constexpr uint32_t kStagers = kBlock - 32;     // threads staging tile rows (warps 0..kWarps-2)
constexpr uint32_t kEvLink = 1u << 24, kEvRight = 1u << 25, kEvLLeaf = 1u << 26, kEvRLeaf = 1u << 27,
                   kEvSplit = 1u << 28, kEvLeaf = 1u << 29, kEvQuit = 1u << 30;

struct StackEntry {
    uint32_t start, end, depth, parent, side;  // side 0 = left child, 1 = right
};

struct BuildArgs {
    const float* x;
    uint32_t n, dim, ld, leaf_cap;
    uint64_t seed;
    KdNodeDev* nodes;
    uint32_t* depth;
    uint8_t* even;
    uint32_t* pidx;
    uint32_t* rtmp;
    uint64_t* sortbuf;  // next_pow2(n) keys, for fallback sorts larger than kSortSmem
    uint32_t* meta;     // [num_nodes, root, leaf_count, max_depth, error]
    const uint8_t* x8;  // exact u8 copy (nullptr: fp32 gathers)
    uint32_t ld8;
    const uint32_t* draws;  // split dimension of the k-th internal node in pre-order
    uint32_t n_draws;
    float* col;  // block path: the node's gathered column, by point_index slot (n floats)
    uint32_t* ltmp;  // cluster path: left side of a partition (n)
};

struct Smem {
    float col[kWarpSubtree];      // warp path: the node's column on its split dim
    uint32_t sub[kWarpSubtree];   // warp path: subtree slice of point_index
    uint32_t sub2[kWarpSubtree];  // warp path: right half during a partition
    uint64_t sortk[kSortSmem];
    uint16_t lidx[kTileMax];  // staged tile: local row index per slot
    uint16_t ltmp[kTileMax];
    StackEntry bstack[kStack];
    StackEntry wstack[kStack];
    uint64_t tstack[kTileStack];
    double red_sum[kWarps];
    int red_top[kWarps], red_lsb[kWarps];
    uint32_t cnt_l[kWarps], cnt_r[kWarps];
    uint32_t dwin[kDrawWin];
    uint32_t dwin_base, draw_idx, node_count, leaf_count, max_depth, error;
    uint32_t t_start, t_size, t_sb;  // staged-tile request to the helper warps (t_size 0: done)
    uint32_t ev_count, ev_tail;      // events emitted by warp 0 / consumed by the record warp
    alignas(16) uint4 ring[kEvRing * 2];
    long long cyc_block, cyc_warp;
    long long ft[16], ft_last;
    uint32_t bsp;
    // broadcast slots for the block path
    uint32_t b_d, b_nl, b_nr, b_mid, b_even;
    float b_split;
    double b_sum;
    int b_exact;
    // cluster coordination (read by the other CTAs of the tree's cluster through DSMEM)
    uint32_t cmd, cmd_id, cmd_d;
    StackEntry cmd_e;
    double cl_sum[kMaxCluster];
    int cl_top[kMaxCluster], cl_lsb[kMaxCluster];
    uint32_t cl_nl[kMaxCluster], cl_nr[kMaxCluster];
    alignas(16) unsigned char stage[kStageBytes];  // staged tile rows
};
static_assert(sizeof(Smem) <= 232448, "forest shared memory exceeds 227 KB");

__device__ __forceinline__ float ldx(const BuildArgs& a, uint32_t p, uint32_t d) {
    return __ldg(a.x + size_t(p) * a.ld + d);
}

// Magnitude/granularity of one value for the exact-sum test.
__device__ __forceinline__ void val_stats(float v, int& top, int& lsb) {
    const uint32_t b = __float_as_uint(v) & 0x7fffffffu;
    if (b == 0) return;
    const uint32_t ex = b >> 23, m = b & 0x7fffffu;
    uint32_t mm;
    int e0;
    if (ex == 0) {
        mm = m;
        e0 = -149;
    } else {
        mm = m | 0x800000u;
        e0 = int(ex) - 150;
    }
    lsb = min(lsb, e0 + __ffs(mm) - 1);
    top = max(top, e0 + 32 - __clz(mm));
}
__device__ __forceinline__ bool sum_is_exact(int top, int lsb, uint32_t size) {
    if (top == INT_MIN) return true;  // all zeros
    const int clog = size <= 1 ? 0 : 32 - __clz(size - 1);
    return top + clog - lsb <= 53;
}

// Orderable (value, id) key; -0 and +0 compare equal like the reference.
__device__ __forceinline__ uint64_t val_id_key(float v, uint32_t id) {
    uint32_t b = __float_as_uint(v);
    if ((b & 0x7fffffffu) == 0) b = 0;
    b = (b & 0x80000000u) ? ~b : (b | 0x80000000u);
    return (uint64_t(b) << 32) | id;
}

// libstdc++ std::midpoint<float> for finite inputs.
__device__ __forceinline__ float midpoint_f(float a, float b) {
    const float aa = fabsf(a), ab = fabsf(b), hi = 3.40282347e38f / 2;
    if (aa <= hi && ab <= hi) return __fdiv_rn(__fadd_rn(a, b), 2.0f);
    if (aa < 1.17549435e-38f * 2) return __fadd_rn(a, __fdiv_rn(b, 2.0f));
    if (ab < 1.17549435e-38f * 2) return __fadd_rn(__fdiv_rn(a, 2.0f), b);
    return __fadd_rn(__fdiv_rn(a, 2.0f), __fdiv_rn(b, 2.0f));
}

// Split dimension of internal node k in pre-order (kd_forest.cpp:53:
// rng_() % dim), read through a shared-memory window over the tree's
// precomputed draw stream (draws_kernel).  Warp-collective.
__device__ uint32_t warp_draw_at(const BuildArgs& a, Smem& s, uint32_t k) {
    __syncwarp();
    if (k < s.dwin_base || k >= s.dwin_base + kDrawWin) {
        const uint32_t base = k & ~(kDrawWin - 1);
        for (uint32_t j = lane_id(); j < kDrawWin; j += 32)
            s.dwin[j] = base + j < a.n_draws ? a.draws[base + j] : 0u;
        __syncwarp();
        if (lane_id() == 0) s.dwin_base = base;
        __syncwarp();
    }
    const uint32_t d = s.dwin[k - s.dwin_base];
    __syncwarp();
    return d;
}
__device__ uint32_t warp_draw(const BuildArgs& a, Smem& s) {
    const uint32_t k = s.draw_idx;
    const uint32_t d = warp_draw_at(a, s, k);
    if (lane_id() == 0) s.draw_idx = k + 1;
    __syncwarp();
    return d;
}

// -------------------------------------------------------------- warp path

#ifdef ANNK_FOREST_TIMING
// phase probes: cycles between consecutive marks accumulate in s.ft[mark]
#define FT_MARK(m)                                                   \
    do {                                                             \
        const long long _t = clock64();                              \
        if (lane_id() == 0) {                                        \
            s.ft[(m)] += _t - s.ft_last;                              \
            s.ft_last = _t;                                          \
        }                                                            \
    } while (0)
#else
#define FT_MARK(m) \
    do {           \
    } while (0)
#endif

// Sorts sub[st, st+size) (subtree-local point ids) by (value, id) on dim d.
__device__ void warp_sort_local(const BuildArgs& a, Smem& s, uint32_t* sub, uint32_t st, uint32_t size,
                                uint32_t d) {
    const uint32_t lane = lane_id();
    const uint32_t m = next_pow2(size);
    uint64_t* k = m <= kSortSmem ? s.sortk : a.sortbuf;
    for (uint32_t j = lane; j < m; j += 32) {
        uint64_t key = kEmptyKey;
        if (j < size) {
            const uint32_t id = sub[st + j];
            key = val_id_key(ldx(a, id, d), id);
        }
        k[j] = key;
    }
    __syncwarp();
    warp_bitonic_sort(k, m);
    for (uint32_t j = lane; j < size; j += 32) sub[st + j] = uint32_t(k[j]);
    __syncwarp();
}

__device__ __forceinline__ float ldv(const BuildArgs& a, uint32_t p, uint32_t d) {
    return a.x8 ? float(__ldg(a.x8 + size_t(p) * a.ld8 + d)) : __ldg(a.x + size_t(p) * a.ld + d);
}

// Points per staged tile (0: staged tiles off — fp32 rows, or rows too wide).
__device__ __forceinline__ uint32_t tile_capacity(const BuildArgs& a) {
    if (!a.x8) return 0u;
    const uint32_t t = min(kTileMax, kStageBytes / (a.ld8 + 4));
    return t >= 64 ? t : 0u;
}

__device__ __forceinline__ void named_bar(uint32_t id, uint32_t count) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// Copies the rows of s.sub[ts, ts+tsz) (u8, ld8 bytes each) into s.stage with
// row stride sb.  Called by the kStagers threads of warps 0..kWarps-2 (warp 0 + the helper warps).
__device__ __forceinline__ void stage_rows(const BuildArgs& a, Smem& s, uint32_t ts, uint32_t tsz, uint32_t sb) {
    const uint32_t parts = a.ld8 / 16;
    const uint32_t total = tsz * parts;
    for (uint32_t j0 = 0; j0 < total; j0 += kStagers * 8) {
        uint4 r[8];
#pragma unroll
        for (uint32_t u = 0; u < 8; ++u) {
            const uint32_t j = j0 + u * kStagers + threadIdx.x;
            if (j < total) {
                const uint32_t row = j / parts, part = j - row * parts;
                r[u] = __ldg(reinterpret_cast<const uint4*>(a.x8 + size_t(s.sub[ts + row]) * a.ld8) + part);
            }
        }
#pragma unroll
        for (uint32_t u = 0; u < 8; ++u) {
            const uint32_t j = j0 + u * kStagers + threadIdx.x;
            if (j < total) {
                const uint32_t row = j / parts, part = j - row * parts;
                uint32_t* dst = reinterpret_cast<uint32_t*>(s.stage + row * sb + part * 16);
                dst[0] = r[u].x;
                dst[1] = r[u].y;
                dst[2] = r[u].z;
                dst[3] = r[u].w;
            }
        }
    }
}

// Helper warps (1..kWarps-1) while warp 0 builds a warp subtree: stage the
// rows of each tile warp 0 requests (named barrier 1 = request, 2 = done).
__device__ void stage_helper(const BuildArgs& a, Smem& s) {
    for (;;) {
        named_bar(1, kStagers);
        const uint32_t ts = s.t_start, tsz = s.t_size;
        if (tsz == 0) break;
        stage_rows(a, s, ts, tsz, s.t_sb);
        named_bar(2, kStagers);
    }
}

// ---- tile events (warp 0 -> the record warp).  An event is two 16-byte halves,
//   A = {node id, parent id, split dim | depth << 16 | flags, seq}
//   B = {column sum (or the split's bits with kEvSplit), point_index position of the node's
//        first point, left size | right size << 11, seq}          (kEvLeaf: left size = size)
// each written by one 128-bit shared-memory store and read by one 128-bit load, so a half
// is seen whole or not at all; seq = event number + 1 marks it valid (the ring starts zeroed).
__device__ __forceinline__ void sts_v4(uint4* p, uint4 v) {
    asm volatile("st.volatile.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(uint32_t(__cvta_generic_to_shared(p))),
                 "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}
__device__ __forceinline__ uint4 lds_v4(const uint4* p) {
    uint4 v;
    asm volatile("ld.volatile.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(uint32_t(__cvta_generic_to_shared(p)))
                 : "memory");
    return v;
}
// warp 0, uniform arguments; ev = events emitted so far
__device__ __forceinline__ void emit_event(Smem& s, uint32_t& ev, uint32_t id, uint32_t par, uint32_t meta,
                                           uint32_t val, uint32_t pos, uint32_t sizes) {
    if ((ev & 31u) == 0) {  // room for the next 32 events
        while (ev + 32u - *reinterpret_cast<volatile uint32_t*>(&s.ev_tail) > kEvRing) {
        }
    }
    if (lane_id() == 0) {
        uint4* slot = s.ring + (ev & (kEvRing - 1)) * 2;
        sts_v4(slot, make_uint4(id, par, meta, ev + 1));
        sts_v4(slot + 1, make_uint4(val, pos, sizes, ev + 1));
    }
    ++ev;
}

// The record warp: every lane takes one pending event; records first, parent links after
// (a link may target a record written by another lane in the same pass).
__device__ void record_warp(const BuildArgs& a, Smem& s) {
    const uint32_t lane = lane_id();
    uint32_t ct = s.ev_tail;
    for (;;) {
        const uint32_t e = ct + lane;
        const uint4* slot = s.ring + (e & (kEvRing - 1)) * 2;
        const uint4 A = lds_v4(slot), B = lds_v4(slot + 1);
        const uint32_t okm = __ballot_sync(0xffffffffu, A.w == e + 1 && B.w == e + 1);
        const uint32_t cnt = okm == 0xffffffffu ? 32u : uint32_t(__ffs(~okm)) - 1u;
        if (cnt == 0) {
            __nanosleep(32);
            continue;
        }
        __threadfence_block();
        const bool mine = lane < cnt;
        const uint32_t id = A.x, meta = A.z;
        const uint32_t cdep = (meta >> 16) & 0xffu;
        if (mine && !(meta & kEvQuit)) {
            if (meta & kEvLeaf) {
                reinterpret_cast<uint4*>(a.nodes)[id] = make_uint4(kLeaf, 0u, B.y, B.y + (B.z & 0x7ffu));
                a.depth[id] = cdep;
                a.even[id] = 0;
            } else {
                const uint32_t nl = B.z & 0x7ffu, nr = B.z >> 11;
                const bool lleaf = meta & kEvLLeaf, rleaf = meta & kEvRLeaf;
                const uint32_t sp = (meta & kEvSplit) ? B.x : __float_as_uint(__fdiv_rn(float(B.x), float(nl + nr)));
                reinterpret_cast<uint4*>(a.nodes)[id] = make_uint4(meta & 0xffffu, sp, id + 1, lleaf ? id + 2 : 0u);
                a.depth[id] = cdep;
                a.even[id] = (meta & kEvSplit) ? 1 : 0;
                if (lleaf) {
                    reinterpret_cast<uint4*>(a.nodes)[id + 1] = make_uint4(kLeaf, 0u, B.y, B.y + nl);
                    a.depth[id + 1] = cdep + 1;
                    a.even[id + 1] = 0;
                    if (rleaf) {
                        reinterpret_cast<uint4*>(a.nodes)[id + 2] = make_uint4(kLeaf, 0u, B.y + nl, B.y + nl + nr);
                        a.depth[id + 2] = cdep + 1;
                        a.even[id + 2] = 0;
                    }
                }
            }
        }
        __syncwarp();
        if (mine && (meta & kEvLink)) {
            if (meta & kEvRight) a.nodes[A.y].right = id;
            else a.nodes[A.y].left = id;
        }
        ct += cnt;
        if (lane == 0) *reinterpret_cast<volatile uint32_t*>(&s.ev_tail) = ct;
        if (__any_sync(0xffffffffu, mine && (meta & kEvQuit))) break;
    }
}

// One tile node of <= 32*C points, all in registers: gather the column,
// integer sum, ballot the sides, then either scatter both sides of li in place
// (balanced split) or sort the rows by (value, global id) (kd_forest.cpp:70-83).
// Returns the split position; writes split / even.
template <int C>
__device__ __forceinline__ uint32_t tile_node_reg(const unsigned char* __restrict__ st, uint16_t* li,
                                                  const uint32_t* gid, uint32_t sb, uint32_t d,
                                                  uint32_t start, uint32_t end, uint32_t& sval, uint8_t& even) {
    const uint32_t lane = lane_id(), ltm = (1u << lane) - 1u;
    const uint32_t size = end - start;
    uint32_t loc[C], v[C];
#pragma unroll
    for (int u = 0; u < C; ++u) {
        const uint32_t p = start + u * 32 + lane;
        loc[u] = p < end ? li[p] : 0u;
    }
    uint32_t is = 0;
#pragma unroll
    for (int u = 0; u < C; ++u) {
        const uint32_t p = start + u * 32 + lane;
        v[u] = p < end ? st[loc[u] * sb + d] : 0u;
        is += v[u];
    }
    const uint32_t isum = __reduce_add_sync(0xffffffffu, is);
    uint32_t bl[C], nl = 0;
#pragma unroll
    for (int u = 0; u < C; ++u) {
        const uint32_t p = start + u * 32 + lane;
        bl[u] = __ballot_sync(0xffffffffu, p < end && v[u] * size <= isum);
        nl += __popc(bl[u]);
    }
    const uint32_t nr = size - nl;
    if (nl != 0 && nr != 0 && max(nl, nr) <= 4u * min(nl, nr)) {
        uint32_t cl = 0, cr = 0;
#pragma unroll
        for (int u = 0; u < C; ++u) {
            const uint32_t p = start + u * 32 + lane;
            const uint32_t pl = __popc(bl[u] & ltm);
            if (p < end) {
                if ((bl[u] >> lane) & 1u) li[start + cl + pl] = uint16_t(loc[u]);
                else li[start + nl + cr + (lane - pl)] = uint16_t(loc[u]);
            }
            const uint32_t c = __popc(bl[u]);
            cl += c;
            cr += min(32u, end - min(end, start + u * 32)) - c;
        }
        sval = isum;  // split = isum / size, divided by the record warp
        even = 0;
        __syncwarp();
        return start + nl;
    }
    uint64_t k[C];
#pragma unroll
    for (int u = 0; u < C; ++u) {
        const uint32_t p = start + u * 32 + lane;
        k[u] = p < end ? (uint64_t(v[u]) << 53) | (uint64_t(gid[loc[u]]) << 11) | loc[u] : kEmptyKey;
    }
    const uint32_t q0 = size / 2 - 1, q1 = size / 2;
    uint32_t a0 = 0, a1 = 0;
    if constexpr (C <= 2) {
        // rank sort: keys are unique, rank = number of smaller keys (independent
        // broadcasts instead of a dependent bitonic network)
        uint32_t rk[C];
#pragma unroll
        for (int u = 0; u < C; ++u) rk[u] = 0;
#pragma unroll
        for (int r = 0; r < C; ++r) {
            const uint32_t cnt = min(32u, size - min(size, uint32_t(r) * 32));
            for (uint32_t j = 0; j < cnt; ++j) {
                const uint64_t kj = shfl_idx_u64(k[r], j);
#pragma unroll
                for (int u = 0; u < C; ++u) rk[u] += kj < k[u] ? 1u : 0u;
            }
        }
#pragma unroll
        for (int u = 0; u < C; ++u) {
            const uint32_t p = start + u * 32 + lane;
            if (p < end) li[start + rk[u]] = uint16_t(loc[u]);
            const uint32_t b0 = __ballot_sync(0xffffffffu, p < end && rk[u] == q0);
            const uint32_t b1 = __ballot_sync(0xffffffffu, p < end && rk[u] == q1);
            const uint32_t x = __shfl_sync(0xffffffffu, v[u], (__ffs(b0) - 1) & 31);
            const uint32_t y = __shfl_sync(0xffffffffu, v[u], (__ffs(b1) - 1) & 31);
            if (b0) a0 = x;
            if (b1) a1 = y;
        }
    } else {
        warp_sort_regs<C>(k);
#pragma unroll
        for (int u = 0; u < C; ++u) {
            const uint32_t p = start + u * 32 + lane;
            if (p < end) li[p] = uint16_t(k[u] & 0x7ffu);
        }
        // values at sorted positions size/2 - 1 and size/2
#pragma unroll
        for (int u = 0; u < C; ++u) {
            const uint32_t x = __shfl_sync(0xffffffffu, uint32_t(k[u] >> 53), q0 & 31);
            const uint32_t y = __shfl_sync(0xffffffffu, uint32_t(k[u] >> 53), q1 & 31);
            if (q0 / 32 == uint32_t(u)) a0 = x;
            if (q1 / 32 == uint32_t(u)) a1 = y;
        }
    }
    sval = __float_as_uint(midpoint_f(float(a0), float(a1)));
    even = 1;
    __syncwarp();
    return start + size / 2;
}

// Builds the whole subtree under `root` (<= tile_max points, u8 datapath)
// from rows staged in shared memory by the whole CTA: every node's column
// gather is then a shared-memory byte read and the partition moves 16-bit
// local row indices; point_index is permuted once at the end.  Same
// pre-order, draws and splits as the warp path.  For a node of `size` points
// with integer sum `isum` (size <= 1024): split = fl32(fl64(isum/size)) ==
// __fdiv_rn(isum, size) (isum, size < 2^24 exact in float, and no double
// rounding since size < 2^28), and for an integer value v,
// v <= split  <=>  v*size <= isum  (the quotient is >= 1/size away from any
// integer it does not equal, far more than half a float ulp below 256).
// `sb` = row stride in bytes (odd word count: consecutive rows in different
// banks).  Node/draw/leaf counters live in registers for the whole tile.
// One tile node of 257..tile points from shared memory: two passes (sum, then
// stable ballot partition through ltmp), degenerate fallback = bitonic sort of
// (value, global id, local row) keys.  Returns the split position.
__device__ __noinline__ uint32_t tile_node_smem(Smem& s, const unsigned char* __restrict__ st, uint16_t* li,
                                                uint16_t* lt, const uint32_t* gid, uint32_t sb, uint32_t d,
                                                uint32_t e_start, uint32_t e_end, uint32_t& sval, uint8_t& even) {
    const uint32_t lane = lane_id(), ltm = (1u << lane) - 1u;
    const uint32_t size = e_end - e_start;
    uint32_t is = 0;
    for (uint32_t p0 = e_start; p0 < e_end; p0 += 256) {
        uint32_t x[8];
#pragma unroll
        for (uint32_t u = 0; u < 8; ++u) {
            const uint32_t p = p0 + u * 32 + lane;
            x[u] = p < e_end ? st[uint32_t(li[p]) * sb + d] : 0u;
        }
#pragma unroll
        for (uint32_t u = 0; u < 8; ++u) is += x[u];
    }
    const uint32_t isum = __reduce_add_sync(0xffffffffu, is);
    uint32_t nl = 0, nr = 0;
    for (uint32_t b0 = e_start; b0 < e_end; b0 += 32) {
        const uint32_t p = b0 + lane;
        const bool valid = p < e_end;
        const uint16_t lc = valid ? li[p] : uint16_t(0);
        const bool left = valid && uint32_t(st[uint32_t(lc) * sb + d]) * size <= isum;
        const uint32_t bl = __ballot_sync(0xffffffffu, left);
        const uint32_t br = __ballot_sync(0xffffffffu, valid && !left);
        if (left) li[e_start + nl + __popc(bl & ltm)] = lc;
        else if (valid) lt[nr + __popc(br & ltm)] = lc;
        nl += __popc(bl);
        nr += __popc(br);
    }
    __syncwarp();
    for (uint32_t j = lane; j < nr; j += 32) li[e_start + nl + j] = lt[j];
    __syncwarp();
    sval = isum;
    uint32_t mid = e_start + nl;
    even = 0;
    if (nl == 0 || nr == 0 || max(nl, nr) > 4u * min(nl, nr)) {
        // kd_forest.cpp:70-83: sort by (value, id); key = value | global id | local row
        const uint32_t m = next_pow2(size);
        uint64_t* k = s.sortk;
        for (uint32_t j = lane; j < m; j += 32) {
            uint64_t key = kEmptyKey;
            if (j < size) {
                const uint32_t lc = li[e_start + j];
                key = (uint64_t(st[lc * sb + d]) << 53) | (uint64_t(gid[lc]) << 11) | lc;
            }
            k[j] = key;
        }
        __syncwarp();
        warp_bitonic_sort(k, m);
        for (uint32_t j = lane; j < size; j += 32) li[e_start + j] = uint16_t(k[j] & 0x7ffu);
        __syncwarp();
        mid = e_start + size / 2;
        sval = __float_as_uint(midpoint_f(float(st[uint32_t(li[mid - 1]) * sb + d]), float(st[uint32_t(li[mid]) * sb + d])));
        even = 1;
    }
    return mid;
}

// Tile stack entry packed in 64 bits: parent id | start(11) | end(11) |
// depth below the tile root(8) | link(2: bit0 = set the parent's child link,
// bit1 = right child).  start/end are relative to the tile.
__device__ __forceinline__ uint64_t tpack(uint32_t parent, uint32_t st, uint32_t en, uint32_t dep, uint32_t link) {
    return (uint64_t(parent) << 32) | (st << 21) | (en << 10) | (dep << 2) | link;
}

__device__ void warp_build_tile(const BuildArgs& a, Smem& s, const StackEntry& root, uint32_t base,
                                uint32_t sb) {
    const uint32_t lane = lane_id();
    const uint32_t ts = root.start, tsz = root.end - root.start;
    FT_MARK(0);
    if (lane == 0) {
        s.t_start = ts;
        s.t_size = tsz;
        s.t_sb = sb;
    }
    __syncwarp();
    named_bar(1, kStagers);
    stage_rows(a, s, ts, tsz, sb);
    for (uint32_t j = lane; j < tsz; j += 32) s.lidx[j] = uint16_t(j);
    named_bar(2, kStagers);
    FT_MARK(13);
    const unsigned char* st = s.stage;
    uint16_t* li = s.lidx;  // indexed by tile-relative slot
    uint16_t* lt = s.ltmp;
    const uint32_t* gid = s.sub + ts;
    const uint32_t lcap = a.leaf_cap, pbase = base + ts, dep0 = root.depth;
    uint32_t nid = s.node_count, kd = s.draw_idx, wb = s.dwin_base, nleaf = s.leaf_count, maxd = s.max_depth;
    uint32_t ev = s.ev_count;
    // the parent's record (written by this warp on the warp path) must be visible before the
    // record warp links the tile root into it
    __threadfence_block();
    // current node in registers; only right siblings go through the stack.
    // Depth inside a tile is bounded (splits are <= 4:1 or even), so the
    // stack cannot overflow: <= log_{5/4}(1024) + 1 entries.
    uint32_t cs = 0, ce = tsz, cdep = root.depth, cpar = root.parent;
    uint32_t clink = kEvLink | (root.side ? kEvRight : 0u);
    uint32_t wsp = 0;
    for (;;) {
        const uint32_t size = ce - cs;
        const uint32_t id = nid++;
        if (size <= lcap) {  // a right child whose left sibling was internal
            emit_event(s, ev, id, cpar, (cdep << 16) | clink | kEvLeaf, 0u, pbase + cs, size);
            ++nleaf;
            maxd = max(maxd, cdep);
        } else {
            FT_MARK(0);
            if (kd - wb >= kDrawWin) {  // refill the draw window (uniform)
                wb = kd & ~(kDrawWin - 1);
                __syncwarp();
                for (uint32_t j = lane; j < kDrawWin; j += 32) s.dwin[j] = wb + j < a.n_draws ? a.draws[wb + j] : 0u;
                __syncwarp();
            }
            const uint32_t d = s.dwin[kd - wb];
            ++kd;
            FT_MARK(8);
            uint32_t sval;
            uint8_t even;
            uint32_t mid;
            if (size <= 32) {
                mid = tile_node_reg<1>(st, li, gid, sb, d, cs, ce, sval, even);
            } else if (size <= 64) {
                mid = tile_node_reg<2>(st, li, gid, sb, d, cs, ce, sval, even);
            } else if (size <= 128) {
                mid = tile_node_reg<4>(st, li, gid, sb, d, cs, ce, sval, even);
            } else if (size <= 256) {
                mid = tile_node_reg<8>(st, li, gid, sb, d, cs, ce, sval, even);
            } else {
                mid = tile_node_smem(s, st, li, lt, gid, sb, d, cs, ce, sval, even);
            }
            FT_MARK(10);
            // the node and its leaf children go to the record warp (left child = id + 1 in
            // pre-order, a leaf right child of a leaf left child = id + 2)
            const bool lleaf = mid - cs <= lcap, rleaf = ce - mid <= lcap;
            const bool both = lleaf && rleaf;
            emit_event(s, ev, id, cpar,
                       d | (cdep << 16) | clink | (lleaf ? kEvLLeaf : 0u) | (rleaf ? kEvRLeaf : 0u) |
                           (even ? kEvSplit : 0u),
                       sval, pbase + cs, (mid - cs) | ((ce - mid) << 11));
            maxd = max(maxd, cdep + 1);
            if (!lleaf) {
                // descend into the left child; the right one waits on the stack
                if (lane == 0) s.tstack[wsp] = tpack(id, mid, ce, cdep + 1 - dep0, 3u);
                ++wsp;
                DCHK(wsp < kTileStack);
                ce = mid;
                cdep += 1;
                cpar = id;
                clink = 0;  // left = id + 1 is already in the record
                FT_MARK(12);
                continue;
            }
            nid += both ? 2u : 1u;
            nleaf += both ? 2u : 1u;
            if (!rleaf) {  // left leaf emitted; the right child (= id + 2) is next
                cs = mid;
                cdep += 1;
                cpar = id;
                clink = 0;
                FT_MARK(12);
                continue;
            }
            FT_MARK(12);
        }
        if (wsp == 0) break;
        __syncwarp();
        --wsp;
        const uint64_t pe = s.tstack[wsp];
        const uint32_t lo = uint32_t(pe);
        cpar = uint32_t(pe >> 32);
        cs = (lo >> 21) & 0x7ffu;
        ce = (lo >> 10) & 0x7ffu;
        cdep = dep0 + ((lo >> 2) & 0xffu);
        clink = ((lo & 1u) ? kEvLink : 0u) | ((lo & 2u) ? kEvRight : 0u);
    }
    if (lane == 0) {
        s.node_count = nid;
        s.draw_idx = kd;
        s.dwin_base = wb;
        s.leaf_count = nleaf;
        s.max_depth = maxd;
        s.ev_count = ev;
    }
    // point_index of the tile in leaf order
    for (uint32_t j = lane; j < tsz; j += 32) s.sub2[j] = gid[s.lidx[j]];
    __syncwarp();
    for (uint32_t j = lane; j < tsz; j += 32) s.sub[ts + j] = s.sub2[j];
    __syncwarp();
    FT_MARK(14);
}

// Builds the subtree rooted at `root` (<= kWarpSubtree points) with warp 0,
// in pre-order (the root's id is assigned here).  The subtree's slice of
// point_index lives in shared memory.  Nodes of <= 256 points gather their
// column into registers (8 independent loads per lane); larger nodes gather
// it into shared memory (s.col) in batches of 8 loads per lane, so neither
// pass waits on one L2 round trip per chunk.  Sum exactly, partition by
// ballots in shared memory.
__device__ void warp_build_subtree(const BuildArgs& a, Smem& s, StackEntry root) {
    const uint32_t lane = lane_id();
    const uint32_t base = root.start, total = root.end - root.start;
    uint32_t* sub = s.sub;
    uint32_t* rtmp = s.sub2;
    float* col = s.col;
    for (uint32_t j = lane; j < total; j += 32) sub[j] = a.pidx[base + j];
    __syncwarp();
    // stage the subtree's rows in L2: every node below gathers from them
    if (a.x8) {
        for (uint32_t j = lane; j < total; j += 32)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(a.x8 + size_t(sub[j]) * a.ld8));
    } else if (size_t(total) * a.ld * 4 <= kPrefetchBytes) {
        const uint32_t lines = (a.ld * 4 + 127) / 128;
        for (uint32_t j = lane; j < total * lines; j += 32) {
            const char* ptr = reinterpret_cast<const char*>(a.x + size_t(sub[j / lines]) * a.ld) + (j % lines) * 128;
            asm volatile("prefetch.global.L2 [%0];" ::"l"(ptr));
        }
    }
    uint32_t wsp = 1;
    if (lane == 0) s.wstack[0] = StackEntry{0, total, root.depth, root.parent, root.side};
    __syncwarp();
    const uint32_t lt = (1u << lane) - 1u;
    // staged-tile path (u8 rows fit shared memory)
    const uint32_t sb = a.ld8 + 4;
    const uint32_t tile_max = tile_capacity(a);
    while (wsp > 0) {
        --wsp;
        const StackEntry e = s.wstack[wsp];
        const uint32_t size = e.end - e.start;
        // (events carry the depth in 8 bits: a tile adds < 64 levels, n < 2^32 gives < 100 above it)
        if (size <= tile_max && size > a.leaf_cap && size >= 64 && e.parent != kInvalidId && e.depth < 160) {
            __syncwarp();
            warp_build_tile(a, s, e, base, sb);
            continue;
        }
        const uint32_t id = s.node_count;
        __syncwarp();
        if (lane == 0) {
            s.node_count = id + 1;
            if (e.parent != kInvalidId) {
                if (e.side == 0) a.nodes[e.parent].left = id;
                else a.nodes[e.parent].right = id;
            }
            a.depth[id] = e.depth;
            s.max_depth = max(s.max_depth, e.depth);
        }
        if (size <= a.leaf_cap) {
            if (lane == 0) {
                a.nodes[id] = KdNodeDev{kLeaf, 0.0f, base + e.start, base + e.end};
                a.even[id] = 0;
                s.leaf_count++;
            }
            __syncwarp();
            continue;
        }
        FT_MARK(0);
        const uint32_t d = warp_draw(a, s);
        FT_MARK(1);
        const uint32_t chunks = (size + 31) / 32;
        float split;
        uint32_t nl = 0, nr = 0;
        if (chunks <= 8) {
            // ---- register path: one gather round
            float v[8];
            uint32_t pid[8];
#pragma unroll
            for (uint32_t u = 0; u < 8; ++u) {
                const uint32_t j = e.start + u * 32 + lane;
                pid[u] = (u < chunks && j < e.end) ? sub[j] : 0;
            }
#pragma unroll
            for (uint32_t u = 0; u < 8; ++u) {
                const uint32_t j = e.start + u * 32 + lane;
                v[u] = (u < chunks && j < e.end) ? ldv(a, pid[u], d) : 0.0f;
            }
            FT_MARK(2);
            double sum;
            if (a.x8) {
                uint32_t is = 0;
#pragma unroll
                for (uint32_t u = 0; u < 8; ++u) is += uint32_t(v[u]);
                sum = double(__reduce_add_sync(0xffffffffu, is));  // exact: integers
            } else {
                sum = 0.0;
                int top = INT_MIN, lsb = INT_MAX;
#pragma unroll
                for (uint32_t u = 0; u < 8; ++u) {
                    sum += double(v[u]);
                    val_stats(v[u], top, lsb);
                }
                for (int o = 16; o > 0; o >>= 1) {
                    sum += __shfl_xor_sync(0xffffffffu, sum, o);
                    top = max(top, __shfl_xor_sync(0xffffffffu, top, o));
                    lsb = min(lsb, __shfl_xor_sync(0xffffffffu, lsb, o));
                }
                if (!sum_is_exact(top, lsb, size)) {  // reference order: sequential over point_index
                    double ser = 0.0;
                    if (lane == 0)
                        for (uint32_t p = e.start; p < e.end; ++p) ser += double(ldv(a, sub[p], d));
                    sum = __shfl_sync(0xffffffffu, ser, 0);
                }
            }
            split = __double2float_rn(__ddiv_rn(sum, double(size)));
            FT_MARK(3);
#pragma unroll
            for (uint32_t u = 0; u < 8; ++u) {
                if (u >= chunks) break;
                const uint32_t j = e.start + u * 32 + lane;
                const bool valid = j < e.end;
                const bool left = valid && v[u] <= split;
                const uint32_t bl = __ballot_sync(0xffffffffu, left);
                const uint32_t br = __ballot_sync(0xffffffffu, valid && !left);
                if (left) sub[e.start + nl + __popc(bl & lt)] = pid[u];
                else if (valid) rtmp[nr + __popc(br & lt)] = pid[u];
                nl += __popc(bl);
                nr += __popc(br);
            }
        } else {
            // ---- shared-memory path (257..4096 points): gather the column once
            double sum = 0.0;
            int top = INT_MIN, lsb = INT_MAX;
            uint32_t is = 0;
            for (uint32_t p0 = e.start; p0 < e.end; p0 += 256) {
                float x[8];
#pragma unroll
                for (uint32_t u = 0; u < 8; ++u) {
                    const uint32_t p = p0 + u * 32 + lane;
                    x[u] = p < e.end ? ldv(a, sub[p], d) : 0.0f;
                }
#pragma unroll
                for (uint32_t u = 0; u < 8; ++u) {
                    const uint32_t p = p0 + u * 32 + lane;
                    if (p < e.end) col[p] = x[u];
                    if (a.x8) is += uint32_t(x[u]);
                    else {
                        sum += double(x[u]);
                        val_stats(x[u], top, lsb);
                    }
                }
            }
            FT_MARK(2);
            if (a.x8) {
                sum = double(__reduce_add_sync(0xffffffffu, is));
            } else {
                for (int o = 16; o > 0; o >>= 1) {
                    sum += __shfl_xor_sync(0xffffffffu, sum, o);
                    top = max(top, __shfl_xor_sync(0xffffffffu, top, o));
                    lsb = min(lsb, __shfl_xor_sync(0xffffffffu, lsb, o));
                }
                if (!sum_is_exact(top, lsb, size)) {
                    __syncwarp();
                    double ser = 0.0;
                    if (lane == 0)
                        for (uint32_t p = e.start; p < e.end; ++p) ser += double(col[p]);
                    sum = __shfl_sync(0xffffffffu, ser, 0);
                }
            }
            split = __double2float_rn(__ddiv_rn(sum, double(size)));
            __syncwarp();
            FT_MARK(3);
            for (uint32_t b0 = e.start; b0 < e.end; b0 += 32) {
                const uint32_t p = b0 + lane;
                const bool valid = p < e.end;
                const uint32_t pid = valid ? sub[p] : 0;
                const bool left = valid && col[p] <= split;
                const uint32_t bl = __ballot_sync(0xffffffffu, left);
                const uint32_t br = __ballot_sync(0xffffffffu, valid && !left);
                if (left) sub[e.start + nl + __popc(bl & lt)] = pid;
                else if (valid) rtmp[nr + __popc(br & lt)] = pid;
                nl += __popc(bl);
                nr += __popc(br);
            }
        }
        FT_MARK(4);
        __syncwarp();
        for (uint32_t j = lane; j < nr; j += 32) sub[e.start + nl + j] = rtmp[j];
        __syncwarp();
        uint32_t mid = e.start + nl;
        uint8_t even = 0;
        FT_MARK(5);
        if (nl == 0 || nr == 0 || max(nl, nr) > 4u * min(nl, nr)) {
            // kd_forest.cpp:70-83 degenerate split: sort by (value, id), split at the median
            warp_sort_local(a, s, sub, e.start, size, d);
            mid = e.start + size / 2;
            split = midpoint_f(ldx(a, sub[mid - 1], d), ldx(a, sub[mid], d));
            even = 1;
        }
        if (lane == 0) {
            a.nodes[id] = KdNodeDev{d, split, 0u, 0u};
            a.even[id] = even;
            s.wstack[wsp] = StackEntry{mid, e.end, e.depth + 1, id, 1u};
            s.wstack[wsp + 1] = StackEntry{e.start, mid, e.depth + 1, id, 0u};
            if (wsp + 2 > kStack - 2) s.error = 1;
        }
        wsp = min(wsp + 2, kStack - 2);
        __syncwarp();
        FT_MARK(6);
    }
    for (uint32_t j = lane; j < total; j += 32) a.pidx[base + j] = sub[j];
    if (tile_max) {  // release the helper warps and the record warp
        if (lane == 0) s.t_size = 0;
        __syncwarp();
        named_bar(1, kStagers);
        uint32_t ev = s.ev_count;
        emit_event(s, ev, 0u, 0u, kEvQuit, 0u, 0u, 0u);
        if (lane == 0) s.ev_count = ev;
        __syncwarp();
    }
    __syncwarp();
}

// ------------------------------------------------------------- block path

__device__ void block_reduce_stats(Smem& s, double& sum, int& top, int& lsb) {
    const uint32_t lane = lane_id(), warp = threadIdx.x / 32;
    for (int o = 16; o > 0; o >>= 1) {
        sum += __shfl_xor_sync(0xffffffffu, sum, o);
        top = max(top, __shfl_xor_sync(0xffffffffu, top, o));
        lsb = min(lsb, __shfl_xor_sync(0xffffffffu, lsb, o));
    }
    if (lane == 0) {
        s.red_sum[warp] = sum;
        s.red_top[warp] = top;
        s.red_lsb[warp] = lsb;
    }
    __syncthreads();
    if (warp == 0) {
        sum = lane < kWarps ? s.red_sum[lane] : 0.0;
        top = lane < kWarps ? s.red_top[lane] : INT_MIN;
        lsb = lane < kWarps ? s.red_lsb[lane] : INT_MAX;
        for (int o = 16; o > 0; o >>= 1) {
            sum += __shfl_xor_sync(0xffffffffu, sum, o);
            top = max(top, __shfl_xor_sync(0xffffffffu, top, o));
            lsb = min(lsb, __shfl_xor_sync(0xffffffffu, lsb, o));
        }
        if (lane == 0) {
            s.red_sum[0] = sum;
            s.red_top[0] = top;
            s.red_lsb[0] = lsb;
        }
    }
    __syncthreads();
    sum = s.red_sum[0];
    top = s.red_top[0];
    lsb = s.red_lsb[0];
    __syncthreads();
}

__device__ void block_sort_node(const BuildArgs& a, Smem& s, uint32_t start, uint32_t size,
                                uint32_t d) {
    const uint32_t m = next_pow2(size);
    uint64_t* k = m <= kSortSmem ? s.sortk : a.sortbuf;
    for (uint32_t j = threadIdx.x; j < m; j += blockDim.x) {
        uint64_t key = kEmptyKey;
        if (j < size) {
            const uint32_t id = a.pidx[start + j];
            key = val_id_key(ldx(a, id, d), id);
        }
        k[j] = key;
    }
    __syncthreads();
    block_bitonic_sort(k, m);
    for (uint32_t j = threadIdx.x; j < size; j += blockDim.x) a.pidx[start + j] = uint32_t(k[j]);
    __syncthreads();
}

// Column value of point p on dim d: u8 copy when present (exact), else fp32.
template <bool U8>
__device__ __forceinline__ float colv(const BuildArgs& a, uint32_t p, uint32_t d) {
    if constexpr (U8) return float(__ldg(a.x8 + size_t(p) * a.ld8 + d));
    else return __ldg(a.x + size_t(p) * a.ld + d);
}

// One node of > kWarpSubtree points with the whole CTA.  Pass 1 gathers the
// column with 8 loads in flight per thread and sums it (u8: integer sum, exact;
// fp32: double sum + exactness test, serial fallback).  Pass 2 is a stable
// partition over chunks of kBlock*8 points, 8 consecutive points per thread,
// with one block-wide scan of packed (left, right) counts per chunk.
template <bool U8>
__device__ void block_split_node(const BuildArgs& a, Smem& s, const StackEntry& e, uint32_t id) {
    constexpr uint32_t kPer = 8, kChunk = kBlock * kPer;
    const uint32_t tid = threadIdx.x, lane = lane_id(), warp = tid / 32;
    const uint32_t size = e.end - e.start;
    if (warp == 0) {
        const uint32_t d = warp_draw(a, s);
        if (lane == 0) s.b_d = d;
    }
    __syncthreads();
    const uint32_t d = s.b_d;
    double sum = 0.0;
    int top = INT_MIN, lsb = INT_MAX;
    uint64_t isum = 0;
    constexpr uint32_t kSumPer = 8;  // gathers in flight per thread in the sum pass (16: no gain)
    for (uint32_t p0 = e.start; p0 < e.end; p0 += kBlock * kSumPer) {
        uint32_t pid[kSumPer];
#pragma unroll
        for (uint32_t u = 0; u < kSumPer; ++u) {
            const uint32_t q = p0 + u * kBlock + tid;
            pid[u] = q < e.end ? a.pidx[q] : 0u;
        }
        float v[kSumPer];
#pragma unroll
        for (uint32_t u = 0; u < kSumPer; ++u) {
            const uint32_t q = p0 + u * kBlock + tid;
            v[u] = q < e.end ? colv<U8>(a, pid[u], d) : 0.0f;
        }
#pragma unroll
        for (uint32_t u = 0; u < kSumPer; ++u) {
            const uint32_t q = p0 + u * kBlock + tid;
            if (q < e.end) a.col[q] = v[u];  // coalesced; read back by the partition pass
            if constexpr (U8) {
                isum += uint32_t(v[u]);
            } else {
                sum += double(v[u]);
                val_stats(v[u], top, lsb);
            }
        }
    }
    if constexpr (U8) {
        for (int o = 16; o > 0; o >>= 1) isum += __shfl_xor_sync(0xffffffffu, isum, o);
        if (lane == 0) s.red_sum[warp] = double(isum);  // < 2^53: exact
        __syncthreads();
        if (tid == 0) {
            double t = 0.0;
            for (uint32_t w = 0; w < kWarps; ++w) t += s.red_sum[w];
            s.b_sum = t;
        }
        __syncthreads();
        sum = s.b_sum;
    } else {
        block_reduce_stats(s, sum, top, lsb);
        if (!sum_is_exact(top, lsb, size)) {
            if (tid == 0) {
                sum = 0.0;
                for (uint32_t p = e.start; p < e.end; ++p) sum += double(ldx(a, a.pidx[p], d));
                s.b_sum = sum;
            }
            __syncthreads();
            sum = s.b_sum;
        }
    }
    float split = __double2float_rn(__ddiv_rn(sum, double(size)));
    uint32_t nl = 0, nr = 0;
    for (uint32_t b0 = e.start; b0 < e.end; b0 += kChunk) {
        const uint32_t q0 = b0 + tid * kPer;
        uint32_t pid[kPer];
        float cv[kPer];
#pragma unroll
        for (uint32_t i = 0; i < kPer; ++i) {
            pid[i] = q0 + i < e.end ? a.pidx[q0 + i] : 0u;
            cv[i] = q0 + i < e.end ? a.col[q0 + i] : 0.0f;
        }
        uint32_t lm = 0, vm = 0;
#pragma unroll
        for (uint32_t i = 0; i < kPer; ++i) {
            if (q0 + i < e.end) {
                vm |= 1u << i;
                if (cv[i] <= split) lm |= 1u << i;
            }
        }
        // block exclusive scan of (lefts | rights << 16)
        const uint32_t x = __popc(lm) | (__popc(vm & ~lm) << 16);
        uint32_t incl = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= uint32_t(o)) incl += y;
        }
        if (lane == 31) s.cnt_l[warp] = incl;
        __syncthreads();
        uint32_t wp = 0, tot = 0;
#pragma unroll
        for (uint32_t w = 0; w < kWarps; ++w) {
            const uint32_t c = s.cnt_l[w];
            wp += w < warp ? c : 0u;
            tot += c;
        }
        const uint32_t ex = wp + incl - x;
        uint32_t ol = e.start + nl + (ex & 0xffffu), orr = e.start + nr + (ex >> 16);
#pragma unroll
        for (uint32_t i = 0; i < kPer; ++i) {
            if ((lm >> i) & 1u) a.pidx[ol++] = pid[i];
            else if ((vm >> i) & 1u) a.rtmp[orr++] = pid[i];
        }
        nl += tot & 0xffffu;
        nr += tot >> 16;
        __syncthreads();
    }
    for (uint32_t j = tid; j < nr; j += kBlock) a.pidx[e.start + nl + j] = a.rtmp[e.start + j];
    __syncthreads();
    uint32_t mid = e.start + nl;
    uint8_t even = 0;
    if (nl == 0 || nr == 0 || max(nl, nr) > 4u * min(nl, nr)) {
        block_sort_node(a, s, e.start, size, d);
        mid = e.start + size / 2;
        split = midpoint_f(ldx(a, a.pidx[mid - 1], d), ldx(a, a.pidx[mid], d));
        even = 1;
    }
    if (tid == 0) {
        a.nodes[id] = KdNodeDev{d, split, 0u, 0u};
        a.even[id] = even;
        s.bstack[s.bsp] = StackEntry{mid, e.end, e.depth + 1, id, 1};
        s.bstack[s.bsp + 1] = StackEntry{e.start, mid, e.depth + 1, id, 0};
        s.bsp += 2;
        if (s.bsp > kStack - 2) s.error = 1;
    }
    __syncthreads();
}

namespace cg = cooperative_groups;

// One node of > kClusterMin points split by the whole cluster (C CTAs, this
// one of rank r).  Each CTA sums its slice of the node (column gathered into
// a.col); the partial sums go to the leader's shared memory through DSMEM and
// every CTA forms the same total, hence the same split.  The stable
// partition needs each slice's left/right counts first (second exchange);
// lefts and rights are then scattered to ltmp / rtmp at their global offsets
// (other slices may still be reading pidx), and copied back to pidx.  The
// leader then handles the degenerate fallback and the node record.
template <bool U8>
__device__ void cluster_split_node(const BuildArgs& a, Smem& s, Smem* lead, const cg::cluster_group& cl,
                                   uint32_t rank, uint32_t C, const StackEntry& e, uint32_t id, uint32_t d) {
    constexpr uint32_t kPer = 8, kChunk = kBlock * kPer;
    const uint32_t tid = threadIdx.x, lane = lane_id(), warp = tid / 32;
    const uint32_t size = e.end - e.start;
    const uint32_t len = (size + C - 1) / C;
    const uint32_t lo = e.start + min(size, rank * len), hi = e.start + min(size, (rank + 1) * len);
    // pass 1: gather + partial sum of this slice
    double sum = 0.0;
    int top = INT_MIN, lsb = INT_MAX;
    uint64_t isum = 0;
    for (uint32_t p0 = lo; p0 < hi; p0 += kChunk) {
        uint32_t pid[kPer];
#pragma unroll
        for (uint32_t u = 0; u < kPer; ++u) {
            const uint32_t q = p0 + u * kBlock + tid;
            pid[u] = q < hi ? a.pidx[q] : 0u;
        }
        float v[kPer];
#pragma unroll
        for (uint32_t u = 0; u < kPer; ++u) {
            const uint32_t q = p0 + u * kBlock + tid;
            v[u] = q < hi ? colv<U8>(a, pid[u], d) : 0.0f;
        }
#pragma unroll
        for (uint32_t u = 0; u < kPer; ++u) {
            const uint32_t q = p0 + u * kBlock + tid;
            if (q < hi) a.col[q] = v[u];
            if constexpr (U8) {
                isum += uint32_t(v[u]);
            } else {
                sum += double(v[u]);
                val_stats(v[u], top, lsb);
            }
        }
    }
    if constexpr (U8) {
        for (int o = 16; o > 0; o >>= 1) isum += __shfl_xor_sync(0xffffffffu, isum, o);
        if (lane == 0) s.red_sum[warp] = double(isum);
        __syncthreads();
        if (tid == 0) {
            double t = 0.0;
            for (uint32_t w = 0; w < kWarps; ++w) t += s.red_sum[w];
            lead->cl_sum[rank] = t;
            lead->cl_top[rank] = INT_MIN;
            lead->cl_lsb[rank] = INT_MAX;
        }
    } else {
        block_reduce_stats(s, sum, top, lsb);
        if (tid == 0) {
            lead->cl_sum[rank] = sum;
            lead->cl_top[rank] = top;
            lead->cl_lsb[rank] = lsb;
        }
    }
    cl.sync();
    if (tid == 0) {
        double t = 0.0;
        int tp = INT_MIN, lb = INT_MAX;
        for (uint32_t r = 0; r < C; ++r) {
            t += lead->cl_sum[r];  // exact: integer / exactly representable partials
            tp = max(tp, lead->cl_top[r]);
            lb = min(lb, lead->cl_lsb[r]);
        }
        s.b_sum = t;
        s.b_exact = U8 ? 1 : int(sum_is_exact(tp, lb, size));
    }
    __syncthreads();
    if (!s.b_exact) {  // uniform across the cluster: the reference's sequential order, by the leader
        cl.sync();
        if (rank == 0 && tid == 0) {
            double t = 0.0;
            for (uint32_t p = e.start; p < e.end; ++p) t += double(ldx(a, a.pidx[p], d));
            s.b_sum = t;
        }
        cl.sync();
        if (tid == 0) s.b_sum = lead->b_sum;
        __syncthreads();
    }
    const float split = __double2float_rn(__ddiv_rn(s.b_sum, double(size)));
    // pass 2a: this slice's left / right counts
    uint32_t cl_ = 0, cr_ = 0;
    for (uint32_t q = lo + tid; q < hi; q += kBlock) {
        if (a.col[q] <= split) ++cl_;
        else ++cr_;
    }
    for (int o = 16; o > 0; o >>= 1) {
        cl_ += __shfl_xor_sync(0xffffffffu, cl_, o);
        cr_ += __shfl_xor_sync(0xffffffffu, cr_, o);
    }
    if (lane == 0) {
        s.cnt_l[warp] = cl_;
        s.cnt_r[warp] = cr_;
    }
    __syncthreads();
    if (tid == 0) {
        uint32_t tl = 0, tr = 0;
        for (uint32_t w = 0; w < kWarps; ++w) {
            tl += s.cnt_l[w];
            tr += s.cnt_r[w];
        }
        lead->cl_nl[rank] = tl;
        lead->cl_nr[rank] = tr;
    }
    cl.sync();
    uint32_t lpre = 0, rpre = 0, NL = 0;
    for (uint32_t r = 0; r < C; ++r) {
        const uint32_t x = lead->cl_nl[r], y = lead->cl_nr[r];
        if (r < rank) {
            lpre += x;
            rpre += y;
        }
        NL += x;
    }
    const uint32_t NR = size - NL;
    // pass 2b: stable scatter of this slice (8 consecutive points per thread)
    uint32_t nl = 0, nr = 0;
    for (uint32_t b0 = lo; b0 < hi; b0 += kChunk) {
        const uint32_t q0 = b0 + tid * kPer;
        uint32_t pid[kPer];
        float cv[kPer];
#pragma unroll
        for (uint32_t i = 0; i < kPer; ++i) {
            pid[i] = q0 + i < hi ? a.pidx[q0 + i] : 0u;
            cv[i] = q0 + i < hi ? a.col[q0 + i] : 0.0f;
        }
        uint32_t lm = 0, vm = 0;
#pragma unroll
        for (uint32_t i = 0; i < kPer; ++i) {
            if (q0 + i < hi) {
                vm |= 1u << i;
                if (cv[i] <= split) lm |= 1u << i;
            }
        }
        const uint32_t x = __popc(lm) | (__popc(vm & ~lm) << 16);
        uint32_t incl = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= uint32_t(o)) incl += y;
        }
        if (lane == 31) s.cnt_l[warp] = incl;
        __syncthreads();
        uint32_t wp = 0, tot = 0;
#pragma unroll
        for (uint32_t w = 0; w < kWarps; ++w) {
            const uint32_t c = s.cnt_l[w];
            wp += w < warp ? c : 0u;
            tot += c;
        }
        const uint32_t ex = wp + incl - x;
        uint32_t ol = e.start + lpre + nl + (ex & 0xffffu), orr = e.start + rpre + nr + (ex >> 16);
#pragma unroll
        for (uint32_t i = 0; i < kPer; ++i) {
            if ((lm >> i) & 1u) a.ltmp[ol++] = pid[i];
            else if ((vm >> i) & 1u) a.rtmp[orr++] = pid[i];
        }
        nl += tot & 0xffffu;
        nr += tot >> 16;
        __syncthreads();
    }
    cl.sync();
    // copy back: positions [e.start, e.start + size) split by rank
    for (uint32_t g = min(size, rank * len) + tid; g < min(size, (rank + 1) * len); g += kBlock)
        a.pidx[e.start + g] = g < NL ? a.ltmp[e.start + g] : a.rtmp[e.start + g - NL];
    cl.sync();
    if (rank == 0) {
        uint32_t mid = e.start + NL;
        uint8_t even = 0;
        float sp = split;
        if (NL == 0 || NR == 0 || max(NL, NR) > 4u * min(NL, NR)) {
            block_sort_node(a, s, e.start, size, d);
            mid = e.start + size / 2;
            sp = midpoint_f(ldx(a, a.pidx[mid - 1], d), ldx(a, a.pidx[mid], d));
            even = 1;
        }
        if (tid == 0) {
            a.nodes[id] = KdNodeDev{d, sp, 0u, 0u};
            a.even[id] = even;
            s.bstack[s.bsp] = StackEntry{mid, e.end, e.depth + 1, id, 1};
            s.bstack[s.bsp + 1] = StackEntry{e.start, mid, e.depth + 1, id, 0};
            s.bsp += 2;
            if (s.bsp > kStack - 2) s.error = 1;
        }
        __syncthreads();
    }
}

__global__ void __launch_bounds__(kBlock, 1) forest_build_kernel(const BuildArgs* __restrict__ args) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Smem& s = *reinterpret_cast<Smem*>(smem_raw);
    const cg::cluster_group cl = cg::this_cluster();
    const uint32_t C = cl.num_blocks(), rank = cl.block_rank();
    const BuildArgs a = args[blockIdx.x / C];
    Smem* lead = cl.map_shared_rank(&s, 0);  // the tree's leader CTA (rank 0) owns the build state
    const uint32_t tid = threadIdx.x;
    for (uint32_t i = rank * kBlock + tid; i < a.n; i += C * kBlock) a.pidx[i] = i;
    for (uint32_t i = tid; i < kEvRing * 2; i += kBlock) s.ring[i] = make_uint4(0u, 0u, 0u, 0u);
    if (tid == 0) {
        s.dwin_base = 0xffffffffu - kDrawWin;  // empty window
        s.ev_count = 0;
        s.ev_tail = 0;
        s.draw_idx = 0;
        s.node_count = 0;
        s.leaf_count = 0;
        s.max_depth = 0;
        s.error = 0;
        s.cyc_block = 0;
        s.cyc_warp = 0;
        for (int q = 0; q < 16; ++q) s.ft[q] = 0;
        s.bstack[0] = StackEntry{0, a.n, 0, kInvalidId, 0};
        s.bsp = 1;
    }
    cl.sync();
    // staged tiles on: the block path runs down to tile size (its chunked
    // partition beats warp 0's streaming path on 1k-4k point nodes)
    const uint32_t warp_limit = tile_capacity(a) ? tile_capacity(a) : kWarpSubtree;
    for (;;) {
        // the leader picks the next pre-order node: 0 done, 1 cluster split,
        // 2 warp subtree / staged tile, 3 block split by the leader alone
        if (rank == 0) {
            if (tid == 0) {
                if (s.bsp == 0 || s.error) {
                    s.cmd = 0;
                } else {
                    const StackEntry e = s.bstack[--s.bsp];
                    const uint32_t size = e.end - e.start;
                    s.cmd_e = e;
                    if (size <= warp_limit) {
                        s.cmd = 2;
                    } else {
                        s.cmd = (C > 1 && size > kClusterMin) ? 1u : 3u;
                        const uint32_t id = s.node_count;
                        s.node_count = id + 1;
                        if (e.parent != kInvalidId) {
                            if (e.side == 0) a.nodes[e.parent].left = id;
                            else a.nodes[e.parent].right = id;
                        }
                        a.depth[id] = e.depth;
                        s.max_depth = max(s.max_depth, e.depth);
                        s.cmd_id = id;
                    }
                }
            }
            __syncthreads();
            if (s.cmd == 1 && tid < 32) {
                const uint32_t d = warp_draw(a, s);
                if (tid == 0) s.cmd_d = d;
            }
        }
        cl.sync();
        const uint32_t cmd = lead->cmd;
        if (cmd == 0) break;
        const StackEntry e = lead->cmd_e;
        if (cmd == 2) {
            if (rank == 0) {
                const long long c0 = clock64();
                if (tid < 32) warp_build_subtree(a, s, e);
                else if (tile_capacity(a)) {
                    if (tid >= kStagers) record_warp(a, s);
                    else stage_helper(a, s);
                }
                if (tid == 0) s.cyc_warp += clock64() - c0;
                __syncthreads();
            }
            continue;
        }
        const long long c1 = clock64();
        if (cmd == 1) {
            if (a.x8) cluster_split_node<true>(a, s, lead, cl, rank, C, e, lead->cmd_id, lead->cmd_d);
            else cluster_split_node<false>(a, s, lead, cl, rank, C, e, lead->cmd_id, lead->cmd_d);
        } else if (rank == 0) {
            if (a.x8) block_split_node<true>(a, s, e, s.cmd_id);
            else block_split_node<false>(a, s, e, s.cmd_id);
        }
        if (rank == 0 && tid == 0) s.cyc_block += clock64() - c1;
    }
    cl.sync();  // the leader's shared memory stays mapped until every CTA is done with it
    if (rank != 0) return;
    __syncthreads();
    if (tid == 0) {
        a.meta[0] = s.node_count;
        a.meta[1] = 0;
        a.meta[2] = s.leaf_count;
        a.meta[3] = s.max_depth;
        a.meta[4] = s.error;
        a.meta[5] = uint32_t(s.cyc_block >> 10);  // phase timing (kcycles), debug/profiling
        a.meta[6] = uint32_t(s.cyc_warp >> 10);
#ifdef ANNK_FOREST_TIMING
        printf("tree %u phases (Mcycles): draw %.1f gather %.1f sum %.1f part %.1f copy %.1f tail %.1f\n",
               blockIdx.x, s.ft[1] / 1e6, s.ft[2] / 1e6, s.ft[3] / 1e6, s.ft[4] / 1e6, s.ft[5] / 1e6, s.ft[6] / 1e6);
        printf("tree %u tile (Mcycles): gap %.1f leaf %.1f stage %.1f draw %.1f sum %.1f part %.1f copy %.1f tail %.1f perm %.1f\n",
               blockIdx.x, s.ft[0] / 1e6, s.ft[15] / 1e6, s.ft[13] / 1e6, s.ft[8] / 1e6, s.ft[9] / 1e6, s.ft[10] / 1e6, s.ft[11] / 1e6,
               s.ft[12] / 1e6, s.ft[14] / 1e6);
#endif
    }
}

// annk_forest_import: pack (split_dim, split_val, left, right) into
// KdNodeDev records and validate them; stats = [leaves, max depth, error bits
// (1 leaf range, 2 split dimension, 4 child id)].
__global__ void import_nodes_kernel(const uint32_t* __restrict__ sd, const float* __restrict__ sv,
                                    const uint32_t* __restrict__ lf, const uint32_t* __restrict__ rt,
                                    const uint32_t* __restrict__ depth, uint32_t m, uint32_t n, uint32_t dim,
                                    KdNodeDev* __restrict__ out, uint32_t* stats) {
    uint32_t leaves = 0, maxd = 0, err = 0;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
        const uint32_t d = sd[i], l = lf[i], r = rt[i];
        out[i] = KdNodeDev{d, sv[i], l, r};
        if (d == kLeaf) {
            ++leaves;
            if (l >= r || r > n) err |= 1u;
        } else {
            if (d >= dim) err |= 2u;
            if (l >= m || r >= m) err |= 4u;
        }
        maxd = max(maxd, depth[i]);
    }
    leaves = __reduce_add_sync(0xffffffffu, leaves);
    maxd = __reduce_max_sync(0xffffffffu, maxd);
    err = __reduce_or_sync(0xffffffffu, err);
    if ((threadIdx.x & 31) == 0) {
        if (leaves) atomicAdd(&stats[0], leaves);
        if (maxd) atomicMax(&stats[1], maxd);
        if (err) atomicOr(&stats[2], err);
    }
}

// The per-tree split-dimension stream: out[t][k] = mt19937_64(substream(seed,t))
// output k mod dim (kd_forest.cpp:53,259).  One CTA per tree; each 312-word
// regeneration is a 3-phase parallel twist, tempering and the modulo are
// per-word parallel.  n draws cover every internal node (<= n-1).
__global__ void draws_kernel(uint64_t seed, uint32_t dim, uint32_t count, uint32_t* __restrict__ out) {
    __shared__ uint64_t mt[312];
    const uint32_t t = blockIdx.x, tid = threadIdx.x;
    uint32_t* o = out + size_t(t) * count;
    if (tid == 0) {
        mt[0] = substream(seed, t);
        for (int i = 1; i < 312; ++i) mt[i] = 6364136223846793005ULL * (mt[i - 1] ^ (mt[i - 1] >> 62)) + uint64_t(i);
    }
    __syncthreads();
    for (uint32_t g = 0; g * 312 < count; ++g) {
        uint64_t v = 0;
        if (tid < 156) v = mt_twist(mt[tid], mt[tid + 1], mt[tid + 156]);
        __syncthreads();
        if (tid < 156) mt[tid] = v;
        __syncthreads();
        if (tid >= 156 && tid < 311) v = mt_twist(mt[tid], mt[tid + 1], mt[tid - 156]);
        __syncthreads();
        if (tid >= 156 && tid < 311) mt[tid] = v;
        __syncthreads();
        if (tid == 0) mt[311] = mt_twist(mt[311], mt[0], mt[155]);
        __syncthreads();
        const uint32_t k = g * 312 + tid;
        if (tid < 312 && k < count) o[k] = uint32_t(mt_temper(mt[tid]) % uint64_t(dim));
        __syncthreads();
    }
}

// parent links and leaf ownership (graph_build.cpp:238-257 tables).
__global__ void forest_links_kernel(const KdNodeDev* __restrict__ nodes, uint32_t num_nodes,
                                    const uint32_t* __restrict__ pidx, uint32_t* __restrict__ parent,
                                    uint32_t* __restrict__ owner) {
    for (uint32_t id = blockIdx.x * blockDim.x + threadIdx.x; id < num_nodes; id += gridDim.x * blockDim.x) {
        const KdNodeDev nd = nodes[id];
        if (nd.split_dim == kLeaf) {
            for (uint32_t p = nd.left; p < nd.right; ++p) owner[pidx[p]] = id;
        } else {
            parent[nd.left] = id;
            parent[nd.right] = id;
        }
    }
}

// Per-leaf sibling lists (CSR over node ids): for a leaf at depth D, entry j
// (0 <= j < D) is the sibling of its ancestor chain at parent depth D-1-j —
// the subtrees graph_build.cpp:266-281 descends into, nearest level first.
__global__ void sib_count_kernel(const KdNodeDev* __restrict__ nodes, const uint32_t* __restrict__ depth,
                                 uint32_t num_nodes, uint32_t* __restrict__ cnt) {
    for (uint32_t id = blockIdx.x * blockDim.x + threadIdx.x; id <= num_nodes; id += gridDim.x * blockDim.x)
        cnt[id] = (id < num_nodes && nodes[id].split_dim == kLeaf) ? depth[id] : 0u;
}
__global__ void sib_fill_kernel(const KdNodeDev* __restrict__ nodes, const uint32_t* __restrict__ parent,
                                uint32_t num_nodes, const uint32_t* __restrict__ off, uint32_t* __restrict__ list) {
    for (uint32_t id = blockIdx.x * blockDim.x + threadIdx.x; id < num_nodes; id += gridDim.x * blockDim.x) {
        if (nodes[id].split_dim != kLeaf) continue;
        uint32_t o = off[id], node = id;
        for (uint32_t par = parent[node]; par != kInvalidId; node = par, par = parent[node]) {
            const KdNodeDev pn = nodes[par];
            list[o++] = pn.left == node ? pn.right : pn.left;
        }
    }
}

// Batched best-bin-first (kd_forest.cpp:276-305).  One thread per query with
// a binary min-heap over (double cost, node) in global scratch.
struct HeapEnt {
    double cost;
    uint32_t node;
    uint32_t pad;
};
__device__ __forceinline__ bool heap_less(const HeapEnt& x, const HeapEnt& y) {
    return x.cost != y.cost ? x.cost < y.cost : x.node < y.node;
}
__global__ void search_leaves_kernel(const KdNodeDev* __restrict__ nodes, uint32_t root,
                                     uint32_t leaf_count, const float* __restrict__ q, uint32_t nq,
                                     uint32_t ld, uint32_t n_leaves, HeapEnt* __restrict__ heaps,
                                     uint32_t heap_cap, uint32_t* __restrict__ out,
                                     uint32_t* __restrict__ counts) {
    const uint32_t qi = blockIdx.x * blockDim.x + threadIdx.x;
    if (qi >= nq) return;
    const float* qq = q + size_t(qi) * ld;
    HeapEnt* h = heaps + size_t(qi) * heap_cap;
    uint32_t hn = 0, cnt = 0;
    const uint32_t want = min(n_leaves, leaf_count);
    uint32_t* o = out + size_t(qi) * n_leaves;
    for (uint32_t j = 0; j < n_leaves; ++j) o[j] = kInvalidId;
    if (want > 0) {
        uint32_t nd = root;
        double cost = 0.0;
        for (;;) {
            for (KdNodeDev x = nodes[nd]; x.split_dim != kLeaf; x = nodes[nd]) {
                const double diff = double(qq[x.split_dim]) - double(x.split_val);
                const HeapEnt v{cost + fabs(diff), diff <= 0.0 ? x.right : x.left, 0};
                uint32_t i = hn++;
                while (i > 0) {
                    const uint32_t p = (i - 1) / 2;
                    if (!heap_less(v, h[p])) break;
                    h[i] = h[p];
                    i = p;
                }
                h[i] = v;
                nd = diff <= 0.0 ? x.left : x.right;
            }
            o[cnt++] = nd;
            if (cnt >= want || hn == 0) break;
            const HeapEnt top = h[0];
            const HeapEnt last = h[--hn];
            uint32_t i = 0;
            for (;;) {
                uint32_t c = 2 * i + 1;
                if (c >= hn) break;
                if (c + 1 < hn && heap_less(h[c + 1], h[c])) ++c;
                if (!heap_less(h[c], last)) break;
                h[i] = h[c];
                i = c;
            }
            if (hn) h[i] = last;
            nd = top.node;
            cost = top.cost;
        }
    }
    counts[qi] = cnt;
}

__global__ void descend_kernel(const KdNodeDev* __restrict__ nodes, const float* __restrict__ q,
                               uint32_t nq, uint32_t ld, const uint32_t* __restrict__ start,
                               uint32_t* __restrict__ out) {
    const uint32_t qi = blockIdx.x * blockDim.x + threadIdx.x;
    if (qi >= nq) return;
    const float* qq = q + size_t(qi) * ld;
    uint32_t nd = start[qi];
    for (KdNodeDev x = nodes[nd]; x.split_dim != kLeaf; x = nodes[nd])
        nd = qq[x.split_dim] <= x.split_val ? x.left : x.right;
    out[qi] = nd;
}

}  // namespace

void forest_ensure_links(annk_forest* f, bool rebuild) {
    if (f->links_ready && !rebuild) return;
    for (auto& t : f->trees) {
        t.parent.alloc(t.num_nodes);
        t.parent.fill_bytes(0xff);
        t.owner.alloc(f->n);
        t.owner.fill_bytes(0xff);
        const uint32_t grid = std::min<uint32_t>((t.num_nodes + 255) / 256, 4096);
        LAUNCH(forest_links_kernel, std::max(grid, 1u), 256, 0, t.nodes.p, t.num_nodes, t.pidx.p,
               t.parent.p, t.owner.p);
        // sibling lists
        t.sib_off.alloc(size_t(t.num_nodes) + 1);
        LAUNCH(sib_count_kernel, std::max(grid, 1u), 256, 0, t.nodes.p, t.depth.p, t.num_nodes, t.sib_off.p);
        size_t tmp = 0;
        CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, t.sib_off.p, t.sib_off.p, t.num_nodes + 1, stream()));
        DevBuf<unsigned char> scratch(std::max<size_t>(tmp, 1));
        CK(cub::DeviceScan::ExclusiveSum(scratch.p, tmp, t.sib_off.p, t.sib_off.p, t.num_nodes + 1, stream()));
        uint32_t total = 0;
        CK(cudaMemcpyAsync(&total, t.sib_off.p + t.num_nodes, 4, cudaMemcpyDeviceToHost, stream()));
        ssync();
        t.sib_list.alloc(std::max<size_t>(total, 1));
        LAUNCH(sib_fill_kernel, std::max(grid, 1u), 256, 0, t.nodes.p, t.parent.p, t.num_nodes, t.sib_off.p,
               t.sib_list.p);
    }
    f->links_ready = true;
    forest_upload_views(f);
}

void forest_upload_views(annk_forest* f) {
    std::vector<TreeView> v(f->n_trees);
    for (uint32_t i = 0; i < f->n_trees; ++i) {
        const TreeDev& t = f->trees[i];
        v[i] = TreeView{t.nodes.p, t.depth.p, t.pidx.p, t.parent.p, t.owner.p, t.sib_off.p, t.sib_list.p,
                        t.root, t.num_nodes, t.leaf_count, t.max_depth};
    }
    f->views.alloc(f->n_trees);
    f->views.upload(v.data(), v.size());
    ssync();
}

}  // namespace annk

using namespace annk;

extern "C" {

int annk_forest_build(const annk_dataset* ds, uint32_t n_trees, uint32_t leaf_cap, uint64_t seed,
                      annk_forest** out) {
    return abi([&] {
        if (!ds || !out) throw_invalid("build_forest: null argument");
        if (ds->n < 1) throw_invalid("build_forest: empty dataset");
        if (n_trees < 1) throw_invalid("build_forest: n_trees must be >= 1");
        if (leaf_cap < 1) throw_invalid("build_forest: leaf_cap must be >= 1");
        auto f = std::make_unique<annk_forest>();
        f->n_trees = n_trees;
        f->n = ds->n;
        f->dim = ds->dim;
        f->leaf_cap = leaf_cap;
        f->seed = seed;
        f->trees.resize(n_trees);
        const uint32_t n = ds->n;
        const size_t cap_nodes = 2 * size_t(n);
        DevBuf<uint32_t> rtmp(size_t(n) * n_trees);
        DevBuf<uint64_t> sortbuf(size_t(next_pow2(n)) * n_trees);
        DevBuf<uint32_t> meta(8 * n_trees);
        DevBuf<uint32_t> draws(size_t(n) * n_trees);
        DevBuf<float> col(size_t(n) * n_trees);
        DevBuf<uint32_t> ltmp(size_t(n) * n_trees);
        LAUNCH(draws_kernel, n_trees, 320, 0, seed, ds->dim, n, draws.p);
        std::vector<BuildArgs> args(n_trees);
        for (uint32_t t = 0; t < n_trees; ++t) {
            TreeDev& tr = f->trees[t];
            tr.nodes.alloc(cap_nodes);
            tr.depth.alloc(cap_nodes);
            tr.even.alloc(cap_nodes);
            tr.pidx.alloc(n);
            args[t] = BuildArgs{ds->data.p, n, ds->dim, ds->ld, leaf_cap, substream(seed, t),
                                tr.nodes.p, tr.depth.p, tr.even.p, tr.pidx.p,
                                rtmp.p + size_t(t) * n, sortbuf.p + size_t(t) * next_pow2(n),
                                meta.p + 8 * t, ds->u8 ? ds->data8.p : nullptr, ds->ld8,
                                draws.p + size_t(t) * n, n, col.p + size_t(t) * n, ltmp.p + size_t(t) * n};
        }
        DevBuf<BuildArgs> dargs(n_trees);
        dargs.upload(args.data(), n_trees);
        const size_t smem = sizeof(Smem);
        CK(cudaFuncSetAttribute(forest_build_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        // one thread-block cluster per tree: the largest size (<= 8) at which all
        // trees' clusters are co-resident (each CTA needs a whole SM's shared memory)
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cudaLaunchConfig_t cfg{};
        cfg.blockDim = dim3(kBlock);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = stream();
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        uint32_t csize = 1;
        const char* env = getenv("ANNK_FOREST_CLUSTER");
        for (uint32_t c = kMaxCluster; c > 1; c /= 2) {
            if (env && uint32_t(atoi(env)) < c) continue;
            attr[0].val.clusterDim.x = c;
            cfg.gridDim = dim3(n_trees * c);
            int ncl = 0;
            if (cudaOccupancyMaxActiveClusters(&ncl, forest_build_kernel, &cfg) == cudaSuccess &&
                ncl >= int(n_trees)) {
                csize = c;
                break;
            }
            (void)cudaGetLastError();
        }
        attr[0].val.clusterDim.x = csize;
        cfg.gridDim = dim3(n_trees * csize);
        prof_begin("forest_build_kernel");
        CK(cudaLaunchKernelEx(&cfg, forest_build_kernel, static_cast<const BuildArgs*>(dargs.p)));
        prof_end();
        note_launch();
        std::vector<uint32_t> hm(8 * n_trees);
        meta.download(hm.data(), hm.size());
        ssync();
        for (uint32_t t = 0; t < n_trees; ++t) {
            if (hm[8 * t + 4]) throw Error(kInternal, "build_forest: traversal stack overflow");
            TreeDev& tr = f->trees[t];
            tr.num_nodes = hm[8 * t + 0];
            tr.root = hm[8 * t + 1];
            tr.leaf_count = hm[8 * t + 2];
            tr.max_depth = hm[8 * t + 3];
            if (getenv("ANNK_DEBUG_FOREST"))
                fprintf(stderr, "tree %u: nodes %u, block-path %u kcycles, warp-path %u kcycles\n", t,
                        tr.num_nodes, hm[8 * t + 5], hm[8 * t + 6]);
        }
        forest_upload_views(f.get());
        *out = f.release();
    });
}

int annk_forest_destroy(annk_forest* f) {
    return abi([&] { delete f; });
}

int annk_forest_info(const annk_forest* f, uint32_t* counts, uint64_t* seed) {
    return abi([&] {
        counts[0] = f->n_trees;
        counts[1] = f->n;
        counts[2] = f->dim;
        counts[3] = f->leaf_cap;
        if (seed) *seed = f->seed;
    });
}

int annk_forest_tree_info(const annk_forest* f, uint32_t t, uint32_t* info) {
    return abi([&] {
        if (t >= f->n_trees) throw_range("forest_tree_info: tree index out of range");
        const TreeDev& tr = f->trees[t];
        info[0] = tr.num_nodes;
        info[1] = tr.root;
        info[2] = tr.leaf_count;
        info[3] = tr.max_depth;
    });
}

int annk_forest_export(const annk_forest* f, uint32_t t, uint32_t* split_dim, float* split_val,
                       uint32_t* left, uint32_t* right, uint32_t* depth, uint8_t* even_split,
                       uint32_t* point_index) {
    return abi([&] {
        if (t >= f->n_trees) throw_range("forest_export: tree index out of range");
        const TreeDev& tr = f->trees[t];
        std::vector<KdNodeDev> nodes(tr.num_nodes);
        tr.nodes.download(nodes.data(), tr.num_nodes);
        if (depth) tr.depth.download(depth, tr.num_nodes);
        if (even_split) tr.even.download(even_split, tr.num_nodes);
        if (point_index) tr.pidx.download(point_index, f->n);
        ssync();
        for (uint32_t i = 0; i < tr.num_nodes; ++i) {
            if (split_dim) split_dim[i] = nodes[i].split_dim;
            if (split_val) split_val[i] = nodes[i].split_val;
            if (left) left[i] = nodes[i].left;
            if (right) right[i] = nodes[i].right;
        }
    });
}

int annk_forest_import(uint32_t n, uint32_t dim, uint32_t leaf_cap, uint64_t seed,
                       uint32_t n_trees, const uint32_t* node_counts, const uint32_t* roots,
                       const uint32_t* split_dim, const float* split_val, const uint32_t* left,
                       const uint32_t* right, const uint32_t* depth, const uint8_t* even_split,
                       const uint32_t* point_index, annk_forest** out) {
    return abi([&] {
        if (n < 1 || dim < 1 || n_trees < 1 || leaf_cap < 1) throw_invalid("forest_import: degenerate header");
        auto f = std::make_unique<annk_forest>();
        f->n_trees = n_trees;
        f->n = n;
        f->dim = dim;
        f->leaf_cap = leaf_cap;
        f->seed = seed;
        f->trees.resize(n_trees);
        // node arrays go up as given (one copy each); a kernel packs KdNodeDev
        // records and validates them (kd_forest.cpp:332-372 checks)
        size_t total = 0;
        for (uint32_t t = 0; t < n_trees; ++t) {
            const uint32_t m = node_counts[t];
            if (m == 0 || m > 2 * n) throw_invalid("forest_import: implausible node count");
            if (roots[t] >= m) throw_invalid("forest_import: bad root");
            total += m;
        }
        DevBuf<uint32_t> sd(total), lf(total), rt(total);
        DevBuf<float> sv(total);
        sd.upload(split_dim, total);
        sv.upload(split_val, total);
        lf.upload(left, total);
        rt.upload(right, total);
        DevBuf<uint32_t> stats(size_t(n_trees) * 4);
        stats.zero();
        size_t off = 0;
        for (uint32_t t = 0; t < n_trees; ++t) {
            TreeDev& tr = f->trees[t];
            const uint32_t m = node_counts[t];
            tr.num_nodes = m;
            tr.root = roots[t];
            tr.nodes.alloc(m);
            tr.depth.alloc(m);
            tr.depth.upload(depth + off, m);
            tr.even.alloc(m);
            tr.even.upload(even_split + off, m);
            tr.pidx.alloc(n);
            tr.pidx.upload(point_index + size_t(t) * n, n);
            LAUNCH(import_nodes_kernel, std::min<uint32_t>((m + 255) / 256, 4096), 256, 0, sd.p + off, sv.p + off,
                   lf.p + off, rt.p + off, tr.depth.p, m, n, dim, tr.nodes.p, stats.p + size_t(t) * 4);
            off += m;
        }
        std::vector<uint32_t> st(size_t(n_trees) * 4);
        stats.download(st.data(), st.size());
        ssync();
        for (uint32_t t = 0; t < n_trees; ++t) {
            const uint32_t err = st[size_t(t) * 4 + 2];
            if (err & 1u) throw_invalid("forest_import: bad leaf range");
            if (err & 2u) throw_invalid("forest_import: split dimension out of range");
            if (err & 4u) throw_invalid("forest_import: child id out of range");
            f->trees[t].leaf_count = st[size_t(t) * 4];
            f->trees[t].max_depth = st[size_t(t) * 4 + 1];
        }
        forest_upload_views(f.get());
        *out = f.release();
    });
}

int annk_search_leaves(const annk_forest* f, uint32_t t, const float* queries, uint32_t nq,
                       uint32_t dim, uint32_t n_leaves, uint32_t* out, uint32_t* out_counts) {
    return abi([&] {
        if (t >= f->n_trees) throw_range("search_leaves: tree index out of range");
        if (dim != f->dim) throw_invalid("search_leaves: query length mismatch");
        if (nq == 0) return;
        const TreeDev& tr = f->trees[t];
        const uint32_t ld = (dim + 3) & ~3u;
        std::vector<float> qh(size_t(nq) * ld, 0.0f);
        for (uint32_t i = 0; i < nq; ++i)
            for (uint32_t j = 0; j < dim; ++j) qh[size_t(i) * ld + j] = queries[size_t(i) * dim + j];
        DevBuf<float> dq(qh.size());
        dq.upload(qh.data(), qh.size());
        const uint32_t nl = std::max(n_leaves, 1u);
        const uint32_t heap_cap = (std::min(n_leaves, tr.leaf_count) + 1) * (tr.max_depth + 1) + 1;
        DevBuf<HeapEnt> heaps(size_t(nq) * heap_cap);
        DevBuf<uint32_t> dout(size_t(nq) * nl), dcnt(nq);
        LAUNCH(search_leaves_kernel, (nq + 127) / 128, 128, 0, tr.nodes.p, tr.root, tr.leaf_count, dq.p,
               nq, ld, n_leaves, heaps.p, heap_cap, dout.p, dcnt.p);
        if (n_leaves) dout.download(out, size_t(nq) * n_leaves);
        dcnt.download(out_counts, nq);
        ssync();
    });
}

int annk_descend_from(const annk_forest* f, uint32_t t, const float* queries, uint32_t nq,
                      uint32_t dim, const uint32_t* start, uint32_t* out) {
    return abi([&] {
        if (t >= f->n_trees) throw_range("descend_from: tree index out of range");
        if (dim != f->dim) throw_invalid("descend_from: query length mismatch");
        const TreeDev& tr = f->trees[t];
        for (uint32_t i = 0; i < nq; ++i)
            if (start[i] >= tr.num_nodes) throw_range("descend_from: node id out of range");
        if (nq == 0) return;
        const uint32_t ld = (dim + 3) & ~3u;
        std::vector<float> qh(size_t(nq) * ld, 0.0f);
        for (uint32_t i = 0; i < nq; ++i)
            for (uint32_t j = 0; j < dim; ++j) qh[size_t(i) * ld + j] = queries[size_t(i) * dim + j];
        DevBuf<float> dq(qh.size());
        dq.upload(qh.data(), qh.size());
        DevBuf<uint32_t> ds(nq), dout(nq);
        ds.upload(start, nq);
        LAUNCH(descend_kernel, (nq + 127) / 128, 128, 0, tr.nodes.p, dq.p, nq, ld, ds.p, dout.p);
        dout.download(out, nq);
        ssync();
    });
}

}  // extern "C"
