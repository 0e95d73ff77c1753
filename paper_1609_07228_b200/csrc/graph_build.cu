// graph_build.cu — divide-and-conquer init + NN-descent on B200.
//
// Reference: proj/src/graph_build.cpp (init_graph :230-292, rebuild_sample_lists
// :59-86, union_reverse_lists + sample_down :38-53,88-103, nn_descent_iteration
// :105-162, finalize :346-373, pool_topk_accuracy :209-226).
//
// Pools are rows of P 64-bit keys (dist_bits << 32 | id) kept sorted, plus a
// flag_new byte per slot.  The reference's NeighborPool insert keeps the top P
// of everything offered, rejecting duplicates (neighbor_pool.hpp:35-53), and
// an entry evicted within a round can never come back (the tail only
// shrinks).  So the pool after a join round is exactly
//       top-P by key of (start pool  U  all offers),
// independent of the order offers arrive.  The GPU join therefore never
// touches the pools: it appends every offer that beats the target's
// start-of-round tail to a per-target buffer, and a merge kernel forms the
// new pools.  Flags follow the reference: an entry already present keeps its
// flag, an entry that arrived this round is new.
//
// The one order-dependent reference quantity is `changes` (accepted inserts,
// counting ones later evicted).  This library reports the order-independent
// count of entries inserted this round that survive in the pools.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <climits>
#include <numeric>
#include <string>
#include <vector>

#include "../../include/annkit_b200.h"
#include "internal.cuh"
#include "join.cuh"

namespace annk {
namespace {

constexpr uint32_t kInitWarps = 4;
constexpr uint32_t kInitCap = 1024;  // fast-path candidate capacity per point
constexpr uint32_t kStageCols = 64;  // fp32 init: floats per staged candidate-row chunk

// ---------------------------------------------------------------- helpers

// Sort + unique n u32 values in smem s (capacity m = pow2 >= n) by one warp.
// Returns the unique count (values compacted to the front).
__device__ uint32_t warp_sort_unique_u32(uint32_t* s, uint32_t n, uint32_t m) {
    const uint32_t lane = lane_id();
    for (uint32_t j = n + lane; j < m; j += 32) s[j] = 0xffffffffu;
    __syncwarp();
    warp_bitonic_sort_u32(s, m);
    uint32_t out = 0;
    for (uint32_t base = 0; base < n; base += 32) {
        const uint32_t j = base + lane;
        const uint32_t v = j < n ? s[j] : 0;
        const bool keep = j < n && (j == 0 || s[j - 1] != v);
        const uint32_t b = __ballot_sync(0xffffffffu, keep);
        __syncwarp();
        if (keep) s[out + __popc(b & ((1u << lane) - 1u))] = v;
        out += __popc(b);
        __syncwarp();
    }
    return out;
}

// Sorted unique ids of s[0..n) (n <= 32 V) written to out; returns the count.
// Register sort + one ballot compaction per register row (no shared-memory passes).
template <int V>
__device__ uint32_t warp_unique_regs_u32(const uint32_t* s, uint32_t n, uint32_t* __restrict__ out) {
    const uint32_t lane = lane_id(), lt = (1u << lane) - 1u;
    uint32_t v[V];
#pragma unroll
    for (int r = 0; r < V; ++r) {
        const uint32_t e = uint32_t(r) * 32 + lane;
        v[r] = e < n ? s[e] : 0xffffffffu;
    }
    warp_sort_regs_u32<V>(v);
    uint32_t cnt = 0;
#pragma unroll
    for (int r = 0; r < V; ++r) {
        uint32_t prev = __shfl_up_sync(0xffffffffu, v[r], 1);
        const uint32_t tail = r > 0 ? __shfl_sync(0xffffffffu, v[r > 0 ? r - 1 : 0], 31) : 0u;
        if (lane == 0) prev = tail;
        const uint32_t e = uint32_t(r) * 32 + lane;
        const bool keep = e < n && (e == 0 || prev != v[r]);
        const uint32_t b = __ballot_sync(0xffffffffu, keep);
        if (keep) out[cnt + __popc(b & lt)] = v[r];
        cnt += __popc(b);
    }
    return cnt;
}

// ----------------------------------------------------------------- init

struct InitArgs {
    const float* x;
    uint32_t n, ld, n_trees, conquer_depth, P;
    const TreeView* trees;
    uint64_t* keys;
    uint8_t* flags;
    uint32_t* sizes;
    unsigned long long* comps;
    uint32_t* overflow;  // [count, ids...]
    const uint8_t* x8;   // exact u8 rows (nullptr: fp32 path)
    uint32_t ld8;
    const int32_t* norms8;
};

// Warp-level scratch for one point's candidate set.
//   table : open-addressing hash set of ids (2*cap u32 slots, EMPTY = ~0u),
//           later reused as the u64 key array (cap keys)
//   uniq  : unique candidate ids in insertion order (cap)
struct InitScratch {
    uint32_t* table;
    uint32_t* uniq;
    uint32_t cap;     // unique-candidate capacity (pow2)
    uint32_t tslots;  // hash slots (pow2, >= cap)
    uint32_t* sib;
    uint32_t sib_cap;
    uint32_t* cnt;  // [0] unique count, [1] sibling count, [2] overflow flag
    const uint8_t* pf_base;  // rows to prefetch into L2 on first insert (nullptr: none)
    uint32_t pf_ld;
    float* stage;  // fp32 path: 32 candidate rows x kStageCols (+4 pad) staging (nullptr: per-lane loads)
};

__device__ __forceinline__ void hs_insert(const InitScratch& w, uint32_t id) {
    const uint32_t mask = w.tslots - 1;
    uint32_t h = (id * 2654435761u) & mask;
    for (uint32_t probe = 0; probe <= mask; ++probe) {
        const uint32_t old = atomicCAS(&w.table[h], 0xffffffffu, id);
        if (old == 0xffffffffu) {
            const uint32_t u = atomicAdd(&w.cnt[0], 1u);
            if (u < w.cap) w.uniq[u] = id;
            else w.cnt[2] = 1;
            // the candidate's row is gathered after collection: start it on its way to L2
            if (w.pf_base) asm volatile("prefetch.global.L2 [%0];" ::"l"(w.pf_base + size_t(id) * w.pf_ld));
            return;
        }
        if (old == id) return;
        h = (h + 1) & mask;
    }
    w.cnt[2] = 1;
}

// Point i's candidate set (graph_build.cpp:266-281): own leaf per tree plus one
// descended leaf per ancestor level >= conquer_depth, deduplicated in a shared
// hash set (self excluded, as the reference skips c == i at :283).  The
// ancestor siblings come from the forest's per-leaf sibling lists, flattened
// over the trees of a 32-tree group so every lane takes independent
// (tree, level) entries; each lane walks kDesc descents interleaved so their
// dependent node loads overlap.
constexpr uint32_t kDesc = 4;
__device__ void init_collect(const InitArgs& a, uint32_t i, const float* q, const InitScratch& w) {
    const uint32_t lane = lane_id();
    const uint8_t* q8 = a.x8 ? a.x8 + size_t(i) * a.ld8 : nullptr;  // used when q is null (u8 path)
    // table <- EMPTY (vectorised)
    uint4* t4 = reinterpret_cast<uint4*>(w.table);
    for (uint32_t j = lane; j < w.tslots / 4; j += 32) t4[j] = make_uint4(~0u, ~0u, ~0u, ~0u);
    if (lane == 0) { w.cnt[0] = 0; w.cnt[1] = 0; w.cnt[2] = 0; }
    __syncwarp();
    for (uint32_t g = 0; g < a.n_trees; g += 32) {
        const uint32_t t = g + lane;
        uint32_t nsib = 0, soff = 0;
        if (t < a.n_trees) {
            const TreeView& tv = a.trees[t];
            const uint32_t leaf = tv.owner[i];
            const KdNodeDev ln = tv.nodes[leaf];
            const uint32_t dl = tv.depth[leaf];
            nsib = dl > a.conquer_depth ? dl - a.conquer_depth : 0u;
            soff = tv.sib_off[leaf];
            for (uint32_t p = ln.left; p < ln.right; ++p) {
                const uint32_t id = tv.pidx[p];
                if (id != i) hs_insert(w, id);
            }
        }
        uint32_t incl = nsib;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= uint32_t(o)) incl += y;
        }
        const uint32_t excl = incl - nsib;
        const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
        for (uint32_t k0 = 0; k0 < total; k0 += 32 * kDesc) {
            uint32_t nd[kDesc];
            const KdNodeDev* nodes[kDesc];
            const uint32_t* pidx[kDesc];
            bool act[kDesc];
#pragma unroll
            for (uint32_t r = 0; r < kDesc; ++r) {
                const uint32_t k = k0 + r * 32 + lane;
                // owner lane of entry k: the last lane whose exclusive prefix is <= k
                uint32_t lo = 0;
#pragma unroll
                for (uint32_t st = 16; st > 0; st >>= 1) {
                    const uint32_t ex = __shfl_sync(0xffffffffu, excl, lo + st);
                    if (ex <= k) lo += st;
                }
                const uint32_t ex_lo = __shfl_sync(0xffffffffu, excl, lo);
                const uint32_t off_lo = __shfl_sync(0xffffffffu, soff, lo);
                act[r] = k < total;
                nd[r] = 0;
                nodes[r] = nullptr;
                pidx[r] = nullptr;
                if (act[r]) {
                    const TreeView& tv = a.trees[g + lo];
                    nodes[r] = tv.nodes;
                    pidx[r] = tv.pidx;
                    nd[r] = tv.sib_list[off_lo + (k - ex_lo)];
                }
            }
            // descend_from(sibling, x_i), kDesc walks interleaved
            KdNodeDev cur[kDesc];
#pragma unroll
            for (uint32_t r = 0; r < kDesc; ++r)
                if (act[r]) cur[r] = nodes[r][nd[r]];
            for (;;) {
                bool more = false;
#pragma unroll
                for (uint32_t r = 0; r < kDesc; ++r) {
                    if (act[r] && cur[r].split_dim != kLeaf) {
                        const float qd = q ? q[cur[r].split_dim] : float(__ldg(q8 + cur[r].split_dim));
                        nd[r] = qd <= cur[r].split_val ? cur[r].left : cur[r].right;
                        more = true;
                    }
                }
                if (!more) break;
#pragma unroll
                for (uint32_t r = 0; r < kDesc; ++r)
                    if (act[r] && cur[r].split_dim != kLeaf) cur[r] = nodes[r][nd[r]];
            }
#pragma unroll
            for (uint32_t r = 0; r < kDesc; ++r) {
                if (!act[r]) continue;
                for (uint32_t p = cur[r].left; p < cur[r].right; ++p) {
                    const uint32_t id = pidx[r][p];
                    if (id != i) hs_insert(w, id);
                }
            }
        }
    }
    __syncwarp();
}

// P-th smallest distance (as fp32 bits) among keys[0..nk), nk >= P, by a
// 4-pass MSB radix select over 256-bin warp histograms.
__device__ uint32_t warp_select_dist(const uint64_t* keys, uint32_t nk, uint32_t P, uint32_t* hist) {
    const uint32_t lane = lane_id();
    uint32_t prefix = 0, pmask = 0, r = P;
    for (int shift = 24; shift >= 0; shift -= 8) {
        for (uint32_t b = lane; b < 256; b += 32) hist[b] = 0;
        __syncwarp();
        for (uint32_t j = lane; j < nk; j += 32) {
            const uint32_t d = uint32_t(keys[j] >> 32);
            if ((d & pmask) == prefix) atomicAdd(&hist[(d >> shift) & 255u], 1u);
        }
        __syncwarp();
        uint32_t local = 0;
        for (uint32_t b = 0; b < 8; ++b) local += hist[lane * 8 + b];
        uint32_t incl = local;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= uint32_t(o)) incl += v;
        }
        const uint32_t excl = incl - local;
        const uint32_t owner = __ffs(__ballot_sync(0xffffffffu, incl >= r)) - 1;
        uint32_t bin = 0, before = 0;
        if (lane == owner) {
            uint32_t acc = excl;
            for (uint32_t b = 0; b < 8; ++b) {
                const uint32_t h = hist[lane * 8 + b];
                if (acc + h >= r) { bin = lane * 8 + b; before = acc; break; }
                acc += h;
            }
        }
        bin = __shfl_sync(0xffffffffu, bin, owner);
        before = __shfl_sync(0xffffffffu, before, owner);
        prefix |= bin << shift;
        pmask |= 255u << shift;
        r -= before;
        __syncwarp();
    }
    return prefix;
}

// The pool from point i's u unique candidate keys (warp scratch): exact top-P by
// (dist, id), all flagged new (graph_build.cpp:282-288).
__device__ void init_select(const InitArgs& a, uint32_t i, uint64_t* keys, uint32_t u, uint32_t* hist) {
    const uint32_t lane = lane_id();
    uint32_t take = min(u, a.P);
    uint64_t* surv = keys;
    uint32_t ns = u;
    if (u > a.P) {
        // keep keys whose distance <= the P-th smallest distance (ties included)
        const uint32_t T = warp_select_dist(keys, u, a.P, hist);
        ns = 0;
        for (uint32_t base = 0; base < u; base += 32) {
            const uint32_t j = base + lane;
            const uint64_t v = j < u ? keys[j] : kEmptyKey;
            const bool keep = j < u && uint32_t(v >> 32) <= T;
            const uint32_t b = __ballot_sync(0xffffffffu, keep);
            __syncwarp();
            if (keep) surv[ns + __popc(b & ((1u << lane) - 1u))] = v;  // in place: target <= j
            ns += __popc(b);
            __syncwarp();
        }
    }
    uint64_t* pk = a.keys + size_t(i) * a.P;
    uint8_t* pf = a.flags + size_t(i) * a.P;
    __syncwarp();
    if (ns <= 128) {
        // the survivors (about P) are sorted in registers and written straight to the pool
        uint64_t v[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const uint32_t e = uint32_t(r) * 32 + lane;
            v[r] = e < ns ? surv[e] : kEmptyKey;
        }
        warp_sort_regs<4>(v);
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const uint32_t e = uint32_t(r) * 32 + lane;
            if (e < a.P) {
                pk[e] = e < take ? v[r] : kEmptyKey;
                pf[e] = e < take ? 1 : 0;
            }
        }
        for (uint32_t j = 128 + lane; j < a.P; j += 32) {
            pk[j] = kEmptyKey;
            pf[j] = 0;
        }
    } else {
        const uint32_t m = next_pow2(max(ns, 1u));
        for (uint32_t j = ns + lane; j < m; j += 32) surv[j] = kEmptyKey;
        __syncwarp();
        warp_bitonic_sort(surv, m);
        for (uint32_t j = lane; j < a.P; j += 32) {
            pk[j] = j < take ? surv[j] : kEmptyKey;
            pf[j] = j < take ? 1 : 0;
        }
    }
    if (lane == 0) {
        a.sizes[i] = take;
        atomicAdd(a.comps, (unsigned long long)u);
    }
    __syncwarp();
}

// Distances, then the pool: exact top-P by (dist, id) of the unique candidates.
__device__ void init_finish(const InitArgs& a, uint32_t i, const float* q, const InitScratch& w, uint32_t* hist) {
    const uint32_t lane = lane_id();
    const uint32_t u = w.cnt[0];
    uint64_t* keys = reinterpret_cast<uint64_t*>(w.table);  // table no longer needed
    __syncwarp();
    if (a.x8) {
        // 8 lanes per candidate row (one coalesced 128-byte segment per step),
        // 4 rows per warp step, kRows steps in flight; dot reduced by shuffles
        constexpr uint32_t kRows = 8;
        const uint32_t sub = lane & 7, grp = lane >> 3;
        const uint8_t* xi = a.x8 + size_t(i) * a.ld8;
        const int32_t ni = a.norms8[i];
        const uint32_t nch = (a.ld8 + 127) / 128;
        uint4 qv0 = make_uint4(0, 0, 0, 0);
        if (sub * 16 < a.ld8) qv0 = *reinterpret_cast<const uint4*>(xi + sub * 16);
        for (uint32_t j0 = 0; j0 < u; j0 += 4 * kRows) {
            uint32_t id[kRows], dot[kRows];
            int32_t nb[kRows];
#pragma unroll
            for (uint32_t r = 0; r < kRows; ++r) {
                const uint32_t j = j0 + r * 4 + grp;
                id[r] = j < u ? w.uniq[j] : i;
                dot[r] = 0;
                nb[r] = sub == 0 ? a.norms8[id[r]] : 0;
            }
            for (uint32_t c = 0; c < nch; ++c) {
                const uint32_t off = (c * 8 + sub) * 16;
                if (off < a.ld8) {
                    const uint4 qv = c == 0 ? qv0 : *reinterpret_cast<const uint4*>(xi + off);
                    uint4 rv[kRows];
#pragma unroll
                    for (uint32_t r = 0; r < kRows; ++r)
                        rv[r] = *reinterpret_cast<const uint4*>(a.x8 + size_t(id[r]) * a.ld8 + off);
#pragma unroll
                    for (uint32_t r = 0; r < kRows; ++r) {
                        dot[r] = __dp4a(qv.x, rv[r].x, dot[r]);
                        dot[r] = __dp4a(qv.y, rv[r].y, dot[r]);
                        dot[r] = __dp4a(qv.z, rv[r].z, dot[r]);
                        dot[r] = __dp4a(qv.w, rv[r].w, dot[r]);
                    }
                }
            }
#pragma unroll
            for (uint32_t r = 0; r < kRows; ++r) {
                dot[r] += __shfl_xor_sync(0xffffffffu, dot[r], 1);
                dot[r] += __shfl_xor_sync(0xffffffffu, dot[r], 2);
                dot[r] += __shfl_xor_sync(0xffffffffu, dot[r], 4);
                const uint32_t j = j0 + r * 4 + grp;
                if (sub == 0 && j < u) keys[j] = make_key(float(ni + nb[r] - 2 * int32_t(dot[r])), id[r]);
            }
        }
    } else {
        if (w.stage) {
            // wide fp32 rows: 32 candidates at a time; their rows pass through shared
            // memory in kStageCols-float chunks loaded coalesced (each load instruction
            // covers 128-byte runs of a few rows instead of 16 bytes of 32 rows), then
            // every lane runs its own candidate's exact sequential chain from there
            constexpr uint32_t SW = kStageCols + 4;  // padded row stride: conflict-free 16-byte reads
            constexpr uint32_t F4 = kStageCols / 4;  // float4 per staged row chunk
            constexpr uint32_t RPI = 32 / F4;        // rows per load instruction
            float* stg = w.stage;
            for (uint32_t j0 = 0; j0 < u; j0 += 32) {
                const uint32_t j = j0 + lane;
                const uint32_t myid = w.uniq[j < u ? j : j0];
                float acc = 0.0f;
                for (uint32_t c0 = 0; c0 < a.ld; c0 += kStageCols) {
                    const uint32_t nc = min(kStageCols, a.ld - c0);  // multiple of 4
#pragma unroll
                    for (uint32_t r0 = 0; r0 < 32; r0 += RPI) {
                        const uint32_t r = r0 + lane / F4, f = lane % F4;
                        const uint32_t rid = __shfl_sync(0xffffffffu, myid, r);
                        if (f * 4 < nc)
                            *reinterpret_cast<float4*>(stg + r * SW + f * 4) =
                                __ldg(reinterpret_cast<const float4*>(a.x + size_t(rid) * a.ld + c0) + f);
                    }
                    __syncwarp();
                    const float* mine = stg + lane * SW;
                    for (uint32_t e = 0; e < nc; e += 4) {
                        const float4 xv = *reinterpret_cast<const float4*>(q + c0 + e);
                        const float4 yv = *reinterpret_cast<const float4*>(mine + e);
                        float d;
                        d = __fsub_rn(xv.x, yv.x); acc = __fadd_rn(acc, __fmul_rn(d, d));
                        d = __fsub_rn(xv.y, yv.y); acc = __fadd_rn(acc, __fmul_rn(d, d));
                        d = __fsub_rn(xv.z, yv.z); acc = __fadd_rn(acc, __fmul_rn(d, d));
                        d = __fsub_rn(xv.w, yv.w); acc = __fadd_rn(acc, __fmul_rn(d, d));
                    }
                    __syncwarp();
                }
                if (j < u) keys[j] = make_key(acc, myid);
            }
        } else {
            for (uint32_t j = lane; j < u; j += 32) {
                const uint32_t id = w.uniq[j];
                keys[j] = make_key(l2_exact_ldg8(q, a.x + size_t(id) * a.ld, a.ld), id);
            }
        }
    }
    __syncwarp();
    init_select(a, i, keys, u, hist);
}

__host__ __device__ __forceinline__ size_t init_warp_bytes(uint32_t cap, uint32_t ld, uint32_t sib_cap) {
    // table (cap u32) + uniq (cap u32) == cap u64 keys, q row, sib (2*sib_cap), hist (256), cnt (4),
    // fp32 path: candidate-row staging (32 rows x (kStageCols + 4) floats)
    return (size_t(cap) * 8 + size_t(ld) * 4 + size_t(sib_cap) * 8 + 256 * 4 + 16 +
            (ld ? size_t(32) * (kStageCols + 4) * 4 : 0) + 15) & ~size_t(15);
}

// u8 datapath: 5 CTAs per SM — 96 registers (no spills) lift residency from 16
// to 20 warps, which the shared-memory scratch also allows (measured: 34.9 ->
// 31.8 ms at cfg2; 6 CTAs force spills and run slower, 45.8 ms).  The fp32
// path's staging scratch limits residency anyway and the cap slows it (cfg3
// init 0.56 -> 0.70 s), so it is instantiated without one.
template <int kMinBlocks>
__global__ void __launch_bounds__(kInitWarps * 32, kMinBlocks) init_kernel_t(InitArgs a, uint32_t sib_cap,
                                                               const uint32_t* __restrict__ order,
                                                               uint32_t n_visit) {
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t warp = threadIdx.x / 32, lane = lane_id();
    // the u8 path reads the point's exact u8 row (L1) for the descents: no fp32 copy in smem
    const uint32_t q_ld = a.x8 ? 0u : a.ld;
    unsigned char* base = smem + warp * init_warp_bytes(kInitCap, q_ld, sib_cap);
    InitScratch w;
    w.table = reinterpret_cast<uint32_t*>(base);
    // one 8 KB region: hash slots [0, 4 KB) + unique list [4 KB, 8 KB); the
    // u64 keys then overwrite it in place (key j covers unique entries
    // 2j-1024 and 2j-1023, already consumed when keys are written in order)
    w.tslots = kInitCap;
    w.uniq = w.table + kInitCap;
    w.cap = kInitCap;
    w.pf_base = a.x8;
    w.pf_ld = a.ld8;
    float* qbase = reinterpret_cast<float*>(w.uniq + kInitCap);
    float* q = q_ld ? qbase : nullptr;
    w.sib = reinterpret_cast<uint32_t*>(qbase + q_ld);
    w.sib_cap = sib_cap;
    uint32_t* hist = w.sib + 2 * sib_cap;
    w.cnt = hist + 256;
    w.stage = q_ld ? reinterpret_cast<float*>(w.cnt + 4) : nullptr;
    for (uint32_t ord = blockIdx.x * kInitWarps + warp; ord < n_visit; ord += gridDim.x * kInitWarps) {
        // visit points in tree-0 leaf order: concurrently processed points share
        // most candidate rows, so the gathers hit L2
        const uint32_t i = order ? order[ord] : ord;
        for (uint32_t j = lane; j < q_ld; j += 32) q[j] = a.x[size_t(i) * a.ld + j];
        __syncwarp();
        init_collect(a, i, q, w);
        if (w.cnt[2]) {  // more unique candidates than the fast path holds
            if (lane == 0) {
                const uint32_t o = atomicAdd(&a.overflow[0], 1u);
                a.overflow[1 + o] = i;
            }
            __syncwarp();
            continue;
        }
        init_finish(a, i, q, w, hist);
    }
}

// Overflow path: one warp per point, scratch in global memory sized for the
// forest's worst case (trees * (max_depth+1) * leaf_cap candidates).
__global__ void init_overflow_kernel(InitArgs a, const uint32_t* list, uint32_t count, uint32_t cap,
                                     uint32_t sib_cap, uint32_t* gscratch, float* gq) {
    __shared__ uint32_t s_misc[256 + 4];
    const uint32_t lane = lane_id();
    for (uint32_t r = blockIdx.x; r < count; r += gridDim.x) {
        const uint32_t i = list[r];
        InitScratch w;
        w.table = gscratch + size_t(blockIdx.x) * (3 * size_t(cap) + 2 * sib_cap);
        w.uniq = w.table + 2 * cap;
        w.cap = cap;
        w.tslots = 2 * cap;
        w.pf_base = nullptr;
        w.pf_ld = 0;
        w.stage = nullptr;
        w.sib = w.uniq + cap;
        w.sib_cap = sib_cap;
        w.cnt = s_misc + 256;
        float* q = gq + size_t(blockIdx.x) * a.ld;
        for (uint32_t j = lane; j < a.ld; j += 32) q[j] = a.x[size_t(i) * a.ld + j];
        __syncwarp();
        init_collect(a, i, q, w);
        init_finish(a, i, q, w, s_misc);
    }
}

// graph_build.cpp:294-326 init_random.  One warp per point i: if P >= n-1 the
// pool is every other point; otherwise draws j = rng() % n from
// mt19937_64(substream(seed, i)), skipping i and repeats, until P distinct ids
// are taken (draw order decides, as in the reference's loop).  The MT state
// (312 words) lives in the warp's shared memory: lane 0 expands the seed, the
// warp twists in 3 phases, lanes consume 32 outputs at a time; a repeat within
// a batch is resolved by __match_any_sync (first lane wins).  The taken ids'
// distances are sorted by (dist, id) into the pool, all flagged new.
__host__ __device__ __forceinline__ size_t init_random_warp_bytes(uint32_t P) {
    // mt[312] + keys[next_pow2(P)] + hash slots (4 * P, pow2) u32
    uint32_t m = 1;
    while (m < P) m <<= 1;
    uint32_t hs = 1;
    while (hs < 4 * P) hs <<= 1;
    return (size_t(312) * 8 + size_t(m) * 8 + size_t(hs) * 4 + 15) & ~size_t(15);
}

__global__ void init_random_kernel(InitArgs a, uint64_t seed) {
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t warp = threadIdx.x / 32, lane = lane_id();
    const uint32_t wpb = blockDim.x / 32;
    const uint32_t P = a.P, n = a.n;
    uint32_t m = 1;
    while (m < P) m <<= 1;
    uint32_t hs = 1;
    while (hs < 4 * P) hs <<= 1;
    unsigned char* base = smem + size_t(warp) * init_random_warp_bytes(P);
    uint64_t* mt = reinterpret_cast<uint64_t*>(base);
    uint64_t* keys = mt + 312;
    uint32_t* hset = reinterpret_cast<uint32_t*>(keys + m);
    for (uint32_t i = blockIdx.x * wpb + warp; i < n; i += gridDim.x * wpb) {
        const uint32_t want = min(P, n - 1);
        const uint8_t* x8i = a.x8 ? a.x8 + size_t(i) * a.ld8 : nullptr;
        const float* xi = a.x + size_t(i) * a.ld;
        auto dist = [&](uint32_t j) -> float {
            return a.x8 ? l2_u8(x8i, a.x8 + size_t(j) * a.ld8, a.ld8, a.norms8[i], a.norms8[j])
                        : l2_exact_ldg(xi, a.x + size_t(j) * a.ld, a.ld);
        };
        uint32_t have = 0;
        if (want == n - 1) {
            for (uint32_t j = lane; j < n; j += 32)
                if (j != i) keys[j < i ? j : j - 1] = make_key(dist(j), j);
            have = n - 1;
        } else {
            for (uint32_t t = lane; t < hs; t += 32) hset[t] = 0xffffffffu;
            if (lane == 0) {
                uint64_t x = substream(seed, i);
                mt[0] = x;
                for (uint32_t t = 1; t < 312; ++t) {
                    x = 6364136223846793005ULL * (x ^ (x >> 62)) + uint64_t(t);
                    mt[t] = x;
                }
            }
            __syncwarp();
            while (have < want) {
                // regenerate 312 words (3 phases: [0,156), [156,311), 311)
                // (uniform trip counts: every lane reaches every __syncwarp)
                for (uint32_t t0 = 0; t0 < 156; t0 += 32) {
                    const uint32_t t = t0 + lane;
                    const uint64_t v = t < 156 ? mt_twist(mt[t], mt[t + 1], mt[t + 156]) : 0ull;
                    __syncwarp();
                    if (t < 156) mt[t] = v;
                }
                __syncwarp();
                for (uint32_t t0 = 156; t0 < 311; t0 += 32) {
                    const uint32_t t = t0 + lane;
                    const uint64_t v = t < 311 ? mt_twist(mt[t], mt[t + 1], mt[t - 156]) : 0ull;
                    __syncwarp();
                    if (t < 311) mt[t] = v;
                }
                __syncwarp();
                if (lane == 0) mt[311] = mt_twist(mt[311], mt[0], mt[155]);
                __syncwarp();
                for (uint32_t b0 = 0; b0 < 312 && have < want; b0 += 32) {
                    const uint32_t t = b0 + lane;
                    const bool ok = t < 312;
                    const uint32_t j = ok ? uint32_t(mt_temper(mt[t]) % uint64_t(n)) : i;
                    // seen before this batch?
                    bool cand = ok && j != i;
                    if (cand) {
                        uint32_t h = (j * 2654435761u) & (hs - 1);
                        for (;;) {
                            const uint32_t e = hset[h];
                            if (e == 0xffffffffu) break;
                            if (e == j) { cand = false; break; }
                            h = (h + 1) & (hs - 1);
                        }
                    }
                    // repeats inside the batch: the lowest lane keeps it
                    const uint32_t same = __match_any_sync(0xffffffffu, cand ? j : 0xffffffffu);
                    cand = cand && (__ffs(same) - 1) == int(lane);
                    const uint32_t bal = __ballot_sync(0xffffffffu, cand);
                    const uint32_t rank = __popc(bal & ((1u << lane) - 1u));
                    cand = cand && have + rank < want;
                    if (cand) {
                        uint32_t h = (j * 2654435761u) & (hs - 1);
                        while (atomicCAS(&hset[h], 0xffffffffu, j) != 0xffffffffu) h = (h + 1) & (hs - 1);
                        keys[have + rank] = uint64_t(j);  // id for now; distance below
                    }
                    have = min(want, have + __popc(bal));
                    __syncwarp();
                }
            }
            for (uint32_t t = lane; t < have; t += 32) {
                const uint32_t j = uint32_t(keys[t]);
                keys[t] = make_key(dist(j), j);
            }
        }
        for (uint32_t t = have + lane; t < m; t += 32) keys[t] = kEmptyKey;
        __syncwarp();
        warp_bitonic_sort(keys, m);
        uint64_t* pk = a.keys + size_t(i) * P;
        uint8_t* pf = a.flags + size_t(i) * P;
        for (uint32_t t = lane; t < P; t += 32) {
            pk[t] = t < have ? keys[t] : kEmptyKey;
            pf[t] = t < have ? 1 : 0;
        }
        if (lane == 0) {
            a.sizes[i] = have;
            atomicAdd(a.comps, (unsigned long long)have);
        }
        __syncwarp();
    }
}

// -------------------------------------------------------------- sampling

struct SampleArgs {
    uint32_t n, P, S;
    const uint64_t* keys;
    uint8_t* flags;
    const uint32_t* sizes;
    uint32_t* fnew;  // n x S
    uint32_t* fold;  // n x P
    uint32_t* cnew;
    uint32_t* cold;
    uint64_t* thr;
    uint32_t lo;  // points [lo, n) are sampled
    uint32_t* rn_cnt;  // reverse-list sizes counted on the way (null: rev_count_kernel does it,
    uint32_t* ro_cnt;  // shard mode, where the other ranks' forward rows arrive later)
};

// graph_build.cpp:71-85: ascending scan until S new entries are taken.
__global__ void sample_kernel(SampleArgs a) {
    const uint32_t lane = lane_id();
    const uint32_t i = a.lo + (blockIdx.x * blockDim.x + threadIdx.x) / 32;
    if (i >= a.n) return;
    const uint32_t sz = a.sizes[i];
    const uint64_t* pk = a.keys + size_t(i) * a.P;
    uint8_t* pf = a.flags + size_t(i) * a.P;
    uint32_t taken = 0, nold = 0;
    for (uint32_t base = 0; base < sz && taken < a.S; base += 32) {
        const uint32_t j = base + lane;
        const bool valid = j < sz;
        const bool isnew = valid && (pf[j] & 1);
        const uint32_t bn = __ballot_sync(0xffffffffu, isnew);
        // entries are scanned while fewer than S news have been taken
        const uint32_t lt = (1u << lane) - 1u;
        const uint32_t rank_new = taken + __popc(bn & lt);  // news before me
        const bool in_scan = valid && rank_new < a.S;
        const uint32_t id = valid ? key_id(pk[j]) : 0;
        const uint32_t bo = __ballot_sync(0xffffffffu, in_scan && !isnew);
        if (in_scan && isnew) {
            a.fnew[size_t(i) * a.S + rank_new] = id;
            pf[j] &= uint8_t(~1u);  // flag_new cleared; `checked` (bit 1) untouched
            if (a.rn_cnt) atomicAdd(&a.rn_cnt[id], 1u);
        } else if (in_scan) {
            a.fold[size_t(i) * a.P + nold + __popc(bo & lt)] = id;
            if (a.ro_cnt) atomicAdd(&a.ro_cnt[id], 1u);
        }
        taken = min(a.S, taken + __popc(bn));
        nold += __popc(bo);
    }
    if (lane == 0) {
        a.cnew[i] = taken;
        a.cold[i] = nold;
        a.thr[i] = sz == a.P ? pk[a.P - 1] : kEmptyKey;
    }
}

// Reverse-list sizes from the forward lists of all points.
// Only targets in [tlo, thi) are counted (shard mode: the owned points).
__global__ void rev_count_kernel(uint32_t n, uint32_t width, const uint32_t* __restrict__ fwd,
                                 const uint32_t* __restrict__ cnt, uint32_t* __restrict__ out, uint32_t tlo,
                                 uint32_t thi) {
    const uint32_t lane = lane_id();
    const uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) / 32;
    if (i >= n) return;
    const uint32_t c = cnt[i];
    for (uint32_t j = lane; j < c; j += 32) {
        const uint32_t id = fwd[size_t(i) * width + j];
        if (id >= tlo && id < thi) atomicAdd(&out[id], 1u);
    }
}

__global__ void reverse_scatter_kernel(uint32_t n, uint32_t width, const uint32_t* __restrict__ fwd,
                                       const uint32_t* __restrict__ cnt, const uint32_t* __restrict__ off,
                                       uint32_t* __restrict__ cursor, uint32_t* __restrict__ data, uint32_t tlo,
                                       uint32_t thi) {
    const uint32_t lane = lane_id();
    const uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) / 32;
    if (i >= n) return;
    const uint32_t c = cnt[i];
    for (uint32_t j = lane; j < c; j += 32) {
        const uint32_t id = fwd[size_t(i) * width + j];
        if (id < tlo || id >= thi) continue;
        const uint32_t pos = atomicAdd(&cursor[id], 1u);
        data[off[id] + pos] = i;
    }
}

// Reverse lists as ascending sets (the reference pushes them in ascending owner
// order, graph_build.cpp:71-85): the scatter above leaves each list in arrival
// order, one warp sorts it in registers (bitonic network over 1/2/4/8 ids per
// lane) up to 256 ids.  Longer lists go on a work list: rev_sort_long_kernel
// sorts those up to kRevSortSmem ids in shared memory, one 256-thread CTA per
// list; a list beyond that (a hub with more than 8192 reverse neighbours) is
// counted in big[0] and the host falls back to the library segmented sort.
constexpr uint32_t kRevSortSmem = 8192, kRevSortWarps = 8, kRevLongThreads = 256;
template <int V>
__device__ __forceinline__ void rev_sort_regs(uint32_t* __restrict__ p, uint32_t len) {
    const uint32_t lane = lane_id();
    uint32_t v[V];
#pragma unroll
    for (int r = 0; r < V; ++r) {
        const uint32_t j = r * 32 + lane;
        v[r] = j < len ? p[j] : 0xffffffffu;
    }
    warp_sort_regs_u32<V>(v);
#pragma unroll
    for (int r = 0; r < V; ++r) {
        const uint32_t j = r * 32 + lane;
        if (j < len) p[j] = v[r];
    }
}
// big: [0] lists the device cannot sort, [1] work-list length; wl: list ids (one slot per list)
__global__ void __launch_bounds__(kRevSortWarps * 32) rev_sort_kernel(const uint32_t* __restrict__ off,
                                                                      uint32_t* __restrict__ data, uint32_t lo,
                                                                      uint32_t hi, uint32_t* __restrict__ big,
                                                                      uint32_t* __restrict__ wl) {
    const uint32_t lane = lane_id(), warp = threadIdx.x / 32;
    const uint32_t i = lo + blockIdx.x * kRevSortWarps + warp;
    if (i >= hi) return;
    const uint32_t b = off[i], len = off[i + 1] - b;
    if (len <= 1) return;
    uint32_t* p = data + b;
    if (len <= 32) rev_sort_regs<1>(p, len);
    else if (len <= 64) rev_sort_regs<2>(p, len);
    else if (len <= 128) rev_sort_regs<4>(p, len);
    else if (len <= 256) rev_sort_regs<8>(p, len);
    else if (lane == 0) {
        if (len > kRevSortSmem) {
            atomicAdd(big, 1u);
        } else {
            wl[atomicAdd(big + 1, 1u)] = i;
        }
    }
}
__global__ void __launch_bounds__(kRevLongThreads) rev_sort_long_kernel(const uint32_t* __restrict__ off,
                                                                        uint32_t* __restrict__ data,
                                                                        const uint32_t* __restrict__ big,
                                                                        const uint32_t* __restrict__ wl) {
    __shared__ uint32_t s[kRevSortSmem];
    const uint32_t cnt = big[1];
    for (uint32_t w = blockIdx.x; w < cnt; w += gridDim.x) {
        const uint32_t i = wl[w];
        const uint32_t b = off[i], len = off[i + 1] - b;
        uint32_t* p = data + b;
        const uint32_t m = next_pow2(len);
        for (uint32_t j = threadIdx.x; j < m; j += kRevLongThreads) s[j] = j < len ? p[j] : 0xffffffffu;
        __syncthreads();
        for (uint32_t k = 2; k <= m; k <<= 1) {
            for (uint32_t j = k >> 1; j > 0; j >>= 1) {
                for (uint32_t e = threadIdx.x; e < m; e += kRevLongThreads) {
                    const uint32_t x = e ^ j;
                    if (x > e) {
                        const uint32_t va = s[e], vb = s[x];
                        if ((va > vb) == ((e & k) == 0)) {
                            s[e] = vb;
                            s[x] = va;
                        }
                    }
                }
                __syncthreads();
            }
        }
        for (uint32_t j = threadIdx.x; j < len; j += kRevLongThreads) p[j] = s[j];
        __syncthreads();
    }
}

struct UnionArgs {
    uint32_t n, P, S;
    uint64_t round_seed;
    const uint32_t *fnew, *fold, *cnew, *cold;
    const uint32_t *rn_off, *rn_data, *ro_off, *ro_data;
    uint32_t* gnew;  // n x 2S
    uint32_t* gold;  // n x (P+S)
    uint32_t* gncnt;
    uint32_t* gocnt;
    unsigned long long* join_rows;
    const uint32_t* samp;  // n x 2 x S sampled reverse lists (rev_sample_kernel), used when longer than S
    uint32_t lo;           // points [lo, n) are unioned
};

// graph_build.cpp:38-48 sample_down for every reverse list longer than S, one
// thread per (point, new/old): the sorted unique list gets a partial
// Fisher-Yates over its first S slots driven by
// std::mt19937_64(substream(round_seed, 2i + kind)).  Output k of a freshly
// seeded mt19937_64 (k < 156) only needs seed words k, k+1 and k+156, so the
// seed expansion is streamed and only words 0..S are kept; swapped positions
// live in a small per-thread overlay in shared memory.
__global__ void rev_sample_kernel(uint32_t n, uint32_t S, uint64_t round_seed, const uint32_t* __restrict__ rn_off,
                                  const uint32_t* __restrict__ rn_data, const uint32_t* __restrict__ ro_off,
                                  const uint32_t* __restrict__ ro_data, uint32_t* __restrict__ samp, uint32_t lo) {
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    const size_t per = size_t(S + 1) * 8 + size_t(4 * S) * 4;
    uint64_t* xs = reinterpret_cast<uint64_t*>(smem + threadIdx.x * per);
    uint32_t* pos = reinterpret_cast<uint32_t*>(xs + S + 1);
    uint32_t* val = pos + 2 * S;
    if (t >= 2 * (n - lo)) return;
    // kind-major: a warp's lanes all sample new lists or all old lists (right after init there
    // are no old lists at all, so interleaving the kinds would idle every other lane)
    const uint32_t kind = t >= n - lo ? 1u : 0u, i = lo + (t - kind * (n - lo));
    const uint32_t* off = kind ? ro_off : rn_off;
    const uint32_t* data = kind ? ro_data : rn_data;
    const uint32_t b = off[i], m = off[i + 1] - b;
    if (m <= S) return;
    const uint32_t* a = data + b;
    uint32_t* out = samp + (size_t(i) * 2 + kind) * S;
    uint64_t x = substream(round_seed, 2 * uint64_t(i) + kind);
    xs[0] = x;
    for (uint32_t k = 1; k <= S; ++k) {
        x = 6364136223846793005ULL * (x ^ (x >> 62)) + uint64_t(k);
        xs[k] = x;
    }
    for (uint32_t k = S + 1; k < 156; ++k) x = 6364136223846793005ULL * (x ^ (x >> 62)) + uint64_t(k);
    // the swaps of the partial Fisher-Yates: positions below S live in head[] (direct), the
    // others in a small overlay searched linearly (at most one new entry per step)
    uint32_t* head = val;
    uint32_t* opos = pos;
    uint32_t* oval = pos + S;
    for (uint32_t k = 0; k < S; ++k) head[k] = a[k];
    uint32_t no = 0;
    for (uint32_t k = 0; k < S; ++k) {
        x = 6364136223846793005ULL * (x ^ (x >> 62)) + uint64_t(156 + k);
        const uint64_t r = mt_temper(mt_twist(xs[k], xs[k + 1], x));
        const uint32_t j = k + uint32_t(r % uint64_t(m - k));
        if (j == k) continue;  // swap with itself
        const uint32_t vk = head[k];
        if (j < S) {
            head[k] = head[j];
            head[j] = vk;
        } else {
            uint32_t q = 0;
            while (q < no && opos[q] != j) ++q;
            if (q == no) {
                opos[no++] = j;
                head[k] = a[j];
            } else {
                head[k] = oval[q];
            }
            oval[q] = vk;
        }
    }
    for (uint32_t k = 0; k < S; ++k) out[k] = head[k];
}

// graph_build.cpp:88-103 per point: sample reverse lists, union, sort-dedup.
__global__ void union_kernel(UnionArgs a, uint32_t m_new, uint32_t m_old) {
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t warp = threadIdx.x / 32, lane = lane_id();
    const uint32_t wpb = blockDim.x / 32;
    uint32_t* sn = reinterpret_cast<uint32_t*>(smem) + warp * (m_new + m_old);
    uint32_t* so = sn + m_new;
    const uint32_t i = a.lo + blockIdx.x * wpb + warp;
    if (i >= a.n) return;
    const uint32_t cn = a.cnew[i], co = a.cold[i];
    for (uint32_t j = lane; j < cn; j += 32) sn[j] = a.fnew[size_t(i) * a.S + j];
    for (uint32_t j = lane; j < co; j += 32) so[j] = a.fold[size_t(i) * a.P + j];
    const uint32_t rnb = a.rn_off[i], rnm = a.rn_off[i + 1] - rnb;
    const uint32_t rob = a.ro_off[i], rom = a.ro_off[i + 1] - rob;
    uint32_t addn = min(rnm, a.S), addo = min(rom, a.S);
    if (rnm <= a.S) {
        for (uint32_t j = lane; j < rnm; j += 32) sn[cn + j] = a.rn_data[rnb + j];
    }
    if (rom <= a.S) {
        for (uint32_t j = lane; j < rom; j += 32) so[co + j] = a.ro_data[rob + j];
    }
    if (rnm > a.S)
        for (uint32_t j = lane; j < a.S; j += 32) sn[cn + j] = a.samp[(size_t(i) * 2) * a.S + j];
    if (rom > a.S)
        for (uint32_t j = lane; j < a.S; j += 32) so[co + j] = a.samp[(size_t(i) * 2 + 1) * a.S + j];
    __syncwarp();
    uint32_t un, uo;
    uint32_t* gn = a.gnew + size_t(i) * 2 * a.S;
    uint32_t* go = a.gold + size_t(i) * (a.P + a.S);
    if (m_new <= 64) {
        un = warp_unique_regs_u32<2>(sn, cn + addn, gn);
    } else {
        un = warp_sort_unique_u32(sn, cn + addn, m_new);
        for (uint32_t j = lane; j < un; j += 32) gn[j] = sn[j];
    }
    if (m_old <= 128) {
        uo = warp_unique_regs_u32<4>(so, co + addo, go);
    } else {
        uo = warp_sort_unique_u32(so, co + addo, m_old);
        for (uint32_t j = lane; j < uo; j += 32) go[j] = so[j];
    }
    if (lane == 0) {
        a.gncnt[i] = un;
        a.gocnt[i] = uo;
        atomicAdd(a.join_rows, (unsigned long long)(un + uo));
    }
}

// --------------------------------------------------------------- finalize

// graph_build.cpp:357-365: pools smaller than k are topped up by scanning ids
// in ascending order (tiny inputs only).  One warp per deficient point.
__global__ void fill_sparse_kernel(const float* __restrict__ x, uint32_t n, uint32_t ld, uint32_t P,
                                   uint32_t k, uint64_t* keys, uint8_t* flags, uint32_t* sizes,
                                   unsigned long long* comps, uint32_t lo, uint32_t hi) {
    const uint32_t lane = lane_id();
    const uint32_t i = lo + (blockIdx.x * blockDim.x + threadIdx.x) / 32;
    if (i >= hi) return;
    uint32_t sz = sizes[i];
    if (sz >= k) return;
    uint64_t* pk = keys + size_t(i) * P;
    uint8_t* pf = flags + size_t(i) * P;
    const float* xi = x + size_t(i) * ld;
    uint32_t added = 0;
    for (uint32_t base = 0; base < n && sz < k; base += 32) {
        const uint32_t j = base + lane;
        bool ok = j < n && j != i;
        for (uint32_t e = 0; ok && e < sz; ++e) ok = key_id(pk[e]) != j;
        const uint32_t b = __ballot_sync(0xffffffffu, ok);
        const uint32_t rank = __popc(b & ((1u << lane) - 1u));
        const uint32_t need = k - sz;
        uint64_t key = kEmptyKey;
        if (ok && rank < need) key = make_key(l2_exact_ldg(xi, x + size_t(j) * ld, ld), j);
        // insertion (sequential, rare path)
        for (uint32_t l = 0; l < 32; ++l) {
            const uint64_t kv = __shfl_sync(0xffffffffu, key, l);
            if (kv == kEmptyKey) continue;
            if (lane == 0) {
                uint32_t p = sz;
                while (p > 0 && pk[p - 1] > kv) { pk[p] = pk[p - 1]; pf[p] = pf[p - 1]; --p; }
                pk[p] = kv;
                pf[p] = 0;
            }
            ++sz;
            ++added;
            __syncwarp();
        }
    }
    if (lane == 0) {
        sizes[i] = sz;
        atomicAdd(comps, (unsigned long long)added);
    }
}

__global__ void finalize_kernel(const uint64_t* __restrict__ keys, uint32_t n, uint32_t P, uint32_t k,
                                uint32_t* __restrict__ ids, float* __restrict__ dists) {
    const size_t t = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    if (t >= size_t(n) * k) return;
    const uint32_t i = uint32_t(t / k), j = uint32_t(t % k);
    const uint64_t key = keys[size_t(i) * P + j];
    ids[t] = key_id(key);
    dists[t] = key_dist(key);
}

// graph_build.cpp:209-226: per-row hit counts (host sums them in row order).
__global__ void topk_hits_kernel(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ sizes,
                                 uint32_t P, uint32_t k, const uint32_t* __restrict__ gt, uint32_t gt_rows,
                                 uint32_t gt_k, const uint32_t* __restrict__ rows, uint32_t* __restrict__ hits) {
    const uint32_t lane = lane_id();
    const uint32_t r = (blockIdx.x * blockDim.x + threadIdx.x) / 32;
    if (r >= gt_rows) return;
    const uint32_t i = rows ? rows[r] : r;
    const uint32_t m = min(k, sizes[i]);
    uint32_t h = 0;
    for (uint32_t j = lane; j < m; j += 32) {
        const uint32_t id = key_id(keys[size_t(i) * P + j]);
        for (uint32_t g = 0; g < gt_k; ++g)
            if (gt[size_t(r) * gt_k + g] == id) { ++h; break; }
    }
    for (int o = 16; o > 0; o >>= 1) h += __shfl_xor_sync(0xffffffffu, h, o);
    if (lane == 0) hits[r] = h;
}

__global__ void split_keys_kernel(const uint64_t* __restrict__ keys, size_t cnt, uint32_t* ids, float* dists) {
    for (size_t t = blockIdx.x * size_t(blockDim.x) + threadIdx.x; t < cnt; t += size_t(gridDim.x) * blockDim.x) {
        const uint64_t k = keys[t];
        ids[t] = key_id(k);
        dists[t] = key_dist(k);
    }
}

// ------------------------------------------------------------ shard mode

__global__ void iota_kernel(uint32_t* __restrict__ out, uint32_t first, uint32_t count) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < count) out[t] = first + t;
}
struct InRange {
    uint32_t lo, hi;
    __host__ __device__ bool operator()(uint32_t v) const { return v >= lo && v < hi; }
};

// Offers held for targets [lo, lo+m): per-target counts (+ a trailing 0 for the scan).
__global__ void offer_counts_kernel(const uint32_t* __restrict__ ocnt, uint32_t lo, uint32_t m,
                                    uint32_t* __restrict__ out) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < m) out[t] = ocnt[lo + t];
    if (t == m) out[m] = 0;
}
// Packs the offers of targets [lo, lo+m) target-major, each target's in slot
// order then its spill segment (the order the replay reads), with their source
// points.  One warp per target.
__global__ void offer_pack_kernel(const uint32_t* __restrict__ ocnt, const uint64_t* __restrict__ obuf,
                                  const uint32_t* __restrict__ osrc, uint32_t cap, const uint32_t* __restrict__ ov_off,
                                  const uint64_t* __restrict__ ov_key, const uint32_t* __restrict__ ov_src,
                                  uint32_t lo, uint32_t m, const uint32_t* __restrict__ off, uint64_t* __restrict__ out,
                                  uint32_t* __restrict__ out_src) {
    const uint32_t lane = lane_id();
    const uint32_t t = (blockIdx.x * blockDim.x + threadIdx.x) / 32;
    if (t >= m) return;
    const uint32_t tgt = lo + t, c = ocnt[tgt], fix = min(c, cap);
    uint64_t* o = out + off[t];
    uint32_t* os = out_src + off[t];
    for (uint32_t j = lane; j < fix; j += 32) {
        o[j] = obuf[size_t(tgt) * cap + j];
        os[j] = osrc[size_t(tgt) * cap + j];
    }
    if (c > fix) {
        const uint64_t* sp = ov_key + ov_off[tgt];
        const uint32_t* ss = ov_src + ov_off[tgt];
        for (uint32_t j = lane; j < c - fix; j += 32) {
            o[fix + j] = sp[j];
            os[fix + j] = ss[j];
        }
    }
}
// Appends received offers for targets [lo, lo+m) to their slots / the spill
// list as one contiguous block per (sender, target): the replay orders blocks
// by source point, and a sender's block keeps its sources' order.
__global__ void offer_add_kernel(uint32_t lo, uint32_t m, const uint32_t* __restrict__ cnt,
                                 const uint32_t* __restrict__ off, const uint64_t* __restrict__ keys,
                                 const uint32_t* __restrict__ srcs, uint32_t* __restrict__ ocnt,
                                 uint64_t* __restrict__ obuf, uint32_t* __restrict__ osrc, uint32_t cap,
                                 uint32_t* __restrict__ ov_cnt, uint32_t* __restrict__ ov_tgt,
                                 uint64_t* __restrict__ ov_key, uint32_t* __restrict__ ov_src, uint32_t ov_cap) {
    const uint32_t lane = lane_id();
    const uint32_t t = (blockIdx.x * blockDim.x + threadIdx.x) / 32;
    if (t >= m) return;
    const uint32_t c = cnt[t];
    if (c == 0) return;
    const uint32_t tgt = lo + t;
    uint32_t base = 0, o0 = 0;
    if (lane == 0) {
        base = atomicAdd(&ocnt[tgt], c);
        const uint32_t nfix = base < cap ? min(c, cap - base) : 0u;
        if (c > nfix) o0 = atomicAdd(ov_cnt, c - nfix);
    }
    base = __shfl_sync(0xffffffffu, base, 0);
    o0 = __shfl_sync(0xffffffffu, o0, 0);
    const uint32_t nfix = base < cap ? min(c, cap - base) : 0u;
    const uint64_t* k = keys + off[t];
    const uint32_t* sr = srcs + off[t];
    for (uint32_t j = lane; j < c; j += 32) {
        if (j < nfix) {
            obuf[size_t(tgt) * cap + base + j] = k[j];
            osrc[size_t(tgt) * cap + base + j] = sr[j];
        } else {
            const uint64_t o = uint64_t(o0) + (j - nfix);
            if (o < ov_cap) {  // the host sized the list for every received offer spilling
                ov_tgt[o] = tgt;
                ov_key[o] = k[j];
                ov_src[o] = sr[j];
            }
        }
    }
}

// --------------------------------------------------------- host helpers

uint32_t grid_for(size_t items, uint32_t per_block) {
    return uint32_t(std::max<size_t>(1, std::min<size_t>((items + per_block - 1) / per_block, 1u << 30)));
}

void exclusive_scan(const uint32_t* in, uint32_t* out, uint32_t n) {
    size_t tmp = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, n + 1, stream()));
    DevBuf<unsigned char> t(tmp);
    prof_begin("cub_exclusive_scan");
    CK(cub::DeviceScan::ExclusiveSum(t.p, tmp, in, out, n + 1, stream()));
    prof_end();
    note_launch();
}

void segmented_sort(uint32_t* data, uint32_t total, const uint32_t* off, uint32_t n) {
    if (total == 0) return;
    DevBuf<uint32_t> out(total);
    size_t tmp = 0;
    CK(cub::DeviceSegmentedSort::SortKeys(nullptr, tmp, data, out.p, total, n, off, off + 1, stream()));
    DevBuf<unsigned char> t(tmp);
    prof_begin("cub_segmented_sort");
    CK(cub::DeviceSegmentedSort::SortKeys(t.p, tmp, data, out.p, total, n, off, off + 1, stream()));
    prof_end();
    note_launch();
    CK(cudaMemcpyAsync(data, out.p, size_t(total) * 4, cudaMemcpyDeviceToDevice, stream()));
}

// Host copy of CSR lists built from fixed-width rows + counts.
void csr_from_rows(const DevBuf<uint32_t>& rows, uint32_t width, const DevBuf<uint32_t>& cnt, uint32_t n,
                   uint32_t* offsets, uint32_t* data) {
    std::vector<uint32_t> c(n);
    cnt.download(c.data(), n);
    std::vector<uint32_t> r;
    if (data) {
        r.resize(size_t(n) * width);
        rows.download(r.data(), r.size());
    }
    ssync();
    uint32_t o = 0;
    for (uint32_t i = 0; i < n; ++i) {
        offsets[i] = o;
        if (data) std::copy(r.begin() + size_t(i) * width, r.begin() + size_t(i) * width + c[i], data + o);
        o += c[i];
    }
    offsets[n] = o;
}

}  // namespace
}  // namespace annk


// ------------------------------------------------------------------ host

using namespace annk;

namespace {

constexpr uint32_t kMaxSample = 64;  // device sample_down keeps 2*S swap slots in registers

void ensure_scratch(annk_state* s) {
    const size_t n = s->n;
    if (s->fnew.n == n * s->S && s->fold.n == n * s->P) return;
    s->fnew.alloc(n * s->S);
    s->fold.alloc(n * s->P);
    s->cnew.alloc(n);
    s->cold.alloc(n);
    s->rn_cnt.alloc(n + 1);
    s->ro_cnt.alloc(n + 1);
    s->rn_off.alloc(n + 1);
    s->ro_off.alloc(n + 1);
    s->rn_cur.alloc(n);
    s->ro_cur.alloc(n);
    s->rn_data.alloc(std::max<size_t>(n * s->S, 1));
    s->ro_data.alloc(std::max<size_t>(n * s->P, 1));
    s->gnew.alloc(n * 2 * s->S);
    s->gold.alloc(n * (s->P + s->S));
    s->gncnt.alloc(n);
    s->gocnt.alloc(n);
    s->thr.alloc(n);
    s->ocnt.alloc(n);
}

uint32_t own_lo(const annk_state* s) { return s->sharded ? s->lo : 0u; }
uint32_t own_hi(const annk_state* s) { return s->sharded ? s->hi : s->n; }

// graph_build.cpp:59-86 forward half: the owned points' pools are scanned and
// their forward lists + start-of-round tails written.
void do_sample(annk_state* s) {
    ensure_scratch(s);
    const uint32_t lo = own_lo(s), hi = own_hi(s);
    SampleArgs a{hi, s->P, s->S, s->keys.p, s->flags.p, s->sizes.p, s->fnew.p, s->fold.p,
                 s->cnew.p, s->cold.p, s->thr.p, lo, nullptr, nullptr};
    s->counts_fused = !s->sharded;
    if (s->counts_fused) {  // every forward row is written here: count the reverse lists on the way
        s->rn_cnt.zero();
        s->ro_cnt.zero();
        a.rn_cnt = s->rn_cnt.p;
        a.ro_cnt = s->ro_cnt.p;
    }
    if (hi > lo) LAUNCH(sample_kernel, grid_for(size_t(hi - lo) * 32, 256), 256, 0, a);
    s->stage = 0;
}

// graph_build.cpp:59-86 reverse half, from the forward lists of ALL points
// (in shard mode the other ranks' rows arrive through annk_state_rows first).
void do_reverse(annk_state* s) {
    ensure_scratch(s);
    const uint32_t n = s->n;
    // reverse lists are needed for the owned points only (all of them unsharded)
    const uint32_t tlo = own_lo(s), thi = own_hi(s);
    if (!s->counts_fused) {
        s->rn_cnt.zero();
        s->ro_cnt.zero();
        LAUNCH(rev_count_kernel, grid_for(size_t(n) * 32, 256), 256, 0, n, s->S, s->fnew.p, s->cnew.p, s->rn_cnt.p,
               tlo, thi);
        LAUNCH(rev_count_kernel, grid_for(size_t(n) * 32, 256), 256, 0, n, s->P, s->fold.p, s->cold.p, s->ro_cnt.p,
               tlo, thi);
    }
    s->counts_fused = false;
    exclusive_scan(s->rn_cnt.p, s->rn_off.p, n);
    exclusive_scan(s->ro_cnt.p, s->ro_off.p, n);
    s->rn_cur.zero();
    s->ro_cur.zero();
    LAUNCH(reverse_scatter_kernel, grid_for(size_t(n) * 32, 256), 256, 0, n, s->S, s->fnew.p, s->cnew.p,
           s->rn_off.p, s->rn_cur.p, s->rn_data.p, tlo, thi);
    LAUNCH(reverse_scatter_kernel, grid_for(size_t(n) * 32, 256), 256, 0, n, s->P, s->fold.p, s->cold.p,
           s->ro_off.p, s->ro_cur.p, s->ro_data.p, tlo, thi);
    // reverse lists as sets in ascending id order (the reference pushes them in
    // ascending owner order, graph_build.cpp:71-85)
    DevBuf<uint32_t> big(4), wl(2 * size_t(n));
    big.zero();
    if (thi > tlo) {
        const uint32_t grid = (thi - tlo + kRevSortWarps - 1) / kRevSortWarps;
        LAUNCH(rev_sort_kernel, grid, kRevSortWarps * 32, 0, s->rn_off.p, s->rn_data.p, tlo, thi, big.p, wl.p);
        LAUNCH(rev_sort_kernel, grid, kRevSortWarps * 32, 0, s->ro_off.p, s->ro_data.p, tlo, thi, big.p + 2,
               wl.p + n);
        const uint32_t lgrid = uint32_t(num_sms()) * 4;
        LAUNCH(rev_sort_long_kernel, lgrid, kRevLongThreads, 0, s->rn_off.p, s->rn_data.p, big.p, wl.p);
        LAUNCH(rev_sort_long_kernel, lgrid, kRevLongThreads, 0, s->ro_off.p, s->ro_data.p, big.p + 2, wl.p + n);
    }
    uint32_t tot[2], hb[4];
    CK(cudaMemcpyAsync(&tot[0], s->rn_off.p + n, 4, cudaMemcpyDeviceToHost, stream()));
    CK(cudaMemcpyAsync(&tot[1], s->ro_off.p + n, 4, cudaMemcpyDeviceToHost, stream()));
    big.download(hb, 4);
    ssync();
    // a list too long for shared memory (a hub with > 8192 reverse neighbours): the whole array
    // goes through the library segmented sort (sorted lists stay sorted)
    if (hb[0]) segmented_sort(s->rn_data.p, tot[0], s->rn_off.p, n);
    if (hb[2]) segmented_sort(s->ro_data.p, tot[1], s->ro_off.p, n);
    s->stage = 1;
}

void do_rebuild(annk_state* s) {
    do_sample(s);
    do_reverse(s);
}

void do_union(annk_state* s) {
    if (s->stage != 1) throw_invalid("union_reverse_lists: call rebuild_sample_lists first");
    const uint32_t n = s->n, lo = own_lo(s), hi = own_hi(s);
    const uint32_t m_new = next_pow2(2 * s->S), m_old = next_pow2(s->P + s->S);
    DevBuf<unsigned long long> rows(1);
    rows.zero();
    const uint64_t round_seed = substream(s->seed, s->iteration);
    DevBuf<uint32_t> samp(size_t(n) * 2 * s->S);
    {
        const uint32_t tpb = 64;
        const size_t per = size_t(s->S + 1) * 8 + size_t(4 * s->S) * 4;
        // S in 32..64 needs more than the default 48 KB of dynamic shared memory (98 KB at S = 64)
        CK(cudaFuncSetAttribute(rev_sample_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(tpb * per)));
        if (hi > lo)
            LAUNCH(rev_sample_kernel, (2 * (hi - lo) + tpb - 1) / tpb, tpb, tpb * per, hi, s->S, round_seed,
                   s->rn_off.p, s->rn_data.p, s->ro_off.p, s->ro_data.p, samp.p, lo);
    }
    UnionArgs a{n, s->P, s->S, round_seed, s->fnew.p, s->fold.p, s->cnew.p, s->cold.p,
                s->rn_off.p, s->rn_data.p, s->ro_off.p, s->ro_data.p, s->gnew.p, s->gold.p,
                s->gncnt.p, s->gocnt.p, rows.p, samp.p, lo};
    a.n = hi;
    const uint32_t wpb = 4;
    if (hi > lo) LAUNCH(union_kernel, (hi - lo + wpb - 1) / wpb, wpb * 32, wpb * (m_new + m_old) * 4, a, m_new, m_old);
    unsigned long long h = 0;
    rows.download(&h, 1);
    ssync();
    s->join_rows = h;
    s->stage = 2;
}

// per-point offer slots: sized from the offer volume seen so far, within a
// 12 GB budget for the keys (offers past the slots spill to a target-sorted
// global list); every offer also carries its source point (4 bytes)
uint32_t offer_cap_max(const annk_state* s) {
    const uint32_t cap_floor = std::max(2 * s->P, 64u);
    uint32_t cap_max = cap_floor;
    // per-target offer slots (12 B each; ~16 B counted) within 32 GB of the
    // 180 GB: at 1M points, 2048 slots -- spilled offers (a radix sort by
    // target per round) 84M -> 21M in round 2 at cfg2
    const char* gb = getenv("ANNK_OFFER_GB");
    const uint64_t budget = (gb ? std::strtoull(gb, nullptr, 10) : 32ull) << 30;
    while (uint64_t(cap_max) * 2 * s->n * 8 <= budget && cap_max < 4096) cap_max *= 2;
    return cap_max;
}
uint32_t g_offer_cap_hint = 0;          // capacities learned by earlier rounds (any state)
uint64_t g_spill_per_point_hint = 8;

// Offers one join launch may hold: the per-target slot counters and the spill
// reservation counter are 32-bit and the spill list is capped (kMaxSpill
// entries, 16 bytes each); a source range that would exceed either is refused
// (returns false, pools untouched) and the caller joins it in smaller pieces.
constexpr uint64_t kMaxJoinOffers = 1ull << 32;
constexpr uint32_t kMaxSpill = 1u << 28;

uint64_t join_offer_limit() {
    const char* lim_env = getenv("ANNK_JOIN_MAX_OFFERS");  // tests: force the piecewise round at small N
    return lim_env ? std::strtoull(lim_env, nullptr, 10) : kMaxJoinOffers;
}

// Join of the owned points whose id lies in [ilo, ihi) (graph_build.cpp:105-162):
// every offer that beats its target's start-of-round tail lands, tagged with
// its source point, in the target's slots or the spill list; pools are not
// touched.  Offers may target any point.
bool join_phase(annk_state* s, const annk_dataset* ds, uint32_t ilo = 0, uint32_t ihi = 0xffffffffu) {
    if (s->stage != 2) throw_invalid("join: call union_reverse_lists first");
    const uint32_t n = s->n;
    const uint32_t cap_floor = std::max(2 * s->P, 64u), cap_max = offer_cap_max(s);
    if (s->offer_cap == 0) s->offer_cap = std::min(cap_max, std::max(cap_floor, g_offer_cap_hint));
    if (s->ov_cap == 0)
        s->ov_cap = uint32_t(std::min<uint64_t>(std::max<uint64_t>(1u << 20, n * g_spill_per_point_hint), kMaxSpill));
    // visit list: tree-0 leaf order (L2 locality), restricted to owned points
    const uint32_t* order = s->sharded ? s->order_own.p : (s->order.n ? s->order.p : nullptr);
    const uint32_t n_visit = own_hi(s) - own_lo(s);
    if (s->ov_count.n != 1) s->ov_count.alloc(1);
    JoinCounters jc;
    for (;;) {
        if (s->obuf.n != size_t(n) * s->offer_cap) {
            s->obuf.alloc(size_t(n) * s->offer_cap);
            s->osrc.alloc(size_t(n) * s->offer_cap);
        }
        if (s->ov_tgt.n != s->ov_cap) {
            s->ov_tgt.alloc(s->ov_cap);
            s->ov_key.alloc(s->ov_cap);
            s->ov_src.alloc(s->ov_cap);
        }
        s->ocnt.zero();
        s->ov_count.zero();
        join_launch(s, ds, order, n_visit, ilo, std::min(ihi, n), kMaxSpill, &jc);
        if (getenv("ANNK_TRACE"))
            fprintf(stderr, "[annk] join [%u,%u): offers %llu spilled %u (cap %u, spill cap %u)\n", ilo,
                    std::min(ihi, n), jc.offers, jc.spilled, s->offer_cap, s->ov_cap);
        // (the offer total bounds the spill count: below 2^32 the 32-bit counter cannot have wrapped)
        if (jc.offers >= join_offer_limit() || jc.spilled > kMaxSpill) {
            s->last_offers = jc.offers;
            return false;
        }
        if (jc.spilled <= s->ov_cap) break;
        s->ov_cap = next_pow2(jc.spilled);  // spill list too small: grow and redo (pools untouched so far)
        g_spill_per_point_hint = std::max<uint64_t>(g_spill_per_point_hint, (uint64_t(s->ov_cap) + n - 1) / n);
    }
    s->spilled = jc.spilled;
    s->spill_sorted = false;
    s->pending_comps = jc.comps;
    s->last_offers = jc.offers;
    s->last_spilled = jc.spilled;
    s->pack_hi = s->pack_lo = 0;
    s->stage = 3;
    return true;
}

// Replays the owned targets' offers into their pools in the reference's order;
// returns the accepted inserts.  Replaying the pieces of a round one after
// another is exact when the pieces are ascending source ranges.
uint64_t merge_offers(annk_state* s) { return replay_offers(s, own_lo(s), own_hi(s)); }

void finish_round(annk_state* s, uint64_t changes) {
    const uint32_t n = s->n;
    const uint32_t cap_floor = std::max(2 * s->P, 64u), cap_max = offer_cap_max(s);
    // slots for ~2.5x the mean offers per target (hub targets take more)
    const uint64_t want = std::max<uint64_t>(cap_floor, (s->last_offers / std::max(n, 1u)) * 10 / 4);
    const uint32_t next = std::min<uint32_t>(cap_max, next_pow2(uint32_t(std::min<uint64_t>(want, 1u << 20))));
    g_offer_cap_hint = std::max(g_offer_cap_hint, next);
    s->offer_cap = std::max(s->offer_cap, next);  // takes effect next round (buffers reallocated)
    s->dist_comps += s->pending_comps;
    s->pending_comps = 0;
    s->iteration += 1;
    s->last_changes = changes;
    s->stage = 2;  // the round's lists stay inspectable (the reference keeps them)
}

uint64_t merge_phase(annk_state* s) {
    if (s->stage != 3) throw_invalid("merge: call join first");
    const uint64_t changes = merge_offers(s);
    finish_round(s, changes);
    return changes;
}

// A round whose offers do not fit one join launch (very large N) is joined in
// ascending source ranges, each replayed into the pools before the next: the
// reference visits the points in ascending order, so this is its order too.
uint64_t do_join_merge(annk_state* s, const annk_dataset* ds) {
    if (s->join_pieces <= 1) {
        if (join_phase(s, ds)) {
            // a spill list past half its cap: the next round (usually more offers while
            // the graph is far from converged) starts in two pieces instead of failing
            const bool heavy = s->spilled > kMaxSpill / 2;
            const uint64_t c = merge_phase(s);
            if (heavy) s->join_pieces = 2;
            return c;
        }
        const uint64_t lim = join_offer_limit();
        s->join_pieces = uint32_t(std::max<uint64_t>(2, (2 * s->last_offers + lim - 1) / lim));
    }
    const uint32_t lo = own_lo(s), hi = own_hi(s);
    uint32_t pieces = s->join_pieces;
    uint64_t comps = 0, offers = 0, spilled = 0, changes = 0, max_piece = 0, max_spill = 0;
    uint32_t pos = lo;
    while (pos < hi) {
        const uint32_t len = std::max(1u, (hi - lo + pieces - 1) / pieces);
        const uint32_t end = std::min(hi, pos + len);
        if (!join_phase(s, ds, pos, end)) {
            if (end - pos <= 1) throw_invalid("join: one point's offers exceed a join launch");
            pieces *= 2;
            continue;
        }
        comps += s->pending_comps;
        offers += s->last_offers;
        spilled += s->spilled;
        max_piece = std::max<uint64_t>(max_piece, s->last_offers);
        max_spill = std::max<uint64_t>(max_spill, s->spilled);
        changes += merge_offers(s);
        s->stage = 2;  // next piece joins against the same lists and start-of-round tails
        pos = end;
    }
    s->pending_comps = comps;
    s->last_offers = offers;
    s->last_spilled = spilled;
    // later rounds start from the piece count this round needed (offer volume
    // usually falls as the graph converges: back to one launch when it fits)
    s->join_pieces = 2 * max_piece * pieces < join_offer_limit() && 2 * max_spill * pieces < kMaxSpill ? 1u : pieces;
    if (max_spill > kMaxSpill / 2) s->join_pieces = std::min(pieces * 2, 1u << 20);  // see the one-launch case
    finish_round(s, changes);
    return changes;
}

// Owned visit order: tree-0 leaf order restricted to [lo, hi) (or lo..hi-1).
void set_shard(annk_state* s, uint32_t lo, uint32_t hi) {
    if (lo > hi || hi > s->n) throw_range("shard: range out of bounds");
    s->lo = lo;
    s->hi = hi;
    s->sharded = !(lo == 0 && hi == s->n);
    if (!s->sharded) {
        s->order_own.release();
        return;
    }
    s->order_own.alloc(std::max<size_t>(hi - lo, 1));
    if (s->order.n == s->n) {
        DevBuf<uint32_t> nsel(1);
        size_t tmp = 0;
        CK(cub::DeviceSelect::If(nullptr, tmp, s->order.p, s->order_own.p, nsel.p, s->n, InRange{lo, hi},
                                 stream()));
        DevBuf<unsigned char> t(std::max<size_t>(tmp, 1));
        CK(cub::DeviceSelect::If(t.p, tmp, s->order.p, s->order_own.p, nsel.p, s->n, InRange{lo, hi}, stream()));
        note_launch();
    } else if (hi > lo) {
        LAUNCH(iota_kernel, (hi - lo + 255) / 256, 256, 0, s->order_own.p, lo, hi - lo);
    }
    ssync();
}

annk_state* new_state(uint32_t n, uint32_t k, uint32_t P, uint32_t S, uint64_t seed) {
    // graph_build.cpp:18-35 make_state
    if (n < 2) throw_invalid("graph build: need at least 2 points");
    if (k < 1) throw_invalid("graph build: k must be >= 1");
    if (P < k) throw_invalid("graph build: pool_cap must be >= k");
    if (S < 1) throw_invalid("graph build: sample_cap must be >= 1");
    if (S > kMaxSample) throw_invalid("graph build: sample_cap > 64 is not supported on the device path");
    auto* s = new annk_state;
    s->n = n;
    s->k = k;
    s->P = P;
    s->S = S;
    s->seed = seed;
    s->keys.alloc(size_t(n) * P);
    s->flags.alloc(size_t(n) * P);
    s->sizes.alloc(n);
    return s;
}

}  // namespace

extern "C" {

}  // extern "C"

namespace {
annk_state* init_graph_impl(const annk_dataset* ds, const annk_forest* fc, uint32_t k, uint32_t conquer_depth,
                            uint32_t pool_cap, uint32_t sample_cap, uint64_t seed, uint32_t lo, uint32_t hi) {
    if (!ds || !fc) throw_invalid("init_graph: null argument");
    if (fc->n != ds->n || fc->dim != ds->dim) throw_invalid("init_graph: forest was built over different data");
    annk_forest* f = const_cast<annk_forest*>(fc);
    std::unique_ptr<annk_state> s(new_state(ds->n, k, pool_cap, sample_cap, seed));
    forest_ensure_links(f, /*rebuild=*/true);  // inside the build, like the reference
    uint32_t max_depth = 0;
    for (const auto& t : f->trees) max_depth = std::max(max_depth, t.max_depth);
    const uint32_t n = ds->n;
    s->order.alloc(n);
    CK(cudaMemcpyAsync(s->order.p, f->trees[0].pidx.p, size_t(n) * 4, cudaMemcpyDeviceToDevice, stream()));
    set_shard(s.get(), lo, hi);
    const uint32_t* visit = s->sharded ? s->order_own.p : s->order.p;
    const uint32_t n_visit = hi - lo;
    DevBuf<unsigned long long> comps(1);
    comps.zero();
    DevBuf<uint32_t> overflow(size_t(n) + 1);
    CK(cudaMemsetAsync(overflow.p, 0, 4, stream()));
    InitArgs a{ds->data.p, n, ds->ld, f->n_trees, conquer_depth, pool_cap, f->views.p,
               s->keys.p, s->flags.p, s->sizes.p, comps.p, overflow.p,
               ds->u8 ? ds->data8.p : nullptr, ds->ld8, ds->u8 ? ds->norms8.p : nullptr};
    const uint32_t sib_full = f->n_trees * (max_depth + 1);
    const uint32_t sib_cap = 0;  // sibling lists come from the forest (sib_list)
    const size_t per_warp = init_warp_bytes(kInitCap, ds->u8 ? 0u : ds->ld, sib_cap);
    const size_t smem = per_warp * kInitWarps;
    void (*init_kernel)(InitArgs, uint32_t, const uint32_t*, uint32_t) =
        ds->u8 ? init_kernel_t<5> : init_kernel_t<1>;
    CK(cudaFuncSetAttribute(reinterpret_cast<const void*>(init_kernel), cudaFuncAttributeMaxDynamicSharedMemorySize,
                            int(smem)));
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, reinterpret_cast<const void*>(init_kernel),
                                                      kInitWarps * 32, smem));
    const uint32_t grid = std::max<uint32_t>(1, std::min<uint32_t>((n_visit + kInitWarps - 1) / kInitWarps,
                                                                    uint32_t(num_sms()) * std::max(per_sm, 1)));
    s->sizes.zero();  // points outside the shard keep empty pools
    if (n_visit) LAUNCH(init_kernel, grid, kInitWarps * 32, smem, a, sib_cap, visit, n_visit);
    uint32_t n_over = 0;
    overflow.download(&n_over, 1);
    ssync();
    if (n_over) {
        const uint32_t cap = next_pow2(f->n_trees * (max_depth + 1) * f->leaf_cap);
        const uint32_t blocks = std::min<uint32_t>(n_over, 1024);
        DevBuf<uint32_t> gscratch(size_t(blocks) * (3 * size_t(cap) + 2 * sib_full));
        DevBuf<float> gq(size_t(blocks) * ds->ld);
        LAUNCH(init_overflow_kernel, blocks, 32, 0, a, overflow.p + 1, n_over, cap, sib_full, gscratch.p, gq.p);
    }
    unsigned long long c = 0;
    comps.download(&c, 1);
    ssync();
    s->dist_comps = c;
    return s.release();
}
}  // namespace

extern "C" {

int annk_init_graph(const annk_dataset* ds, const annk_forest* fc, uint32_t k, uint32_t conquer_depth,
                    uint32_t pool_cap, uint32_t sample_cap, uint64_t seed, annk_state** out) {
    return abi([&] {
        if (!ds || !out) throw_invalid("init_graph: null argument");
        *out = init_graph_impl(ds, fc, k, conquer_depth, pool_cap, sample_cap, seed, 0, ds->n);
    });
}

int annk_init_random(const annk_dataset* ds, uint32_t k, uint32_t pool_cap, uint32_t sample_cap, uint64_t seed,
                     annk_state** out) {
    return abi([&] {
        if (!ds || !out) throw_invalid("init_random: null argument");
        std::unique_ptr<annk_state> s(new_state(ds->n, k, pool_cap, sample_cap, seed));
        const uint32_t n = ds->n;
        DevBuf<unsigned long long> comps(1);
        comps.zero();
        InitArgs a{ds->data.p, n, ds->ld, 0, 0, pool_cap, nullptr, s->keys.p, s->flags.p, s->sizes.p, comps.p,
                   nullptr, ds->u8 ? ds->data8.p : nullptr, ds->ld8, ds->u8 ? ds->norms8.p : nullptr};
        const uint32_t wpb = 4;
        const size_t sm = init_random_warp_bytes(pool_cap) * wpb;
        if (sm > 200 * 1024) throw_invalid("init_random: pool_cap too large for the device path");
        CK(cudaFuncSetAttribute(init_random_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
        LAUNCH(init_random_kernel, std::min<uint32_t>((n + wpb - 1) / wpb, uint32_t(num_sms()) * 16), wpb * 32,
               sm, a, seed);
        unsigned long long c = 0;
        comps.download(&c, 1);
        ssync();
        s->dist_comps = c;
        *out = s.release();
    });
}

int annk_init_graph_shard(const annk_dataset* ds, const annk_forest* fc, uint32_t k, uint32_t conquer_depth,
                          uint32_t pool_cap, uint32_t sample_cap, uint64_t seed, uint32_t lo, uint32_t hi,
                          annk_state** out) {
    return abi([&] {
        if (!ds || !out) throw_invalid("init_graph: null argument");
        if (lo > hi || hi > ds->n) throw_range("init_graph: shard range out of bounds");
        *out = init_graph_impl(ds, fc, k, conquer_depth, pool_cap, sample_cap, seed, lo, hi);
    });
}

int annk_state_set_shard(annk_state* s, uint32_t lo, uint32_t hi) {
    return abi([&] {
        if (!s) throw_invalid("set_shard: null state");
        set_shard(s, lo, hi);
    });
}

int annk_state_rows(annk_state* s, int which, int put, uint32_t lo, uint32_t hi, void* buf) {
    return abi([&] {
        if (!s || (!buf && hi > lo)) throw_invalid("state_rows: null argument");
        if (lo > hi || hi > s->n) throw_range("state_rows: row range out of bounds");
        ensure_scratch(s);
        char* dev;
        size_t row_bytes;
        switch (which) {
            case ANNK_ROWS_FNEW: dev = reinterpret_cast<char*>(s->fnew.p); row_bytes = size_t(s->S) * 4; break;
            case ANNK_ROWS_CNEW: dev = reinterpret_cast<char*>(s->cnew.p); row_bytes = 4; break;
            case ANNK_ROWS_FOLD: dev = reinterpret_cast<char*>(s->fold.p); row_bytes = size_t(s->P) * 4; break;
            case ANNK_ROWS_COLD: dev = reinterpret_cast<char*>(s->cold.p); row_bytes = 4; break;
            case ANNK_ROWS_THR: dev = reinterpret_cast<char*>(s->thr.p); row_bytes = 8; break;
            default: throw_invalid("state_rows: unknown row buffer");
        }
        const size_t bytes = size_t(hi - lo) * row_bytes;
        char* d = dev + size_t(lo) * row_bytes;
        if (bytes) CK(cudaMemcpyAsync(put ? d : buf, put ? buf : d, bytes, cudaMemcpyDefault, stream()));
        ssync();
    });
}

int annk_shard_sample(annk_state* s) {
    return abi([&] { do_sample(s); });
}

int annk_shard_union(annk_state* s) {
    return abi([&] {
        do_reverse(s);
        do_union(s);
    });
}

int annk_shard_join(annk_state* s, const annk_dataset* ds, uint64_t* comps) {
    return abi([&] {
        if (!s || !ds || ds->n != s->n) throw_invalid("join: state/dataset mismatch");
        if (!join_phase(s, ds))
            throw_invalid("join: this shard's offers exceed one join launch (" +
                          std::to_string(join_offer_limit()) + " offers); join it in source ranges "
                          "(annk_shard_join_range)");
        if (comps) *comps = s->pending_comps;
    });
}

int annk_shard_join_range(annk_state* s, const annk_dataset* ds, uint32_t ilo, uint32_t ihi, uint64_t* comps,
                          uint64_t* offers, uint32_t* ok) {
    return abi([&] {
        if (!s || !ds || ds->n != s->n || !ok) throw_invalid("join: state/dataset mismatch");
        if (ilo > ihi || ihi > s->n) throw_range("join: source range out of bounds");
        if (s->stage == 3) s->stage = 2;  // a refused or earlier piece: the lists are still valid
        *ok = join_phase(s, ds, ilo, ihi) ? 1u : 0u;
        if (comps) *comps = *ok ? s->pending_comps : 0;
        if (offers) *offers = s->last_offers;
    });
}

int annk_shard_offers_count(annk_state* s, uint32_t lo, uint32_t hi, uint64_t* total) {
    return abi([&] {
        if (!s || !total) throw_invalid("offers_count: null argument");
        if (s->stage != 3) throw_invalid("offers_count: call join first");
        if (lo > hi || hi > s->n) throw_range("offers_count: target range out of bounds");
        group_spills(s);
        const uint32_t m = hi - lo;
        s->pack_cnt.alloc(size_t(m) + 1);
        s->pack_off.alloc(size_t(m) + 1);
        LAUNCH(offer_counts_kernel, (m + 1 + 255) / 256, 256, 0, s->ocnt.p, lo, m, s->pack_cnt.p);
        exclusive_scan(s->pack_cnt.p, s->pack_off.p, m);
        uint32_t t = 0;
        CK(cudaMemcpyAsync(&t, s->pack_off.p + m, 4, cudaMemcpyDeviceToHost, stream()));
        ssync();
        s->pack_lo = lo;
        s->pack_hi = hi;
        *total = t;
    });
}

int annk_shard_offers_pack(annk_state* s, uint32_t lo, uint32_t hi, uint32_t* counts, uint64_t* keys,
                           uint32_t* srcs) {
    return abi([&] {
        if (!s) throw_invalid("offers_pack: null state");
        if (s->stage != 3 || s->pack_lo != lo || s->pack_hi != hi || s->pack_cnt.n != size_t(hi - lo) + 1)
            throw_invalid("offers_pack: call offers_count for the same range first");
        const uint32_t m = hi - lo;
        uint32_t total = 0;
        CK(cudaMemcpyAsync(&total, s->pack_off.p + m, 4, cudaMemcpyDeviceToHost, stream()));
        ssync();
        DevBuf<uint64_t> out(std::max<uint32_t>(total, 1));
        DevBuf<uint32_t> out_src(std::max<uint32_t>(total, 1));
        if (m)
            LAUNCH(offer_pack_kernel, grid_for(size_t(m) * 32, 256), 256, 0, s->ocnt.p, s->obuf.p, s->osrc.p,
                   s->offer_cap, s->ov_off.p, s->ov_key.p, s->ov_src.p, lo, m, s->pack_off.p, out.p, out_src.p);
        if (counts && m) CK(cudaMemcpyAsync(counts, s->pack_cnt.p, size_t(m) * 4, cudaMemcpyDefault, stream()));
        if (keys && total) CK(cudaMemcpyAsync(keys, out.p, size_t(total) * 8, cudaMemcpyDefault, stream()));
        if (srcs && total) CK(cudaMemcpyAsync(srcs, out_src.p, size_t(total) * 4, cudaMemcpyDefault, stream()));
        ssync();
    });
}

int annk_shard_offers_add(annk_state* s, uint32_t lo, uint32_t hi, const uint32_t* counts, const uint64_t* keys,
                          const uint32_t* srcs) {
    return abi([&] {
        if (!s || (!counts && hi > lo)) throw_invalid("offers_add: null argument");
        if (s->stage != 3) throw_invalid("offers_add: call join first");
        if (lo < own_lo(s) || hi > own_hi(s) || lo > hi) throw_range("offers_add: targets outside the shard");
        const uint32_t m = hi - lo;
        if (m == 0) return;
        DevBuf<uint32_t> cnt(size_t(m) + 1), off(size_t(m) + 1);
        CK(cudaMemcpyAsync(cnt.p, counts, size_t(m) * 4, cudaMemcpyDefault, stream()));
        CK(cudaMemsetAsync(cnt.p + m, 0, 4, stream()));
        {  // received total in 64 bits (the u32 scan below could wrap)
            std::vector<uint32_t> hc(m);
            CK(cudaMemcpyAsync(hc.data(), counts, size_t(m) * 4, cudaMemcpyDefault, stream()));
            ssync();
            uint64_t t = 0;
            for (uint32_t v : hc) t += v;
            if (t >= join_offer_limit()) throw_invalid("offers_add: more received offers than one round may hold");
        }
        exclusive_scan(cnt.p, off.p, m);
        uint32_t total = 0;
        CK(cudaMemcpyAsync(&total, off.p + m, 4, cudaMemcpyDeviceToHost, stream()));
        ssync();
        if (total == 0) return;
        if (!keys || !srcs) throw_invalid("offers_add: null keys");
        DevBuf<uint64_t> k(total);
        DevBuf<uint32_t> sr(total);
        CK(cudaMemcpyAsync(k.p, keys, size_t(total) * 8, cudaMemcpyDefault, stream()));
        CK(cudaMemcpyAsync(sr.p, srcs, size_t(total) * 4, cudaMemcpyDefault, stream()));
        // room for the worst case (every received offer spills); keep what is there
        const uint64_t need = uint64_t(s->spilled) + total;
        if (need > kMaxSpill) throw_invalid("offers_add: spill list would exceed its cap; join in source ranges");
        if (need > s->ov_cap) {
            const uint32_t cap = next_pow2(uint32_t(need));
            DevBuf<uint32_t> t2(cap), s2(cap);
            DevBuf<uint64_t> k2(cap);
            if (s->spilled) {
                CK(cudaMemcpyAsync(t2.p, s->ov_tgt.p, size_t(s->spilled) * 4, cudaMemcpyDeviceToDevice, stream()));
                CK(cudaMemcpyAsync(k2.p, s->ov_key.p, size_t(s->spilled) * 8, cudaMemcpyDeviceToDevice, stream()));
                CK(cudaMemcpyAsync(s2.p, s->ov_src.p, size_t(s->spilled) * 4, cudaMemcpyDeviceToDevice, stream()));
            }
            std::swap(s->ov_tgt, t2);
            std::swap(s->ov_key, k2);
            std::swap(s->ov_src, s2);
            s->ov_cap = cap;
        }
        // received offers append after the (target-grouped) spill list; grouping it again is a
        // stable sort, so every target keeps slot order, then its own spills, then these
        CK(cudaMemcpyAsync(s->ov_count.p, &s->spilled, 4, cudaMemcpyHostToDevice, stream()));
        LAUNCH(offer_add_kernel, grid_for(size_t(m) * 32, 256), 256, 0, lo, m, cnt.p, off.p, k.p, sr.p, s->ocnt.p,
               s->obuf.p, s->osrc.p, s->offer_cap, s->ov_count.p, s->ov_tgt.p, s->ov_key.p, s->ov_src.p, s->ov_cap);
        uint32_t sp = 0;
        s->ov_count.download(&sp, 1);
        ssync();
        s->spilled = sp;
        s->last_spilled = sp;
        s->spill_sorted = false;
        s->pack_lo = s->pack_hi = 0;
    });
}

int annk_shard_merge(annk_state* s, uint64_t* changes) {
    return abi([&] {
        const uint64_t c = merge_phase(s);
        if (changes) *changes = c;
    });
}

// One piece of a round joined in source ranges: the owned pools take the
// piece's offers (exact when pieces arrive in ascending source order); the
// round ends with annk_shard_finish_round.
int annk_shard_merge_piece(annk_state* s, uint64_t* changes) {
    return abi([&] {
        if (s->stage != 3) throw_invalid("merge: call join first");
        const uint64_t c = merge_offers(s);
        s->piece_changes += c;
        s->piece_comps += s->pending_comps;
        s->pending_comps = 0;
        s->stage = 2;
        if (changes) *changes = c;
    });
}

int annk_shard_finish_round(annk_state* s, uint64_t* changes) {
    return abi([&] {
        if (s->stage != 2) throw_invalid("finish_round: call union_reverse_lists first");
        s->pending_comps = s->piece_comps;
        const uint64_t c = s->piece_changes;
        s->piece_comps = s->piece_changes = 0;
        finish_round(s, c);
        if (changes) *changes = c;
    });
}

int annk_state_import(uint32_t n, uint32_t k, uint32_t pool_cap, uint32_t sample_cap, uint64_t seed,
                      uint32_t iteration, uint64_t dist_comps, const uint32_t* sizes, const uint32_t* ids,
                      const float* dists, const uint8_t* flags, annk_state** out) {
    return abi([&] {
        std::unique_ptr<annk_state> s(new_state(n, k, pool_cap, sample_cap, seed));
        s->iteration = iteration;
        s->dist_comps = dist_comps;
        std::vector<uint64_t> keys(size_t(n) * pool_cap, kEmptyKey);
        std::vector<uint8_t> fl(size_t(n) * pool_cap, 0);
        std::vector<uint32_t> sz(n);
        for (uint32_t i = 0; i < n; ++i) {
            // reference NeighborPool::insert semantics (sorted, dedup, capped)
            std::vector<std::pair<uint64_t, uint8_t>> row;
            for (uint32_t j = 0; j < std::min(sizes[i], pool_cap); ++j) {
                const size_t o = size_t(i) * pool_cap + j;
                if (ids[o] >= n) throw_range("state_import: id out of range");
                row.emplace_back(make_key(dists[o], ids[o]), flags[o]);
            }
            std::stable_sort(row.begin(), row.end(), [](auto& x, auto& y) { return x.first < y.first; });
            row.erase(std::unique(row.begin(), row.end(), [](auto& x, auto& y) { return x.first == y.first; }),
                      row.end());
            if (row.size() > pool_cap) row.resize(pool_cap);
            sz[i] = uint32_t(row.size());
            for (size_t j = 0; j < row.size(); ++j) {
                keys[size_t(i) * pool_cap + j] = row[j].first;
                fl[size_t(i) * pool_cap + j] = row[j].second;
            }
        }
        s->keys.upload(keys.data(), keys.size());
        s->flags.upload(fl.data(), fl.size());
        s->sizes.upload(sz.data(), n);
        ssync();
        *out = s.release();
    });
}

int annk_state_destroy(annk_state* s) {
    return abi([&] { delete s; });
}

int annk_state_meta(const annk_state* s, uint64_t* meta) {
    return abi([&] {
        meta[0] = s->n;
        meta[1] = s->k;
        meta[2] = s->P;
        meta[3] = s->S;
        meta[4] = s->seed;
        meta[5] = s->iteration;
        meta[6] = s->dist_comps;
        meta[7] = s->last_changes;
    });
}

int annk_state_export(const annk_state* s, uint32_t* sizes, uint32_t* ids, float* dists, uint8_t* flags) {
    return abi([&] {
        const size_t cnt = size_t(s->n) * s->P;
        if (sizes) s->sizes.download(sizes, s->n);
        if (flags) s->flags.download(flags, cnt);
        if (ids || dists) {
            DevBuf<uint32_t> di(cnt);
            DevBuf<float> dd(cnt);
            LAUNCH(split_keys_kernel, grid_for(cnt, 256), 256, 0, s->keys.p, cnt, di.p, dd.p);
            if (ids) di.download(ids, cnt);
            if (dists) dd.download(dists, cnt);
            ssync();
        }
        ssync();
    });
}

int annk_state_lists(const annk_state* s, int which, uint32_t* offsets, uint32_t* data) {
    return abi([&] {
        if (which < 0 || which > 3) throw_invalid("state_lists: which must be 0..3");
        const uint32_t n = s->n;
        if (s->stage == 0) {
            for (uint32_t i = 0; i <= n; ++i) offsets[i] = 0;
            return;
        }
        if (which == 0) {
            if (s->stage >= 2) csr_from_rows(s->gnew, 2 * s->S, s->gncnt, n, offsets, data);
            else csr_from_rows(s->fnew, s->S, s->cnew, n, offsets, data);
        } else if (which == 1) {
            if (s->stage >= 2) csr_from_rows(s->gold, s->P + s->S, s->gocnt, n, offsets, data);
            else csr_from_rows(s->fold, s->P, s->cold, n, offsets, data);
        } else {
            const DevBuf<uint32_t>& off = which == 2 ? s->rn_off : s->ro_off;
            const DevBuf<uint32_t>& dat = which == 2 ? s->rn_data : s->ro_data;
            off.download(offsets, n + 1);
            ssync();
            if (data && offsets[n]) dat.download(data, offsets[n]);
            ssync();
        }
    });
}

int annk_rebuild_sample_lists(annk_state* s) {
    return abi([&] { do_rebuild(s); });
}

int annk_union_reverse_lists(annk_state* s) {
    return abi([&] { do_union(s); });
}

int annk_nn_descent_iteration(annk_state* s, const annk_dataset* ds, uint64_t* changes) {
    return abi([&] {
        if (!s || !ds || ds->n != s->n) throw_invalid("nn_descent_iteration: state/dataset mismatch");
        do_rebuild(s);
        do_union(s);
        const uint64_t c = do_join_merge(s, ds);
        if (changes) *changes = c;
    });
}

int annk_refine_nn_descent(annk_state* s, const annk_dataset* ds, uint32_t max_iters, double min_change_rate,
                           uint32_t* iters_run) {
    return abi([&] {
        if (!s || !ds || ds->n != s->n) throw_invalid("refine_nn_descent: state/dataset mismatch");
        const double threshold = min_change_rate * double(s->n) * double(s->P);
        uint32_t it = 0;
        while (it < max_iters) {
            do_rebuild(s);
            do_union(s);
            const uint64_t c = do_join_merge(s, ds);
            ++it;
            if (double(c) < threshold) break;
        }
        if (iters_run) *iters_run = it;
    });
}

namespace {
void finalize_impl(annk_state* s, const annk_dataset* ds, uint32_t k, uint32_t* ids, float* dists) {
    {
        const uint32_t n = s->n;
        if (n < 2 || n - 1 < k) throw_invalid("finalize: need n-1 >= k");
        if (k > s->P) throw_invalid("finalize: k exceeds pool capacity");
        if (!ds || ds->n != n) throw_invalid("finalize: dataset mismatch");
        // shard mode: rows [lo, hi) only, written as (hi - lo) x k
        const uint32_t lo = own_lo(s), m = own_hi(s) - lo;
        DevBuf<unsigned long long> comps(1);
        comps.zero();
        const size_t pk = size_t(lo) * s->P;
        if (m)
            LAUNCH(fill_sparse_kernel, grid_for(size_t(m) * 32, 256), 256, 0, ds->data.p, n, ds->ld, s->P, k,
                   s->keys.p, s->flags.p, s->sizes.p, comps.p, lo, lo + m);
        DevBuf<uint32_t> di(size_t(m) * k);
        DevBuf<float> dd(size_t(m) * k);
        if (m) LAUNCH(finalize_kernel, grid_for(size_t(m) * k, 256), 256, 0, s->keys.p + pk, m, s->P, k, di.p, dd.p);
        unsigned long long c = 0;
        comps.download(&c, 1);
        if (ids) CK(cudaMemcpyAsync(ids, di.p, size_t(m) * k * 4, cudaMemcpyDefault, stream()));
        if (dists) CK(cudaMemcpyAsync(dists, dd.p, size_t(m) * k * 4, cudaMemcpyDefault, stream()));
        ssync();
        s->dist_comps += c;
    }
}
}  // namespace

int annk_finalize(annk_state* s, const annk_dataset* ds, uint32_t k, uint32_t* ids, float* dists) {
    return abi([&] {
        if (!s) throw_invalid("finalize: null state");
        finalize_impl(s, ds, k, ids, dists);
    });
}

// The last round of a build and finalize as one call: once the join has run,
// every target's replay touches only that target's pool, so the targets are
// replayed in ascending chunks and each chunk's rows are finalized and copied
// to the host (second stream) while the next chunk replays.  Same pools,
// flags, `changes`, dist_comps and rows as annk_nn_descent_iteration followed
// by annk_finalize.
static cudaStream_t copy_stream() {
    static cudaStream_t cs = nullptr;
    if (!cs) CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    return cs;
}

int annk_nn_descent_iteration_finalize(annk_state* s, const annk_dataset* ds, uint32_t k, uint32_t* ids,
                                       float* dists, uint64_t* changes, uint64_t* round_dist_comps) {
    return abi([&] {
        if (!s || !ds || ds->n != s->n) throw_invalid("nn_descent_iteration: state/dataset mismatch");
        const uint32_t n = s->n;
        if (n < 2 || n - 1 < k) throw_invalid("finalize: need n-1 >= k");
        if (k > s->P) throw_invalid("finalize: k exceeds pool capacity");
        do_rebuild(s);
        do_union(s);
        bool one_launch = false;
        if (!s->sharded && s->join_pieces <= 1) {
            one_launch = join_phase(s, ds);
            if (!one_launch) {  // as do_join_merge: this round goes in pieces
                const uint64_t lim = join_offer_limit();
                s->join_pieces = uint32_t(std::max<uint64_t>(2, (2 * s->last_offers + lim - 1) / lim));
            }
        }
        if (!one_launch) {  // sharded states and rounds joined in pieces: the two steps one after the other
            const uint64_t c = do_join_merge(s, ds);
            if (changes) *changes = c;
            if (round_dist_comps) *round_dist_comps = s->dist_comps;
            finalize_impl(s, ds, k, ids, dists);
            return;
        }
        const char* ce = getenv("ANNK_FUSED_CHUNKS");  // experiments
        const uint32_t chunks = std::max(1u, std::min(ce ? uint32_t(atoi(ce)) : 8u, n / 32768u));
        DevBuf<unsigned long long> comps(1);
        comps.zero();
        DevBuf<uint32_t> di(size_t(n) * k);
        DevBuf<float> dd(size_t(n) * k);
        std::vector<cudaEvent_t> evs(chunks);
        uint64_t total = 0;
        for (uint32_t c = 0; c < chunks; ++c) {
            const uint32_t lo = uint32_t(uint64_t(n) * c / chunks), hi = uint32_t(uint64_t(n) * (c + 1) / chunks);
            total += replay_offers(s, lo, hi);
            const uint32_t m = hi - lo;
            LAUNCH(fill_sparse_kernel, grid_for(size_t(m) * 32, 256), 256, 0, ds->data.p, n, ds->ld, s->P, k,
                   s->keys.p, s->flags.p, s->sizes.p, comps.p, lo, hi);
            LAUNCH(finalize_kernel, grid_for(size_t(m) * k, 256), 256, 0, s->keys.p + size_t(lo) * s->P, m, s->P, k,
                   di.p + size_t(lo) * k, dd.p + size_t(lo) * k);
            CK(cudaEventCreateWithFlags(&evs[c], cudaEventDisableTiming));
            CK(cudaEventRecord(evs[c], stream()));
            CK(cudaStreamWaitEvent(copy_stream(), evs[c], 0));
            if (ids)
                CK(cudaMemcpyAsync(ids + size_t(lo) * k, di.p + size_t(lo) * k, size_t(m) * k * 4, cudaMemcpyDefault,
                                   copy_stream()));
            if (dists)
                CK(cudaMemcpyAsync(dists + size_t(lo) * k, dd.p + size_t(lo) * k, size_t(m) * k * 4,
                                   cudaMemcpyDefault, copy_stream()));
        }
        finish_round(s, total);
        if (changes) *changes = total;
        if (round_dist_comps) *round_dist_comps = s->dist_comps;
        unsigned long long fc = 0;
        comps.download(&fc, 1);
        ssync();
        CK(cudaStreamSynchronize(copy_stream()));
        for (cudaEvent_t e : evs) cudaEventDestroy(e);
        s->dist_comps += fc;
    });
}

int annk_pool_topk_accuracy(const annk_state* s, const uint32_t* gt_ids, uint32_t gt_rows, uint32_t gt_k,
                            const uint32_t* rows, double* acc) {
    return abi([&] {
        if (!rows && gt_rows != s->n) throw_invalid("accuracy hook: ground truth shape");
        if (gt_rows == 0 || gt_k == 0) throw_invalid("accuracy hook: empty ground truth");
        DevBuf<uint32_t> dgt(size_t(gt_rows) * gt_k), drows(rows ? gt_rows : 0), hits(gt_rows);
        dgt.upload(gt_ids, size_t(gt_rows) * gt_k);
        if (rows) {
            for (uint32_t r = 0; r < gt_rows; ++r)
                if (rows[r] >= s->n) throw_range("accuracy hook: row out of range");
            drows.upload(rows, gt_rows);
        }
        LAUNCH(topk_hits_kernel, grid_for(size_t(gt_rows) * 32, 256), 256, 0, s->keys.p, s->sizes.p, s->P, s->k,
               dgt.p, gt_rows, gt_k, rows ? drows.p : nullptr, hits.p);
        std::vector<uint32_t> h(gt_rows);
        hits.download(h.data(), gt_rows);
        ssync();
        double sum = 0.0;  // graph_build.cpp:213-225 summation order
        for (uint32_t r = 0; r < gt_rows; ++r) sum += double(h[r]) / double(gt_k);
        *acc = sum / gt_rows;
    });
}

int annk_state_stats(const annk_state* s, uint64_t* out) {
    return abi([&] {
        out[0] = s->join_rows;
        out[1] = s->last_offers;
        out[2] = s->last_spilled;
        out[3] = s->offer_cap;
    });
}

int annk_state_join_rows(const annk_state* s, uint64_t* rows) {
    return abi([&] { *rows = s->join_rows; });
}

}  // extern "C"
