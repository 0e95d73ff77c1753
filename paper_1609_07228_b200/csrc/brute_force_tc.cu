// brute_force_tc.cu — exact kNN on the 5th-generation tensor cores (tcgen05).
//
// Reference: proj/src/eval.cpp:17-80 (exact_row / brute_force_knn /
// brute_force_graph): per query, a NeighborPool(k) over every base id in
// ascending order, keyed by (l2_sq, id) (neighbor_pool.hpp:17-20).
//
// Exactness: on the u8 datapath every value is an integer in
// [0,255] and dim * 255^2 < 2^24, so dist = |q|^2 + |b|^2 - 2 q.b computed in
// int32 equals the reference's sequential fp32 l2_sq bit-for-bit.  The dot
// products come from tcgen05.mma.kind::i8 (u8 x u8 -> s32, exact), so the
// keys and therefore the top-k ids and distances are identical.
//
// Structure (one CTA per SM, persistent over work items):
//   work item   = 256 queries (two M=128 blocks) x one slice of base tiles
//   base tile   = 128 rows x 128 bytes, TMA (SWIZZLE_128B) into a 6-stage ring,
//                 with the tile's squared norms and -(norm >> 1) (bulk copies)
//   warp 16     = TMA producer (one elected lane)
//   warp 17     = TMEM allocator + MMA issuer (one elected lane): per tile, two
//                 M=128 N=128 K=32 MMA chains (one per query block) into a
//                 double-buffered accumulator (4 x 128 TMEM columns = 512)
//   warps 0..15 = epilogue: warp w reads query block (w/4)%2, TMEM lanes
//                 32*(w%4)..+31 and column half w/8 of every tile, i.e. ONE query
//                 per thread and one candidate list per (query, half).  Per
//                 group of 4 columns one VIADDMNMX chain bounds max(dot - norm/2);
//                 only flagged groups get the exact integer test, and the few
//                 survivors' keys are appended to the list; a full list is sorted
//                 by the whole warp in registers and cut back to k.  The two
//                 halves and the base slices are merged by bf_merge_kernel.
// The MMAs of tile t+1 overlap the epilogue of tile t.
//
// Cell-ordered scan (large inputs): a query's list threshold only falls when a
// closer row arrives, and in arbitrary row order that happens k ln(n/k) times
// per query, spread over the whole scan -- about 60% of a warp's 32x32 chunks
// then leave the one-instruction-per-pair filter for the exact test.  Rows and
// queries are therefore grouped by their nearest of ~n/1024 pivot rows (one
// extra pass of this kernel with k = 1), and a query block starts its scan at
// the tiles of its own cell: the lists converge within the first few tiles and
// the rest of the scan stays on the filter.  The visiting order never changes
// the result -- the top k by (distance, original id) of all rows -- only how
// soon the threshold reaches it.
#include <cuda.h>
#include <cub/cub.cuh>
#include <cudaTypedefs.h>

#include <algorithm>
#include <climits>
#include <cstdlib>

#include "../../include/annkit_b200.h"
#include "internal.cuh"
#include "tcgen05.cuh"

namespace annk {
namespace {

using namespace tc;

constexpr uint32_t kQB = 128;              // queries per MMA block (M)
constexpr uint32_t kNQB = 2;               // query blocks per work item
constexpr uint32_t kTQ = kQB * kNQB;       // queries per work item
constexpr uint32_t kTB = 64;               // base rows per tile (N)
constexpr uint32_t kRow = 128;             // bytes per row (K): ld8 == 128
constexpr uint32_t kStages = 12;
constexpr uint32_t kAcc = 512 / (kNQB * kTB);  // TMEM accumulator buffers (4 x 2 x 64 columns)
constexpr uint32_t kEpiWarps = 16;
constexpr uint32_t kThreadsTC = (kEpiWarps + 2) * 32;
constexpr uint32_t kTileBytes = kTB * kRow;  // 8 KB
constexpr uint32_t kABytes = kTQ * kRow;     // 32 KB
constexpr uint32_t kCB = 192;              // candidate list per (query, half), global memory
constexpr int kSortV = 8;                  // keys per lane in the list sorts (next pow2 of kCB, / 32)
constexpr uint32_t kChunks = kTB / 64;     // 32-column chunks per warp per tile (two warps per row)
constexpr uint32_t kStageStride = 36;     // words per lane in the survivor staging area (conflict-free v4)
constexpr uint32_t kRingWords = 3 * kTB;  // per stage: the tile's norms, -(norm >> 1), original row ids
constexpr uint32_t kNormBytes = kStages * kRingWords * 4;
constexpr uint32_t kStageBytes = kEpiWarps * 32 * kStageStride * 4;
constexpr uint32_t kSmemTC = 1024 + kABytes + kStages * kTileBytes + kNormBytes + kStageBytes + kTQ * 2 * 8;

// Instruction descriptor, kind::i8: D s32 (bits 4-5 = 2), A/B unsigned (0),
// both K-major, N >> 3 at bits 17-22, M >> 4 at bits 24-28.
constexpr uint32_t kIdesc = (2u << 4) | ((kTB >> 3) << 17) | ((kQB >> 4) << 24);

constexpr uint32_t kEndTile = 0xffffffffu;  // stage marker: the item has no more tiles

struct TcArgs {
    const int32_t* bnorm;
    const int32_t* nhalf;  // -(bnorm >> 1)
    uint32_t nb;
    const int32_t* qnorm;
    uint32_t nq;
    const uint32_t* self_ids;
    uint32_t k;
    uint32_t splits;
    uint32_t tiles_per_split;
    uint32_t n_items;
    uint64_t* cand;  // gridDim.x x kTQ x kCB
    uint64_t* out;   // nq x out_lists x k; this launch fills lists out_first + (split * 2 + half)
    uint32_t out_lists, out_first;
    // pruned scan (all null otherwise): base rows / queries are stored grouped by cell
    const uint32_t* bperm;       // stored base row -> original id (the id of the keys)
    const uint32_t* qperm;       // stored query -> original query index (the output row)
    const uint2* item_range;     // per query block: the tile range [x, y) to visit (splits == 1)
    const uint32_t* tile_bits;   // per query block: bitmap of the tiles to visit (splits == 1)
    uint32_t words_per_item;
    const uint32_t* tile_list;   // per query block: the tiles to visit, in order (list_stride entries, splits == 1)
    const uint32_t* tile_count;
    uint32_t list_stride;
    const uint64_t* thr0;        // per stored query: a key its k-th neighbour is known to be below
    int32_t* blockmin;           // blockmin mode (no lists): per (query block, base row) the smallest distance
    uint64_t* argmin;            // argmin mode (no lists, splits == 1): per query the key of its nearest base row
    uint32_t dbg;                // timing experiments only (ANNK_BF_DBG): 1 = no filter, 2 = filter, never a hit
};

// Fallback cut (more than kCB - 32 keys tie at the k-th distance): sort the
// list with the whole warp and keep exactly its k best.
__device__ __noinline__ uint32_t flush_sort(uint64_t* b, uint32_t cnt, uint32_t k, uint32_t lane) {
    uint64_t v[kSortV];
#pragma unroll
    for (int r = 0; r < kSortV; ++r) {
        const uint32_t e = uint32_t(r) * 32 + lane;
        v[r] = e < cnt ? b[e] : kEmptyKey;
    }
    warp_sort_regs<kSortV>(v);
    __syncwarp();
    const uint32_t keep = min(cnt, k);
#pragma unroll
    for (int r = 0; r < kSortV; ++r) {
        const uint32_t e = uint32_t(r) * 32 + lane;
        if (e < keep) b[e] = v[r];
    }
    __syncwarp();
    return keep;
}

struct Cut {
    uint32_t n;     // keys kept (>= k)
    uint64_t tkey;  // every key of the list that can still matter is <= tkey
};

// Cut a full candidate list (cnt > k keys) back to the keys whose distance is
// at most T = its k-th smallest distance (ties kept, so at least k remain; the
// list stays unsorted).  T is found by a warp-wide binary search on the integer
// distance (< 2^24 on the u8 datapath) between the list's min and max: at most
// 24 rounds (about log2 of the span) of count(d <= mid) with one
// REDUX each — a fraction of a full sort's work.  The new filter bound is
// (T, max id): any later key with a larger distance cannot reach the top k.
__device__ __noinline__ Cut flush_buffer(uint64_t* b, uint32_t cnt, uint32_t k, uint32_t lane) {
    constexpr int V = kCB / 32;
    uint64_t v[V];
    uint32_t dv[V];
#pragma unroll
    for (int r = 0; r < V; ++r) {
        const uint32_t e = uint32_t(r) * 32 + lane;
        v[r] = e < cnt ? b[e] : kEmptyKey;
        dv[r] = e < cnt ? uint32_t(key_dist(v[r])) : 0xffffffffu;
    }
    // smallest T with #{d <= T} >= k lies in [min d, max d] of the list (cnt > k):
    // the list's own span is far narrower than 2^24 once it has converged
    uint32_t mn = 0xffffffffu, mx = 0;
#pragma unroll
    for (int r = 0; r < V; ++r) {
        const uint32_t e = uint32_t(r) * 32 + lane;
        if (e < cnt) {
            mn = min(mn, dv[r]);
            mx = max(mx, dv[r]);
        }
    }
    uint32_t lo = __reduce_min_sync(0xffffffffu, mn), hi = __reduce_max_sync(0xffffffffu, mx);
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        uint32_t c = 0;
#pragma unroll
        for (int r = 0; r < V; ++r) c += dv[r] <= mid ? 1u : 0u;
        if (__reduce_add_sync(0xffffffffu, c) >= k) hi = mid;
        else lo = mid + 1;
    }
    uint32_t n = 0;
    const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
    for (int r = 0; r < V; ++r) {
        const bool keep = dv[r] <= lo;
        const uint32_t bal = __ballot_sync(0xffffffffu, keep);
        if (keep) b[n + __popc(bal & lt)] = v[r];
        n += __popc(bal);
    }
    __syncwarp();
    return Cut{n, (uint64_t(__float_as_uint(float(lo))) << 32) | 0xffffffffull};
}

// Write the k best keys of a candidate buffer (cnt <= kCB keys, distinct ids), unsorted, padded
// with kEmptyKey: the k-th smallest key is found by a warp-wide binary search on the distance
// and, only if several keys tie at it, on the id -- a few hundred instructions where a sort of
// the list costs thousands; whoever merges the lists orders them.
__device__ __noinline__ void emit_topk(const uint64_t* b, uint32_t cnt, uint32_t k, uint64_t* o, uint32_t lane) {
    constexpr int V = kCB / 32;
    uint64_t v[V];
#pragma unroll
    for (int r = 0; r < V; ++r) {
        const uint32_t e = uint32_t(r) * 32 + lane;
        v[r] = e < cnt ? b[e] : kEmptyKey;
    }
    uint64_t kth = kEmptyKey - 1;  // keep key <= kth
    if (cnt > k && k == 1) {
        uint64_t m = v[0];
#pragma unroll
        for (int r = 1; r < V; ++r) m = min(m, v[r]);
        for (int o = 16; o > 0; o >>= 1) m = min(m, __shfl_xor_sync(0xffffffffu, m, o));
        kth = m;
    } else if (cnt > k) {
        uint32_t dv[V];  // integer distances; empty slots above every bound
        uint32_t mn = 0xffffffffu, mx = 0;
#pragma unroll
        for (int r = 0; r < V; ++r) {
            dv[r] = v[r] != kEmptyKey ? uint32_t(key_dist(v[r])) : 0xffffffffu;
            mn = min(mn, dv[r]);
            if (v[r] != kEmptyKey) mx = max(mx, dv[r]);
        }
        uint32_t lo = __reduce_min_sync(0xffffffffu, mn), hi = __reduce_max_sync(0xffffffffu, mx);
        while (lo < hi) {  // smallest T with #{d <= T} >= k
            const uint32_t mid = (lo + hi) >> 1;
            uint32_t c = 0;
#pragma unroll
            for (int r = 0; r < V; ++r) c += dv[r] <= mid ? 1u : 0u;
            if (__reduce_add_sync(0xffffffffu, c) >= k) hi = mid;
            else lo = mid + 1;
        }
        uint32_t c_lt = 0, c_le = 0;
#pragma unroll
        for (int r = 0; r < V; ++r) {
            c_lt += dv[r] < lo ? 1u : 0u;
            c_le += dv[r] <= lo ? 1u : 0u;
        }
        c_lt = __reduce_add_sync(0xffffffffu, c_lt);
        c_le = __reduce_add_sync(0xffffffffu, c_le);
        uint32_t id_hi = 0xffffffffu;
        if (c_le > k) {  // ties at T: the k - c_lt smallest ids among them
            const uint32_t want = k - c_lt;
            uint32_t a0 = 0, a1 = 0xffffffffu;
            while (a0 < a1) {  // smallest id bound with #{d == T, id <= bound} >= want
                const uint32_t mid = a0 + (a1 - a0) / 2;
                uint32_t c = 0;
#pragma unroll
                for (int r = 0; r < V; ++r)
                    c += (dv[r] == lo && uint32_t(v[r]) <= mid) ? 1u : 0u;
                if (__reduce_add_sync(0xffffffffu, c) >= want) a1 = mid;
                else a0 = mid + 1;
            }
            id_hi = a0;
        }
        kth = make_key(float(lo), id_hi);
    }
    uint32_t n = 0;
    const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
    for (int r = 0; r < V; ++r) {
        const bool keep = v[r] <= kth;
        const uint32_t bal = __ballot_sync(0xffffffffu, keep);
        if (keep) o[n + __popc(bal & lt)] = v[r];
        n += __popc(bal);
    }
    for (uint32_t e = n + lane; e < k; e += 32) o[e] = kEmptyKey;
    __syncwarp();
}

__global__ void __launch_bounds__(kThreadsTC, 1)
bf_tc_u8_kernel(const __grid_constant__ CUtensorMap tm_base, const __grid_constant__ CUtensorMap tm_q, TcArgs a) {
    extern __shared__ unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t full_bar[kStages], empty_bar[kStages], tfull_bar[kAcc], tempty_bar[kAcc];
    __shared__ __align__(8) uint64_t afull_bar, aempty_bar;
    __shared__ uint32_t tmem_base_s;
    __shared__ uint32_t stage_tile[kStages];  // the tile each stage holds (kEndTile: end of the item)

    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t sbase = (smem_u32(smem_raw) + 1023u) & ~1023u;  // 1024-aligned (swizzle atoms)
    const uint32_t sA = sbase, sB = sbase + kABytes, sN = sB + kStages * kTileBytes;
    const uint32_t n_tiles = (a.nb + kTB - 1) / kTB;

    if (tid == 0) {
        for (uint32_t s = 0; s < kStages; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&empty_bar[s], 1 + kEpiWarps);  // MMA commit + every epilogue warp (norms)
        }
        for (uint32_t b = 0; b < kAcc; ++b) {
            mbar_init(&tfull_bar[b], 1);
            mbar_init(&tempty_bar[b], kEpiWarps);
        }
        mbar_init(&afull_bar, 1);
        mbar_init(&aempty_bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (warp == kEpiWarps + 1) {  // TMEM: 4 accumulators of 128 columns
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                         smem_u32(&tmem_base_s))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base_s;

    // The producer decides which tiles an item visits (a slice of the base, a tile
    // range, or the set bits of a bitmap) and labels every stage with its tile; an
    // end marker closes the item.  The MMA lane and the epilogue warps follow the labels.
    if (warp == kEpiWarps) {
        // ------------------------------------------------------------ TMA producer
        // (lane 0 issues; the warp reads an item's tile bitmap 32 words at a time)
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm_base)) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm_q)) : "memory");
        }
        uint32_t it = 0, ni = 0;
        auto push = [&](uint32_t tile) {  // lane 0 only
            const uint32_t s = it % kStages;
            mbar_wait_backoff(&empty_bar[s], ((it / kStages) & 1) ^ 1);
            stage_tile[s] = tile;
            if (tile == kEndTile) {
                mbar_arrive(&full_bar[s]);
            } else {
                mbar_expect_tx(&full_bar[s], kTileBytes + kTB * (a.bperm ? 12 : 8));
                tma_load_2d(sB + s * kTileBytes, &tm_base, &full_bar[s], 0, int32_t(tile * kTB));
                // (norm and id arrays are padded to whole tiles: rows past the end read as sentinels)
                bulk_load(sN + s * kRingWords * 4, a.bnorm + size_t(tile) * kTB, kTB * 4, &full_bar[s]);
                bulk_load(sN + s * kRingWords * 4 + kTB * 4, a.nhalf + size_t(tile) * kTB, kTB * 4, &full_bar[s]);
                if (a.bperm)
                    bulk_load(sN + s * kRingWords * 4 + kTB * 8, a.bperm + size_t(tile) * kTB, kTB * 4, &full_bar[s]);
            }
            ++it;
        };
        for (uint32_t item = blockIdx.x; item < a.n_items; item += gridDim.x, ++ni) {
            const uint32_t qb = item / a.splits, split = item % a.splits;
            if (lane == 0) {
                mbar_wait_backoff(&aempty_bar, (ni & 1) ^ 1);
                mbar_expect_tx(&afull_bar, kABytes);
                for (uint32_t h = 0; h < kNQB; ++h)
                    tma_load_2d(sA + h * kQB * kRow, &tm_q, &afull_bar, 0, int32_t(qb * kTQ + h * kQB));
            }
            if (a.tile_list) {
                const uint32_t* l = a.tile_list + size_t(qb) * a.list_stride;
                const uint32_t n = __ldg(a.tile_count + qb);
                for (uint32_t e0 = 0; e0 < n; e0 += 32) {
                    const uint32_t mine = e0 + lane < n ? __ldg(l + e0 + lane) : 0u;
                    for (uint32_t e = 0; e < min(32u, n - e0); ++e) {
                        const uint32_t tile = __shfl_sync(0xffffffffu, mine, e);
                        if (lane == 0) push(tile);
                    }
                    __syncwarp();
                }
            } else if (a.tile_bits) {
                const uint32_t* w = a.tile_bits + size_t(qb) * a.words_per_item;
                for (uint32_t w0 = 0; w0 < a.words_per_item; w0 += 32) {
                    const uint32_t mine = w0 + lane < a.words_per_item ? __ldg(w + w0 + lane) : 0u;
                    uint32_t nz = __ballot_sync(0xffffffffu, mine != 0);
                    while (nz) {
                        const uint32_t src = __ffs(nz) - 1;
                        nz &= nz - 1;
                        uint32_t bits = __shfl_sync(0xffffffffu, mine, src);
                        if (lane == 0)
                            for (; bits; bits &= bits - 1) push((w0 + src) * 32 + __ffs(bits) - 1);
                        __syncwarp();
                    }
                }
            } else if (lane == 0) {
                uint32_t t0 = split * a.tiles_per_split, t1 = min(n_tiles, t0 + a.tiles_per_split);
                if (a.item_range) {
                    t0 = a.item_range[qb].x;
                    t1 = a.item_range[qb].y;
                }
                for (uint32_t t = t0; t < t1; ++t) push(t);
            }
            if (lane == 0) push(kEndTile);
            __syncwarp();
        }
    } else if (warp == kEpiWarps + 1) {
        // ------------------------------------------------------------ MMA issuer
        if (lane == 0) {
            uint32_t it = 0, ia = 0, ni = 0;
            for (uint32_t item = blockIdx.x; item < a.n_items; item += gridDim.x, ++ni) {
                mbar_wait_backoff(&afull_bar, ni & 1);
                tc_fence_after();
                for (;; ++it) {
                    const uint32_t s = it % kStages;
                    mbar_wait(&full_bar[s], (it / kStages) & 1);  // the MMA lane polls without backoff
                    if (stage_tile[s] == kEndTile) {
                        mbar_arrive(&empty_bar[s]);
                        ++it;
                        break;
                    }
                    const uint32_t b = ia % kAcc;
                    mbar_wait(&tempty_bar[b], ((ia / kAcc) & 1) ^ 1);
                    tc_fence_after();
#pragma unroll
                    for (uint32_t h = 0; h < kNQB; ++h)
#pragma unroll
                        for (uint32_t kk = 0; kk < kRow / 32; ++kk)
                            mma_i8(tmem + (b * kNQB + h) * kTB, sdesc_sw128(sA + h * kQB * kRow + kk * 32),
                                   sdesc_sw128(sB + s * kTileBytes + kk * 32), kIdesc, kk);
                    tc_commit(&empty_bar[s]);  // smem stage free once these MMAs have read it
                    tc_commit(&tfull_bar[b]);  // accumulator b ready for the epilogue
                    ++ia;
                }
                tc_commit(&aempty_bar);  // query tiles free once the item's MMAs are done
            }
        }
    } else {
        // ------------------------------------------------------------ epilogue
        // warp w: query block h, TMEM lane quarter, column half of every tile; each
        // (query, half) keeps its own candidate list (merged with the splits on the host)
        const uint32_t h = (warp >> 2) & 1, quarter = warp & 3, half = warp >> 3;
        const uint32_t row = h * kQB + quarter * 32 + lane;  // query within the item
        const size_t cbase = (size_t(blockIdx.x) * 2 + half) * kTQ;  // this half's candidate lists
        uint64_t* buf = a.cand + (cbase + row) * kCB;
        const int32_t* ring = reinterpret_cast<const int32_t*>(smem_raw + (sN - smem_u32(smem_raw)));
        uint32_t* st = reinterpret_cast<uint32_t*>(smem_raw + (sN + kNormBytes - smem_u32(smem_raw))) +
                       (warp * 32 + lane) * kStageStride;
        // each half publishes its list's k-th key; the other half filters with the smaller one
        // (the union's k-th is at most either), which roughly halves the survivors
        uint64_t* share = reinterpret_cast<uint64_t*>(smem_raw + (sN + kNormBytes + kStageBytes - smem_u32(smem_raw)));
        uint64_t* my_share = share + row * 2 + half;
        const uint64_t* other_share = share + row * 2 + (half ^ 1);
        uint32_t it = 0, ia = 0;
        for (uint32_t item = blockIdx.x; item < a.n_items; item += gridDim.x) {
            const uint32_t qb = item / a.splits, split = item % a.splits;
            const uint32_t qi = qb * kTQ + row;
            const bool qvalid = qi < a.nq;
            const int32_t qn = qvalid ? a.qnorm[qi] : 0;
            const uint32_t self = (a.self_ids && qvalid) ? a.self_ids[qi] : kInvalidId;
            uint32_t cnt = 0;
            int32_t best_v = INT_MAX, best_j = 0;  // argmin mode: smallest bn - 2 dot and its row
            uint64_t thr = (a.thr0 && qvalid) ? a.thr0[qi] : kEmptyKey;
            // keep iff qn + bn - 2 dot <= T  <=>  2 dot - bn >= qn - T = lim (ties settled by the key).
            // Necessary condition with h = bn >> 1: dot - h >= ceil(lim / 2) = L, evaluated per
            // group of 4 columns as max(dot + (-h)) with one VIADDMNMX per pair.
            int32_t lim = qvalid ? (thr == kEmptyKey ? INT_MIN : qn - int32_t(key_dist(thr))) : INT_MAX;
            int32_t L = qvalid ? (lim == INT_MIN ? INT_MIN / 2 : (lim + 1) >> 1) : INT_MAX;
            *my_share = thr;
            asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * 32) : "memory");  // shares reset for this item
            for (;; ++it) {
                const uint32_t s = it % kStages;
                mbar_wait(&full_bar[s], (it / kStages) & 1);  // stage label and column norms landed
                const uint32_t tile = stage_tile[s];
                if (tile == kEndTile) {
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&empty_bar[s]);
                    ++it;
                    break;
                }
                const uint32_t b = ia % kAcc;
                {
                    const uint64_t o = *reinterpret_cast<const volatile uint64_t*>(other_share);
                    if (qvalid && o < thr) {
                        thr = o;
                        lim = qn - int32_t(key_dist(thr));
                        L = (lim + 1) >> 1;
                    }
                }
                mbar_wait(&tfull_bar[b], (ia / kAcc) & 1);
                tc_fence_after();
                const uint32_t taddr = tmem + ((quarter * 32) << 16) + (b * kNQB + h) * kTB;
#pragma unroll 1
                for (uint32_t c = half * kChunks; c < (half + 1) * kChunks; ++c) {
                    uint32_t d[32];
                    tmem_ld32_async(taddr + c * 32, d);
                    tmem_wait(d);
                    if (c == (half + 1) * kChunks - 1) {  // our columns of accumulator b read: release
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&tempty_bar[b]);
                    }
                    if (a.dbg & 1) continue;
                    const uint32_t j0 = tile * kTB + c * 32;
                    const int32_t* rowp = ring + s * kRingWords + c * 32;  // exact norms; + kTB: -(norm >> 1); + 2 kTB: ids
                    if (a.blockmin) {
                        // blockmin mode: the smallest distance of this warp's 32 queries to every column
                        int32_t mine = INT_MAX;
#pragma unroll
                        for (int e = 0; e < 32; ++e) {
                            const int32_t v = qvalid ? qn - 2 * int32_t(d[e]) : INT_MAX / 2;
                            const int32_t r = __reduce_min_sync(0xffffffffu, v);
                            if (lane == uint32_t(e)) mine = r;
                        }
                        if (j0 + lane < a.nb) atomicMin(a.blockmin + size_t(qb) * a.nb + j0 + lane, mine + rowp[lane]);
                        continue;
                    }
                    if (a.argmin) {
                        // argmin mode: running minimum of bn - 2 dot over the columns (padding rows carry
                        // sentinel norms); the first of equal values wins within a list
#pragma unroll
                        for (int g4 = 0; g4 < 8; ++g4) {
                            const int4 bv = *reinterpret_cast<const int4*>(rowp + 4 * g4);
                            const int32_t x0 = bv.x - 2 * int32_t(d[4 * g4]), x1 = bv.y - 2 * int32_t(d[4 * g4 + 1]);
                            const int32_t x2 = bv.z - 2 * int32_t(d[4 * g4 + 2]), x3 = bv.w - 2 * int32_t(d[4 * g4 + 3]);
                            if (x0 < best_v) { best_v = x0; best_j = int32_t(j0 + 4 * g4); }
                            if (x1 < best_v) { best_v = x1; best_j = int32_t(j0 + 4 * g4 + 1); }
                            if (x2 < best_v) { best_v = x2; best_j = int32_t(j0 + 4 * g4 + 2); }
                            if (x3 < best_v) { best_v = x3; best_j = int32_t(j0 + 4 * g4 + 3); }
                        }
                        continue;
                    }
                    int32_t g[8];
#pragma unroll
                    for (int gi = 0; gi < 8; ++gi) {
                        const int4 hv = *reinterpret_cast<const int4*>(rowp + kTB + 4 * gi);
                        g[gi] = __viaddmax_s32(int32_t(d[4 * gi]), hv.x,
                                               __viaddmax_s32(int32_t(d[4 * gi + 1]), hv.y,
                                                              __viaddmax_s32(int32_t(d[4 * gi + 2]), hv.z,
                                                                             int32_t(d[4 * gi + 3]) + hv.w)));
                    }
                    const int32_t mx = max(max(max(g[0], g[1]), max(g[2], g[3])), max(max(g[4], g[5]), max(g[6], g[7])));
                    const bool hit = mx >= L && !(a.dbg & 2);
                    if (!__any_sync(0xffffffffu, hit)) continue;
                    // groups that may hold survivors; the row chunk is staged for their exact test
                    uint32_t gm = 0;
                    if (hit) {
#pragma unroll
                        for (int gi = 0; gi < 8; ++gi) gm |= uint32_t(g[gi] >= L) << gi;
#pragma unroll
                        for (int v = 0; v < 32; v += 4)
                            *reinterpret_cast<uint4*>(st + v) = make_uint4(d[v], d[v + 1], d[v + 2], d[v + 3]);
                    }
                    // room for up to 4 survivors per flagged group in every buffer that takes some
                    uint32_t need = __ballot_sync(0xffffffffu, cnt + 4 * __popc(gm) > kCB);
                    while (need) {
                        const uint32_t src = __ffs(need) - 1;
                        need &= need - 1;
                        uint64_t* sb = a.cand + (cbase + row - lane + src) * kCB;
                        const uint32_t sc = __shfl_sync(0xffffffffu, cnt, src);
                        Cut cut = flush_buffer(sb, sc, a.k, lane);
                        if (cut.n + 32 > kCB) {  // too many ties at the k-th distance: exact cut
                            cut.n = flush_sort(sb, cut.n, a.k, lane);  // (the cut compacted the list to cut.n keys)
                            cut.tkey = sb[a.k - 1];
                        }
                        if (lane == src) {
                            cnt = cut.n;
                            if (cut.tkey < thr) {
                                thr = cut.tkey;
                                lim = qn - int32_t(key_dist(thr));
                                L = (lim + 1) >> 1;
                                *reinterpret_cast<volatile uint64_t*>(my_share) = thr;
                            }
                        }
                    }
                    while (gm) {  // exact test of the flagged groups' columns
                        const uint32_t gi = __ffs(gm) - 1;
                        gm &= gm - 1;
                        const uint4 dv = *reinterpret_cast<const uint4*>(st + 4 * gi);
                        const uint32_t jg = j0 + 4 * gi;
                        const int4 bv = *reinterpret_cast<const int4*>(rowp + 4 * gi);
                        const int32_t xs[4] = {int32_t(2 * dv.x) - bv.x, int32_t(2 * dv.y) - bv.y,
                                               int32_t(2 * dv.z) - bv.z, int32_t(2 * dv.w) - bv.w};
#pragma unroll
                        for (int e2 = 0; e2 < 4; ++e2) {
                            if (xs[e2] >= lim && jg + e2 < a.nb) {
                                const uint32_t j = a.bperm ? uint32_t(rowp[2 * kTB + 4 * gi + e2]) : jg + e2;
                                const uint64_t key = make_key(float(qn - xs[e2]), j);
                                if (j != self && key < thr) {
                                    DCHK(cnt < kCB);
                                    buf[cnt++] = key;
                                }
                            }
                        }
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty_bar[s]);  // this tile's column norms are no longer read
                ++ia;
            }
            if (a.blockmin) continue;
            if (a.argmin) {  // the two column halves of a query meet in shared memory
                const uint64_t mine = (uint64_t(uint32_t(best_v) ^ 0x80000000u) << 32) | uint32_t(best_j);
                if (half == 1) *my_share = mine;
                asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * 32) : "memory");
                if (half == 0 && qvalid) {
                    const uint64_t o = *other_share, m = min(mine, o);
                    const int32_t v = int32_t(uint32_t(m >> 32) ^ 0x80000000u);
                    a.argmin[qi] = make_key(float(qn + v), uint32_t(m));
                }
                asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * 32) : "memory");  // read before the next item's reset
                continue;
            }
            // final top-k of every query of this warp, written in (query, split) order
#pragma unroll 1
            for (uint32_t src = 0; src < 32; ++src) {
                const uint32_t sq = qb * kTQ + row - lane + src;
                if (sq >= a.nq) break;
                const uint64_t* sb = a.cand + (cbase + row - lane + src) * kCB;
                const uint32_t sc = __shfl_sync(0xffffffffu, cnt, src);
                const uint32_t oq = a.qperm ? a.qperm[sq] : sq;
                uint64_t* o = a.out + (size_t(oq) * a.out_lists + a.out_first + split * 2 + half) * a.k;
                if (sc == 0) {
                    for (uint32_t e = lane; e < a.k; e += 32) o[e] = kEmptyKey;
                    __syncwarp();
                } else {
                    emit_topk(sb, sc, a.k, o, lane);
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == kEpiWarps + 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
    }
}

// Tile-padded copies of the base norms and of -(norm >> 1), optionally through
// a row permutation; entries past the end hold sentinels (the exact test then
// rejects them by index).
__global__ void pad_norms_kernel(const int32_t* __restrict__ n, const uint32_t* __restrict__ perm, uint32_t cnt,
                                 uint32_t padded, int32_t* __restrict__ norms, int32_t* __restrict__ nhalf) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < padded; i += gridDim.x * blockDim.x) {
        const int32_t v = i < cnt ? n[perm ? perm[i] : i] : 0;
        norms[i] = i < cnt ? v : INT_MAX / 2;
        nhalf[i] = i < cnt ? -(v >> 1) : INT_MIN / 2;
    }
}

// ---- pruned scan: helpers

// sum of the rows' distances to their nearest pivot (the high word of their k = 1 key)
__global__ void near_sum_kernel(const uint64_t* __restrict__ keys, uint32_t n, unsigned long long* __restrict__ sum) {
    unsigned long long v = 0;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        v += uint32_t(key_dist(keys[i]));
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(sum, v);
}

// cell of every row = its nearest pivot; a row farther than twice the mean
// nearest-pivot distance goes to the outlier cell C (never pruned, so it
// needs no radius).  r2[c] = largest squared distance of a member to pivot c.
__global__ void cells_kernel(const uint64_t* __restrict__ keys, uint32_t n, uint32_t C,
                             const unsigned long long* __restrict__ sum, uint32_t sum_n,
                             uint32_t* __restrict__ cells, uint32_t* __restrict__ vals, int32_t* __restrict__ r2) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint64_t key = keys[i];
    const uint32_t d = uint32_t(key_dist(key)), c = uint32_t(key);
    const bool far = (unsigned long long)(d) * sum_n > 2ull * *sum || c >= C;
    cells[i] = far ? C : c;
    vals[i] = i;
    if (!far && r2) atomicMax(r2 + c, int32_t(d));
}

// out row p = in row perm[p] (128-byte rows, 8 threads per row), with the rows' norms and self ids
__global__ void gather_cells_kernel(const uint8_t* __restrict__ in, const uint32_t* __restrict__ perm, uint32_t n,
                                    uint8_t* __restrict__ out, const int32_t* __restrict__ nin,
                                    int32_t* __restrict__ nout, const uint32_t* __restrict__ sin,
                                    uint32_t* __restrict__ sout) {
    const uint32_t e = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t r = e >> 3, c = e & 7;
    if (r >= n) return;
    const uint32_t src = perm[r];
    reinterpret_cast<uint4*>(out + size_t(r) * kRow)[c] = __ldg(reinterpret_cast<const uint4*>(in + size_t(src) * kRow) + c);
    if (c == 0) {
        if (nout) nout[r] = nin[src];
        if (sout) sout[r] = sin[src];
    }
}

// pivot rows: evenly spaced base rows
__global__ void pivots_kernel(const uint8_t* __restrict__ in, const int32_t* __restrict__ nin, uint32_t n, uint32_t C,
                              uint8_t* __restrict__ out, int32_t* __restrict__ nout) {
    const uint32_t e = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t r = e >> 3, c = e & 7;
    if (r >= C) return;
    const uint32_t src = uint32_t(uint64_t(r) * n / C);
    reinterpret_cast<uint4*>(out + size_t(r) * kRow)[c] = __ldg(reinterpret_cast<const uint4*>(in + size_t(src) * kRow) + c);
    if (c == 0) nout[r] = nin[src];
}

// start[c] = first stored base row of cell c, c = 0..C+1 (start[C+1] = n)
__global__ void cell_starts_kernel(const uint32_t* __restrict__ sorted_cells, uint32_t n, uint32_t C,
                                   uint32_t* __restrict__ start) {
    const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c > C + 1) return;
    uint32_t lo = 0, hi = n;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (sorted_cells[mid] < c) lo = mid + 1;
        else hi = mid;
    }
    start[c] = lo;
}

// Home tiles of a query block: the tiles of the n_home cells whose pivots are
// nearest to the block (smallest blockmin), nearest cell first -- for clustered
// rows the first of these are the cells of the queries' own clusters, where
// their lists converge, and the farther ones then pass on the filter alone.
constexpr uint32_t kHomeSel = 256;  // cells selected per block at most
__global__ void home_kernel(const int32_t* __restrict__ blockmin, const uint32_t* __restrict__ cell_start,
                            uint32_t C, uint32_t n_home, uint32_t words, uint32_t* __restrict__ bits,
                            uint32_t* __restrict__ list, uint32_t list_stride, uint32_t* __restrict__ count,
                            unsigned long long* __restrict__ home_tiles) {
    extern __shared__ uint32_t hs[];
    uint32_t* bm = hs;                                      // words
    int32_t* M = reinterpret_cast<int32_t*>(hs + words);    // C (INT_MAX for empty cells)
    __shared__ uint32_t cnt_s, nsel_s, sel[kHomeSel], ord[kHomeSel];
    const uint32_t qb = blockIdx.x;
    for (uint32_t w = threadIdx.x; w < words; w += blockDim.x) bm[w] = 0;
    for (uint32_t c = threadIdx.x; c < C; c += blockDim.x)
        M[c] = cell_start[c] == cell_start[c + 1] ? INT_MAX : blockmin[size_t(qb) * C + c];
    if (threadIdx.x == 0) nsel_s = 0;
    __syncthreads();
    // smallest v with #{M <= v} >= n_home (or every non-empty cell when there are fewer)
    uint32_t lo = 0, hi = 0x7ffffffeu;
    while (lo < hi) {
        const uint32_t mid = lo + (hi - lo) / 2;
        if (threadIdx.x == 0) cnt_s = 0;
        __syncthreads();
        uint32_t c_ = 0;
        for (uint32_t c = threadIdx.x; c < C; c += blockDim.x) c_ += uint32_t(M[c]) <= mid ? 1u : 0u;
        if (c_) atomicAdd(&cnt_s, c_);
        __syncthreads();
        const uint32_t tot = cnt_s;
        __syncthreads();
        if (tot >= n_home) hi = mid;
        else lo = mid + 1;
    }
    for (uint32_t c = threadIdx.x; c < C; c += blockDim.x)
        if (uint32_t(M[c]) <= lo) {
            const uint32_t q = atomicAdd(&nsel_s, 1u);
            if (q < kHomeSel) sel[q] = c;
        }
    __syncthreads();
    const uint32_t ns = min(nsel_s, kHomeSel);
    for (uint32_t t = threadIdx.x; t < ns; t += blockDim.x) {  // rank by (M, cell)
        const uint32_t c = sel[t];
        uint32_t rank = 0;
        for (uint32_t u = 0; u < ns; ++u) {
            const uint32_t o = sel[u];
            rank += (M[o] < M[c] || (M[o] == M[c] && o < c)) ? 1u : 0u;
        }
        ord[rank] = c;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t n = 0;
        for (uint32_t r = 0; r < ns; ++r) {
            const uint32_t c = ord[r];
            const uint32_t t0 = cell_start[c] / kTB, t1 = (cell_start[c + 1] - 1) / kTB;
            if (n + (t1 - t0 + 1) > list_stride) break;
            for (uint32_t t = t0; t <= t1; ++t)
                if (!(bm[t >> 5] >> (t & 31) & 1u)) {
                    bm[t >> 5] |= 1u << (t & 31);
                    list[size_t(qb) * list_stride + n++] = t;
                }
        }
        count[qb] = n;
        if (home_tiles) atomicAdd(home_tiles, (unsigned long long)n);
    }
    __syncthreads();
    for (uint32_t w = threadIdx.x; w < words; w += blockDim.x) bits[size_t(qb) * words + w] = bm[w];
}

// thr0 of a stored query = the k-th key of its home-tile list (kEmptyKey if it holds fewer)
__global__ void thr0_kernel(const uint64_t* __restrict__ fin, uint32_t lists, uint32_t k,
                            const uint32_t* __restrict__ qperm, uint32_t nq, uint64_t* __restrict__ thr0) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < nq) thr0[i] = fin[(size_t(qperm[i]) * lists) * k + k - 1];
}

// The tiles a query block still has to visit after its home tiles.  Cell c
// (pivot p, radius^2 R over its members) can hold no top-k row of any query q
// of the block when d(q, p) - sqrt(R) > sqrt(T) for the block's largest
// threshold T (triangle inequality; every distance is an exact integer
// square): with M = min_q d^2(q, p) that is M > T + R + 2 sqrt(T R), tested
// with the square root rounded up.  The outlier cell is always visited.
__global__ void prune_kernel(const int32_t* __restrict__ blockmin, const int32_t* __restrict__ r2,
                             const uint32_t* __restrict__ cell_start, uint32_t C, const uint64_t* __restrict__ thr0,
                             uint32_t nq, const uint32_t* __restrict__ home_bits, uint32_t words,
                             uint32_t* __restrict__ bits, unsigned long long* __restrict__ kept_tiles) {
    extern __shared__ uint32_t bm[];
    __shared__ uint32_t tmax_s;
    const uint32_t qb = blockIdx.x;
    if (threadIdx.x == 0) tmax_s = 0;
    for (uint32_t w = threadIdx.x; w < words; w += blockDim.x) bm[w] = 0;
    __syncthreads();
    {
        uint32_t t = 0;
        for (uint32_t q = qb * kTQ + threadIdx.x; q < min(nq, (qb + 1) * kTQ); q += blockDim.x) {
            const uint64_t key = thr0[q];
            t = max(t, key == kEmptyKey ? 0xffffffffu : uint32_t(key_dist(key)));
        }
        atomicMax(&tmax_s, t);
    }
    __syncthreads();
    const uint32_t T = tmax_s;
    for (uint32_t c = threadIdx.x; c <= C; c += blockDim.x) {
        const uint32_t b0 = cell_start[c], b1 = cell_start[c + 1];
        if (b0 == b1) continue;
        bool keep = true;
        if (c < C && T != 0xffffffffu) {
            const int64_t M = blockmin[size_t(qb) * C + c], R = r2[c];
            const uint64_t tr = uint64_t(T) * uint64_t(R);
            uint64_t sq = uint64_t(sqrt(double(tr)));
            while (sq * sq < tr) ++sq;  // ceil(sqrt(T R)) whatever the rounding of the double root
            keep = !(M > int64_t(T) + R + 2 * int64_t(sq));
        }
        if (keep)
            for (uint32_t t = b0 / kTB; t <= (b1 - 1) / kTB; ++t) atomicOr(&bm[t >> 5], 1u << (t & 31));
    }
    __syncthreads();
    unsigned long long cnt = 0;
    for (uint32_t w = threadIdx.x; w < words; w += blockDim.x) {
        const uint32_t v = bm[w] & ~home_bits[size_t(qb) * words + w];  // the home tiles are done
        bits[size_t(qb) * words + w] = v;
        cnt += __popc(v);
    }
    if (kept_tiles && cnt) atomicAdd(kept_tiles, cnt);
}

// rows x 128 u8 matrix, boxes of 128 rows x 128 bytes, 128-byte swizzle; rows
// past the end read as zeros.
CUtensorMap make_map(const uint8_t* p, uint32_t rows, uint32_t box_rows) {
    CUtensorMap m;
    const cuuint64_t dims[2] = {kRow, rows};
    const cuuint64_t strides[1] = {kRow};
    const cuuint32_t box[2] = {kRow, box_rows};
    const cuuint32_t es[2] = {1, 1};
    const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(p), dims, strides,
                                   box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
    return m;
}

struct TcProblem {
    const uint8_t* b8;      // nb x 128 bytes
    const int32_t* bnorm;   // nb
    uint32_t nb;
    const uint8_t* q8;      // nq x 128 bytes
    const int32_t* qnorm;   // nq
    uint32_t nq;
    const uint32_t* self_ids;
    uint32_t k;
};

struct TcMode {  // how one launch walks the base (defaults: every tile, or slices when queries are few)
    const uint32_t* bperm = nullptr;
    const uint32_t* qperm = nullptr;
    const uint2* item_range = nullptr;
    const uint32_t* tile_bits = nullptr;
    uint32_t words_per_item = 0;
    const uint32_t* tile_list = nullptr;
    const uint32_t* tile_count = nullptr;
    uint32_t list_stride = 0;
    const uint64_t* thr0 = nullptr;
    int32_t* blockmin = nullptr;
    uint64_t* argmin = nullptr;
    uint64_t* out = nullptr;  // nq x out_lists x k (null: a private buffer merged into out_keys)
    uint32_t out_lists = 0, out_first = 0;
    bool whole_items = false;  // one item per query block (no base slices)
};

// One launch of the kernel over `pr`; without m.out the lists are merged into out_keys.
void tc_launch(const TcProblem& pr, const TcMode& m, uint64_t* out_keys) {
    const uint32_t nb = pr.nb, nq = pr.nq, k = pr.k;
    const uint32_t n_tiles = (nb + kTB - 1) / kTB;
    const uint32_t qblocks = (nq + kTQ - 1) / kTQ;
    const uint32_t sms = uint32_t(num_sms());
    // split the base range only when there are too few query blocks to fill the GPU
    uint32_t splits = std::max(1u, std::min(n_tiles, (sms + qblocks - 1) / qblocks));
    splits = std::min(splits, std::max(1u, 2048u / k));  // 2 lists per split: merge list fits a warp
    if (m.whole_items) splits = 1;
    const uint32_t tps = (n_tiles + splits - 1) / splits;
    splits = (n_tiles + tps - 1) / tps;
    const uint32_t n_items = qblocks * splits;
    const uint32_t grid = std::min(n_items, sms);
    const uint32_t padded = n_tiles * kTB;
    DevBuf<int32_t> norms(padded), nhalf(padded);
    LAUNCH(pad_norms_kernel, std::min((padded + 255) / 256, 4096u), 256, 0, pr.bnorm, nullptr, nb, padded, norms.p,
           nhalf.p);
    const CUtensorMap tb = make_map(pr.b8, nb, kTB);
    const CUtensorMap tq = make_map(pr.q8, nq, kQB);
    DevBuf<uint64_t> cand(m.blockmin || m.argmin ? 0 : size_t(grid) * 2 * kTQ * kCB);
    DevBuf<uint64_t> part(m.out || m.blockmin || m.argmin ? 0 : size_t(nq) * splits * 2 * k);  // per (query, split, column half)
    const char* dbg = getenv("ANNK_BF_DBG");
    TcArgs args{norms.p, nhalf.p, nb, pr.qnorm, nq, pr.self_ids, k, splits, tps, n_items, cand.p,
                m.out ? m.out : part.p, m.out ? m.out_lists : splits * 2, m.out ? m.out_first : 0u,
                m.bperm, m.qperm, m.item_range, m.tile_bits, m.words_per_item, m.tile_list, m.tile_count,
                m.list_stride, m.thr0, m.blockmin, m.argmin,
                dbg ? uint32_t(atoi(dbg)) : 0u};
    CK(cudaFuncSetAttribute(bf_tc_u8_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kSmemTC)));
    LAUNCH(bf_tc_u8_kernel, grid, kThreadsTC, kSmemTC, tb, tq, args);
    if (!m.out && !m.blockmin && !m.argmin) merge_split_lists(part.p, nq, splits * 2, k, out_keys);
}

// Sort ids by cell (stable: ascending id inside a cell).
void sort_by_cell(DevBuf<uint32_t>& cells, DevBuf<uint32_t>& vals, uint32_t n, uint32_t C) {
    DevBuf<uint32_t> c2(n), v2((n + kTB - 1) / kTB * kTB);  // (ids padded to whole tiles: the kernel stages them per tile)
    int bits = 1;
    while ((1u << bits) <= C) ++bits;  // cell ids 0..C
    size_t tmp = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp, cells.p, c2.p, vals.p, v2.p, int(n), 0, bits, stream()));
    DevBuf<unsigned char> t(tmp);
    CK(cub::DeviceRadixSort::SortPairs(t.p, tmp, cells.p, c2.p, vals.p, v2.p, int(n), 0, bits, stream()));
    cells = std::move(c2);
    vals = std::move(v2);
}

struct Cells {
    DevBuf<uint32_t> cell, perm;  // sorted cell ids, stored row -> original row
};

// Nearest-pivot cell of every row of (r8, rnorm, n) and the rows' order by cell.  `sum`
// accumulates the rows' nearest-pivot distances when these are the base rows (it sets the
// outlier threshold for the queries as well).
void assign_and_sort(const uint8_t* piv8, const int32_t* pivn, uint32_t C, const uint8_t* r8, const int32_t* rnorm,
                     uint32_t n, unsigned long long* sum, uint32_t sum_n, bool is_base, int32_t* r2, Cells& out) {
    DevBuf<uint64_t> near(n);
    {
        TcMode m;
        m.argmin = near.p;
        m.whole_items = true;
        tc_launch(TcProblem{piv8, pivn, C, r8, rnorm, n, nullptr, 1}, m, nullptr);
    }
    if (is_base) LAUNCH(near_sum_kernel, 296, 256, 0, near.p, n, sum);
    out.cell.alloc(n);
    out.perm.alloc(n);
    LAUNCH(cells_kernel, (n + 255) / 256, 256, 0, near.p, n, C, sum, sum_n, out.cell.p, out.perm.p, r2);
    sort_by_cell(out.cell, out.perm, n, C);
}

// Tile counts of the last tcgen05 u8 run (annk_bf_last_scan): the device counters
// land in a pinned host triple behind the run, read after a synchronize.
uint64_t g_last_tiles_total = 0;
bool g_last_pruned = false;
unsigned long long* g_last_counts = nullptr;  // pinned: [0] pivot distance sum, [1] tiles kept by the pruning, [2] home tiles

// Exact top-k with most of the base pruned away:
//  1. cells: rows (and queries) grouped by their nearest of C pivot rows;
//  2. per (query block, pivot) the block's smallest distance to the pivot (blockmin pass);
//  3. home pass: every block scans the tiles of its own cells -> thresholds;
//  4. the cells whose members provably lie beyond every threshold of a block are dropped
//     (triangle inequality on exact integer squares), the rest is scanned with the
//     thresholds in place; home and rest lists are merged.
// The result is the same top k by (distance, original id) as the full scan's.
struct PhaseTimer {  // ANNK_BF_STATS: per-phase device times (synchronises at the end)
    bool on = getenv("ANNK_BF_STATS") != nullptr;
    std::vector<std::pair<const char*, cudaEvent_t>> ev;
    void mark(const char* name) {
        if (!on) return;
        cudaEvent_t e;
        CK(cudaEventCreate(&e));
        CK(cudaEventRecord(e, stream()));
        ev.emplace_back(name, e);
    }
    void report() {
        if (!on || ev.empty()) return;
        CK(cudaEventSynchronize(ev.back().second));
        for (size_t i = 1; i < ev.size(); ++i) {
            float ms = 0;
            CK(cudaEventElapsedTime(&ms, ev[i - 1].second, ev[i].second));
            fprintf(stderr, "[annk]   %-10s %8.3f ms\n", ev[i].first, ms);
        }
        for (auto& e : ev) cudaEventDestroy(e.second);
    }
};

void tc_run_pruned(const TcProblem& pr, uint64_t* out_keys) {
    PhaseTimer pt;
    pt.mark("start");
    const uint32_t nb = pr.nb, nq = pr.nq, k = pr.k;
    const uint32_t n_tiles = (nb + kTB - 1) / kTB, qblocks = (nq + kTQ - 1) / kTQ;
    const char* ce = getenv("ANNK_BF_CELL_ROWS");
    const uint32_t cell_rows = ce ? std::max(1, atoi(ce)) : 128;  // mean rows per cell
    const uint32_t C = std::min(8192u, std::max(64u, (nb / cell_rows + 63) / 64 * 64));
    DevBuf<uint8_t> piv8(size_t(C) * kRow);
    DevBuf<int32_t> pivn(C), r2(C);
    DevBuf<unsigned long long> sum(3);  // [0] nearest-pivot distance sum, [1] tiles kept by the pruning, [2] home tiles
    sum.zero();
    r2.zero();
    LAUNCH(pivots_kernel, (C * 8 + 255) / 256, 256, 0, pr.b8, pr.bnorm, nb, C, piv8.p, pivn.p);
    Cells bc, qc_own;
    assign_and_sort(piv8.p, pivn.p, C, pr.b8, pr.bnorm, nb, sum.p, nb, true, r2.p, bc);
    DevBuf<uint8_t> sb8(size_t(nb) * kRow), sq8;
    DevBuf<int32_t> sbn(nb), sqn;
    DevBuf<uint32_t> sself;
    const bool same = pr.q8 == pr.b8 && nq == nb;  // the queries are the base rows: one order serves both
    if (same && pr.self_ids) sself.alloc(nq);
    LAUNCH(gather_cells_kernel, (nb * 8 + 255) / 256, 256, 0, pr.b8, bc.perm.p, nb, sb8.p, pr.bnorm, sbn.p,
           same ? pr.self_ids : nullptr, same && pr.self_ids ? sself.p : nullptr);
    const Cells* qc = &bc;
    const uint8_t* q8 = sb8.p;
    const int32_t* qn = sbn.p;
    if (!same) {
        assign_and_sort(piv8.p, pivn.p, C, pr.q8, pr.qnorm, nq, sum.p, nb, false, nullptr, qc_own);
        sq8.alloc(size_t(nq) * kRow);
        sqn.alloc(nq);
        if (pr.self_ids) sself.alloc(nq);
        LAUNCH(gather_cells_kernel, (nq * 8 + 255) / 256, 256, 0, pr.q8, qc_own.perm.p, nq, sq8.p, pr.qnorm, sqn.p,
               pr.self_ids, pr.self_ids ? sself.p : nullptr);
        qc = &qc_own;
        q8 = sq8.p;
        qn = sqn.p;
    }
    pt.mark("cells");
    const uint32_t* self = pr.self_ids ? sself.p : nullptr;
    DevBuf<uint32_t> cstart(C + 2);
    LAUNCH(cell_starts_kernel, (C + 2 + 127) / 128, 128, 0, bc.cell.p, nb, C, cstart.p);
    // blockmin pass: stored queries x pivots
    DevBuf<int32_t> bmin(size_t(qblocks) * C);
    bmin.fill_bytes(0x7f);
    {
        TcMode m;
        m.blockmin = bmin.p;
        m.whole_items = true;
        tc_launch(TcProblem{piv8.p, pivn.p, C, q8, qn, nq, nullptr, 1}, m, nullptr);
    }
    pt.mark("blockmin");
    // home pass
    const uint32_t words = (n_tiles + 31) / 32;
    DevBuf<uint32_t> hbits(size_t(qblocks) * words), bits(size_t(qblocks) * words);
    const char* he = getenv("ANNK_BF_HOME_CELLS");
    CK(cudaFuncSetAttribute(home_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int((words + C) * 4)));
    CK(cudaFuncSetAttribute(prune_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(words * 4)));
    const uint32_t hstride = 1024;
    DevBuf<uint32_t> hlist(size_t(qblocks) * hstride), hcount(qblocks);
    LAUNCH(home_kernel, qblocks, 256, (words + C) * 4, bmin.p, cstart.p, C, he ? uint32_t(atoi(he)) : std::min(128u, std::max(16u, C / 64)), words,
           hbits.p, hlist.p, hstride, hcount.p, sum.p + 2);
    const TcProblem sp{sb8.p, sbn.p, nb, q8, qn, nq, self, k};
    DevBuf<uint64_t> fin(size_t(nq) * 3 * k);  // per query: home top-k, then the rest pass's two half lists
    {
        DevBuf<uint64_t> home(size_t(nq) * 2 * k);
        TcMode m;
        m.bperm = bc.perm.p;
        m.qperm = qc->perm.p;
        m.tile_list = hlist.p;
        m.tile_count = hcount.p;
        m.list_stride = hstride;
        m.whole_items = true;
        m.out = home.p;
        m.out_lists = 2;
        tc_launch(sp, m, nullptr);
        merge_split_lists(home.p, nq, 2, k, fin.p, 3 * k);
    }
    pt.mark("home");
    DevBuf<uint64_t> thr0(nq);
    LAUNCH(thr0_kernel, (nq + 255) / 256, 256, 0, fin.p, 3u, k, qc->perm.p, nq, thr0.p);
    LAUNCH(prune_kernel, qblocks, 256, words * 4, bmin.p, r2.p, cstart.p, C, thr0.p, nq, hbits.p, words, bits.p,
           sum.p + 1);
    pt.mark("prune");
    {
        TcMode m;
        m.bperm = bc.perm.p;
        m.qperm = qc->perm.p;
        m.tile_bits = bits.p;
        m.words_per_item = words;
        m.thr0 = thr0.p;
        m.whole_items = true;
        m.out = fin.p;
        m.out_lists = 3;
        m.out_first = 1;
        tc_launch(sp, m, nullptr);
    }
    pt.mark("rest");
    merge_split_lists(fin.p, nq, 3, k, out_keys, 0, true);
    pt.mark("merge");
    pt.report();
    if (!g_last_counts) CK(cudaMallocHost(&g_last_counts, 3 * sizeof(unsigned long long)));
    CK(cudaMemcpyAsync(g_last_counts, sum.p, 3 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, stream()));
    g_last_tiles_total = uint64_t(qblocks) * n_tiles;
    g_last_pruned = true;
    if (getenv("ANNK_BF_STATS")) {  // (synchronises) how much of the base the rest pass visited
        ssync();
        fprintf(stderr, "[annk] pruned exact kNN: %u cells, tiles visited %llu of %llu (home %llu)\n", C,
                g_last_counts[1] + g_last_counts[2], (unsigned long long)g_last_tiles_total, g_last_counts[2]);
    }
}

void tc_run(const TcProblem& pr, uint64_t* out_keys) {
    const uint32_t n_tiles = (pr.nb + kTB - 1) / kTB, qblocks = (pr.nq + kTQ - 1) / kTQ;
    const char* env = getenv("ANNK_BF_CELLS");  // 1: also for small inputs (tests), 0: never
    const bool force = env && atoi(env) == 1, off = env && atoi(env) == 0;
    // pruned scan: inputs large enough to pay for the extra passes
    const bool pruned = !off && n_tiles >= 8 && pr.nb > pr.k + 2 * kTB &&
                        (force || (qblocks >= uint32_t(num_sms()) && pr.nb >= 16384));
    if (pruned) tc_run_pruned(pr, out_keys);
    else {
        tc_launch(pr, TcMode{}, out_keys);
        g_last_tiles_total = uint64_t(qblocks) * n_tiles;
        g_last_pruned = false;
    }
}

}  // namespace

// Exact kNN on tcgen05 for the u8 datapath with 128-byte rows; returns false
// (nothing launched) when the shape is not supported.
bool brute_force_tc(const annk_dataset* base, uint32_t nq, const uint32_t* self_ids, uint32_t k,
                    uint64_t* out_keys, const uint8_t* q8, const int32_t* qnorm) {
    if (!base->u8 || q8 == nullptr || base->ld8 != kRow || k == 0 || k > 128 || nq == 0) return false;
    if (getenv("ANNK_BF_MMA_SYNC")) return false;
    tc_run(TcProblem{base->data8.p, base->norms8.p, base->n, q8, qnorm, nq, self_ids, k}, out_keys);
    return true;
}

// (query block, base tile) pairs of the last brute_force_tc run: all of them, and
// the ones its MMA passes visited (home + rest pass of the pruned scan; the
// blockmin pass over the pivots is not counted).  Synchronises.
void brute_force_tc_last_scan(uint64_t* total, uint64_t* visited, int* pruned) {
    ssync();
    *total = g_last_tiles_total;
    *visited = g_last_pruned && g_last_counts ? g_last_counts[1] + g_last_counts[2] : g_last_tiles_total;
    *pruned = g_last_pruned ? 1 : 0;
}

}  // namespace annk
