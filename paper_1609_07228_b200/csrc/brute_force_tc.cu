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
#include <cuda.h>
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
constexpr uint32_t kNormBytes = kStages * kTB * 8;  // per stage: the tile's norms, then -(norm >> 1)
constexpr uint32_t kStageBytes = kEpiWarps * 32 * kStageStride * 4;
constexpr uint32_t kSmemTC = 1024 + kABytes + kStages * kTileBytes + kNormBytes + kStageBytes + kTQ * 2 * 8;

// Instruction descriptor, kind::i8: D s32 (bits 4-5 = 2), A/B unsigned (0),
// both K-major, N >> 3 at bits 17-22, M >> 4 at bits 24-28.
constexpr uint32_t kIdesc = (2u << 4) | ((kTB >> 3) << 17) | ((kQB >> 4) << 24);

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
    uint64_t* out;   // (nq x splits) x k
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

// Sort a candidate buffer (cnt keys) with the whole warp and write its k best.
__device__ __noinline__ void emit_topk(const uint64_t* b, uint32_t cnt, uint32_t k, uint64_t* o, uint32_t lane) {
    uint64_t v[kSortV];
#pragma unroll
    for (int r = 0; r < kSortV; ++r) {
        const uint32_t e = uint32_t(r) * 32 + lane;
        v[r] = e < cnt ? b[e] : kEmptyKey;
    }
    warp_sort_regs<kSortV>(v);
#pragma unroll
    for (int r = 0; r < kSortV; ++r) {
        const uint32_t e = uint32_t(r) * 32 + lane;
        if (e < k) o[e] = v[r];
    }
    __syncwarp();
}

__global__ void __launch_bounds__(kThreadsTC, 1)
bf_tc_u8_kernel(const __grid_constant__ CUtensorMap tm_base, const __grid_constant__ CUtensorMap tm_q, TcArgs a) {
    extern __shared__ unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t full_bar[kStages], empty_bar[kStages], tfull_bar[kAcc], tempty_bar[kAcc];
    __shared__ __align__(8) uint64_t afull_bar, aempty_bar;
    __shared__ uint32_t tmem_base_s;

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

    if (warp == kEpiWarps) {
        // ------------------------------------------------------------ TMA producer
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm_base)) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm_q)) : "memory");
            uint32_t it = 0, ni = 0;
            for (uint32_t item = blockIdx.x; item < a.n_items; item += gridDim.x, ++ni) {
                const uint32_t qb = item / a.splits, split = item % a.splits;
                const uint32_t t0 = split * a.tiles_per_split, t1 = min(n_tiles, t0 + a.tiles_per_split);
                mbar_wait_backoff(&aempty_bar, (ni & 1) ^ 1);
                mbar_expect_tx(&afull_bar, kABytes);
                for (uint32_t h = 0; h < kNQB; ++h)
                    tma_load_2d(sA + h * kQB * kRow, &tm_q, &afull_bar, 0, int32_t(qb * kTQ + h * kQB));
                for (uint32_t t = t0; t < t1; ++t, ++it) {
                    const uint32_t s = it % kStages;
                    mbar_wait_backoff(&empty_bar[s], ((it / kStages) & 1) ^ 1);
                    mbar_expect_tx(&full_bar[s], kTileBytes + kTB * 8);
                    tma_load_2d(sB + s * kTileBytes, &tm_base, &full_bar[s], 0, int32_t(t * kTB));
                    // (norm arrays are padded to whole tiles: rows past the end read as sentinels)
                    bulk_load(sN + s * kTB * 8, a.bnorm + size_t(t) * kTB, kTB * 4, &full_bar[s]);
                    bulk_load(sN + s * kTB * 8 + kTB * 4, a.nhalf + size_t(t) * kTB, kTB * 4, &full_bar[s]);
                }
            }
        }
    } else if (warp == kEpiWarps + 1) {
        // ------------------------------------------------------------ MMA issuer
        if (lane == 0) {
            uint32_t it = 0, ni = 0;
            for (uint32_t item = blockIdx.x; item < a.n_items; item += gridDim.x, ++ni) {
                const uint32_t split = item % a.splits;
                const uint32_t t0 = split * a.tiles_per_split, t1 = min(n_tiles, t0 + a.tiles_per_split);
                mbar_wait_backoff(&afull_bar, ni & 1);
                tc_fence_after();
                for (uint32_t t = t0; t < t1; ++t, ++it) {
                    const uint32_t s = it % kStages, b = it % kAcc;
                    mbar_wait(&full_bar[s], (it / kStages) & 1);  // the MMA lane polls without backoff
                    mbar_wait(&tempty_bar[b], ((it / kAcc) & 1) ^ 1);
                    tc_fence_after();
#pragma unroll
                    for (uint32_t h = 0; h < kNQB; ++h)
#pragma unroll
                        for (uint32_t kk = 0; kk < kRow / 32; ++kk)
                            mma_i8(tmem + (b * kNQB + h) * kTB, sdesc_sw128(sA + h * kQB * kRow + kk * 32),
                                   sdesc_sw128(sB + s * kTileBytes + kk * 32), kIdesc, kk);
                    tc_commit(&empty_bar[s]);  // smem stage free once these MMAs have read it
                    tc_commit(&tfull_bar[b]);  // accumulator b ready for the epilogue
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
        uint32_t it = 0;
        for (uint32_t item = blockIdx.x; item < a.n_items; item += gridDim.x) {
            const uint32_t qb = item / a.splits, split = item % a.splits;
            const uint32_t t0 = split * a.tiles_per_split, t1 = min(n_tiles, t0 + a.tiles_per_split);
            const uint32_t qi = qb * kTQ + row;
            const bool qvalid = qi < a.nq;
            const int32_t qn = qvalid ? a.qnorm[qi] : 0;
            const uint32_t self = (a.self_ids && qvalid) ? a.self_ids[qi] : kInvalidId;
            uint32_t cnt = 0;
            uint64_t thr = kEmptyKey;
            // keep iff qn + bn - 2 dot <= T  <=>  2 dot - bn >= qn - T = lim (ties settled by the key).
            // Necessary condition with h = bn >> 1: dot - h >= ceil(lim / 2) = L, evaluated per
            // group of 4 columns as max(dot + (-h)) with one VIADDMNMX per pair.
            int32_t lim = qvalid ? INT_MIN : INT_MAX;
            int32_t L = qvalid ? (lim + 1) >> 1 : INT_MAX;
            *my_share = kEmptyKey;
            asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * 32) : "memory");  // shares reset for this item
            for (uint32_t t = t0; t < t1; ++t, ++it) {
                const uint32_t b = it % kAcc, s = it % kStages;
                {
                    const uint64_t o = *reinterpret_cast<const volatile uint64_t*>(other_share);
                    if (qvalid && o < thr) {
                        thr = o;
                        lim = qn - int32_t(key_dist(thr));
                        L = (lim + 1) >> 1;
                    }
                }
                mbar_wait(&tfull_bar[b], (it / kAcc) & 1);
                tc_fence_after();
                mbar_wait(&full_bar[s], (it / kStages) & 1);  // column norms landed
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
                    const uint32_t j0 = t * kTB + c * 32;
                    const int32_t* rowp = ring + s * 2 * kTB + c * 32;  // exact norms; rowp + kTB: -(norm >> 1)
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
                    const bool hit = mx >= L;
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
                            cut.n = flush_sort(sb, sc, a.k, lane);
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
                            const uint32_t j = jg + e2;
                            if (xs[e2] >= lim && j < a.nb && j != self) {
                                const uint64_t key = make_key(float(qn - xs[e2]), j);
                                if (key < thr) {
                                    DCHK(cnt < kCB);
                                    buf[cnt++] = key;
                                }
                            }
                        }
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty_bar[s]);  // this tile's column norms are no longer read
            }
            // final top-k of every query of this warp, written in (query, split) order
#pragma unroll 1
            for (uint32_t src = 0; src < 32; ++src) {
                const uint32_t sq = qb * kTQ + row - lane + src;
                if (sq >= a.nq) break;
                const uint64_t* sb = a.cand + (cbase + row - lane + src) * kCB;
                const uint32_t sc = __shfl_sync(0xffffffffu, cnt, src);
                emit_topk(sb, sc, a.k, a.out + ((size_t(sq) * a.splits + split) * 2 + half) * a.k, lane);
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

// Tile-padded copies of the base norms and of -(norm >> 1); entries past the
// end hold sentinels (the exact test then rejects them by index).
__global__ void pad_norms_kernel(const int32_t* __restrict__ n, uint32_t cnt, uint32_t padded,
                                 int32_t* __restrict__ norms, int32_t* __restrict__ nhalf) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < padded; i += gridDim.x * blockDim.x) {
        norms[i] = i < cnt ? n[i] : INT_MAX / 2;
        nhalf[i] = i < cnt ? -(n[i] >> 1) : INT_MIN / 2;
    }
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

}  // namespace

// Exact kNN on tcgen05 for the u8 datapath with 128-byte rows; returns false
// (nothing launched) when the shape is not supported.
bool brute_force_tc(const annk_dataset* base, uint32_t nq, const uint32_t* self_ids, uint32_t k,
                    uint64_t* out_keys, const uint8_t* q8, const int32_t* qnorm) {
    if (!base->u8 || q8 == nullptr || base->ld8 != kRow || k == 0 || k > 128 || nq == 0) return false;
    if (getenv("ANNK_BF_MMA_SYNC")) return false;
    const uint32_t nb = base->n;
    const uint32_t n_tiles = (nb + kTB - 1) / kTB;
    const uint32_t qblocks = (nq + kTQ - 1) / kTQ;
    const uint32_t sms = uint32_t(num_sms());
    // split the base range only when there are too few query blocks to fill the GPU
    uint32_t splits = std::max(1u, std::min(n_tiles, (sms + qblocks - 1) / qblocks));
    splits = std::min(splits, std::max(1u, 2048u / k));  // 2 lists per split: merge list fits a warp
    const uint32_t tps = (n_tiles + splits - 1) / splits;
    splits = (n_tiles + tps - 1) / tps;
    const uint32_t n_items = qblocks * splits;
    const uint32_t grid = std::min(n_items, sms);
    const CUtensorMap tb = make_map(base->data8.p, nb, kTB);
    const CUtensorMap tq = make_map(q8, nq, kQB);
    DevBuf<uint64_t> cand(size_t(grid) * 2 * kTQ * kCB);
    DevBuf<uint64_t> part(size_t(nq) * splits * 2 * k);  // per (query, split, column half)
    const uint32_t padded = n_tiles * kTB;
    DevBuf<int32_t> norms(padded), nhalf(padded);
    LAUNCH(pad_norms_kernel, std::min((padded + 255) / 256, 4096u), 256, 0, base->norms8.p, nb, padded, norms.p,
           nhalf.p);
    TcArgs args{norms.p, nhalf.p, nb, qnorm, nq, self_ids, k, splits, tps, n_items, cand.p,
                part.p};
    CK(cudaFuncSetAttribute(bf_tc_u8_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kSmemTC)));
    LAUNCH(bf_tc_u8_kernel, grid, kThreadsTC, kSmemTC, tb, tq, args);
    merge_split_lists(part.p, nq, splits * 2, k, out_keys);
    return true;
}

}  // namespace annk
