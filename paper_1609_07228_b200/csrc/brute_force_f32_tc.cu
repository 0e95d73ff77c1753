// brute_force_f32_tc.cu — exact kNN for fp32 rows on the tensor cores.
//
// Reference: proj/src/eval.cpp:17-80 (exact_row / brute_force_knn /
// brute_force_graph): per query, a NeighborPool(k) over every base id keyed by
// (l2_sq, id) — l2_sq being the sequential fp32 chain of dataset.hpp:67-74.
//
// Two passes:
//  1. Candidates on tcgen05.  D' = |q|^2 + |b|^2 - 2 q.b with the dot product
//     from a bf16x3 split: x = hi + lo + e (hi = bf16(x), lo = bf16(x - hi),
//     |e| <= 2^-18 |x|), q.b ~ hi.hi + hi.lo + lo.hi, three kind::f16 MMA
//     chains into one fp32 TMEM accumulator.  A certified bound
//         |l2_sq(q, b) - D'| <= M_q (1 + g) + g D'
//     (M_q = c1 (|q|^2 + max|b|^2) covers the dropped lo.lo / e terms, the
//     tensor core's fp32 accumulation over 3*K products and the fp32 rounding
//     of D'; g = (dim + 3) 2^-24 bounds the reference chain's own rounding)
//     turns the k-th smallest D' of a candidate list into a cut: a base row
//     whose D' exceeds cut(D'_k) = (1+g)(D'_k + 2 M_q)/(1-g) has an exact
//     distance above k others' and can never be in the top k.  Each
//     (query, column half) list keeps every row under its current cut.
//  2. Exact re-rank (rerank_kernel): per query the union of its lists under the
//     smallest cut, exact distances with the reference's sequential chain, keys
//     (dist, id) sorted, first k written.  Ids and distances are therefore
//     bit-identical to the reference.  A query whose lists saturate with rows
//     inside the margin (massive near-ties) is flagged and recomputed by the
//     exact CUDA-core kernel.
//
// Kernel structure (one CTA per SM, persistent over work items):
//   work item  = 128 queries (M) x one slice of base tiles
//   base tile  = 256 rows (N); K streamed in 64-element chunks (128-byte bf16
//                rows, SWIZZLE_128B); a stage holds A hi/lo (2 x 16 KB) and B
//                hi/lo (2 x 32 KB); 2 stages
//   warp 8     = TMA producer; warp 9 = TMEM owner + MMA issuer (12 MMAs
//                128x256x16 per stage); accumulators double-buffered (2 x 256
//                TMEM columns) so the epilogue of tile t overlaps tile t+1
//   warps 0..7 = epilogue: warp w reads TMEM lane quarter w%4 (one query per
//                thread) and column half w/4 of every tile.
#include <cuda_bf16.h>

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <vector>

#include "../../include/annkit_b200.h"
#include "internal.cuh"
#include "tcgen05.cuh"

namespace annk {
namespace {

using namespace tc;

constexpr uint32_t kFQ = 128;                              // queries per item (MMA M)
constexpr uint32_t kFB = 256;                              // base rows per tile (MMA N)
constexpr uint32_t kFK = 64;                               // bf16 elements per K chunk (128 bytes)
constexpr uint32_t kFStages = 2;
constexpr uint32_t kFAB = kFQ * 128;                       // one A operand (hi or lo) per stage
constexpr uint32_t kFBB = kFB * 128;                       // one B operand per stage
constexpr uint32_t kFStageBytes = 2 * kFAB + 2 * kFBB;     // 96 KB
constexpr uint32_t kFEpiWarps = 8;
constexpr uint32_t kFThreads = (kFEpiWarps + 2) * 32;
constexpr uint32_t kFCB = 256;                             // candidate list per (query, column half)
constexpr uint32_t kFSmem = 1024 + kFStages * kFStageBytes + kFQ * 2 * 4;
constexpr uint32_t kRR = 1024;                             // re-rank candidates per query
constexpr float kSentinelNorm = 1e30f;                     // norms of the padding rows past the end
// kind::f16 instruction descriptor: D f32 (bits 4-5 = 1), A/B bf16 (bits 7-9,
// 10-12 = 1), both K-major, N >> 3 at bits 17-22, M >> 4 at bits 24-28.
constexpr uint32_t kFIdesc = (1u << 4) | (1u << 7) | (1u << 10) | ((kFB >> 3) << 17) | ((kFQ >> 4) << 24);

// Per-dimension mean of the base rows (double sums): the rows are centred on it
// before the split, which leaves every difference q - b unchanged but shrinks
// the norms the error bound scales with.
__global__ void col_sum_kernel(const float* __restrict__ x, uint32_t n, uint32_t ld, uint32_t dim,
                               double* __restrict__ sum) {
    for (uint32_t c = threadIdx.x; c < dim; c += blockDim.x) {
        double s = 0.0;
        for (uint32_t r = blockIdx.x; r < n; r += gridDim.x) s += double(x[size_t(r) * ld + c]);
        atomicAdd(&sum[c], s);
    }
}

// One warp per row: r = x - mu (exact in double), hi = bf16(r), lo = bf16(r - hi)
// (r - hi is exact), zero padded to kp elements; |r - hi - lo| <= 2^-18 |r|.  The
// squared norm of r is summed in double and rounded once.  Rows in [n,
// rows_pad) only get the sentinel norm.
__global__ void split_rows_kernel(const float* __restrict__ x, uint32_t n, uint32_t ld, uint32_t dim, uint32_t kp,
                                  uint32_t rows_pad, const double* __restrict__ musum, double inv_n,
                                  __nv_bfloat162* __restrict__ hi, __nv_bfloat162* __restrict__ lo,
                                  float* __restrict__ norms, uint32_t* __restrict__ stat) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t w0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    uint32_t bad = 0, nmax = 0;
    for (uint32_t r = w0; r < rows_pad; r += nw) {
        if (r >= n) {
            if (lane == 0) norms[r] = kSentinelNorm;
            continue;
        }
        const float* xr = x + size_t(r) * ld;
        double s = 0.0;
        for (uint32_t c = 2 * lane; c < kp; c += 64) {
            double v[2];
            __nv_bfloat16 h[2], l[2];
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const uint32_t cc = c + e;
                const float xv = cc < dim ? xr[cc] : 0.0f;
                bad |= isfinite(xv) ? 0u : 1u;
                const double mu = cc < dim ? double(float(musum[cc] * inv_n)) : 0.0;
                v[e] = double(xv) - mu;
                h[e] = __float2bfloat16_rn(float(v[e]));
                l[e] = __float2bfloat16_rn(float(v[e] - double(__bfloat162float(h[e]))));
                s += v[e] * v[e];
            }
            hi[(size_t(r) * kp + c) >> 1] = __halves2bfloat162(h[0], h[1]);
            lo[(size_t(r) * kp + c) >> 1] = __halves2bfloat162(l[0], l[1]);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        const float nf = float(s);
        if (lane == 0) norms[r] = nf;
        nmax = max(nmax, __float_as_uint(nf));  // non-negative floats order as their bits
    }
    bad = __reduce_or_sync(0xffffffffu, bad);
    nmax = __reduce_max_sync(0xffffffffu, nmax);
    if (lane == 0) {
        if (bad) atomicOr(&stat[0], 1u);
        atomicMax(&stat[1], nmax);
    }
}

struct FArgs {
    const float* bnorm;  // padded to whole tiles (sentinels past the end)
    uint32_t nb;
    const float* qnorm;
    uint32_t nq;
    const uint32_t* self_ids;
    uint32_t k, splits, tiles_per_split, n_items, kchunks;
    float c1, bnmax, g;  // M_q = c1 (|q|^2 + bnmax); cut(D'_k) = (D'_k + 2 M_q) g
    uint64_t* cand;      // gridDim.x x kFQ x 2 x kFCB
    uint64_t* out;       // (nq x splits x 2) x kFCB
    uint32_t* out_cnt;   // nq x splits x 2
    float* out_cut;      // nq x splits x 2
    uint8_t* ovf;        // nq: lists saturated, recompute exactly
};

struct FCut {
    uint32_t n;
    float cut;
};

// Cut a candidate list (cnt > k keys, unsorted) back to the keys under
// cut(D'_k): D'_k (the list's k-th smallest D') is found by a warp-wide binary
// search on the keys' distance bits (non-negative floats order as integers).
__device__ __noinline__ FCut fflush(uint64_t* b, uint32_t cnt, uint32_t k, float m2, float g, uint32_t lane) {
    constexpr int V = kFCB / 32;
    uint64_t v[V];
    uint32_t dv[V];
    uint32_t mn = 0xffffffffu, mx = 0;
#pragma unroll
    for (int r = 0; r < V; ++r) {
        const uint32_t e = uint32_t(r) * 32 + lane;
        v[r] = e < cnt ? b[e] : kEmptyKey;
        dv[r] = uint32_t(v[r] >> 32);
        if (e < cnt) {
            mn = min(mn, dv[r]);
            mx = max(mx, dv[r]);
        }
    }
    uint32_t lo = __reduce_min_sync(0xffffffffu, mn), hi = __reduce_max_sync(0xffffffffu, mx);
    while (lo < hi) {
        const uint32_t mid = lo + ((hi - lo) >> 1);
        uint32_t c = 0;
#pragma unroll
        for (int r = 0; r < V; ++r) c += dv[r] <= mid ? 1u : 0u;
        if (__reduce_add_sync(0xffffffffu, c) >= k) hi = mid;
        else lo = mid + 1;
    }
    const float cut = (__uint_as_float(lo) + m2) * g;
    const uint32_t cb = __float_as_uint(cut);
    uint32_t n = 0;
    const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
    for (int r = 0; r < V; ++r) {
        const bool keep = dv[r] <= cb;
        const uint32_t bal = __ballot_sync(0xffffffffu, keep);
        if (keep) b[n + __popc(bal & lt)] = v[r];
        n += __popc(bal);
    }
    __syncwarp();
    return FCut{n, cut};
}

// group-filter bound: fl(qn + v) <= cut implies v <= lim_of(cut, qn)
__device__ __forceinline__ float lim_of(float cut, float qn) {
    return cut >= FLT_MAX ? FLT_MAX : (cut < 0.0f ? -FLT_MAX : (cut - qn) + (cut + qn) * 2.4e-7f);
}

__global__ void __launch_bounds__(kFThreads, 1)
bf_tc_f32_kernel(const __grid_constant__ CUtensorMap tm_bh, const __grid_constant__ CUtensorMap tm_bl,
                 const __grid_constant__ CUtensorMap tm_qh, const __grid_constant__ CUtensorMap tm_ql, FArgs a) {
    extern __shared__ unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t full_bar[kFStages], empty_bar[kFStages], tfull_bar[2], tempty_bar[2];
    __shared__ uint32_t tmem_base_s;

    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t sbase = (smem_u32(smem_raw) + 1023u) & ~1023u;
    const uint32_t n_tiles = (a.nb + kFB - 1) / kFB;
    float* share = reinterpret_cast<float*>(smem_raw + (sbase + kFStages * kFStageBytes - smem_u32(smem_raw)));

    if (tid == 0) {
        for (uint32_t s = 0; s < kFStages; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&empty_bar[s], 1);
        }
        for (uint32_t b = 0; b < 2; ++b) {
            mbar_init(&tfull_bar[b], 1);
            mbar_init(&tempty_bar[b], kFEpiWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (warp == kFEpiWarps + 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                         smem_u32(&tmem_base_s))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base_s;

    if (warp == kFEpiWarps) {
        // ------------------------------------------------------------ TMA producer
        if (lane == 0) {
            uint32_t st = 0;
            for (uint32_t item = blockIdx.x; item < a.n_items; item += gridDim.x) {
                const uint32_t qb = item / a.splits, split = item % a.splits;
                const uint32_t t0 = split * a.tiles_per_split, t1 = min(n_tiles, t0 + a.tiles_per_split);
                for (uint32_t t = t0; t < t1; ++t) {
                    for (uint32_t kc = 0; kc < a.kchunks; ++kc, ++st) {
                        const uint32_t s = st % kFStages;
                        mbar_wait_backoff(&empty_bar[s], ((st / kFStages) & 1) ^ 1);
                        mbar_expect_tx(&full_bar[s], kFStageBytes);
                        const uint32_t so = sbase + s * kFStageBytes;
                        const int32_t x = int32_t(kc * kFK);
                        tma_load_2d(so, &tm_qh, &full_bar[s], x, int32_t(qb * kFQ));
                        tma_load_2d(so + kFAB, &tm_ql, &full_bar[s], x, int32_t(qb * kFQ));
                        tma_load_2d(so + 2 * kFAB, &tm_bh, &full_bar[s], x, int32_t(t * kFB));
                        tma_load_2d(so + 2 * kFAB + kFBB, &tm_bl, &full_bar[s], x, int32_t(t * kFB));
                    }
                }
            }
        }
    } else if (warp == kFEpiWarps + 1) {
        // ------------------------------------------------------------ MMA issuer
        if (lane == 0) {
            uint32_t st = 0, it = 0;
            for (uint32_t item = blockIdx.x; item < a.n_items; item += gridDim.x) {
                const uint32_t split = item % a.splits;
                const uint32_t t0 = split * a.tiles_per_split, t1 = min(n_tiles, t0 + a.tiles_per_split);
                for (uint32_t t = t0; t < t1; ++t, ++it) {
                    const uint32_t b = it & 1;
                    mbar_wait(&tempty_bar[b], ((it >> 1) & 1) ^ 1);
                    tc_fence_after();
                    const uint32_t d = tmem + b * kFB;
                    for (uint32_t kc = 0; kc < a.kchunks; ++kc, ++st) {
                        const uint32_t s = st % kFStages;
                        mbar_wait(&full_bar[s], (st / kFStages) & 1);
                        tc_fence_after();
                        const uint32_t so = sbase + s * kFStageBytes;
#pragma unroll
                        for (uint32_t kk = 0; kk < kFK / 16; ++kk) {
                            const uint64_t ah = sdesc_sw128(so + kk * 32), al = sdesc_sw128(so + kFAB + kk * 32);
                            const uint64_t bh = sdesc_sw128(so + 2 * kFAB + kk * 32);
                            const uint64_t bl = sdesc_sw128(so + 2 * kFAB + kFBB + kk * 32);
                            // the small cross terms first, then hi.hi
                            mma_bf16(d, ah, bl, kFIdesc, (kc | kk) != 0);
                            mma_bf16(d, al, bh, kFIdesc, 1);
                            mma_bf16(d, ah, bh, kFIdesc, 1);
                        }
                        tc_commit(&empty_bar[s]);  // stage free once these MMAs have read it
                    }
                    tc_commit(&tfull_bar[b]);  // accumulator b holds the tile's dot products
                }
            }
        }
    } else {
        // ------------------------------------------------------------ epilogue
        const uint32_t quarter = warp & 3, half = warp >> 2;
        const uint32_t row = quarter * 32 + lane;
        uint64_t* buf = a.cand + ((size_t(blockIdx.x) * kFQ + row) * 2 + half) * kFCB;
        float* my_share = share + row * 2 + half;
        const float* other_share = share + row * 2 + (half ^ 1);
        uint32_t it = 0;
        for (uint32_t item = blockIdx.x; item < a.n_items; item += gridDim.x) {
            const uint32_t qb = item / a.splits, split = item % a.splits;
            const uint32_t t0 = split * a.tiles_per_split, t1 = min(n_tiles, t0 + a.tiles_per_split);
            const uint32_t qi = qb * kFQ + row;
            const bool qvalid = qi < a.nq;
            const float qn = qvalid ? a.qnorm[qi] : 0.0f;
            const uint32_t self = (a.self_ids && qvalid) ? a.self_ids[qi] : kInvalidId;
            const float m2 = 2.0f * a.c1 * (qn + a.bnmax);
            uint32_t cnt = 0;
            bool dead = !qvalid;
            float cut = qvalid ? FLT_MAX : -FLT_MAX;
            float lim = lim_of(cut, qn);
            *reinterpret_cast<volatile float*>(my_share) = FLT_MAX;
            asm volatile("bar.sync 1, %0;" ::"n"(kFEpiWarps * 32) : "memory");
            for (uint32_t t = t0; t < t1; ++t, ++it) {
                const uint32_t b = it & 1;
                {
                    const float o = *reinterpret_cast<const volatile float*>(other_share);
                    if (!dead && o < cut) {
                        cut = o;
                        lim = lim_of(cut, qn);
                    }
                }
                mbar_wait(&tfull_bar[b], (it >> 1) & 1);
                tc_fence_after();
                const uint32_t taddr = tmem + ((quarter * 32) << 16) + b * kFB + half * (kFB / 2);
#pragma unroll 1
                for (uint32_t c = 0; c < kFB / 64; ++c) {
                    uint32_t d[32];
                    tmem_ld32_async(taddr + c * 32, d);
                    tmem_wait(d);
                    if (c == kFB / 64 - 1) {  // our columns of accumulator b are read: release it
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&tempty_bar[b]);
                    }
                    const uint32_t j0 = t * kFB + half * (kFB / 2) + c * 32;
                    const float4* bn4 = reinterpret_cast<const float4*>(a.bnorm + j0);
                    float v[32];
                    float gmin[8];
#pragma unroll
                    for (int gi = 0; gi < 8; ++gi) {
                        const float4 bn = __ldg(bn4 + gi);
                        v[4 * gi + 0] = fmaf(-2.0f, __uint_as_float(d[4 * gi + 0]), bn.x);
                        v[4 * gi + 1] = fmaf(-2.0f, __uint_as_float(d[4 * gi + 1]), bn.y);
                        v[4 * gi + 2] = fmaf(-2.0f, __uint_as_float(d[4 * gi + 2]), bn.z);
                        v[4 * gi + 3] = fmaf(-2.0f, __uint_as_float(d[4 * gi + 3]), bn.w);
                        gmin[gi] = fminf(fminf(v[4 * gi], v[4 * gi + 1]), fminf(v[4 * gi + 2], v[4 * gi + 3]));
                    }
                    uint32_t gm = 0;
#pragma unroll
                    for (int gi = 0; gi < 8; ++gi) gm |= uint32_t(gmin[gi] <= lim) << gi;
                    if (!__any_sync(0xffffffffu, gm != 0)) continue;
                    // room for up to 4 survivors per flagged group in every list that takes some
                    uint32_t need = __ballot_sync(0xffffffffu, cnt + 4 * __popc(gm) > kFCB);
                    while (need) {
                        const uint32_t src = __ffs(need) - 1;
                        need &= need - 1;
                        uint64_t* sb = a.cand + ((size_t(blockIdx.x) * kFQ + row - lane + src) * 2 + half) * kFCB;
                        const uint32_t sc = __shfl_sync(0xffffffffu, cnt, src);
                        const float sm2 = __shfl_sync(0xffffffffu, m2, src);
                        const FCut fc = fflush(sb, sc, a.k, sm2, a.g, lane);
                        if (lane == src) {
                            if (fc.n + 32 > kFCB) {  // saturated with rows inside the margin
                                dead = true;
                                cnt = 0;
                                cut = -FLT_MAX;
                                lim = -FLT_MAX;
                                gm = 0;
                                a.ovf[qi] = 1;
                            } else {
                                cnt = fc.n;
                                if (fc.cut < cut) {
                                    cut = fc.cut;
                                    lim = lim_of(cut, qn);
                                    *reinterpret_cast<volatile float*>(my_share) = cut;
                                }
                            }
                        }
                    }
#pragma unroll
                    for (int gi = 0; gi < 8; ++gi) {
                        if ((gm >> gi) & 1) {
#pragma unroll
                            for (int e = 0; e < 4; ++e) {
                                const float dd = qn + v[4 * gi + e];
                                const uint32_t j = j0 + 4 * gi + e;
                                if (dd <= cut && j < a.nb && j != self) {
                                    DCHK(cnt < kFCB);
                                    buf[cnt++] = make_key(fmaxf(dd, 0.0f), j);
                                }
                            }
                        }
                    }
                }
            }
            // final cut of every list of this warp, then the lists go out in (query, split, half) order
            uint32_t need = __ballot_sync(0xffffffffu, !dead && cnt > a.k);
            while (need) {
                const uint32_t src = __ffs(need) - 1;
                need &= need - 1;
                uint64_t* sb = a.cand + ((size_t(blockIdx.x) * kFQ + row - lane + src) * 2 + half) * kFCB;
                const uint32_t sc = __shfl_sync(0xffffffffu, cnt, src);
                const float sm2 = __shfl_sync(0xffffffffu, m2, src);
                const FCut fc = fflush(sb, sc, a.k, sm2, a.g, lane);
                if (lane == src) {
                    cnt = fc.n;
                    cut = fminf(cut, fc.cut);
                }
            }
#pragma unroll 1
            for (uint32_t src = 0; src < 32; ++src) {
                const uint32_t sq = qb * kFQ + row - lane + src;
                if (sq >= a.nq) break;
                const uint64_t* sb = a.cand + ((size_t(blockIdx.x) * kFQ + row - lane + src) * 2 + half) * kFCB;
                const uint32_t sc = __shfl_sync(0xffffffffu, dead ? 0u : cnt, src);
                const float scut = __shfl_sync(0xffffffffu, cut, src);
                const size_t li = (size_t(sq) * a.splits + split) * 2 + half;
                uint64_t v[kFCB / 32];  // sorted, so the re-rank can count by binary search
#pragma unroll
                for (int r = 0; r < int(kFCB / 32); ++r) {
                    const uint32_t e = uint32_t(r) * 32 + lane;
                    v[r] = e < sc ? sb[e] : kEmptyKey;
                }
                warp_sort_regs<kFCB / 32>(v);
#pragma unroll
                for (int r = 0; r < int(kFCB / 32); ++r) {
                    const uint32_t e = uint32_t(r) * 32 + lane;
                    if (e < sc) a.out[li * kFCB + e] = v[r];
                }
                if (lane == 0) {
                    a.out_cnt[li] = sc;
                    a.out_cut[li] = scut;
                }
            }
            __syncwarp();
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == kFEpiWarps + 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
    }
}

// number of keys of a sorted list whose distance bits are <= t
__device__ __forceinline__ uint32_t count_le(const uint64_t* l, uint32_t n, uint32_t t) {
    uint32_t lo = 0, hi = n;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (uint32_t(l[mid] >> 32) <= t) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// One warp per query.  Its L sorted lists (one per base slice and column half)
// each bound the query's exact k-th distance; the union's own k-th smallest D'
// (found by bisection on the distance bits, counting with a binary search per
// list) gives the tightest cut.  The keys under it get their exact distance
// (the reference's sequential chain); sorted keys, first k.
__global__ void __launch_bounds__(256) rerank_kernel(const uint64_t* __restrict__ lists,
                                                     const uint32_t* __restrict__ lcnt,
                                                     const float* __restrict__ lcut, uint32_t L,
                                                     const float* __restrict__ q, const float* __restrict__ qnorm,
                                                     const float* __restrict__ base, uint32_t ld, uint32_t nq,
                                                     uint32_t k, float c1, float bnmax, float g,
                                                     uint8_t* __restrict__ ovf, uint64_t* __restrict__ out) {
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31, lt = (1u << lane) - 1u;
    uint64_t* s = reinterpret_cast<uint64_t*>(smem) + size_t(warp) * kRR;
    const uint32_t qi = blockIdx.x * (blockDim.x >> 5) + warp;
    if (qi >= nq || ovf[qi]) return;
    const uint64_t* ql = lists + size_t(qi) * L * kFCB;
    const uint32_t* qc = lcnt + size_t(qi) * L;
    float tau = FLT_MAX;
    for (uint32_t l = lane; l < L; l += 32) tau = fminf(tau, lcut[size_t(qi) * L + l]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tau = fminf(tau, __shfl_xor_sync(0xffffffffu, tau, o));
    // the union's k-th smallest D' (keys above tau cannot matter)
    uint32_t lo = 0, hi = __float_as_uint(tau);
    {
        uint32_t c = 0;
        for (uint32_t l = lane; l < L; l += 32) c += count_le(ql + size_t(l) * kFCB, qc[l], hi);
        if (__reduce_add_sync(0xffffffffu, c) < k) lo = hi;  // fewer than k under tau: keep them all
    }
    while (lo < hi) {
        const uint32_t mid = lo + ((hi - lo) >> 1);
        uint32_t c = 0;
        for (uint32_t l = lane; l < L; l += 32) c += count_le(ql + size_t(l) * kFCB, qc[l], mid);
        if (__reduce_add_sync(0xffffffffu, c) >= k) hi = mid;
        else lo = mid + 1;
    }
    tau = fminf(tau, (__uint_as_float(lo) + 2.0f * c1 * (qnorm[qi] + bnmax)) * g);
    const uint32_t tb = __float_as_uint(tau);
    uint32_t n = 0;
    for (uint32_t l = 0; l < L; ++l) {
        const uint64_t* lp = ql + size_t(l) * kFCB;
        const uint32_t c = qc[l];
        for (uint32_t e0 = 0; e0 < c; e0 += 32) {
            const uint32_t e = e0 + lane;
            const uint64_t key = e < c ? lp[e] : kEmptyKey;
            const bool keep = e < c && uint32_t(key >> 32) <= tb;
            const uint32_t bal = __ballot_sync(0xffffffffu, keep);
            if (keep && n + __popc(bal & lt) < kRR) s[n + __popc(bal & lt)] = key;
            n += __popc(bal);
            if (bal != 0xffffffffu) break;  // sorted: the rest of the list is above the cut
        }
    }
    if (n > kRR) {
        if (lane == 0) ovf[qi] = 1;
        return;
    }
    __syncwarp();
    const float* qr = q + size_t(qi) * ld;
    for (uint32_t e = lane; e < n; e += 32) {
        const uint32_t id = key_id(s[e]);
        s[e] = make_key(l2_exact_ldg8(qr, base + size_t(id) * ld, ld), id);
    }
    DCHK(n <= kRR);
    const uint32_t np2 = next_pow2(max(n, k));
    for (uint32_t e = n + lane; e < np2; e += 32) s[e] = kEmptyKey;
    __syncwarp();
    warp_bitonic_sort(s, np2);
    for (uint32_t e = lane; e < k; e += 32) out[size_t(qi) * k + e] = s[e];
}

__global__ void gather_f32_rows_kernel(const float* __restrict__ src, uint32_t ld, const uint32_t* __restrict__ rows,
                                       uint32_t nr, const uint32_t* __restrict__ self, float* __restrict__ dst,
                                       uint32_t* __restrict__ dself) {
    const uint32_t r = blockIdx.x;
    if (r >= nr) return;
    const float* s = src + size_t(rows[r]) * ld;
    float* d = dst + size_t(r) * ld;
    for (uint32_t j = threadIdx.x; j < ld; j += blockDim.x) d[j] = s[j];
    if (threadIdx.x == 0 && self) dself[r] = self[rows[r]];
}

__global__ void scatter_keys_kernel(const uint64_t* __restrict__ src, const uint32_t* __restrict__ rows, uint32_t nr,
                                    uint32_t k, uint64_t* __restrict__ dst) {
    const uint32_t r = blockIdx.x;
    if (r >= nr) return;
    for (uint32_t j = threadIdx.x; j < k; j += blockDim.x) dst[size_t(rows[r]) * k + j] = src[size_t(r) * k + j];
}

CUtensorMap make_bf16_map(const void* p, uint32_t kp, uint32_t rows, uint32_t box_rows) {
    CUtensorMap m;
    const cuuint64_t dims[2] = {kp, std::max(rows, 1u)};
    const cuuint64_t strides[1] = {cuuint64_t(kp) * 2};
    const cuuint32_t box[2] = {kFK, box_rows};
    const cuuint32_t es[2] = {1, 1};
    const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(p), dims, strides, box,
                                   es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
    return m;
}

}  // namespace

uint32_t g_bf_f32_overflow = 0;  // queries recomputed on the CUDA cores by the last call (tests)

// Exact kNN of fp32 rows on tcgen05 (see the header); false (nothing launched)
// when the input is not supported: k > 128, non-finite values, or norms so
// large that the error bound is meaningless.
bool brute_force_tc_f32(const annk_dataset* base, const float* qdata, uint32_t nq, const uint32_t* self_ids,
                        uint32_t k, uint64_t* out_keys) {
    g_bf_f32_overflow = 0;
    if (k == 0 || k > 128 || nq == 0 || base->n == 0 || getenv("ANNK_BF_CUDA_CORE")) return false;
    const uint32_t nb = base->n, dim = base->dim, ld = base->ld;
    const uint32_t kp = (dim + kFK - 1) / kFK * kFK;
    const uint32_t n_tiles = (nb + kFB - 1) / kFB;
    const uint32_t padded = n_tiles * kFB;
    DevBuf<__nv_bfloat16> bh(size_t(nb) * kp), bl(size_t(nb) * kp), qh(size_t(nq) * kp), ql(size_t(nq) * kp);
    DevBuf<float> bnorm(padded), qnorm(nq);
    DevBuf<uint32_t> stat(4);
    stat.zero();
    const uint32_t sms = uint32_t(num_sms());
    DevBuf<double> musum(dim);
    musum.zero();
    LAUNCH(col_sum_kernel, std::min<uint32_t>(nb, sms * 8), 256, 0, base->data.p, nb, ld, dim, musum.p);
    const double inv_n = 1.0 / double(nb);
    LAUNCH(split_rows_kernel, sms * 4, 256, 0, base->data.p, nb, ld, dim, kp, padded, musum.p, inv_n,
           reinterpret_cast<__nv_bfloat162*>(bh.p), reinterpret_cast<__nv_bfloat162*>(bl.p), bnorm.p, stat.p);
    LAUNCH(split_rows_kernel, sms * 4, 256, 0, qdata, nq, ld, dim, kp, nq, musum.p, inv_n,
           reinterpret_cast<__nv_bfloat162*>(qh.p), reinterpret_cast<__nv_bfloat162*>(ql.p), qnorm.p, stat.p + 2);
    uint32_t st[4];
    stat.download(st, 4);
    ssync();
    float bnmax, qnmax;
    memcpy(&bnmax, &st[1], 4);
    memcpy(&qnmax, &st[3], 4);
    if (st[0] || st[2] || !(bnmax < 1e30f) || !(qnmax < 1e30f)) return false;
    // certified margins (see the header): the dropped lo.lo and split residues
    // (< 3.5 2^-18 sum|q_i b_i|), fp32 accumulation of 3 dim products (zero
    // padding adds exactly; 17/16 per 16-product MMA, factor 1.1 spare), the
    // roundings of the norms and of D'
    const double u = std::ldexp(1.0, -24);
    const double c_dot = 3.5 * std::ldexp(1.0, -18) + 3.4 * (dim + 16) * std::ldexp(1.0, -23);
    const double c1 = c_dot + 16 * u;
    const double gam = (dim + 3) * u * 1.01 + 8 * u;
    const double g = (1 + gam) / (1 - gam) * (1 + std::ldexp(1.0, -20));
    // work split: query blocks x base slices, sized so the items fill whole waves of SMs
    const uint32_t qblocks = (nq + kFQ - 1) / kFQ;
    uint32_t splits = 1;
    double best = 1e300;
    for (uint32_t s = 1; s <= std::min<uint32_t>(32, n_tiles); ++s) {
        const double waves = double((uint64_t(qblocks) * s + sms - 1) / sms);
        const double span = waves * double((n_tiles + s - 1) / s);
        if (span < best * 0.98) {
            best = span;
            splits = s;
        }
    }
    const uint32_t tps = (n_tiles + splits - 1) / splits;
    splits = (n_tiles + tps - 1) / tps;
    const uint32_t n_items = qblocks * splits;
    const uint32_t grid = std::min(n_items, sms);
    const CUtensorMap mbh = make_bf16_map(bh.p, kp, nb, kFB), mbl = make_bf16_map(bl.p, kp, nb, kFB);
    const CUtensorMap mqh = make_bf16_map(qh.p, kp, nq, kFQ), mql = make_bf16_map(ql.p, kp, nq, kFQ);
    const uint32_t L = splits * 2;
    DevBuf<uint64_t> cand(size_t(grid) * kFQ * 2 * kFCB), lists(size_t(nq) * L * kFCB);
    DevBuf<uint32_t> lcnt(size_t(nq) * L);
    DevBuf<float> lcut(size_t(nq) * L);
    DevBuf<uint8_t> ovf(nq);
    ovf.zero();
    FArgs args{bnorm.p, nb, qnorm.p, nq, self_ids, k, splits, tps, n_items, kp / kFK, float(c1), bnmax, float(g),
               cand.p, lists.p, lcnt.p, lcut.p, ovf.p};
    CK(cudaFuncSetAttribute(bf_tc_f32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kFSmem)));
    LAUNCH(bf_tc_f32_kernel, grid, kFThreads, kFSmem, mbh, mbl, mqh, mql, args);
    const bool trace = getenv("ANNK_TRACE") != nullptr;
    if (trace) {
        std::vector<uint8_t> h(nq);
        ovf.download(h.data(), nq);
        std::vector<uint32_t> hc(size_t(nq) * L);
        lcnt.download(hc.data(), hc.size());
        std::vector<float> hcut(size_t(nq) * L);
        lcut.download(hcut.data(), hcut.size());
        ssync();
        size_t o = 0, tot = 0;
        for (uint32_t i = 0; i < nq; ++i) o += h[i];
        for (auto c : hc) tot += c;
        fprintf(stderr, "[annk] bf_tc_f32: %u queries x %u lists, %zu saturated in the kernel, mean list %.1f, "
                "c1 %.3g bnmax %.4g g-1 %.3g; q0 cuts:", nq, L, o, double(tot) / hc.size(), c1, bnmax, g - 1);
        for (uint32_t l = 0; l < std::min(L, 8u); ++l) fprintf(stderr, " %.5g/%u", hcut[l], hc[l]);
        fprintf(stderr, "\n");
    }
    cand.release();
    bh.release();
    bl.release();
    qh.release();
    ql.release();
    const size_t rsm = size_t(8) * kRR * 8;
    CK(cudaFuncSetAttribute(rerank_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(rsm)));
    LAUNCH(rerank_kernel, (nq + 7) / 8, 256, rsm, lists.p, lcnt.p, lcut.p, L, qdata, qnorm.p, base->data.p, ld, nq,
           k, float(c1), bnmax, float(g), ovf.p, out_keys);
    // queries whose candidate lists saturated: exact CUDA-core kernel
    std::vector<uint8_t> hov(nq);
    ovf.download(hov.data(), nq);
    ssync();
    std::vector<uint32_t> rows;
    for (uint32_t i = 0; i < nq; ++i)
        if (hov[i]) rows.push_back(i);
    g_bf_f32_overflow = uint32_t(rows.size());
    if (trace) fprintf(stderr, "[annk] bf_tc_f32: %zu queries recomputed on the CUDA cores\n", rows.size());
    if (!rows.empty()) {
        const uint32_t nr = uint32_t(rows.size());
        DevBuf<uint32_t> drows(nr), dself(self_ids ? nr : 0);
        drows.upload(rows.data(), nr);
        DevBuf<float> qsub(size_t(nr) * ld);
        LAUNCH(gather_f32_rows_kernel, nr, 128, 0, qdata, ld, drows.p, nr, self_ids, qsub.p, dself.p);
        DevBuf<uint64_t> ksub(size_t(nr) * k);
        brute_force_f32_tiles(base, qsub.p, nr, self_ids ? dself.p : nullptr, k, ksub.p);
        LAUNCH(scatter_keys_kernel, nr, 128, 0, ksub.p, drows.p, nr, k, out_keys);
        ssync();
    }
    return true;
}

}  // namespace annk
