// join.cu — NN-descent local join and the exact-order pool replay on B200.
//
// Reference: proj/src/graph_build.cpp nn_descent_iteration :105-162 and
// NeighborPool::insert (proj/include/annkit/neighbor_pool.hpp:35-53).
//
// The reference (one worker) walks the points i = 0..n-1; for each i it takes
// the pairs of its lists in the order
//     for a in new:  for b > a in new: (a, b);   for l in old, l != new[a]: (a, l)
// and for every pair offers the second member to the first member's pool,
// then the first to the second's.  `changes` counts the offers a pool
// accepts, including entries evicted again later in the round, so it depends
// on that order.  This file reproduces it exactly:
//
//  * join: one CTA per point computes every pair distance of the point's
//    lists into a shared-memory matrix D (u8 rows: IMMA `mma.sync` m16n8k32,
//    exact integer arithmetic; fp32 rows: the reference's sequential chain per
//    pair), then emits the offers that beat their target's start-of-round tail
//    in exactly the reference's pair order, and hands them to the targets'
//    offer slots with ONE global atomic per (point, target) — a stable
//    counting sort keeps each target's offers from this point contiguous and
//    in order.  Every offer carries its source point.
//  * replay: one warp per target restores the global order — source point
//    ascending (runs of one source are already in pair order) — and replays
//    the offers against the start pool with NeighborPool::insert semantics,
//    32 offers at a time: a window's candidates (keys below the current tail)
//    are accepted iff not a duplicate and #(pool ∪ earlier distinct
//    candidates below the key) < P, which is exactly the sequential insert
//    outcome; the accepted keys are merged into the pool in one step.
//    Pools, flags and `changes` equal the reference's bit-for-bit.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdlib>

#include "join.cuh"

namespace annk {
namespace {

constexpr uint32_t kJT = 256;           // join threads per CTA
constexpr uint32_t kJW = kJT / 32;      // join warps per CTA
constexpr uint32_t kXG = 4;             // fp32 staged rows: x rows per work item
constexpr uint32_t kWX = 8;             // wide fp32 rows: interleaved chains per lane
enum : int { kModeU8 = 0, kModeF32 = 1, kModeWide = 2 };

__host__ __device__ __forceinline__ size_t al16(size_t v) { return (v + 15) & ~size_t(15); }
__host__ __device__ __forceinline__ uint32_t rup(uint32_t v, uint32_t m) { return (v + m - 1) / m * m; }

struct JArgs {
    const float* x;
    const uint8_t* x8;
    const int32_t* norms;
    uint32_t ld, ld8, P, S, cap;
    const uint32_t *gnew, *gold, *gncnt, *gocnt;
    const uint64_t* thr;
    const uint32_t* order;
    uint32_t n_visit, ilo, ihi;
    uint32_t* ocnt;
    uint64_t* obuf;
    uint32_t* osrc;
    uint32_t* ov_cnt;
    uint32_t* ov_tgt;
    uint64_t* ov_key;
    uint32_t* ov_src;
    uint32_t ov_cap;
    unsigned long long* counters;  // [0] comps, [1] offers
    uint32_t rmax;   // list capacity 3S + P
    uint32_t rn;     // per-member array length (rmax rounded up to 32)
    uint32_t rs;     // D row stride (floats)
    uint32_t xc;     // D rows per chunk (multiple of 16)
    uint32_t ol;     // offer buffer capacity
    uint32_t rsb;    // staged row stride in bytes (0: rows not staged)
};

struct JLayout {
    size_t thr, bkey, ids, nrm, mb, mf, ms, wc, rowcnt, canon, bmem, D, rows, total;
};

__host__ __device__ inline JLayout j_layout(const JArgs& a) {
    JLayout L;
    size_t o = 0;
    L.thr = o;    o += al16(size_t(a.rn) * 8);
    L.bkey = o;   o += al16(size_t(a.ol) * 8);
    L.ids = o;    o += al16(size_t(a.rn) * 4);
    L.nrm = o;    o += al16(size_t(a.rn) * 4);
    L.mb = o;     o += al16(size_t(a.rn) * 4);
    L.mf = o;     o += al16(size_t(a.rn) * 4);
    L.ms = o;     o += al16(size_t(a.rn) * 4);
    L.wc = o;     o += al16(size_t(kJW) * a.rn * 4);
    L.rowcnt = o; o += al16(size_t(a.xc + 2) * 4 * 3);  // rowcnt, rowbase, sub-chunk bounds
    L.canon = o;  o += al16(size_t(a.rn) * 2);
    L.bmem = o;   o += al16(size_t(a.ol) * 2);
    L.D = o;      o += al16(size_t(a.xc) * a.rs * 4);
    L.rows = o;   o += size_t(a.rsb) * a.rn;
    L.total = o;
    return L;
}

__device__ __forceinline__ void mma_u8(int32_t (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                       uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t lds32(const unsigned char* p) { return *reinterpret_cast<const uint32_t*>(p); }

// D[x - xb][y] for x in [xb, xe), y in (x, R): the squared distance of list
// members x and y (lower-triangle cells of a tile are computed and ignored).
template <int MODE>
__device__ void join_distances(const JArgs& a, const unsigned char* rows, const uint32_t* ids, const int32_t* nrm,
                               float* D, uint32_t xb, uint32_t xe, uint32_t R) {
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t yb0 = (xb + 1) / 32, nyb = (R + 31) / 32 - yb0;
    if (MODE == kModeU8) {
        // Gram of the rows by IMMA: tile = 16 x-rows x 32 y-columns, K = row bytes.
        const uint32_t g = lane >> 2, t = lane & 3;
        const uint32_t nmt = (xe - xb + 15) / 16, ntiles = nmt * nyb;
        const uint32_t kb = a.rsb - 16;  // row bytes rounded up to 32 (zero padded)
        for (uint32_t tile = warp; tile < ntiles; tile += kJW) {
            const uint32_t m0 = xb + (tile / nyb) * 16, n0 = (yb0 + tile % nyb) * 32;
            if (n0 + 31 <= m0) continue;  // no y > x in this tile
            int32_t acc[4][4];
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[q][0] = acc[q][1] = acc[q][2] = acc[q][3] = 0;
            const unsigned char* ra0 = rows + size_t(m0 + g) * a.rsb + t * 4;
            const unsigned char* ra1 = ra0 + size_t(8) * a.rsb;
            const unsigned char* rb = rows + size_t(n0 + g) * a.rsb + t * 4;
            for (uint32_t k0 = 0; k0 < kb; k0 += 32) {
                const uint32_t a0 = lds32(ra0 + k0), a1 = lds32(ra1 + k0);
                const uint32_t a2 = lds32(ra0 + k0 + 16), a3 = lds32(ra1 + k0 + 16);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const unsigned char* r = rb + size_t(q * 8) * a.rsb + k0;
                    mma_u8(acc[q], a0, a1, a2, a3, lds32(r), lds32(r + 16));
                }
            }
            const uint32_t r0 = m0 + g, r1 = r0 + 8;
            const int32_t n_0 = nrm[r0], n_1 = nrm[r1];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint32_t c = n0 + q * 8 + 2 * t;
                const int32_t nc0 = nrm[c], nc1 = nrm[c + 1];
                if (r0 < xe) {
                    float2 v = make_float2(float(n_0 + nc0 - 2 * acc[q][0]), float(n_0 + nc1 - 2 * acc[q][1]));
                    *reinterpret_cast<float2*>(D + size_t(r0 - xb) * a.rs + c) = v;
                }
                if (r1 < xe) {
                    float2 v = make_float2(float(n_1 + nc0 - 2 * acc[q][2]), float(n_1 + nc1 - 2 * acc[q][3]));
                    *reinterpret_cast<float2*>(D + size_t(r1 - xb) * a.rs + c) = v;
                }
            }
        }
    } else if (MODE == kModeF32) {
        // rows staged in shared memory: each lane owns a y column and runs kXG
        // exact sequential fp32 chains (graph_build.cpp l2_sq order).
        const uint32_t nxg = (xe - xb + kXG - 1) / kXG, items = nxg * nyb;
        for (uint32_t it = warp; it < items; it += kJW) {
            const uint32_t x0 = xb + (it / nyb) * kXG, y = (yb0 + it % nyb) * 32 + lane;
            if ((yb0 + it % nyb) * 32 + 31 <= x0) continue;
            const float* yr = reinterpret_cast<const float*>(rows + size_t(y < R ? y : 0) * a.rsb);
            const float* xr[kXG];
#pragma unroll
            for (uint32_t k = 0; k < kXG; ++k)
                xr[k] = reinterpret_cast<const float*>(rows + size_t(min(x0 + k, xe - 1)) * a.rsb);
            float acc[kXG];
#pragma unroll
            for (uint32_t k = 0; k < kXG; ++k) acc[k] = 0.0f;
            for (uint32_t c = 0; c < a.ld; c += 4) {
                const float4 b = *reinterpret_cast<const float4*>(yr + c);
#pragma unroll
                for (uint32_t k = 0; k < kXG; ++k) {
                    const float4 v = *reinterpret_cast<const float4*>(xr[k] + c);
                    float d;
                    d = __fsub_rn(v.x, b.x); acc[k] = __fadd_rn(acc[k], __fmul_rn(d, d));
                    d = __fsub_rn(v.y, b.y); acc[k] = __fadd_rn(acc[k], __fmul_rn(d, d));
                    d = __fsub_rn(v.z, b.z); acc[k] = __fadd_rn(acc[k], __fmul_rn(d, d));
                    d = __fsub_rn(v.w, b.w); acc[k] = __fadd_rn(acc[k], __fmul_rn(d, d));
                }
            }
            if (y < R) {
#pragma unroll
                for (uint32_t k = 0; k < kXG; ++k)
                    if (x0 + k < xe) D[size_t(x0 + k - xb) * a.rs + y] = acc[k];
            }
        }
    } else {
        // wide fp32 rows streamed from L2: the lane's y row and kWX broadcast x
        // rows, kWX interleaved exact chains per lane.
        const uint32_t nxg = (xe - xb + kWX - 1) / kWX, items = nxg * nyb;
        for (uint32_t it = warp; it < items; it += kJW) {
            const uint32_t x0 = xb + (it / nyb) * kWX, y = (yb0 + it % nyb) * 32 + lane;
            if ((yb0 + it % nyb) * 32 + 31 <= x0) continue;
            const float4* yrow = reinterpret_cast<const float4*>(a.x + size_t(ids[y < R ? y : 0]) * a.ld);
            const float4* xrow[kWX];
#pragma unroll
            for (uint32_t k = 0; k < kWX; ++k)
                xrow[k] = reinterpret_cast<const float4*>(a.x + size_t(ids[min(x0 + k, xe - 1)]) * a.ld);
            float acc[kWX];
#pragma unroll
            for (uint32_t k = 0; k < kWX; ++k) acc[k] = 0.0f;
            for (uint32_t c = 0; c < a.ld / 4; ++c) {
                const float4 b = __ldg(yrow + c);
#pragma unroll
                for (uint32_t k = 0; k < kWX; ++k) {
                    const float4 v = __ldg(xrow[k] + c);
                    float d;
                    d = __fsub_rn(v.x, b.x); acc[k] = __fadd_rn(acc[k], __fmul_rn(d, d));
                    d = __fsub_rn(v.y, b.y); acc[k] = __fadd_rn(acc[k], __fmul_rn(d, d));
                    d = __fsub_rn(v.z, b.z); acc[k] = __fadd_rn(acc[k], __fmul_rn(d, d));
                    d = __fsub_rn(v.w, b.w); acc[k] = __fadd_rn(acc[k], __fmul_rn(d, d));
                }
            }
            if (y < R) {
#pragma unroll
                for (uint32_t k = 0; k < kWX; ++k)
                    if (x0 + k < xe) D[size_t(x0 + k - xb) * a.rs + y] = acc[k];
            }
        }
    }
}

// The offers of pair (x, y) (graph_build.cpp:139-151): y to x's pool, then x
// to y's pool, each only if it beats the target's start-of-round tail (a key
// at or above it is rejected by every pool state of the round).
struct PairOffers {
    bool valid, ox, oy;
    uint64_t kx, ky;
};
__device__ __forceinline__ PairOffers pair_offers(const float* Dr, const uint32_t* ids, const uint64_t* thr_s,
                                                  uint32_t x, uint32_t idx, uint64_t tx, uint32_t y, uint32_t R) {
    PairOffers p;
    const bool in = y < R;
    const uint32_t idy = in ? ids[y] : idx;
    p.valid = in && idy != idx;  // graph_build.cpp:146 (l == j is skipped)
    const float d = p.valid ? Dr[y] : 0.0f;
    p.kx = make_key(d, idy);
    p.ky = make_key(d, idx);
    p.ox = p.valid && p.kx < tx;
    p.oy = p.valid && p.ky < thr_s[in ? y : x];
    return p;
}

template <int MODE>
__global__ void __launch_bounds__(kJT) join_kernel(JArgs a) {
    extern __shared__ __align__(16) unsigned char sm[];
    __shared__ uint32_t s_nsub;
    const JLayout L = j_layout(a);
    uint64_t* thr_s = reinterpret_cast<uint64_t*>(sm + L.thr);
    uint64_t* bkey = reinterpret_cast<uint64_t*>(sm + L.bkey);
    uint32_t* ids = reinterpret_cast<uint32_t*>(sm + L.ids);
    int32_t* nrm = reinterpret_cast<int32_t*>(sm + L.nrm);
    uint32_t* mb = reinterpret_cast<uint32_t*>(sm + L.mb);
    uint32_t* mf = reinterpret_cast<uint32_t*>(sm + L.mf);
    uint32_t* ms = reinterpret_cast<uint32_t*>(sm + L.ms);
    uint32_t* wc = reinterpret_cast<uint32_t*>(sm + L.wc);
    uint32_t* rowcnt = reinterpret_cast<uint32_t*>(sm + L.rowcnt);
    uint32_t* rowbase = rowcnt + a.xc + 2;
    uint32_t* sub = rowbase + a.xc + 2;
    uint16_t* canon = reinterpret_cast<uint16_t*>(sm + L.canon);
    uint16_t* bmem = reinterpret_cast<uint16_t*>(sm + L.bmem);
    float* D = reinterpret_cast<float*>(sm + L.D);
    unsigned char* rows = sm + L.rows;
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, lt = (1u << lane) - 1u;
    uint32_t* wcw = wc + warp * a.rn;
    unsigned long long comps = 0, offers = 0;
    for (uint32_t j = tid; j < kJW * a.rn; j += kJT) wc[j] = 0;
    for (uint32_t j = tid; j < a.rn; j += kJT) nrm[j] = 0;
    for (uint32_t ord = blockIdx.x; ord < a.n_visit; ord += gridDim.x) {
        const uint32_t i = a.order ? a.order[ord] : ord;
        if (i < a.ilo || i >= a.ihi) continue;
        const uint32_t A = a.gncnt[i], B = a.gocnt[i], R = A + B;
        if (A == 0) continue;
        __syncthreads();  // the previous point is done with shared memory
        const uint32_t* nw = a.gnew + size_t(i) * 2 * a.S;
        const uint32_t* od = a.gold + size_t(i) * (a.P + a.S);
        for (uint32_t r = tid; r < R; r += kJT) {
            const uint32_t id = r < A ? nw[r] : od[r - A];
            ids[r] = id;
            thr_s[r] = a.thr[id];
            if (MODE == kModeU8) nrm[r] = a.norms[id];
        }
        __syncthreads();
        // a member present in both lists (new[a] == old[l]) is one pool: its
        // offers are counted under its new-list position
        for (uint32_t r = tid; r < R; r += kJT) {
            uint32_t c = r;
            if (r >= A) {
                const uint32_t v = ids[r];
                uint32_t lo = 0, hi = A;
                while (lo < hi) {
                    const uint32_t mid = (lo + hi) >> 1;
                    if (ids[mid] < v) lo = mid + 1;
                    else hi = mid;
                }
                if (lo < A && ids[lo] == v) c = lo;
            }
            canon[r] = uint16_t(c);
        }
        if (MODE == kModeU8) {
            const uint32_t kb = a.rsb - 16, v16 = kb / 16, l16 = a.ld8 / 16;
            for (uint32_t j = tid; j < R * v16; j += kJT) {
                const uint32_t r = j / v16, c = j % v16;
                uint4 v = make_uint4(0, 0, 0, 0);
                if (c < l16) v = __ldg(reinterpret_cast<const uint4*>(a.x8 + size_t(ids[r]) * a.ld8) + c);
                *reinterpret_cast<uint4*>(rows + size_t(r) * a.rsb + c * 16) = v;
            }
        } else if (MODE == kModeF32) {
            const uint32_t v4 = a.ld / 4;
            for (uint32_t j = tid; j < R * v4; j += kJT) {
                const uint32_t r = j / v4, c = j % v4;
                *reinterpret_cast<float4*>(rows + size_t(r) * a.rsb + c * 16) =
                    __ldg(reinterpret_cast<const float4*>(a.x + size_t(ids[r]) * a.ld) + c);
            }
        }
        __syncthreads();
        for (uint32_t xb = 0; xb < A; xb += a.xc) {
            const uint32_t xe = min(A, xb + a.xc), nrow = xe - xb;
            join_distances<MODE>(a, rows, ids, nrm, D, xb, xe, R);
            __syncthreads();
            // offers per row x (and the pairs counted as distance computations)
            for (uint32_t x = xb + warp; x < xe; x += kJW) {
                const uint32_t idx = ids[x];
                const uint64_t tx = thr_s[x];
                const float* Dr = D + size_t(x - xb) * a.rs;
                uint32_t cnt = 0, pairs = 0;
                for (uint32_t y0 = x + 1; y0 < R; y0 += 32) {
                    const PairOffers p = pair_offers(Dr, ids, thr_s, x, idx, tx, y0 + lane, R);
                    cnt += __popc(__ballot_sync(0xffffffffu, p.ox)) + __popc(__ballot_sync(0xffffffffu, p.oy));
                    pairs += __popc(__ballot_sync(0xffffffffu, p.valid));
                }
                if (lane == 0) {
                    rowcnt[x - xb] = cnt;
                    comps += pairs;
                }
            }
            __syncthreads();
            // row offsets and sub-chunks whose offers fit the buffer
            if (warp == 0) {
                uint32_t run = 0;
                for (uint32_t r0 = 0; r0 < nrow; r0 += 32) {
                    const uint32_t r = r0 + lane;
                    const uint32_t c = r < nrow ? rowcnt[r] : 0u;
                    uint32_t incl = c;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
                        if (lane >= uint32_t(o)) incl += v;
                    }
                    if (r < nrow) rowbase[r] = run + incl - c;
                    run += __shfl_sync(0xffffffffu, incl, 31);
                }
                if (lane == 0) {
                    rowbase[nrow] = run;
                    uint32_t ns = 0;
                    sub[ns++] = 0;
                    if (run > a.ol) {  // rare: greedy split at row boundaries (a row has <= 2 rmax offers)
                        uint32_t acc = 0;
                        for (uint32_t r = 0; r < nrow; ++r) {
                            if (acc + rowcnt[r] > a.ol) {
                                sub[ns++] = r;
                                acc = 0;
                            }
                            acc += rowcnt[r];
                        }
                    }
                    sub[ns] = nrow;
                    s_nsub = ns;
                }
            }
            __syncthreads();
            const uint32_t nsub = s_nsub;
            for (uint32_t sc = 0; sc < nsub; ++sc) {
                const uint32_t sb = sub[sc], se = sub[sc + 1];
                const uint32_t c = rowbase[se] - rowbase[sb];
                if (c == 0) continue;  // uniform
                // emit in the reference's pair order: row x, y ascending, y->x before x->y
                for (uint32_t x = xb + sb + warp; x < xb + se; x += kJW) {
                    const uint32_t idx = ids[x];
                    const uint64_t tx = thr_s[x];
                    const uint16_t cx = canon[x];
                    const float* Dr = D + size_t(x - xb) * a.rs;
                    uint32_t pos = rowbase[x - xb] - rowbase[sb];
                    for (uint32_t y0 = x + 1; y0 < R; y0 += 32) {
                        const uint32_t y = y0 + lane;
                        const PairOffers p = pair_offers(Dr, ids, thr_s, x, idx, tx, y, R);
                        const uint32_t bx = __ballot_sync(0xffffffffu, p.ox);
                        const uint32_t by = __ballot_sync(0xffffffffu, p.oy);
                        const uint32_t q = pos + __popc(bx & lt) + __popc(by & lt);
                        if (p.ox) {
                            bkey[q] = p.kx;
                            bmem[q] = cx;
                        }
                        if (p.oy) {
                            bkey[q + (p.ox ? 1 : 0)] = p.ky;
                            bmem[q + (p.ox ? 1 : 0)] = canon[y];
                        }
                        pos += __popc(bx) + __popc(by);
                    }
                }
                __syncthreads();
                // flush: stable counting sort by target; one global reservation per target
                const uint32_t seg = (c + kJW - 1) / kJW;
                const uint32_t s0 = min(c, warp * seg), s1 = min(c, s0 + seg);
                for (uint32_t e0 = s0; e0 < s1; e0 += 32) {
                    const uint32_t e = e0 + lane;
                    const bool v = e < s1;
                    const uint32_t m = v ? bmem[e] : 0xffffu;
                    const uint32_t mask = __match_any_sync(0xffffffffu, m);
                    if (v && (mask & lt) == 0) wcw[m] += __popc(mask);
                }
                __syncthreads();
                for (uint32_t m = tid; m < R; m += kJT) {
                    uint32_t run = 0;
#pragma unroll
                    for (uint32_t w = 0; w < kJW; ++w) {
                        const uint32_t t = wc[w * a.rn + m];
                        wc[w * a.rn + m] = run;
                        run += t;
                    }
                    if (run) {
                        const uint32_t base = atomicAdd(&a.ocnt[ids[m]], run);
                        const uint32_t fix = base < a.cap ? min(run, a.cap - base) : 0u;
                        mb[m] = base;
                        mf[m] = fix;
                        ms[m] = run > fix ? atomicAdd(a.ov_cnt, run - fix) : 0u;
                    }
                }
                __syncthreads();
                for (uint32_t e0 = s0; e0 < s1; e0 += 32) {
                    const uint32_t e = e0 + lane;
                    const bool v = e < s1;
                    const uint32_t m = v ? bmem[e] : 0xffffu;
                    const uint32_t mask = __match_any_sync(0xffffffffu, m);
                    const uint32_t r = v ? wcw[m] + __popc(mask & lt) : 0u;
                    __syncwarp();
                    if (v) {
                        if ((mask & lt) == 0) wcw[m] += __popc(mask);
                        const uint32_t tgt = ids[m];
                        const uint64_t key = bkey[e];
                        if (r < mf[m]) {
                            const size_t slot = size_t(tgt) * a.cap + mb[m] + r;
                            a.obuf[slot] = key;
                            a.osrc[slot] = i;
                        } else {
                            const uint32_t o = ms[m] + (r - mf[m]);
                            if (o < a.ov_cap) {
                                a.ov_tgt[o] = tgt;
                                a.ov_key[o] = key;
                                a.ov_src[o] = i;
                            }
                        }
                    }
                    __syncwarp();
                }
                __syncthreads();
                for (uint32_t m = tid; m < R; m += kJT) {
#pragma unroll
                    for (uint32_t w = 0; w < kJW; ++w) wc[w * a.rn + m] = 0;
                }
                if (tid == 0) offers += c;
                __syncthreads();
            }
        }
    }
    for (int o = 16; o > 0; o >>= 1) comps += __shfl_xor_sync(0xffffffffu, comps, o);
    if (lane == 0 && comps) atomicAdd(&a.counters[0], comps);
    if (tid == 0 && offers) atomicAdd(&a.counters[1], offers);
}

// ------------------------------------------------------------------ replay

struct RArgs {
    uint32_t lo, hi, P, cap;
    uint64_t* keys;
    uint8_t* flags;
    uint32_t* sizes;
    const uint32_t* ocnt;
    const uint64_t* obuf;
    const uint32_t* osrc;
    const uint32_t* ov_off;
    const uint64_t* ov_key;
    const uint32_t* ov_src;
    unsigned long long* changes;
    uint32_t* next;       // work counter
    uint32_t runmax;      // runs held in shared memory per warp
    uint32_t* big;        // first pass: targets with more runs, deferred
    uint32_t* nbig;
    const uint32_t* big_list;  // second pass: deferred targets, runs in global scratch
    uint32_t big_n;
    const uint64_t* big_off;   // per deferred target: scratch start (units of entries)
    uint64_t* g_runkey;
    uint32_t* g_pstart;
    uint32_t* g_seqoff;
};

__host__ __device__ inline size_t replay_warp_bytes(uint32_t P, uint32_t runmax) {
    return al16(size_t(P) * 8) * 2 + al16(size_t(P)) * 2 + 32 * 8 + al16(size_t(runmax) * 8) +
           al16(size_t(runmax + 1) * 4) * 2;
}

__device__ __forceinline__ uint32_t lower_bound64(const uint64_t* a, uint32_t n, uint64_t v) {
    uint32_t lo = 0, hi = n;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (a[mid] < v) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// Replays target t's offers.  Returns false (pool untouched) when the target
// has more than `runmax` source runs and no scratch was given.
__device__ bool replay_target(const RArgs& a, uint32_t t, uint64_t* S, uint64_t* T, uint8_t* SF, uint8_t* TF,
                              uint64_t* accs, uint64_t* runkey, uint32_t* pstart, uint32_t* seqoff, uint32_t runmax,
                              unsigned long long& changes) {
    const uint32_t lane = threadIdx.x & 31, lt = (1u << lane) - 1u;
    const uint32_t m = a.ocnt[t];
    if (m == 0) return true;
    const uint32_t cf = min(m, a.cap);
    const uint64_t* k0 = a.obuf + size_t(t) * a.cap;
    const uint32_t* s0 = a.osrc + size_t(t) * a.cap;
    const uint32_t spill = m > cf ? a.ov_off[t] : 0u;
    const uint64_t* k1 = a.ov_key + spill;
    const uint32_t* s1 = a.ov_src + spill;
    // runs: maximal stretches of one source (a segment boundary always starts one)
    uint32_t nr = 0, lastsrc = 0;
    for (uint32_t q0 = 0; q0 < m; q0 += 32) {
        const uint32_t q = q0 + lane;
        const bool v = q < m;
        const uint32_t src = v ? (q < cf ? s0[q] : s1[q - cf]) : 0u;
        uint32_t prev = __shfl_up_sync(0xffffffffu, src, 1);
        if (lane == 0) prev = lastsrc;
        const bool start = v && (q == 0 || q == cf || src != prev);
        const uint32_t b = __ballot_sync(0xffffffffu, start);
        if (start) {
            const uint32_t idx = nr + __popc(b & lt);
            if (idx < runmax) {
                runkey[idx] = (uint64_t(src) << 32) | idx;
                pstart[idx] = q;
            }
        }
        nr += __popc(b);
        lastsrc = __shfl_sync(0xffffffffu, src, 31);
    }
    if (nr > runmax) return false;
    const uint32_t np2 = next_pow2(nr);
    for (uint32_t j = nr + lane; j < np2; j += 32) runkey[j] = ~0ull;
    if (lane == 0) pstart[nr] = m;
    __syncwarp();
    if (np2 <= 32) {
        uint64_t v[1] = {lane < np2 ? runkey[lane] : ~0ull};
        warp_sort_regs<1>(v);
        if (lane < np2) runkey[lane] = v[0];
    } else if (np2 <= 64) {
        uint64_t v[2] = {runkey[lane], runkey[32 + lane]};
        warp_sort_regs<2>(v);
        runkey[lane] = v[0];
        runkey[32 + lane] = v[1];
    } else if (np2 <= 128) {
        uint64_t v[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) v[r] = runkey[r * 32 + lane];
        warp_sort_regs<4>(v);
#pragma unroll
        for (int r = 0; r < 4; ++r) runkey[r * 32 + lane] = v[r];
    } else {
        warp_bitonic_sort(runkey, np2);
    }
    __syncwarp();
    // sequence offsets of the runs in (source, position) order
    {
        uint32_t run = 0;
        for (uint32_t r0 = 0; r0 < nr; r0 += 32) {
            const uint32_t r = r0 + lane;
            uint32_t len = 0;
            if (r < nr) {
                const uint32_t idx = uint32_t(runkey[r]);
                len = pstart[idx + 1] - pstart[idx];
            }
            uint32_t incl = len;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= uint32_t(o)) incl += v;
            }
            if (r < nr) seqoff[r] = run + incl - len;
            run += __shfl_sync(0xffffffffu, incl, 31);
        }
    }
    // start pool
    uint32_t sz = a.sizes[t];
    const uint64_t* pk = a.keys + size_t(t) * a.P;
    const uint8_t* pf = a.flags + size_t(t) * a.P;
    for (uint32_t j = lane; j < sz; j += 32) {
        S[j] = pk[j];
        SF[j] = pf[j];
    }
    __syncwarp();
    uint64_t tail = sz == a.P ? S[a.P - 1] : kEmptyKey;
    uint32_t accepted = 0;
    for (uint32_t q0 = 0; q0 < m; q0 += 32) {
        const uint32_t q = q0 + lane;
        uint64_t c = kEmptyKey;
        if (q < m) {
            uint32_t lo = 0, hi = nr;  // last run with seqoff <= q
            while (hi - lo > 1) {
                const uint32_t mid = (lo + hi) >> 1;
                if (seqoff[mid] <= q) lo = mid;
                else hi = mid;
            }
            const uint32_t pos = pstart[uint32_t(runkey[lo])] + (q - seqoff[lo]);
            c = pos < cf ? k0[pos] : k1[pos - cf];
        }
        const bool cand = c < tail;
        const uint32_t cm = __ballot_sync(0xffffffffu, cand);
        if (cm == 0) continue;
        uint32_t rS = 0;
        bool dup = false;
        if (cand) {
            rS = lower_bound64(S, sz, c);
            dup = rS < sz && S[rS] == c;
        }
        // candidates in sequence order: a later equal key is a duplicate; an
        // earlier distinct candidate below the key counts towards its rank
        uint32_t below = 0;
        for (uint32_t bits = cm; bits; bits &= bits - 1) {
            const uint32_t s = __ffs(bits) - 1;
            const uint64_t cs = shfl_idx_u64(c, s);
            const bool ds = __shfl_sync(0xffffffffu, dup, s);
            if (lane > s) {
                if (cs == c) dup = true;
                else if (!ds && cs < c) ++below;
            }
        }
        const bool acc = cand && !dup && rS + below < a.P;
        const uint32_t am = __ballot_sync(0xffffffffu, acc);
        if (am == 0) continue;
        const uint32_t na = __popc(am);
        // merge: accepted keys sorted by rank among themselves, then pool
        // entries shifted by the accepted keys below them
        uint32_t arank = 0;
        for (uint32_t bits = am; bits; bits &= bits - 1) {
            const uint32_t s = __ffs(bits) - 1;
            const uint64_t cs = shfl_idx_u64(c, s);
            if (acc && cs < c) ++arank;
        }
        if (acc) accs[arank] = c;
        __syncwarp();
        for (uint32_t p = lane; p < sz; p += 32) {
            const uint64_t v = S[p];
            const uint32_t np = p + lower_bound64(accs, na, v);
            if (np < a.P) {
                T[np] = v;
                TF[np] = SF[p];
            }
        }
        if (acc && rS + arank < a.P) {
            T[rS + arank] = c;
            TF[rS + arank] = 1;  // arrived this round: flag_new
        }
        __syncwarp();
        sz = min(a.P, sz + na);
        uint64_t* tk = S;
        S = T;
        T = tk;
        uint8_t* tf = SF;
        SF = TF;
        TF = tf;
        accepted += na;
        tail = sz == a.P ? S[a.P - 1] : kEmptyKey;
    }
    if (accepted) {
        uint64_t* wk = a.keys + size_t(t) * a.P;
        uint8_t* wf = a.flags + size_t(t) * a.P;
        for (uint32_t j = lane; j < a.P; j += 32) {
            wk[j] = j < sz ? S[j] : kEmptyKey;
            wf[j] = j < sz ? SF[j] : 0;
        }
        if (lane == 0) a.sizes[t] = sz;
        changes += accepted;
    }
    return true;
}

__global__ void replay_kernel(RArgs a) {
    extern __shared__ __align__(16) unsigned char sm[];
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned char* base = sm + size_t(warp) * replay_warp_bytes(a.P, a.runmax);
    uint64_t* S = reinterpret_cast<uint64_t*>(base);
    uint64_t* T = reinterpret_cast<uint64_t*>(base + al16(size_t(a.P) * 8));
    uint8_t* SF = base + al16(size_t(a.P) * 8) * 2;
    uint8_t* TF = SF + al16(a.P);
    uint64_t* accs = reinterpret_cast<uint64_t*>(TF + al16(a.P));
    uint64_t* runkey = accs + 32;
    uint32_t* pstart = reinterpret_cast<uint32_t*>(runkey + a.runmax);
    uint32_t* seqoff = reinterpret_cast<uint32_t*>(reinterpret_cast<unsigned char*>(pstart) +
                                                   al16(size_t(a.runmax + 1) * 4));
    unsigned long long changes = 0;
    if (a.big_list) {
        const uint32_t b = (blockIdx.x * blockDim.x + threadIdx.x) / 32;
        if (b < a.big_n) {
            const uint64_t o = a.big_off[b];
            replay_target(a, a.big_list[b], S, T, SF, TF, accs, a.g_runkey + o, a.g_pstart + o, a.g_seqoff + o,
                          0xffffffffu, changes);
        }
    } else {
        for (;;) {
            uint32_t w = 0;
            if (lane == 0) w = atomicAdd(a.next, 1u);
            const uint32_t t = a.lo + __shfl_sync(0xffffffffu, w, 0);
            if (t >= a.hi) break;
            if (!replay_target(a, t, S, T, SF, TF, accs, runkey, pstart, seqoff, a.runmax, changes)) {
                if (lane == 0) a.big[atomicAdd(a.nbig, 1u)] = t;
            }
        }
    }
    if (lane == 0 && changes) atomicAdd(a.changes, changes);
}

__global__ void big_sizes_kernel(const uint32_t* __restrict__ big, uint32_t nb, const uint32_t* __restrict__ ocnt,
                                 uint64_t* __restrict__ out) {
    const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b < nb) out[b] = uint64_t(next_pow2(ocnt[big[b]] + 1)) + 1;
    if (b == nb) out[nb] = 0;
}

// spill grouping: stable sort of (target, index) then gather of keys and sources
__global__ void spill_counts_kernel2(const uint32_t* __restrict__ ocnt, uint32_t n, uint32_t cap,
                                     uint32_t* __restrict__ out) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = ocnt[i] > cap ? ocnt[i] - cap : 0;
    if (i == n) out[n] = 0;
}
__global__ void iota_u32_kernel(uint32_t* __restrict__ out, uint32_t count) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < count) out[t] = t;
}
__global__ void gather_spill_kernel(const uint32_t* __restrict__ perm, uint32_t count,
                                    const uint64_t* __restrict__ key, const uint32_t* __restrict__ src,
                                    uint64_t* __restrict__ key2, uint32_t* __restrict__ src2) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < count) {
        const uint32_t p = perm[t];
        key2[t] = key[p];
        src2[t] = src[p];
    }
}

uint32_t gridn(size_t items, uint32_t per) {
    return uint32_t(std::max<size_t>(1, std::min<size_t>((items + per - 1) / per, 1u << 30)));
}

template <class T>
void ex_scan(const T* in, T* out, uint32_t n) {
    size_t tmp = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, n + 1, stream()));
    DevBuf<unsigned char> t(std::max<size_t>(tmp, 1));
    CK(cub::DeviceScan::ExclusiveSum(t.p, tmp, in, out, n + 1, stream()));
    note_launch();
}

}  // namespace

void join_launch(annk_state* s, const annk_dataset* ds, const uint32_t* order, uint32_t n_visit, uint32_t ilo,
                 uint32_t ihi, JoinCounters* out) {
    JArgs a{};
    a.x = ds->data.p;
    a.x8 = ds->u8 ? ds->data8.p : nullptr;
    a.norms = ds->u8 ? ds->norms8.p : nullptr;
    a.ld = ds->ld;
    a.ld8 = ds->ld8;
    a.P = s->P;
    a.S = s->S;
    a.cap = s->offer_cap;
    a.gnew = s->gnew.p;
    a.gold = s->gold.p;
    a.gncnt = s->gncnt.p;
    a.gocnt = s->gocnt.p;
    a.thr = s->thr.p;
    a.order = order;
    a.n_visit = n_visit;
    a.ilo = ilo;
    a.ihi = ihi;
    a.ocnt = s->ocnt.p;
    a.obuf = s->obuf.p;
    a.osrc = s->osrc.p;
    a.ov_cnt = s->ov_count.p;
    a.ov_tgt = s->ov_tgt.p;
    a.ov_key = s->ov_key.p;
    a.ov_src = s->ov_src.p;
    a.ov_cap = s->ov_cap;
    DevBuf<unsigned long long> counters(2);
    counters.zero();
    a.counters = counters.p;
    a.rmax = 3 * s->S + s->P;
    a.rn = rup(a.rmax, 32);
    a.rs = a.rn + 8;
    const uint32_t amax = 2 * s->S;
    a.xc = std::max(16u, std::min(rup(amax, 16), (24576u / (a.rs * 4)) / 16 * 16));
    a.ol = rup(std::max(1024u, 2 * a.rmax), 32);
    int mode;
    const size_t f32_rsb = size_t(ds->ld + 4) * 4;
    if (ds->u8) {
        mode = kModeU8;
        a.rsb = rup(ds->ld8, 32) + 16;
    } else if (f32_rsb * a.rn <= 96 * 1024) {
        mode = kModeF32;
        a.rsb = uint32_t(f32_rsb);
    } else {
        mode = kModeWide;
        a.rsb = 0;
    }
    const size_t smem = j_layout(a).total;
    if (smem > size_t(max_smem_optin())) throw_invalid("join: list capacity too large for the device path");
    const void* fn = mode == kModeU8    ? reinterpret_cast<const void*>(join_kernel<kModeU8>)
                     : mode == kModeF32 ? reinterpret_cast<const void*>(join_kernel<kModeF32>)
                                        : reinterpret_cast<const void*>(join_kernel<kModeWide>);
    CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kJT, smem));
    const uint32_t grid = std::max(1u, std::min<uint32_t>(n_visit, uint32_t(num_sms()) * std::max(per_sm, 1)));
    if (n_visit) {
        if (mode == kModeU8) LAUNCH(join_kernel<kModeU8>, grid, kJT, smem, a);
        else if (mode == kModeF32) LAUNCH(join_kernel<kModeF32>, grid, kJT, smem, a);
        else LAUNCH(join_kernel<kModeWide>, grid, kJT, smem, a);
    }
    unsigned long long c[2] = {0, 0};
    CK(cudaMemcpyAsync(c, counters.p, 16, cudaMemcpyDeviceToHost, stream()));
    uint32_t sp = 0;
    CK(cudaMemcpyAsync(&sp, s->ov_count.p, 4, cudaMemcpyDeviceToHost, stream()));
    ssync();
    out->comps = c[0];
    out->offers = c[1];
    out->spilled = sp;
}

void group_spills(annk_state* s) {
    const uint32_t n = s->n;
    if (s->ov_off.n != size_t(n) + 1) s->ov_off.alloc(size_t(n) + 1);
    if (s->spill_sorted) return;
    if (s->spilled) {
        DevBuf<uint32_t> counts(size_t(n) + 1);
        LAUNCH(spill_counts_kernel2, gridn(size_t(n) + 1, 256), 256, 0, s->ocnt.p, n, s->offer_cap, counts.p);
        ex_scan(counts.p, s->ov_off.p, n);
        const uint32_t m = s->spilled;
        DevBuf<uint32_t> idx(m), idx2(m), tgt2(m);
        LAUNCH(iota_u32_kernel, gridn(m, 256), 256, 0, idx.p, m);
        int bits = 1;
        while ((uint64_t(1) << bits) < n) ++bits;
        size_t tmp = 0;
        CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp, s->ov_tgt.p, tgt2.p, idx.p, idx2.p, m, 0, bits, stream()));
        DevBuf<unsigned char> t(std::max<size_t>(tmp, 1));
        prof_begin("cub_radix_sort_spill");
        CK(cub::DeviceRadixSort::SortPairs(t.p, tmp, s->ov_tgt.p, tgt2.p, idx.p, idx2.p, m, 0, bits, stream()));
        prof_end();
        note_launch();
        DevBuf<uint64_t> key2(s->ov_cap);
        DevBuf<uint32_t> src2(s->ov_cap);
        LAUNCH(gather_spill_kernel, gridn(m, 256), 256, 0, idx2.p, m, s->ov_key.p, s->ov_src.p, key2.p, src2.p);
        CK(cudaMemcpyAsync(s->ov_tgt.p, tgt2.p, size_t(m) * 4, cudaMemcpyDeviceToDevice, stream()));
        std::swap(s->ov_key, key2);
        std::swap(s->ov_src, src2);
    }
    s->spill_sorted = true;
}

uint64_t replay_offers(annk_state* s, uint32_t lo, uint32_t hi) {
    if (hi <= lo) return 0;
    group_spills(s);
    RArgs a{};
    a.lo = lo;
    a.hi = hi;
    a.P = s->P;
    a.cap = s->offer_cap;
    a.keys = s->keys.p;
    a.flags = s->flags.p;
    a.sizes = s->sizes.p;
    a.ocnt = s->ocnt.p;
    a.obuf = s->obuf.p;
    a.osrc = s->osrc.p;
    a.ov_off = s->ov_off.p;
    a.ov_key = s->ov_key.p;
    a.ov_src = s->ov_src.p;
    DevBuf<unsigned long long> changes(1);
    DevBuf<uint32_t> ctr(2);  // [0] work counter, [1] deferred count
    DevBuf<uint32_t> big(size_t(hi - lo));
    changes.zero();
    ctr.zero();
    a.changes = changes.p;
    a.next = ctr.p;
    a.nbig = ctr.p + 1;
    a.big = big.p;
    a.runmax = 256;
    uint32_t wpb = 8;
    while (wpb > 1 && replay_warp_bytes(a.P, a.runmax) * wpb > 96 * 1024) wpb /= 2;
    const size_t smem = replay_warp_bytes(a.P, a.runmax) * wpb;
    if (smem > size_t(max_smem_optin())) throw_invalid("refine: pool_cap too large for the device path");
    CK(cudaFuncSetAttribute(replay_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, replay_kernel, wpb * 32, smem));
    const uint32_t grid = std::min<uint32_t>((hi - lo + wpb - 1) / wpb, uint32_t(num_sms()) * std::max(per_sm, 1));
    LAUNCH(replay_kernel, grid, wpb * 32, smem, a);
    uint32_t nb = 0;
    CK(cudaMemcpyAsync(&nb, ctr.p + 1, 4, cudaMemcpyDeviceToHost, stream()));
    ssync();
    if (nb) {
        // targets with more source runs than fit shared memory: runs in global scratch
        DevBuf<uint64_t> sizes(size_t(nb) + 1), off(size_t(nb) + 1);
        LAUNCH(big_sizes_kernel, gridn(size_t(nb) + 1, 256), 256, 0, big.p, nb, s->ocnt.p, sizes.p);
        ex_scan(sizes.p, off.p, nb);
        uint64_t total = 0;
        CK(cudaMemcpyAsync(&total, off.p + nb, 8, cudaMemcpyDeviceToHost, stream()));
        ssync();
        DevBuf<uint64_t> rk(total);
        DevBuf<uint32_t> ps(total), so(total);
        a.big_list = big.p;
        a.big_n = nb;
        a.big_off = off.p;
        a.g_runkey = rk.p;
        a.g_pstart = ps.p;
        a.g_seqoff = so.p;
        LAUNCH(replay_kernel, gridn(size_t(nb) * 32, wpb * 32), wpb * 32, smem, a);
    }
    unsigned long long c = 0;
    changes.download(&c, 1);
    ssync();
    return c;
}

}  // namespace annk
