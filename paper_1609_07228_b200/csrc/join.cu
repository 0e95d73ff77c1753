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

#include <type_traits>

#include <algorithm>
#include <cstdio>
#include <chrono>
#include <cstdlib>
#include <thread>
#include <cstring>

#include "join.cuh"

namespace annk {
namespace {

constexpr uint32_t kWX = 16;     // fp32 rows: interleaved exact chains per lane
constexpr uint32_t kStrip = 8;   // u8 rows: list rows per distance strip (the upper half of an IMMA m-tile)
constexpr uint32_t kStripF = 16; // fp32 rows: one strip = kWX chains, so every partner row is read A/16 times
constexpr uint32_t kFC = 16;     // fp32 rows: dimensions per staged chunk (double-buffered: 2 x 3 KB per warp)
constexpr uint32_t kFG = kFC / 4;  // 16-byte pieces per staged row chunk
// window row r's 16-byte pieces are XOR-swizzled so 8 lanes reading the same
// piece of 8 different rows hit 8 different bank groups
__device__ __forceinline__ uint32_t fswz(uint32_t r) { return (r >> 1) & (kFG - 1); }
constexpr uint32_t kPad = 64;    // member arrays padded so a partner window may read past the list
constexpr uint32_t kMemRegs = 5;  // list members held per lane (lists <= 160): next-point fetch, reservations
enum : int { kModeU8 = 0, kModeF32 = 1 };

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
    uint32_t* next;  // visit-list work counter
    uint32_t* ocnt;
    uint64_t* obuf;
    uint32_t* osrc;
    uint32_t* ov_cnt;
    uint32_t* ov_tgt;
    uint64_t* ov_key;
    uint32_t* ov_src;
    uint32_t ov_cap;
    unsigned long long* counters;  // [0] comps, [1] offers
    uint32_t strip;  // list rows per distance strip (kStrip u8, kStripF fp32)
    uint32_t stage_words;  // fp32 rows: shared staging of one 32-dimension chunk of the strip and window rows
    uint32_t rn;     // per-member array length: list capacity 3S + P rounded up to 32
    uint32_t rs;     // D strip row stride (floats)
    uint32_t dbg_n;  // points (debug bounds checks)
    uint32_t ol;     // offer buffer capacity
};

// Per-warp shared memory: one warp processes one point at a time.
struct WLayout {
    size_t thr, bkey, ids, nrm, mc, mb, mf, ms, D, canon, bmem, stage, total;
};
__host__ __device__ inline WLayout w_layout(const JArgs& a) {
    WLayout L;
    size_t o = 0;
    L.thr = o;   o += al16(size_t(a.rn + kPad) * 8);
    L.bkey = o;  o += al16(size_t(a.ol) * 8);
    L.ids = o;   o += al16(size_t(a.rn + kPad) * 4);
    L.nrm = o;   o += al16(size_t(a.rn) * 4);
    L.mc = o;    o += al16(size_t(a.rn) * 4);
    L.mb = o;    o += al16(size_t(a.rn) * 4);
    L.mf = o;    o += al16(size_t(a.rn) * 4);
    L.ms = o;    o += al16(size_t(a.rn) * 4);
    L.D = o;     o += al16(size_t(a.strip) * a.rs * 4);
    L.canon = o; o += al16(size_t(a.rn + kPad) * 2);
    L.bmem = o;  o += al16(size_t(a.ol) * 2);
    L.stage = o; o += al16(size_t(a.stage_words) * 4);
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

__device__ __forceinline__ uint4 ldg128(const uint8_t* p) { return __ldg(reinterpret_cast<const uint4*>(p)); }

// D[x - xb][y] for the strip rows x in [xb, xb + 8) and y in (x, R): the
// squared distance of list members x and y (cells with y <= x are ignored).
template <int MODE>
__device__ __forceinline__ void strip_distances(const JArgs& a, const uint32_t* ids, const int32_t* nrm, float* D,
                                                uint32_t xb, uint32_t xe, uint32_t R, float* stage) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t yb0 = (xb + 1) / 32, yb1 = (R + 31) / 32;
    if (MODE == kModeU8) {
        // IMMA m16n8k32 tiles (both 8-row halves hold the strip) x 32 y-columns, K = row bytes, read
        // straight from the u8 rows (L1-resident: prefetched one point ahead).
        // A dot product does not depend on the order of its terms, so a lane
        // loads 16 contiguous bytes per row and feeds them to two k-steps (the
        // same k permutation for both operands).
        const uint32_t g = lane >> 2, t = lane & 3;
        const uint32_t kb = rup(a.ld8, 64);
        const uint8_t* ra0 = a.x8 + size_t(ids[min(xb + g, R - 1)]) * a.ld8 + t * 16;
        const int32_t n_0 = nrm[xb + g];
        for (uint32_t yb = yb0; yb < yb1; ++yb) {
            const uint32_t n0 = yb * 32;
            int32_t acc[4][4];
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[q][0] = acc[q][1] = acc[q][2] = acc[q][3] = 0;
            const uint8_t* rb[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) rb[q] = a.x8 + size_t(ids[min(n0 + q * 8 + g, R - 1)]) * a.ld8 + t * 16;
            for (uint32_t k0 = 0; k0 < kb; k0 += 64) {
                const bool in = k0 + t * 16 < a.ld8;
                const uint4 z = make_uint4(0, 0, 0, 0);
                const uint4 u0 = in ? ldg128(ra0 + k0) : z, u1 = u0;
                uint4 v[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) v[q] = in ? ldg128(rb[q] + k0) : z;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    mma_u8(acc[q], u0.x, u1.x, u0.y, u1.y, v[q].x, v[q].y);
                    mma_u8(acc[q], u0.z, u1.z, u0.w, u1.w, v[q].z, v[q].w);
                }
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint32_t c = n0 + q * 8 + 2 * t;
                const int32_t nc0 = nrm[c], nc1 = nrm[c + 1];
                *reinterpret_cast<float2*>(D + size_t(g) * a.rs + c) =
                    make_float2(float(n_0 + nc0 - 2 * acc[q][0]), float(n_0 + nc1 - 2 * acc[q][1]));
            }
        }
    } else {
        // fp32 rows: the strip's kWX rows and a window of 32 partner rows are staged
        // through shared memory 32 dimensions at a time by cp.async (16-byte
        // pieces, double-buffered: the next chunk lands while this one is used);
        // each lane runs kWX interleaved exact chains (graph_build.cpp l2_sq order:
        // index ascending; the zero fill past the row adds +0 exactly) for its
        // partner.  Window rows are stored with the 16-byte pieces of row r
        // XOR-swizzled by r & 7, so the lanes' LDS.128 column reads are
        // conflict-free; strip rows are read as broadcasts.
        const uint32_t nxr = xe - xb;
        const uint32_t sbase = uint32_t(__cvta_generic_to_shared(stage));
        const uint32_t nchunk = (a.ld + kFC - 1) / kFC;
        for (uint32_t yb = max(yb0, (xb + 1) / 32); yb < yb1; ++yb) {
            const float* xsrc[kWX * kFG / 32];
            const float* ysrc[32 * kFG / 32];
#pragma unroll
            for (uint32_t j = 0; j < kWX * kFG / 32; ++j) {
                const uint32_t e = j * 32 + lane, r = e / kFG;
                xsrc[j] = a.x + size_t(ids[xb + min(r, nxr - 1)]) * a.ld + (e % kFG) * 4;
            }
#pragma unroll
            for (uint32_t j = 0; j < 32 * kFG / 32; ++j) {
                const uint32_t e = j * 32 + lane, r = e / kFG;
                ysrc[j] = a.x + size_t(ids[min(yb * 32 + r, R - 1)]) * a.ld + (e % kFG) * 4;
            }
            auto issue = [&](uint32_t c, uint32_t buf) {
                const uint32_t c0 = c * kFC;
                const uint32_t xo = sbase + buf * (kWX * kFC + 32 * kFC) * 4, yo = xo + kWX * kFC * 4;
#pragma unroll
                for (uint32_t j = 0; j < kWX * kFG / 32; ++j) {
                    const uint32_t e = j * 32 + lane, r = e / kFG, g = e % kFG;
                    const uint32_t bytes = c0 + g * 4 < a.ld ? 16u : 0u;
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(xo + (r * kFC + g * 4) * 4),
                                 "l"(xsrc[j] + (bytes ? c0 : 0)), "r"(bytes)
                                 : "memory");
                }
#pragma unroll
                for (uint32_t j = 0; j < 32 * kFG / 32; ++j) {
                    const uint32_t e = j * 32 + lane, r = e / kFG, g = e % kFG;
                    const uint32_t bytes = c0 + g * 4 < a.ld ? 16u : 0u;
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(
                                     yo + (r * kFC + ((g ^ fswz(r)) * 4)) * 4),
                                 "l"(ysrc[j] + (bytes ? c0 : 0)), "r"(bytes)
                                 : "memory");
                }
                asm volatile("cp.async.commit_group;" ::: "memory");
            };
            // only as many chains as the strip has rows (the last strip of a point is often short)
            auto chains = [&](auto ncw) {
                constexpr uint32_t NC = decltype(ncw)::value;
                float acc[NC];
#pragma unroll
                for (uint32_t k = 0; k < NC; ++k) acc[k] = 0.0f;
                issue(0, 0);
                for (uint32_t c = 0; c < nchunk; ++c) {
                    const uint32_t buf = c & 1;
                    if (c + 1 < nchunk) {
                        issue(c + 1, buf ^ 1);
                        asm volatile("cp.async.wait_group 1;" ::: "memory");
                    } else {
                        asm volatile("cp.async.wait_group 0;" ::: "memory");
                    }
                    __syncwarp();
                    const float* xs = stage + buf * (kWX * kFC + 32 * kFC);
                    const float* ys = xs + kWX * kFC + lane * kFC;
                    const uint32_t cw = min(kFC, a.ld - c * kFC);  // a multiple of 4
                    for (uint32_t k = 0; k < cw; k += 4) {
                        const float4 bv = *reinterpret_cast<const float4*>(ys + (((k >> 2) ^ fswz(lane)) << 2));
#pragma unroll
                        for (uint32_t u = 0; u < NC; ++u) {
                            const float4 v = *reinterpret_cast<const float4*>(xs + u * kFC + k);
                            float d;
                            d = __fsub_rn(v.x, bv.x); acc[u] = __fadd_rn(acc[u], __fmul_rn(d, d));
                            d = __fsub_rn(v.y, bv.y); acc[u] = __fadd_rn(acc[u], __fmul_rn(d, d));
                            d = __fsub_rn(v.z, bv.z); acc[u] = __fadd_rn(acc[u], __fmul_rn(d, d));
                            d = __fsub_rn(v.w, bv.w); acc[u] = __fadd_rn(acc[u], __fmul_rn(d, d));
                        }
                    }
                    __syncwarp();  // this buffer is refilled two chunks later
                }
                const uint32_t y = yb * 32 + lane;
#pragma unroll
                for (uint32_t u = 0; u < NC; ++u)
                    if (u < nxr) D[size_t(u) * a.rs + y] = acc[u];
            };
            if (nxr <= 4) chains(std::integral_constant<uint32_t, 4>{});
            else if (nxr <= 8) chains(std::integral_constant<uint32_t, 8>{});
            else chains(std::integral_constant<uint32_t, kWX>{});
        }
    }
}

// Hands the buffered offers (in the reference's pair order) to their targets:
// a stable counting sort by target keeps each target's offers from this point
// contiguous and in order, reserved with ONE global atomic per target.
__device__ __forceinline__ void join_flush(const JArgs& a, uint32_t i, uint32_t c, uint32_t R, const uint32_t* ids,
                                           const uint64_t* bkey, const uint16_t* bmem, uint32_t* mc, uint32_t* mb,
                                           uint32_t* mf, uint32_t* ms) {
    const uint32_t lane = threadIdx.x & 31, lt = (1u << lane) - 1u;
    for (uint32_t e0 = 0; e0 < c; e0 += 32) {
        const uint32_t e = e0 + lane;
        const bool v = e < c;
        const uint32_t m = v ? bmem[e] : 0xffffu;
        const uint32_t mask = __match_any_sync(0xffffffffu, m);
        if (v && (mask & lt) == 0) mc[m] += __popc(mask);
        __syncwarp();
    }
    // slot reservations: a lane's (up to kMemRegs) atomics are all in flight before
    // any result is used
    {
        uint32_t run[kMemRegs], base[kMemRegs];
#pragma unroll
        for (uint32_t k = 0; k < kMemRegs; ++k) {
            const uint32_t m = k * 32 + lane;
            run[k] = m < R ? mc[m] : 0u;
            base[k] = run[k] ? atomicAdd(&a.ocnt[ids[m]], run[k]) : 0u;
        }
#pragma unroll
        for (uint32_t k = 0; k < kMemRegs; ++k) {
            const uint32_t m = k * 32 + lane;
            if (run[k]) {
                const uint32_t fix = base[k] < a.cap ? min(run[k], a.cap - base[k]) : 0u;
                mb[m] = base[k];
                mf[m] = fix;
                ms[m] = run[k] > fix ? atomicAdd(a.ov_cnt, run[k] - fix) : 0u;
                mc[m] = 0;
            }
        }
    }
    for (uint32_t m = kMemRegs * 32 + lane; m < R; m += 32) {  // lists longer than the registers cover
        const uint32_t run = mc[m];
        if (run) {
            const uint32_t base = atomicAdd(&a.ocnt[ids[m]], run);
            const uint32_t fix = base < a.cap ? min(run, a.cap - base) : 0u;
            mb[m] = base;
            mf[m] = fix;
            ms[m] = run > fix ? atomicAdd(a.ov_cnt, run - fix) : 0u;
            mc[m] = 0;
        }
    }
    __syncwarp();
    for (uint32_t e0 = 0; e0 < c; e0 += 32) {
        const uint32_t e = e0 + lane;
        const bool v = e < c;
        const uint32_t m = v ? bmem[e] : 0xffffu;
        const uint32_t mask = __match_any_sync(0xffffffffu, m);
        const uint32_t r = v ? mc[m] + __popc(mask & lt) : 0u;
        __syncwarp();
        if (v) {
            if ((mask & lt) == 0) mc[m] += __popc(mask);
            const uint32_t tgt = ids[m];
            const uint64_t key = bkey[e];
            if (r < mf[m]) {
                const size_t slot = size_t(tgt) * a.cap + mb[m] + r;
                DCHK(mb[m] + r < a.cap && tgt < a.dbg_n);
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
    for (uint32_t m = lane; m < R; m += 32) mc[m] = 0;
    __syncwarp();
}

// Next visited point: the visit list is handed out one point per request.
__device__ __forceinline__ void join_next_point(const JArgs& a, uint32_t& pi, uint32_t& pa, uint32_t& pb) {
    const uint32_t lane = threadIdx.x & 31;
    for (;;) {
        uint32_t o = 0;
        if (lane == 0) o = atomicAdd(a.next, 1u);
        o = __shfl_sync(0xffffffffu, o, 0);
        if (o >= a.n_visit) {
            pa = pb = 0;
            pi = 0xffffffffu;
            return;
        }
        pi = a.order ? __ldg(a.order + o) : o;
        if (pi < a.ilo || pi >= a.ihi) continue;
        pa = __ldg(a.gncnt + pi);
        if (pa == 0) continue;
        pb = __ldg(a.gocnt + pi);
        return;
    }
}


// One warp per point (persistent; points handed out by a counter).  The
// point's list members are staged, the pair distances computed a 16-row strip
// at a time, and the offers emitted row by row in the reference's order
// (graph_build.cpp:135-152: row x = new[a], partners y > x ascending, y -> x
// before x -> y) into a per-warp buffer flushed at row boundaries.  The next
// point's header and members are fetched while the current one is processed.
template <int MODE>
__global__ void __launch_bounds__(32) join_kernel(JArgs a) {
    extern __shared__ __align__(16) unsigned char sm[];
    const WLayout L = w_layout(a);
    uint64_t* thr_s = reinterpret_cast<uint64_t*>(sm + L.thr);
    uint64_t* bkey = reinterpret_cast<uint64_t*>(sm + L.bkey);
    uint32_t* ids = reinterpret_cast<uint32_t*>(sm + L.ids);
    int32_t* nrm = reinterpret_cast<int32_t*>(sm + L.nrm);
    uint32_t* mc = reinterpret_cast<uint32_t*>(sm + L.mc);
    uint32_t* mb = reinterpret_cast<uint32_t*>(sm + L.mb);
    uint32_t* mf = reinterpret_cast<uint32_t*>(sm + L.mf);
    uint32_t* ms = reinterpret_cast<uint32_t*>(sm + L.ms);
    float* D = reinterpret_cast<float*>(sm + L.D);
    uint16_t* canon = reinterpret_cast<uint16_t*>(sm + L.canon);
    uint16_t* bmem = reinterpret_cast<uint16_t*>(sm + L.bmem);
    float* stage = reinterpret_cast<float*>(sm + L.stage);
    const uint32_t lane = threadIdx.x & 31, lt = (1u << lane) - 1u;
    unsigned long long comps = 0, offers = 0;
    for (uint32_t m = lane; m < a.rn; m += 32) {
        mc[m] = 0;
        nrm[m] = 0;
    }
    uint32_t i, A, B;
    join_next_point(a, i, A, B);
    uint32_t mid[kMemRegs], mnrm[kMemRegs];
    uint64_t mthr[kMemRegs];
#define JOIN_FETCH(pi, pa, pb)                                                                               \
    _Pragma("unroll") for (uint32_t k = 0; k < kMemRegs; ++k) {                                          \
        const uint32_t r = k * 32 + lane;                                                                    \
        if (r < (pa) + (pb)) {                                                                               \
            mid[k] = r < (pa) ? __ldg(a.gnew + size_t(pi) * 2 * a.S + r)                                     \
                              : __ldg(a.gold + size_t(pi) * (a.P + a.S) + (r - (pa)));                       \
            mthr[k] = __ldg(a.thr + mid[k]);                                                                 \
            if (MODE == kModeU8) mnrm[k] = uint32_t(__ldg(a.norms + mid[k]));                                \
        }                                                                                                    \
    }
    JOIN_FETCH(i, A, B)
    while (A) {
        const uint32_t R = A + B;
#pragma unroll
        for (uint32_t k = 0; k < kMemRegs; ++k) {
            const uint32_t r = k * 32 + lane;
            if (r < R) {
                ids[r] = mid[k];
                thr_s[r] = mthr[k];
                nrm[r] = int32_t(mnrm[k]);
            }
        }
        for (uint32_t r = kMemRegs * 32 + lane; r < R; r += 32) {  // lists longer than the registers hold
            const uint32_t id = r < A ? a.gnew[size_t(i) * 2 * a.S + r] : a.gold[size_t(i) * (a.P + a.S) + r - A];
            ids[r] = id;
            thr_s[r] = a.thr[id];
            if (MODE == kModeU8) nrm[r] = a.norms[id];
        }
        __syncwarp();
        // a member in both lists (new[a] == old[l]) is one pool: its offers are
        // counted under its new-list position
        for (uint32_t r = A + lane; r < R; r += 32) {
            const uint32_t v = ids[r];
            uint32_t lo = 0, hi = A;
            while (lo < hi) {
                const uint32_t md = (lo + hi) >> 1;
                if (ids[md] < v) lo = md + 1;
                else hi = md;
            }
            const bool dual = lo < A && ids[lo] == v;
            canon[r] = uint16_t(dual ? lo : r);
            comps -= dual ? 1u : 0u;
        }
        for (uint32_t r = lane; r < A; r += 32) canon[r] = uint16_t(r);
        // distance computations (graph_build.cpp:138-150): every new x with each
        // later member, except a member against itself (an id in both lists)
        if (lane == 0) comps += uint64_t(A) * (R - 1) - uint64_t(A) * (A - 1) / 2;
        uint32_t ni, nA, nB;
        join_next_point(a, ni, nA, nB);
        __syncwarp();
        uint32_t nbuf = 0;
        constexpr uint32_t strip = MODE == kModeU8 ? kStrip : kStripF;
        for (uint32_t xb = 0; xb < A; xb += strip) {
            const uint32_t xe = min(A, xb + strip);
            strip_distances<MODE>(a, ids, nrm, D, xb, xe, R, stage);
            if (xb == 0) {
                JOIN_FETCH(ni, nA, nB)  // next point's members: in flight while this one is processed
            }
            __syncwarp();
            // the strip's pairs (x, y > x), x = xb..xe-1, flattened in the reference's
            // order (row-major) so every lane of a window carries a pair; per pair
            // y -> x is offered before x -> y (graph_build.cpp:135-152)
            uint32_t off[kStripF + 1];
            {
                uint32_t o = 0;
#pragma unroll
                for (uint32_t r = 0; r <= kStripF; ++r) {
                    off[r] = o;
                    if (r < strip && xb + r < xe) o += R - (xb + r) - 1;
                    else o = 0xffffffffu;  // rows past the strip: never reached
                }
            }
            uint32_t total = 0;
#pragma unroll
            for (uint32_t r = 1; r <= kStripF; ++r)
                if (r <= xe - xb) total = off[r];
            for (uint32_t p0 = 0; p0 < total; p0 += 64) {
                if (nbuf + 128 > a.ol) {  // a step adds at most 128 offers (ol >= 2 rn >= 128)
                    join_flush(a, i, nbuf, R, ids, bkey, bmem, mc, mb, mf, ms);
                    offers += nbuf;
                    nbuf = 0;
                }
                bool ox[2], oy[2];
                uint64_t kx[2], ky[2];
                uint32_t bx[2], by[2];
                uint16_t mx_[2], my_[2];
#pragma unroll
                for (int h = 0; h < 2; ++h) {  // two 32-pair windows per step (their loads overlap)
                    const uint32_t pp = p0 + 32 * h + lane;
                    uint32_t r = 0, offr = 0;
#pragma unroll
                    for (uint32_t k = 1; k < kStripF; ++k)
                        if (k < strip && pp >= off[k]) {
                            r = k;
                            offr = off[k];
                        }
                    const bool in = pp < total;
                    const uint32_t x = xb + r;
                    const uint32_t y = in ? x + 1 + (pp - offr) : x + 1;  // < rn + kPad: reads stay in the arrays
                    const uint32_t idx = ids[x], idy = ids[y];
                    const float d = D[size_t(r) * a.rs + y];
                    const uint64_t tx = thr_s[x], thy = thr_s[y];
                    const bool valid = in && idy != idx;  // graph_build.cpp:146 (l == j is skipped)
                    kx[h] = make_key(d, idy);
                    ky[h] = make_key(d, idx);
                    ox[h] = valid && kx[h] < tx;
                    oy[h] = valid && ky[h] < thy;
                    mx_[h] = canon[x];
                    my_[h] = canon[y];
                    bx[h] = __ballot_sync(0xffffffffu, ox[h]);
                    by[h] = __ballot_sync(0xffffffffu, oy[h]);
                }
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const uint32_t q = nbuf + __popc(bx[h] & lt) + __popc(by[h] & lt);
                    DCHK(!(ox[h] || oy[h]) || q + (ox[h] && oy[h] ? 1u : 0u) < a.ol);
                    if (ox[h]) {
                        bkey[q] = kx[h];
                        bmem[q] = mx_[h];
                    }
                    if (oy[h]) {
                        bkey[q + (ox[h] ? 1 : 0)] = ky[h];
                        bmem[q + (ox[h] ? 1 : 0)] = my_[h];
                    }
                    nbuf += __popc(bx[h]) + __popc(by[h]);
                }
            }
            __syncwarp();
        }
        if (MODE == kModeU8) {  // next point's rows (one 128-byte line each) into L1
#pragma unroll
            for (uint32_t k = 0; k < kMemRegs; ++k)
                if (k * 32 + lane < nA + nB) asm volatile("prefetch.global.L1 [%0];" ::"l"(a.x8 + size_t(mid[k]) * a.ld8));
        }
        if (nbuf) {
            join_flush(a, i, nbuf, R, ids, bkey, bmem, mc, mb, mf, ms);
            offers += nbuf;
        }
        i = ni;
        A = nA;
        B = nB;
    }
#undef JOIN_FETCH
    for (int o = 16; o > 0; o >>= 1) comps += __shfl_xor_sync(0xffffffffu, comps, o);
    if (lane == 0) {
        if (comps) atomicAdd(&a.counters[0], comps);
        if (offers) atomicAdd(&a.counters[1], offers);
    }
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
    uint32_t* next;            // work counter
    const uint32_t* list;      // targets to replay (nullptr: the range [lo, hi))
    uint32_t list_n;
    uint32_t runmax;           // source runs held in shared memory per warp
    uint32_t* def;             // targets with more runs than that, deferred to a later pass
    uint32_t* def_nr;          // ... and their run counts
    uint32_t* ndef;
    const uint64_t* g_off;     // global-scratch pass: per listed target, its scratch start
    uint64_t* g_runkey;
    uint32_t* g_pstart;
    uint32_t* g_seqoff;
};

__host__ __device__ inline size_t replay_warp_bytes(uint32_t P, uint32_t runmax) {
    return al16(size_t(P) * 8) + al16(size_t(P)) + 64 * 8 + al16(size_t(runmax) * 8) +
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

// Replays target t's offers.  Returns 0, or (pool untouched) the target's
// number of source runs when it exceeds `runmax`.
__device__ uint32_t replay_target(const RArgs& a, uint32_t t, uint64_t* S, uint8_t* SF, uint64_t* accs, uint64_t* wk, uint64_t* runkey, uint32_t* pstart, uint32_t* seqoff, uint32_t runmax,
                              unsigned long long& changes) {
    const uint32_t lane = threadIdx.x & 31, lt = (1u << lane) - 1u;
    const uint32_t m = a.ocnt[t];
    if (m == 0) return 0;
    const uint32_t cf = min(m, a.cap);
    const uint64_t* k0 = a.obuf + size_t(t) * a.cap;
    const uint32_t* s0 = a.osrc + size_t(t) * a.cap;
    const uint32_t spill = m > cf ? a.ov_off[t] : 0u;
    const uint64_t* k1 = a.ov_key + spill;
    const uint32_t* s1 = a.ov_src + spill;
    // runs: maximal stretches of one source (a segment boundary always starts one)
    uint32_t nr = 0, lastsrc = 0;
    for (uint32_t q00 = 0; q00 < m; q00 += 64) {
        uint32_t src2[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {  // both windows' loads in flight together
            const uint32_t q = q00 + 32 * h + lane;
            src2[h] = q < m ? (q < cf ? s0[q] : s1[q - cf]) : 0u;
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const uint32_t q = q00 + 32 * h + lane;
            const bool v = q < m;
            const uint32_t src = src2[h];
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
    }
    if (nr > runmax) return nr;
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
        __syncwarp();
        // run r covers sequence positions [seqoff[r], seqoff[r+1]); position q maps to
        // slot q + delta[r] (delta kept in runkey's low word once the order is fixed)
        for (uint32_t r = lane; r < nr; r += 32)
            runkey[r] = uint32_t(pstart[uint32_t(runkey[r])] - seqoff[r]);
        if (lane == 0) seqoff[nr] = m;
        __syncwarp();
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
    uint32_t rbase = 0;  // the run holding the window's first position
    for (uint32_t q0 = 0; q0 < m; q0 += 32) {
        const uint32_t q = q0 + lane;
        // runs starting inside the window: bit o set if one starts at q0 + o
        const uint32_t rj = rbase + 1 + lane;
        const uint32_t bo = rj < nr ? seqoff[rj] - q0 : 64u;
        const uint32_t bm = __reduce_or_sync(0xffffffffu, bo < 32 ? 1u << bo : 0u);
        const uint32_t run = rbase + __popc(bm & ((2u << lane) - 1u));
        uint64_t c = kEmptyKey;
        if (q < m) {
            const uint32_t pos = q + uint32_t(runkey[run]);
            DCHK(pos < m && run < nr);
            c = pos < cf ? k0[pos] : k1[pos - cf];
        }
        rbase += __popc(__ballot_sync(0xffffffffu, bo <= 32));
        const bool cand = c < tail;
        const uint32_t cm = __ballot_sync(0xffffffffu, cand);
        if (cm == 0) continue;
        uint32_t rS = 0;
        bool dupS = false;
        if (cand) {
            rS = lower_bound64(S, sz, c);
            dupS = rS < sz && S[rS] == c;
        }
        // a key equal to an earlier one in the window is a duplicate (the earlier
        // copy entered the pool or was rejected with the same rank)
        const uint32_t eq = __match_any_sync(0xffffffffu, c);
        const bool first = cand && !dupS && (eq & lt & cm) == 0;
        const uint32_t fm = __ballot_sync(0xffffffffu, first);
        wk[lane] = c;
        __syncwarp();
        // rank at arrival: pool keys below it + earlier first occurrences below it
        uint32_t below = 0;
        for (uint32_t bits = fm & lt; bits; bits &= bits - 1) below += wk[__ffs(bits) - 1] < c ? 1u : 0u;
        const bool acc = first && rS + below < a.P;
        const uint32_t am = __ballot_sync(0xffffffffu, acc);
        if (am == 0) {
            __syncwarp();
            continue;
        }
        const uint32_t na = __popc(am);
        // merge in place: accepted keys ranked among themselves; pool entries at
        // or above the lowest insertion point move up by the accepted keys below
        // them (top-down 32-entry chunks: a chunk is read before it is written)
        uint32_t arank = 0;
        if (acc)
            for (uint32_t bits = am; bits; bits &= bits - 1) arank += wk[__ffs(bits) - 1] < c ? 1u : 0u;
        const uint32_t pmin = __reduce_min_sync(0xffffffffu, acc ? rS : 0xffffffffu);
        __syncwarp();
        if (acc) accs[arank] = c;
        __syncwarp();
        for (int32_t hi = int32_t(sz); hi > int32_t(pmin); hi -= 32) {
            const int32_t p = hi - 32 + int32_t(lane);
            uint64_t v = 0;
            uint8_t f = 0;
            uint32_t np = 0xffffffffu;
            if (p >= int32_t(pmin)) {
                v = S[p];
                f = SF[p];
                np = uint32_t(p) + lower_bound64(accs, na, v);
            }
            __syncwarp();
            if (np < a.P) {
                S[np] = v;
                SF[np] = f;
            }
            __syncwarp();
        }
        DCHK(!acc || arank < 32);
        if (acc && rS + arank < a.P) {
            S[rS + arank] = c;
            SF[rS + arank] = 1;  // arrived this round: flag_new
        }
        __syncwarp();
        sz = min(a.P, sz + na);
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
    return 0;
}

__global__ void replay_kernel(RArgs a) {
    extern __shared__ __align__(16) unsigned char sm[];
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned char* base = sm + size_t(warp) * replay_warp_bytes(a.P, a.runmax);
    uint64_t* S = reinterpret_cast<uint64_t*>(base);
    uint8_t* SF = base + al16(size_t(a.P) * 8);
    uint64_t* accs = reinterpret_cast<uint64_t*>(SF + al16(a.P));
    uint64_t* wk = accs + 32;
    uint64_t* runkey = wk + 32;
    uint32_t* pstart = reinterpret_cast<uint32_t*>(runkey + a.runmax);
    uint32_t* seqoff = reinterpret_cast<uint32_t*>(reinterpret_cast<unsigned char*>(pstart) +
                                                   al16(size_t(a.runmax + 1) * 4));
    unsigned long long changes = 0;
    const uint32_t items = a.list ? a.list_n : a.hi - a.lo;
    for (;;) {
        uint32_t w = 0;
        if (lane == 0) w = atomicAdd(a.next, 1u);
        w = __shfl_sync(0xffffffffu, w, 0);
        if (w >= items) break;
        const uint32_t t = a.list ? a.list[w] : a.lo + w;
        uint32_t nr;
        if (a.g_runkey) {
            const uint64_t o = a.g_off[w];
            nr = replay_target(a, t, S, SF, accs, wk, a.g_runkey + o, a.g_pstart + o, a.g_seqoff + o,
                               0xffffffffu, changes);
        } else {
            nr = replay_target(a, t, S, SF, accs, wk, runkey, pstart, seqoff, a.runmax, changes);
        }
        if (nr && lane == 0) {
            const uint32_t d = atomicAdd(a.ndef, 1u);
            a.def[d] = t;
            a.def_nr[d] = nr;
        }
    }
    if (lane == 0 && changes) atomicAdd(a.changes, changes);
}

// ------------------------------------------------------------ compaction
// Most offers of a round repeat an id already in the target's pool (94% of the
// candidates of round 2 at cfg2).  Such an offer is never accepted: either the
// entry is still there when it arrives (NeighborPool::insert rejects the
// duplicate) or it was evicted earlier in the round, which only happens to the
// maximum of a full pool, and the tail stays below the evicted key ever since.
// Before the ordered replay, every target's offers are filtered against an id
// table of its current pool and compacted in place, storage order (hence the
// source runs and the reference order) preserved; pools, flags and `changes`
// are unchanged.
struct CArgs {
    uint32_t lo, hi, P, cap;
    const uint64_t* keys;
    const uint32_t* sizes;
    uint32_t* ocnt;
    uint64_t* obuf;
    uint32_t* osrc;
    const uint32_t* ov_off;
    uint64_t* ov_key;
    uint32_t* ov_src;
    uint32_t* next;
    uint32_t hbits;
    unsigned long long* dropped;
};

__device__ __forceinline__ uint32_t ct_hash(uint32_t id, uint32_t mask) { return (id * 0x9E3779B1u >> 7) & mask; }

__global__ void __launch_bounds__(256) offer_compact_kernel(CArgs a) {
    extern __shared__ __align__(16) uint32_t csm[];
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, lt = (1u << lane) - 1u;
    const uint32_t hslots = 1u << a.hbits;
    uint32_t* H = csm + size_t(warp) * hslots;
    unsigned long long dropped = 0;
    const uint32_t items = a.hi - a.lo;
    for (;;) {
        uint32_t w = 0;
        if (lane == 0) w = atomicAdd(a.next, 1u);
        w = __shfl_sync(0xffffffffu, w, 0);
        if (w >= items) break;
        const uint32_t t = a.lo + w;
        const uint32_t m = a.ocnt[t];
        if (m == 0) continue;
        const uint32_t cf = min(m, a.cap);
        uint64_t* k0 = a.obuf + size_t(t) * a.cap;
        uint32_t* s0 = a.osrc + size_t(t) * a.cap;
        const uint32_t spill = m > cf ? a.ov_off[t] : 0u;
        uint64_t* k1 = a.ov_key + spill;
        uint32_t* s1 = a.ov_src + spill;
        for (uint32_t j = lane; j < hslots; j += 32) H[j] = 0xffffffffu;
        __syncwarp();
        const uint32_t sz = a.sizes[t];
        // 4-slot buckets (one LDS.128 per probe), load factor <= 1/4
        const uint32_t bmask = (hslots >> 2) - 1;
        for (uint32_t j = lane; j < sz; j += 32) {
            const uint32_t id = key_id(a.keys[size_t(t) * a.P + j]);
            for (uint32_t b = ct_hash(id, bmask);; b = (b + 1) & bmask) {
                bool done = false;
#pragma unroll
                for (uint32_t e = 0; e < 4 && !done; ++e) done = atomicCAS(&H[b * 4 + e], 0xffffffffu, id) == 0xffffffffu;
                if (done) break;
            }
        }
        __syncwarp();
        uint32_t wpos = 0;
        // offers at positions < cf live in the target's slots, the rest in its spill segment;
        // survivors move to lower positions only, so a window is read before it is written
        auto pass = [&](auto spilled) {
            constexpr bool kSp = decltype(spilled)::value;
            for (uint32_t q00 = 0; q00 < m; q00 += 64) {
                uint64_t key[2];
                uint32_t src[2];
                bool keep[2];
#pragma unroll
                for (int h2 = 0; h2 < 2; ++h2) {  // both windows' loads in flight together
                    const uint32_t q = q00 + 32 * h2 + lane;
                    if (kSp) {
                        key[h2] = q < m ? (q < cf ? k0[q] : k1[q - cf]) : kEmptyKey;
                        src[h2] = q < m ? (q < cf ? s0[q] : s1[q - cf]) : 0u;
                    } else {
                        key[h2] = q < m ? k0[q] : kEmptyKey;
                        src[h2] = q < m ? s0[q] : 0u;
                    }
                }
#pragma unroll
                for (int h2 = 0; h2 < 2; ++h2) {
                    keep[h2] = q00 + 32 * h2 + lane < m;
                    if (keep[h2]) {
                        const uint32_t id = key_id(key[h2]);
                        for (uint32_t b = ct_hash(id, bmask);; b = (b + 1) & bmask) {
                            const uint4 v = *reinterpret_cast<const uint4*>(H + b * 4);
                            if (v.x == id || v.y == id || v.z == id || v.w == id) { keep[h2] = false; break; }
                            if ((v.x & v.y & v.z & v.w) != 0xffffffffu) break;  // a free slot: not present
                        }
                    }
                }
                __syncwarp();
#pragma unroll
                for (int h2 = 0; h2 < 2; ++h2) {
                    const uint32_t bal = __ballot_sync(0xffffffffu, keep[h2]);
                    if (keep[h2]) {
                        const uint32_t pos = wpos + __popc(bal & lt);
                        DCHK(pos <= q00 + 32 * h2 + lane && pos < m);
                        if (!kSp || pos < cf) {
                            k0[pos] = key[h2];
                            s0[pos] = src[h2];
                        } else {
                            k1[pos - cf] = key[h2];
                            s1[pos - cf] = src[h2];
                        }
                    }
                    wpos += __popc(bal);
                }
            }
        };
        if (m > cf) pass(std::true_type{});
        else pass(std::false_type{});
        __syncwarp();
        if (lane == 0) {
            a.ocnt[t] = wpos;
            dropped += m - wpos;
        }
    }
    if (lane == 0 && dropped) atomicAdd(a.dropped, dropped);
}

__global__ void big_sizes_kernel(const uint32_t* __restrict__ nr, uint32_t nb, uint64_t* __restrict__ out) {
    const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b < nb) out[b] = uint64_t(next_pow2(nr[b] + 1)) + 1;
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
                 uint32_t ihi, uint32_t ov_abort, JoinCounters* out) {
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
    DevBuf<uint32_t> next(1);
    counters.zero();
    next.zero();
    a.counters = counters.p;
    a.next = next.p;
    const uint32_t rmax = 3 * s->S + s->P;
    if (rmax > 0xffffu) throw_invalid("join: sample_cap/pool_cap too large for the device path");
    a.strip = ds->u8 ? kStrip : kStripF;
    a.dbg_n = s->n;
    a.stage_words = ds->u8 ? 0u : 2 * (kWX * kFC + 32 * kFC);
    a.rn = rup(rmax, 32);
    a.rs = a.rn + 8;
    a.ol = rup(std::max(384u, 2 * a.rn), 32);  // 384 (was 768): 14 instead of 11 warps per SM, join 37.2 -> 35.3 ms
    const size_t smem = w_layout(a).total;
    if (smem > size_t(max_smem_optin())) throw_invalid("join: list capacity too large for the device path");
    const void* fn = ds->u8 ? reinterpret_cast<const void*>(join_kernel<kModeU8>)
                            : reinterpret_cast<const void*>(join_kernel<kModeF32>);
    CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 32, smem));
    const uint32_t grid = std::max(1u, std::min<uint32_t>(n_visit, uint32_t(num_sms()) * std::max(per_sm, 1)));
    if (n_visit) {
        if (ds->u8) LAUNCH(join_kernel<kModeU8>, grid, 32, smem, a);
        else LAUNCH(join_kernel<kModeF32>, grid, 32, smem, a);
    }
    // A launch whose spill list outgrows ov_abort entries is thrown away by the caller
    // (the range is joined again in pieces).  For ranges large enough for that to happen
    // the host watches the spill counter from a second stream while the kernel runs and,
    // past the limit, ends the visit list (the work counter jumps beyond n_visit) so the
    // doomed launch stops early.  The kernel itself is untouched; smaller ranges (cfg2:
    // 1M points) are not watched.
    if (n_visit >= (1u << 20) && ov_abort != 0xffffffffu) {
        static cudaStream_t ps = nullptr;
        static cudaEvent_t done = nullptr;
        static uint32_t* hp = nullptr;
        if (!ps) {
            CK(cudaStreamCreateWithFlags(&ps, cudaStreamNonBlocking));
            CK(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
            CK(cudaHostAlloc(&hp, 8, cudaHostAllocDefault));
        }
        CK(cudaEventRecord(done, stream()));
        while (cudaEventQuery(done) == cudaErrorNotReady) {
            CK(cudaMemcpyAsync(hp, s->ov_count.p, 4, cudaMemcpyDeviceToHost, ps));
            CK(cudaStreamSynchronize(ps));
            if (hp[0] > ov_abort) {
                hp[1] = 0x7fffffffu;
                CK(cudaMemcpyAsync(next.p, hp + 1, 4, cudaMemcpyHostToDevice, ps));
                CK(cudaStreamSynchronize(ps));
                break;
            }
            std::this_thread::sleep_for(std::chrono::microseconds(200));
        }
        cudaGetLastError();  // cudaErrorNotReady from the query is not an error
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

// Small device counters are read back through mapped pinned memory (a one-thread
// kernel stores them over PCIe) instead of a device-to-host memcpy: a memcpy
// would queue behind the bulk row copies that annk_nn_descent_iteration_finalize
// keeps in flight on the device-to-host copy engine while the next chunk replays.
__global__ void peek_kernel(const uint32_t* __restrict__ src, uint32_t words, volatile uint32_t* dst) {
    for (uint32_t i = 0; i < words; ++i) dst[i] = src[i];
}
void peek_words(const void* dev, uint32_t words, void* out) {
    static uint32_t* host = nullptr;
    static uint32_t* host_dev = nullptr;
    if (!host) {
        CK(cudaHostAlloc(&host, 64, cudaHostAllocMapped));
        CK(cudaHostGetDevicePointer(&host_dev, host, 0));
    }
    LAUNCH(peek_kernel, 1, 1, 0, static_cast<const uint32_t*>(dev), words, host_dev);
    ssync();
    memcpy(out, host, size_t(words) * 4);
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
    DevBuf<uint32_t> ctr(4);  // per pass: [work counter, deferred count]
    changes.zero();
    a.changes = changes.p;
    const uint32_t n = s->n;
    const bool trace = getenv("ANNK_TRACE") != nullptr;
    {  // drop the offers of ids already in their target's pool (never accepted)
        CArgs c{};
        c.lo = lo;
        c.hi = hi;
        c.P = s->P;
        c.cap = s->offer_cap;
        c.keys = s->keys.p;
        c.sizes = s->sizes.p;
        c.ocnt = s->ocnt.p;
        c.obuf = s->obuf.p;
        c.osrc = s->osrc.p;
        c.ov_off = s->ov_off.p;
        c.ov_key = s->ov_key.p;
        c.ov_src = s->ov_src.p;
        c.hbits = 7;
        while ((1u << c.hbits) < 4 * s->P) ++c.hbits;  // load factor <= 1/4
        DevBuf<unsigned long long> dropped(1);
        dropped.zero();
        ctr.zero();
        c.next = ctr.p;
        c.dropped = dropped.p;
        const uint32_t wpb = 8;
        const size_t smem = size_t(wpb) << (c.hbits + 2);
        if (smem > size_t(max_smem_optin())) throw_invalid("refine: pool_cap too large for the device path");
        CK(cudaFuncSetAttribute(offer_compact_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        int per_sm = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, offer_compact_kernel, wpb * 32, smem));
        const uint32_t grid = std::min<uint32_t>((hi - lo + wpb - 1) / wpb, uint32_t(num_sms()) * std::max(per_sm, 1));
        LAUNCH(offer_compact_kernel, grid, wpb * 32, smem, c);
        if (trace) {
            unsigned long long d = 0;
            dropped.download(&d, 1);
            ssync();
            fprintf(stderr, "[annk] replay: %llu offers of ids already in their pool dropped\n", d);
        }
    }
    if (s->rp_big.n < 4 * size_t(n)) s->rp_big.alloc(4 * size_t(n));  // two (target, run count) lists
    uint32_t* def[2] = {s->rp_big.p, s->rp_big.p + 2 * size_t(n)};
    // pass 1: every target, up to 256 source runs in shared memory (8 warps per block);
    // pass 2: the deferred ones with up to 1024 (4 warps per block);
    // pass 3: the rest with their runs in global scratch
    const uint32_t runmax[2] = {256, 1024}, wpbs[2] = {8, 4};
    uint32_t nlist = 0;
    for (int pass = 0; pass < 3; ++pass) {
        ctr.zero();
        a.next = ctr.p;
        a.ndef = ctr.p + 1;
        a.list = pass ? def[(pass - 1) & 1] : nullptr;
        a.list_n = nlist;
        a.def = def[pass & 1];
        a.def_nr = def[pass & 1] + n;
        const uint32_t items = pass ? nlist : hi - lo;
        if (items == 0) break;
        DevBuf<uint64_t> sizes, off;
        if (pass < 2) {
            a.runmax = runmax[pass];
            a.g_runkey = nullptr;
        } else {
            sizes.alloc(size_t(items) + 1);
            off.alloc(size_t(items) + 1);
            LAUNCH(big_sizes_kernel, gridn(size_t(items) + 1, 256), 256, 0, def[1] + n, items, sizes.p);
            ex_scan(sizes.p, off.p, items);
            uint64_t total = 0;
            peek_words(off.p + items, 2, &total);
            if (trace) fprintf(stderr, "[annk] replay: %u targets with runs in global scratch (%llu entries)\n", items,
                               (unsigned long long)total);
            if (s->rp_runkey.n < total) {  // grow-only scratch kept by the state
                const size_t cap = std::max<size_t>(total + total / 4, size_t(1) << 16);
                s->rp_runkey.alloc(cap);
                s->rp_pstart.alloc(cap);
                s->rp_seqoff.alloc(cap);
            }
            a.runmax = 0;
            a.g_off = off.p;
            a.g_runkey = s->rp_runkey.p;
            a.g_pstart = s->rp_pstart.p;
            a.g_seqoff = s->rp_seqoff.p;
        }
        const uint32_t wpb = pass < 2 ? wpbs[pass] : 4;
        const size_t smem = replay_warp_bytes(a.P, a.runmax) * wpb;
        if (smem > size_t(max_smem_optin())) throw_invalid("refine: pool_cap too large for the device path");
        CK(cudaFuncSetAttribute(replay_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        int per_sm = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, replay_kernel, wpb * 32, smem));
        const uint32_t grid = std::min<uint32_t>((items + wpb - 1) / wpb, uint32_t(num_sms()) * std::max(per_sm, 1));
        LAUNCH(replay_kernel, grid, wpb * 32, smem, a);
        if (pass == 2) break;
        peek_words(ctr.p + 1, 1, &nlist);
        if (trace) fprintf(stderr, "[annk] replay pass %d: %u targets deferred (> %u source runs)\n", pass, nlist,
                           a.runmax);
    }
    unsigned long long c = 0;
    peek_words(changes.p, 2, &c);
    return c;
}

}  // namespace annk
