// brute_force.cu — exact kNN (reference: proj/src/eval.cpp:17-80).
//
// v1 path: register-tiled CUDA-core distance tiles with a fused per-query
// top-k filter.  Each CTA owns QT queries x one slice of the base set; each
// thread accumulates a 2 x 4 block of pair distances over shared-memory
// staged dimension chunks, in index order with separate mul/add (bit-exact
// with the reference's l2_sq).  Candidates below the query's running k-th key
// are appended to a per-query shared buffer, which is compacted (bitonic sort,
// keep k) whenever it cannot absorb another tile.  Slices are merged by a
// second kernel.  Keys order by (dist, id), so ties break by id exactly like
// NeighborPool (neighbor_pool.hpp:17-20).
#include <algorithm>
#include <climits>
#include <cstdlib>

#include "../../include/annkit_b200.h"
#include "internal.cuh"

namespace annk {
namespace {

constexpr int QT = 32;   // queries per CTA
constexpr int BT = 64;   // base rows per tile
constexpr int DC = 64;   // dims per smem chunk
constexpr int kThreads = 256;
constexpr uint32_t kBigK = 512;

__global__ void __launch_bounds__(kThreads)
bf_tile_kernel(const float* __restrict__ base, uint32_t nb, uint32_t ld, const float* __restrict__ q,
               uint32_t nq, const uint32_t* __restrict__ self_ids, uint32_t k, uint32_t cb,
               uint32_t splits, uint32_t tiles_per_split, uint64_t* __restrict__ out) {
    extern __shared__ __align__(16) unsigned char smem[];
    uint64_t* buf = reinterpret_cast<uint64_t*>(smem);                   // QT x cb
    uint64_t* thr = buf + size_t(QT) * cb;                               // QT
    uint32_t* cnt = reinterpret_cast<uint32_t*>(thr + QT);              // QT
    uint32_t* selfq = cnt + QT;                                          // QT
    float* sq = reinterpret_cast<float*>(selfq + QT);                    // QT x (DC+1)
    float* sb = sq + QT * (DC + 1);                                      // BT x (DC+1)

    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t q0 = blockIdx.x * QT;
    const uint32_t split = blockIdx.y;
    const uint32_t n_tiles = (nb + BT - 1) / BT;
    const uint32_t t_begin = split * tiles_per_split;
    const uint32_t t_end = min(n_tiles, t_begin + tiles_per_split);
    if (tid < QT) {
        cnt[tid] = 0;
        thr[tid] = kEmptyKey;
        const uint32_t qi = q0 + tid;
        selfq[tid] = (self_ids && qi < nq) ? self_ids[qi] : kInvalidId;
    }
    const uint32_t tq = tid >> 4, tb = tid & 15;  // queries tq, tq+16; rows tb+16m
    __syncthreads();

    for (uint32_t t = t_begin; t < t_end; ++t) {
        const uint32_t b0 = t * BT;
        float acc[2][4];
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) acc[a][b] = 0.0f;
        for (uint32_t c0 = 0; c0 < ld; c0 += DC) {
            const uint32_t cw = min(uint32_t(DC), ld - c0);
            // stage (float4, coalesced): cw is a multiple of 4
            const uint32_t v4 = cw / 4;
            for (uint32_t j = tid; j < QT * v4; j += kThreads) {
                const uint32_t r = j / v4, c = (j % v4) * 4;
                float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
                if (q0 + r < nq) v = __ldg(reinterpret_cast<const float4*>(q + size_t(q0 + r) * ld + c0 + c));
                float* d = sq + r * (DC + 1) + c;
                d[0] = v.x; d[1] = v.y; d[2] = v.z; d[3] = v.w;
            }
            for (uint32_t j = tid; j < BT * v4; j += kThreads) {
                const uint32_t r = j / v4, c = (j % v4) * 4;
                float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
                if (b0 + r < nb) v = __ldg(reinterpret_cast<const float4*>(base + size_t(b0 + r) * ld + c0 + c));
                float* d = sb + r * (DC + 1) + c;
                d[0] = v.x; d[1] = v.y; d[2] = v.z; d[3] = v.w;
            }
            __syncthreads();
            const float* qa = sq + tq * (DC + 1);
            const float* qb = sq + (tq + 16) * (DC + 1);
            const float* ba = sb + tb * (DC + 1);
#pragma unroll 4
            for (uint32_t i = 0; i < cw; ++i) {
                const float x0 = qa[i], x1 = qb[i];
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    const float y = ba[b * 16 * (DC + 1) + i];
                    const float d0 = __fsub_rn(x0, y), d1 = __fsub_rn(x1, y);
                    acc[0][b] = __fadd_rn(acc[0][b], __fmul_rn(d0, d0));
                    acc[1][b] = __fadd_rn(acc[1][b], __fmul_rn(d1, d1));
                }
            }
            __syncthreads();
        }
        // fused top-k filter
#pragma unroll
        for (int a = 0; a < 2; ++a) {
            const uint32_t ql = tq + 16 * a;
            if (q0 + ql >= nq) continue;
            const uint64_t th = thr[ql];
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                const uint32_t bj = b0 + tb + 16 * b;
                if (bj >= nb || bj == selfq[ql]) continue;
                const uint64_t key = make_key(acc[a][b], bj);
                if (key < th) {
                    const uint32_t slot = atomicAdd(&cnt[ql], 1u);
                    buf[size_t(ql) * cb + slot] = key;
                }
            }
        }
        __syncthreads();
        // compact buffers that could not absorb another tile
        for (uint32_t ql = warp; ql < QT; ql += kThreads / 32) {
            const uint32_t c = cnt[ql];
            if (c + BT <= cb) continue;
            uint64_t* bq = buf + size_t(ql) * cb;
            for (uint32_t j = c + lane; j < cb; j += 32) bq[j] = kEmptyKey;
            __syncwarp();
            warp_bitonic_sort(bq, cb);
            if (lane == 0) {
                const uint32_t keep = min(c, k);
                cnt[ql] = keep;
                if (keep == k) thr[ql] = bq[k - 1];
            }
            __syncwarp();
        }
        __syncthreads();
    }
    // final: sorted first k of each buffer
    for (uint32_t ql = warp; ql < QT; ql += kThreads / 32) {
        const uint32_t qi = q0 + ql;
        if (qi >= nq) continue;
        const uint32_t c = cnt[ql];
        uint64_t* bq = buf + size_t(ql) * cb;
        for (uint32_t j = c + lane; j < cb; j += 32) bq[j] = kEmptyKey;
        __syncwarp();
        warp_bitonic_sort(bq, cb);
        uint64_t* o = out + (size_t(qi) * splits + split) * k;
        for (uint32_t j = lane; j < k; j += 32) o[j] = bq[j];
        __syncwarp();
    }
}

// Exact u8 datapath (see annk_dataset::u8): whole rows staged as 32-bit words
// (stride W+4 keeps 16-byte loads conflict-free), each thread accumulates a
// 2 x 4 block of dp4a dot products; dist = |q|^2 + |b|^2 - 2 q.b exactly.
__global__ void __launch_bounds__(kThreads)
bf_tile_u8_kernel(const uint8_t* __restrict__ base8, const int32_t* __restrict__ bnorm, uint32_t nb,
                  uint32_t ld8, const uint8_t* __restrict__ q8, const int32_t* __restrict__ qnorm, uint32_t nq,
                  const uint32_t* __restrict__ self_ids, uint32_t k, uint32_t cb, uint32_t splits,
                  uint32_t tiles_per_split, uint64_t* __restrict__ out) {
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t W = ld8 / 4, WS = W + 4;
    uint64_t* buf = reinterpret_cast<uint64_t*>(smem);                   // QT x cb
    uint64_t* thr = buf + size_t(QT) * cb;                               // QT
    uint32_t* cnt = reinterpret_cast<uint32_t*>(thr + QT);              // QT
    uint32_t* selfq = cnt + QT;                                          // QT
    int32_t* qn = reinterpret_cast<int32_t*>(selfq + QT);                // QT
    int32_t* bn = qn + QT;                                               // BT
    uint32_t* sq = reinterpret_cast<uint32_t*>(bn + BT);                 // QT x WS (16 B aligned)
    uint32_t* sb = sq + QT * WS;                                         // BT x WS

    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t q0 = blockIdx.x * QT;
    const uint32_t split = blockIdx.y;
    const uint32_t n_tiles = (nb + BT - 1) / BT;
    const uint32_t t_begin = split * tiles_per_split;
    const uint32_t t_end = min(n_tiles, t_begin + tiles_per_split);
    if (tid < QT) {
        cnt[tid] = 0;
        thr[tid] = kEmptyKey;
        const uint32_t qi = q0 + tid;
        selfq[tid] = (self_ids && qi < nq) ? self_ids[qi] : kInvalidId;
        qn[tid] = qi < nq ? qnorm[qi] : 0;
    }
    const uint32_t w4 = W / 4;  // uint4 per row
    for (uint32_t j = tid; j < QT * w4; j += kThreads) {
        const uint32_t r = j / w4, c = (j % w4) * 4;
        uint4 v = make_uint4(0, 0, 0, 0);
        if (q0 + r < nq) v = __ldg(reinterpret_cast<const uint4*>(q8 + size_t(q0 + r) * ld8) + j % w4);
        *reinterpret_cast<uint4*>(sq + r * WS + c) = v;
    }
    const uint32_t tq = tid >> 4, tb = tid & 15;
    __syncthreads();
    for (uint32_t t = t_begin; t < t_end; ++t) {
        const uint32_t b0 = t * BT;
        for (uint32_t j = tid; j < BT * w4; j += kThreads) {
            const uint32_t r = j / w4, c = (j % w4) * 4;
            uint4 v = make_uint4(0, 0, 0, 0);
            if (b0 + r < nb) v = __ldg(reinterpret_cast<const uint4*>(base8 + size_t(b0 + r) * ld8) + j % w4);
            *reinterpret_cast<uint4*>(sb + r * WS + c) = v;
        }
        if (tid < BT) bn[tid] = b0 + tid < nb ? bnorm[b0 + tid] : 0;
        __syncthreads();
        uint32_t dot[2][4] = {{0, 0, 0, 0}, {0, 0, 0, 0}};
        const uint32_t* qa = sq + tq * WS;
        const uint32_t* qb = sq + (tq + 16) * WS;
#pragma unroll 2
        for (uint32_t w = 0; w < W; w += 4) {
            const uint4 x0 = *reinterpret_cast<const uint4*>(qa + w);
            const uint4 x1 = *reinterpret_cast<const uint4*>(qb + w);
#pragma unroll
            for (int m = 0; m < 4; ++m) {
                const uint4 y = *reinterpret_cast<const uint4*>(sb + (tb + 16 * m) * WS + w);
                dot[0][m] = __dp4a(x0.x, y.x, dot[0][m]);
                dot[0][m] = __dp4a(x0.y, y.y, dot[0][m]);
                dot[0][m] = __dp4a(x0.z, y.z, dot[0][m]);
                dot[0][m] = __dp4a(x0.w, y.w, dot[0][m]);
                dot[1][m] = __dp4a(x1.x, y.x, dot[1][m]);
                dot[1][m] = __dp4a(x1.y, y.y, dot[1][m]);
                dot[1][m] = __dp4a(x1.z, y.z, dot[1][m]);
                dot[1][m] = __dp4a(x1.w, y.w, dot[1][m]);
            }
        }
#pragma unroll
        for (int a2 = 0; a2 < 2; ++a2) {
            const uint32_t ql = tq + 16 * a2;
            if (q0 + ql >= nq) continue;
            const uint64_t th = thr[ql];
#pragma unroll
            for (int m = 0; m < 4; ++m) {
                const uint32_t bj = b0 + tb + 16 * m;
                if (bj >= nb || bj == selfq[ql]) continue;
                const float d = float(qn[ql] + bn[tb + 16 * m] - 2 * int32_t(dot[a2][m]));
                const uint64_t key = make_key(d, bj);
                if (key < th) {
                    const uint32_t slot = atomicAdd(&cnt[ql], 1u);
                    buf[size_t(ql) * cb + slot] = key;
                }
            }
        }
        __syncthreads();
        for (uint32_t ql = warp; ql < QT; ql += kThreads / 32) {
            const uint32_t c = cnt[ql];
            if (c + BT <= cb) continue;
            uint64_t* bq = buf + size_t(ql) * cb;
            for (uint32_t j = c + lane; j < cb; j += 32) bq[j] = kEmptyKey;
            __syncwarp();
            warp_bitonic_sort(bq, cb);
            if (lane == 0) {
                const uint32_t keep = min(c, k);
                cnt[ql] = keep;
                if (keep == k) thr[ql] = bq[k - 1];
            }
            __syncwarp();
        }
        __syncthreads();
    }
    for (uint32_t ql = warp; ql < QT; ql += kThreads / 32) {
        const uint32_t qi = q0 + ql;
        if (qi >= nq) continue;
        const uint32_t c = cnt[ql];
        uint64_t* bq = buf + size_t(ql) * cb;
        for (uint32_t j = c + lane; j < cb; j += 32) bq[j] = kEmptyKey;
        __syncwarp();
        warp_bitonic_sort(bq, cb);
        uint64_t* o = out + (size_t(qi) * splits + split) * k;
        for (uint32_t j = lane; j < k; j += 32) o[j] = bq[j];
        __syncwarp();
    }
}

// ---------------------------------------------------- tensor-core u8 path
// Exact kNN on the integer tensor cores: mma.sync.m16n8k32 u8 x u8 -> s32 is
// exact (products <= 255^2, dim <= 128), so dist = |q|^2 + |b|^2 - 2 q.b equals
// the reference's fp32 l2_sq bit-for-bit on the u8 datapath.
// A CTA owns 64 queries; every warp keeps all 64 queries' A fragments in
// registers for the whole base sweep.  Base tiles of 128 rows are staged in
// shared memory with cp.async (double buffered, 144-byte padded stride so the
// 32-bit B-fragment loads are conflict-free); each warp takes two 8-row column
// blocks of the tile, 4 MMAs per B fragment.  The epilogue feeds the same
// threshold filter and per-query sorted buffers as the CUDA-core kernels.
constexpr int MQ = 32, MB = 128, MTHREADS = 256;  // queries per CTA (2 row groups)
constexpr uint32_t kMmaStride = 144;  // bytes per staged base row (>= 128, 16-aligned, 4 mod 32 words)

__device__ __forceinline__ void mma_u8(int32_t (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc, bool valid) {
    const uint32_t d = uint32_t(__cvta_generic_to_shared(smem_dst));
    const int n = valid ? 16 : 0;  // zero-fill rows past the base set
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(gsrc), "r"(n));
}

constexpr uint32_t kMmaStages = 4;  // cp.async ring depth


template <int KS>  // 32-byte k-steps per row (ld8 <= 32 * KS)
__global__ void __launch_bounds__(MTHREADS, 1)
bf_mma_u8_kernel(const uint8_t* __restrict__ base8, const int32_t* __restrict__ bnorm, uint32_t nb,
                 uint32_t ld8, const uint8_t* __restrict__ q8, const int32_t* __restrict__ qnorm, uint32_t nq,
                 const uint32_t* __restrict__ self_ids, uint32_t k, uint32_t cb, uint32_t splits,
                 uint32_t tiles_per_split, uint64_t* __restrict__ out) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ uint32_t need_flush;
    uint64_t* buf = reinterpret_cast<uint64_t*>(smem);       // MQ x cb
    uint64_t* thr = buf + size_t(MQ) * cb;                   // MQ
    uint32_t* cnt = reinterpret_cast<uint32_t*>(thr + MQ);   // MQ
    int32_t* bn = reinterpret_cast<int32_t*>(cnt + MQ);      // stages x MB base norms
    unsigned char* sb = reinterpret_cast<unsigned char*>(bn + kMmaStages * MB);  // stages x MB x stride

    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t g = lane >> 2, t4 = lane & 3;
    const uint32_t q0 = blockIdx.x * MQ, split = blockIdx.y;
    const uint32_t n_tiles = (nb + MB - 1) / MB;
    const uint32_t t_begin = split * tiles_per_split, t_end = min(n_tiles, t_begin + tiles_per_split);
    if (tid < MQ) {
        cnt[tid] = 0;
        thr[tid] = kEmptyKey;
    }
    if (tid == 0) need_flush = 0;
    for (uint32_t j = tid; j < kMmaStages * MB; j += MTHREADS)
        for (uint32_t c = ld8; c < 32u * KS; c += 4) *reinterpret_cast<uint32_t*>(sb + j * kMmaStride + c) = 0;
    constexpr int RG = MQ / 16;
    uint32_t a[RG][KS][4];
    int32_t qn_r[2 * RG];
    uint32_t self_r[2 * RG];
#pragma unroll
    for (int rg = 0; rg < RG; ++rg) {
#pragma unroll
        for (int hr = 0; hr < 2; ++hr) {
            const uint32_t qi = q0 + rg * 16 + g + 8 * hr;
            qn_r[rg * 2 + hr] = qi < nq ? qnorm[qi] : 0;
            self_r[rg * 2 + hr] = (self_ids && qi < nq) ? self_ids[qi] : kInvalidId;
        }
#pragma unroll
        for (int ks = 0; ks < KS; ++ks)
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const uint32_t qi = q0 + rg * 16 + g + ((r & 1) ? 8 : 0);
                const uint32_t kb = ks * 32 + ((r & 2) ? 16 : 0) + t4 * 4;
                a[rg][ks][r] = (qi < nq && kb < ld8)
                                   ? __ldg(reinterpret_cast<const uint32_t*>(q8 + size_t(qi) * ld8 + kb))
                                   : 0u;
            }
    }
    const uint32_t chunks = ld8 / 16;  // 16-byte chunks per base row
    const bool pow2_chunks = chunks == 2 * KS && (chunks & (chunks - 1)) == 0;
    const uint32_t cshift = 31 - __clz(max(chunks, 1u));
    auto stage = [&](uint32_t t) {
        if (t < t_end) {
            const uint32_t b0 = t * MB, st = (t - t_begin) % kMmaStages;
            unsigned char* dst = sb + size_t(st) * MB * kMmaStride;
            for (uint32_t j = tid; j < MB * chunks; j += MTHREADS) {
                const uint32_t r = pow2_chunks ? (j >> cshift) : j / chunks;
                const uint32_t c = j - r * chunks;
                const bool ok = b0 + r < nb;
                cp_async16(dst + r * kMmaStride + c * 16, base8 + size_t(ok ? b0 + r : 0) * ld8 + c * 16, ok);
            }
            if (tid < MB) {
                const bool ok = b0 + tid < nb;
                const uint32_t d = uint32_t(__cvta_generic_to_shared(bn + st * MB + tid));
                asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(d),
                             "l"(bnorm + (ok ? b0 + tid : 0)), "r"(ok ? 4 : 0));
            }
        }
        asm volatile("cp.async.commit_group;");  // (empty groups keep the count uniform)
    };
#pragma unroll
    for (uint32_t p = 0; p < kMmaStages - 1; ++p) stage(t_begin + p);
    // keep iff qn + bn - 2 dot <= T  <=>  2 dot >= (qn - T) + bn; lim = qn - T (T = current
    // k-th distance, an exact integer; ties pass and are settled by the exact key test)
    int32_t lim[2 * RG];
    uint64_t thr_k[2 * RG];
#pragma unroll
    for (int j = 0; j < 2 * RG; ++j) {
        lim[j] = INT_MIN;
        thr_k[j] = kEmptyKey;
    }
    const bool self_mode = self_ids != nullptr;
    for (uint32_t t = t_begin; t < t_end; ++t) {
        asm volatile("cp.async.wait_group %0;" ::"n"(kMmaStages - 2));
        __syncthreads();  // tile t visible; buffers and thresholds settled; tile t-1's stage free
        stage(t + kMmaStages - 1);
#pragma unroll
        for (int rg = 0; rg < RG; ++rg)
#pragma unroll
            for (int hr = 0; hr < 2; ++hr) {
                const uint64_t tk = thr[rg * 16 + g + 8 * hr];
                thr_k[rg * 2 + hr] = tk;
                lim[rg * 2 + hr] = tk == kEmptyKey ? INT_MIN : qn_r[rg * 2 + hr] - int32_t(key_dist(tk));
            }
        const uint32_t st = (t - t_begin) % kMmaStages;
        const uint32_t b0 = t * MB;
        const unsigned char* tile = sb + size_t(st) * MB * kMmaStride;
        const bool full = b0 + MB <= nb;
#pragma unroll
        for (int half = 0; half < 2; ++half) {
            const uint32_t cbk = warp + 8 * half;  // 8-row column block of the tile
            const uint32_t col0 = cbk * 8 + 2 * t4, bj0 = b0 + col0;
            const int32_t bn0 = bn[st * MB + col0], bn1 = bn[st * MB + col0 + 1];
            int32_t acc[RG][4];
#pragma unroll
            for (int rg = 0; rg < RG; ++rg)
#pragma unroll
                for (int r = 0; r < 4; ++r) acc[rg][r] = 0;
            const unsigned char* brow = tile + (cbk * 8 + g) * kMmaStride + t4 * 4;
#pragma unroll
            for (int ks = 0; ks < KS; ++ks) {
                const uint32_t b0r = *reinterpret_cast<const uint32_t*>(brow + ks * 32);
                const uint32_t b1r = *reinterpret_cast<const uint32_t*>(brow + ks * 32 + 16);
#pragma unroll
                for (int rg = 0; rg < RG; ++rg) mma_u8(acc[rg], a[rg][ks], b0r, b1r);
            }
#pragma unroll
            for (int rg = 0; rg < RG; ++rg) {
#pragma unroll
                for (int hr = 0; hr < 2; ++hr) {
                    const int qq = rg * 2 + hr;
#pragma unroll
                    for (int hc = 0; hc < 2; ++hc) {
                        const int32_t two_dot = 2 * acc[rg][hr * 2 + hc];
                        if (two_dot < lim[qq] + (hc ? bn1 : bn0)) continue;  // cheap reject (most pairs)
                        const uint32_t bj = bj0 + hc;
                        const uint32_t ql = rg * 16 + g + 8 * hr;
                        if (q0 + ql >= nq || (!full && bj >= nb) || (self_mode && bj == self_r[qq])) continue;
                        const uint64_t key = make_key(float(qn_r[qq] + (hc ? bn1 : bn0) - two_dot), bj);
                        if (key < thr_k[qq]) {
                            const uint32_t slot = atomicAdd(&cnt[ql], 1u);
                            buf[size_t(ql) * cb + slot] = key;
                            if (slot + 1 + MB > cb) need_flush = 1;
                        }
                    }
                }
            }
        }
        __syncthreads();
        if (need_flush) {  // uniform: read after the barrier
            for (uint32_t ql = warp; ql < MQ; ql += MTHREADS / 32) {
                const uint32_t c = cnt[ql];
                if (c + MB <= cb) continue;
                uint64_t* bq = buf + size_t(ql) * cb;
                for (uint32_t j = c + lane; j < cb; j += 32) bq[j] = kEmptyKey;
                __syncwarp();
                warp_bitonic_sort(bq, cb);
                if (lane == 0) {
                    const uint32_t keep = min(c, k);
                    cnt[ql] = keep;
                    if (keep == k) thr[ql] = bq[k - 1];
                }
                __syncwarp();
            }
            __syncthreads();
            if (tid == 0) need_flush = 0;
        }
    }
    asm volatile("cp.async.wait_group 0;");
    __syncthreads();
    for (uint32_t ql = warp; ql < MQ; ql += MTHREADS / 32) {
        const uint32_t qi = q0 + ql;
        if (qi >= nq) continue;
        const uint32_t c = cnt[ql];
        uint64_t* bq = buf + size_t(ql) * cb;
        for (uint32_t j = c + lane; j < cb; j += 32) bq[j] = kEmptyKey;
        __syncwarp();
        warp_bitonic_sort(bq, cb);
        uint64_t* o = out + (size_t(qi) * splits + split) * k;
        for (uint32_t j = lane; j < k; j += 32) o[j] = bq[j];
        __syncwarp();
    }
}

__global__ void gather_rows_u8_kernel(const uint8_t* __restrict__ src, const int32_t* __restrict__ norms,
                                      uint32_t ld8, const uint32_t* __restrict__ rows, uint32_t nr,
                                      uint8_t* __restrict__ dst, int32_t* __restrict__ dnorms) {
    const uint32_t r = blockIdx.x;
    if (r >= nr) return;
    const uint8_t* s = src + size_t(rows[r]) * ld8;
    uint8_t* d = dst + size_t(r) * ld8;
    for (uint32_t j = threadIdx.x; j < ld8; j += blockDim.x) d[j] = s[j];
    if (threadIdx.x == 0) dnorms[r] = norms[rows[r]];
}

// Merge `splits` sorted k-lists per query into the final k.
__global__ void bf_merge_kernel(const uint64_t* __restrict__ part, uint32_t nq, uint32_t splits,
                                uint32_t k, uint32_t m, uint64_t* __restrict__ out, uint32_t out_stride,
                                uint32_t first_sorted) {
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t qi = blockIdx.x * (blockDim.x / 32) + warp;
    uint64_t* s = reinterpret_cast<uint64_t*>(smem) + size_t(warp) * m;
    if (qi >= nq) return;
    if (first_sorted) {
        // list 0 is sorted and the other lists hold their keys first (kEmptyKey after them):
        // when those are all empty the result is list 0
        bool empty = true;
        for (uint32_t l = 1 + lane; l < splits; l += 32) empty &= part[(size_t(qi) * splits + l) * k] == kEmptyKey;
        if (__all_sync(0xffffffffu, empty)) {
            for (uint32_t j = lane; j < k; j += 32) out[size_t(qi) * out_stride + j] = part[size_t(qi) * splits * k + j];
            return;
        }
    }
    for (uint32_t j = lane; j < m; j += 32) s[j] = j < splits * k ? part[size_t(qi) * splits * k + j] : kEmptyKey;
    __syncwarp();
    warp_bitonic_sort(s, m);
    for (uint32_t j = lane; j < k; j += 32) out[size_t(qi) * out_stride + j] = s[j];
}

// Large-k path (k > kBigK, small inputs only): all keys, then a block sort per query.
__global__ void bf_allkeys_kernel(const float* __restrict__ base, uint32_t nb, uint32_t ld,
                                  const float* __restrict__ q, uint32_t dim_pad,
                                  const uint32_t* __restrict__ self_ids, uint32_t m,
                                  uint64_t* __restrict__ keys) {
    const uint32_t qi = blockIdx.x;
    const float* qq = q + size_t(qi) * ld;
    const uint32_t self = self_ids ? self_ids[qi] : kInvalidId;
    uint64_t* kq = keys + size_t(qi) * m;
    for (uint32_t j = threadIdx.x; j < m; j += blockDim.x) {
        uint64_t key = kEmptyKey;
        if (j < nb && j != self) key = make_key(l2_exact_ldg(qq, base + size_t(j) * ld, dim_pad), j);
        kq[j] = key;
    }
}
__global__ void bf_block_sort_kernel(uint64_t* keys, uint32_t m, uint32_t k, uint64_t* out) {
    uint64_t* kq = keys + size_t(blockIdx.x) * m;
    block_bitonic_sort(kq, m);
    for (uint32_t j = threadIdx.x; j < k; j += blockDim.x) out[size_t(blockIdx.x) * k + j] = kq[j];
}

__global__ void gather_rows_kernel(const float* __restrict__ src, uint32_t ld, const uint32_t* __restrict__ rows,
                                   uint32_t nr, float* __restrict__ dst) {
    const uint32_t r = blockIdx.x;
    if (r >= nr) return;
    const float* s = src + size_t(rows[r]) * ld;
    float* d = dst + size_t(r) * ld;
    for (uint32_t j = threadIdx.x; j < ld; j += blockDim.x) d[j] = s[j];
}

__global__ void keys_to_ids_kernel(const uint64_t* __restrict__ keys, size_t n, uint32_t* __restrict__ ids,
                                   float* __restrict__ dists) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
        const uint64_t k = keys[i];
        ids[i] = key_id(k);
        if (dists) dists[i] = key_dist(k);
    }
}

}  // namespace

// eval.cpp:129-155 accuracy_vs_k, membership part: for row i, the rank of each
// graph id in the exact row truth[i] (k_max ids, ascending (dist, id)) via a
// shared-memory hash (id -> rank), then per k' in k_list: hits += rank < k'.
// One CTA per row (grid-stride); per-k' hit counts are 64-bit atomics.
__global__ void accuracy_hits_kernel(const uint32_t* __restrict__ graph, uint32_t n, uint32_t k,
                                     const uint32_t* __restrict__ truth, uint32_t kmax,
                                     const uint32_t* __restrict__ klist, uint32_t nk, uint32_t slots,
                                     unsigned long long* __restrict__ hits) {
    extern __shared__ __align__(16) unsigned char smem[];
    uint64_t* tab = reinterpret_cast<uint64_t*>(smem);  // (id << 32 | rank), empty = ~0
    unsigned long long* local = reinterpret_cast<unsigned long long*>(tab + slots);
    const uint32_t mask = slots - 1;
    for (uint32_t j = threadIdx.x; j < nk; j += blockDim.x) local[j] = 0;
    for (uint32_t i = blockIdx.x; i < n; i += gridDim.x) {
        for (uint32_t j = threadIdx.x; j < slots; j += blockDim.x) tab[j] = ~0ull;
        __syncthreads();
        const uint32_t* tr = truth + size_t(i) * kmax;
        for (uint32_t r = threadIdx.x; r < kmax; r += blockDim.x) {
            const uint32_t id = tr[r];
            uint32_t h = (id * 2654435761u) & mask;
            const uint64_t v = (uint64_t(id) << 32) | r;
            while (atomicCAS(reinterpret_cast<unsigned long long*>(&tab[h]), ~0ull, v) != ~0ull) h = (h + 1) & mask;
        }
        __syncthreads();
        const uint32_t* gr = graph + size_t(i) * k;
        for (uint32_t j = threadIdx.x; j < k; j += blockDim.x) {
            const uint32_t id = gr[j];
            uint32_t h = (id * 2654435761u) & mask, rank = 0xffffffffu;
            for (;;) {
                const uint64_t e = tab[h];
                if (e == ~0ull) break;
                if (uint32_t(e >> 32) == id) { rank = uint32_t(e); break; }
                h = (h + 1) & mask;
            }
            if (rank != 0xffffffffu)
                for (uint32_t q = 0; q < nk; ++q)
                    if (rank < klist[q]) atomicAdd(&local[q], 1ull);
        }
        __syncthreads();
    }
    __syncthreads();
    for (uint32_t j = threadIdx.x; j < nk; j += blockDim.x)
        if (local[j]) atomicAdd(&hits[j], local[j]);
}

void merge_split_lists(const uint64_t* part, uint32_t nq, uint32_t splits, uint32_t k, uint64_t* out_keys,
                       uint32_t out_stride, bool first_sorted) {
    if (out_stride == 0) out_stride = k;
    const uint32_t m = next_pow2(splits * k);
    const uint32_t wpb = std::max(1u, std::min(8u, uint32_t(64 * 1024 / (m * 8))));
    CK(cudaFuncSetAttribute(bf_merge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(wpb * m * 8)));
    LAUNCH(bf_merge_kernel, (nq + wpb - 1) / wpb, wpb * 32, wpb * m * 8, part, nq, splits, k, m, out_keys, out_stride, first_sorted ? 1u : 0u);
}

void brute_force_tiles(const annk_dataset* base, const float* qdata, uint32_t nq, const uint32_t* self_ids,
                       uint32_t k, uint64_t* out_keys, const uint8_t* q8, const int32_t* qnorm);

void brute_force_device(const annk_dataset* base, const float* qdata, uint32_t q_ld, uint32_t nq,
                        const uint32_t* self_ids, uint32_t k, uint64_t* out_keys, const uint8_t* q8,
                        const int32_t* qnorm) {
    if (nq == 0) return;
    const uint32_t nb = base->n, ld = base->ld;
    if (q_ld != ld) throw_invalid("brute_force: query stride mismatch");
    if (k > kBigK) {
        const uint32_t m = next_pow2(nb);
        if (double(nq) * m * 8 > 8e9) throw_invalid("brute_force: k too large for this input size");
        DevBuf<uint64_t> keys(size_t(nq) * m);
        LAUNCH(bf_allkeys_kernel, nq, 256, 0, base->data.p, nb, ld, qdata, ld, self_ids, m, keys.p);
        LAUNCH(bf_block_sort_kernel, nq, 1024, 0, keys.p, m, k, out_keys);
        ssync();
        return;
    }
    const bool u8 = base->u8 && q8 != nullptr;
    if (u8 && brute_force_tc(base, nq, self_ids, k, out_keys, q8, qnorm)) return;  // tcgen05 path
    if (!u8 && brute_force_tc_f32(base, qdata, nq, self_ids, k, out_keys)) return;  // tcgen05 bf16x3 + exact re-rank
    if (u8 && base->ld8 <= 128 && k <= 128 && !getenv("ANNK_BF_DP4A")) {
        // tensor-core path
        // buffer room past the kept k decides how often a query's buffer is sorted
        const uint32_t cbm = std::max(next_pow2(k + MB), 512u);
        const size_t smem = size_t(MQ) * cbm * 8 + MQ * 8 + MQ * 4 + kMmaStages * MB * 4 +
                            size_t(kMmaStages) * MB * kMmaStride;
        const uint32_t ks = (base->ld8 + 31) / 32;
        const void* fn = ks == 1 ? reinterpret_cast<const void*>(bf_mma_u8_kernel<1>)
                         : ks == 2 ? reinterpret_cast<const void*>(bf_mma_u8_kernel<2>)
                         : ks == 3 ? reinterpret_cast<const void*>(bf_mma_u8_kernel<3>)
                                   : reinterpret_cast<const void*>(bf_mma_u8_kernel<4>);
        CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        int per_sm = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, MTHREADS, smem));
        const uint32_t qtiles = (nq + MQ - 1) / MQ;
        const uint32_t n_tiles = (nb + MB - 1) / MB;
        const uint32_t want = uint32_t(num_sms()) * std::max(per_sm, 1) * 2;
        uint32_t splits = std::max(1u, std::min(n_tiles, (want + qtiles - 1) / qtiles));
        splits = std::min(splits, std::max(1u, 4096u / k));
        const uint32_t tps = (n_tiles + splits - 1) / splits;
        splits = (n_tiles + tps - 1) / tps;
        DevBuf<uint64_t> part(splits == 1 ? 0 : size_t(nq) * splits * k);
        uint64_t* dst = splits == 1 ? out_keys : part.p;
        const dim3 grid(qtiles, splits);
        if (ks == 1)
            LAUNCH(bf_mma_u8_kernel<1>, grid, MTHREADS, smem, base->data8.p, base->norms8.p, nb, base->ld8, q8,
                   qnorm, nq, self_ids, k, cbm, splits, tps, dst);
        else if (ks == 2)
            LAUNCH(bf_mma_u8_kernel<2>, grid, MTHREADS, smem, base->data8.p, base->norms8.p, nb, base->ld8, q8,
                   qnorm, nq, self_ids, k, cbm, splits, tps, dst);
        else if (ks == 3)
            LAUNCH(bf_mma_u8_kernel<3>, grid, MTHREADS, smem, base->data8.p, base->norms8.p, nb, base->ld8, q8,
                   qnorm, nq, self_ids, k, cbm, splits, tps, dst);
        else
            LAUNCH(bf_mma_u8_kernel<4>, grid, MTHREADS, smem, base->data8.p, base->norms8.p, nb, base->ld8, q8,
                   qnorm, nq, self_ids, k, cbm, splits, tps, dst);
        if (splits > 1) merge_split_lists(part.p, nq, splits, k, out_keys);
        return;
    }
    brute_force_tiles(base, qdata, nq, self_ids, k, out_keys, u8 ? q8 : nullptr, qnorm);
}

// The CUDA-core tile kernels (fp32 rows: the exact sequential chain; u8 rows:
// dp4a) with the slice merge.
void brute_force_tiles(const annk_dataset* base, const float* qdata, uint32_t nq, const uint32_t* self_ids,
                       uint32_t k, uint64_t* out_keys, const uint8_t* q8, const int32_t* qnorm) {
    const uint32_t nb = base->n, ld = base->ld;
    const bool u8 = q8 != nullptr;
    const uint32_t cb = next_pow2(k + BT);
    const size_t smem =
        u8 ? size_t(QT) * cb * 8 + QT * 8 + QT * 4 * 3 + BT * 4 + size_t(QT + BT) * (base->ld8 / 4 + 4) * 4
           : size_t(QT) * cb * 8 + QT * 8 + QT * 4 * 2 + size_t(QT + BT) * (DC + 1) * 4;
    int per_sm = 0;
    if (u8) {
        CK(cudaFuncSetAttribute(bf_tile_u8_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, bf_tile_u8_kernel, kThreads, smem));
    } else {
        CK(cudaFuncSetAttribute(bf_tile_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, bf_tile_kernel, kThreads, smem));
    }
    const uint32_t qtiles = (nq + QT - 1) / QT;
    const uint32_t n_tiles = (nb + BT - 1) / BT;
    const uint32_t want = uint32_t(num_sms()) * std::max(per_sm, 1) * 2;
    uint32_t splits = std::max(1u, std::min(n_tiles, (want + qtiles - 1) / qtiles));
    splits = std::min(splits, std::max(1u, 4096u / k));  // merge list fits 32 KB per warp
    const uint32_t tps = (n_tiles + splits - 1) / splits;
    splits = (n_tiles + tps - 1) / tps;
    DevBuf<uint64_t> part(splits == 1 ? 0 : size_t(nq) * splits * k);
    uint64_t* dst = splits == 1 ? out_keys : part.p;
    if (u8) {
        LAUNCH(bf_tile_u8_kernel, dim3(qtiles, splits), kThreads, smem, base->data8.p, base->norms8.p, nb,
               base->ld8, q8, qnorm, nq, self_ids, k, cb, splits, tps, dst);
    } else {
        LAUNCH(bf_tile_kernel, dim3(qtiles, splits), kThreads, smem, base->data.p, nb, ld, qdata, nq, self_ids,
               k, cb, splits, tps, dst);
    }
    if (splits > 1) {
        const uint32_t m = next_pow2(splits * k);
        const uint32_t wpb = std::max(1u, std::min(8u, uint32_t(64 * 1024 / (m * 8))));
        CK(cudaFuncSetAttribute(bf_merge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(wpb * m * 8)));
        LAUNCH(bf_merge_kernel, (nq + wpb - 1) / wpb, wpb * 32, wpb * m * 8, part.p, nq, splits, k, m, out_keys, k, 0u);
    }
}

void brute_force_f32_tiles(const annk_dataset* base, const float* qdata, uint32_t nq, const uint32_t* self_ids,
                           uint32_t k, uint64_t* out_keys) {
    brute_force_tiles(base, qdata, nq, self_ids, k, out_keys, nullptr, nullptr);
}

}  // namespace annk

using namespace annk;

namespace {
void finish_keys(const DevBuf<uint64_t>& keys, size_t count, uint32_t* ids, float* dists) {
    DevBuf<uint32_t> di(count);
    DevBuf<float> dd(dists ? count : 0);
    const uint32_t grid = uint32_t(std::min<size_t>((count + 255) / 256, 65535));
    LAUNCH(keys_to_ids_kernel, std::max(grid, 1u), 256, 0, keys.p, count, di.p, dists ? dd.p : nullptr);
    di.download(ids, count);
    if (dists) dd.download(dists, count);
    ssync();
}
}  // namespace

extern "C" {

int annk_brute_force_knn(const annk_dataset* base, const annk_dataset* queries, uint32_t k,
                         uint32_t* out_ids, float* out_dists, uint64_t* dist_comps) {
    return abi([&] {
        if (!base) throw_invalid("brute_force_knn: null base");
        const bool self = queries == nullptr;
        if (base->n == 0) throw_invalid("brute_force_knn: empty base set");
        if (!self && queries->dim != base->dim) throw_invalid("brute_force_knn: query dim mismatch");
        const uint32_t limit = self ? base->n - 1 : base->n;
        if (k < 1 || k > limit)
            throw_invalid("brute_force_knn: k=" + std::to_string(k) + " out of range (max " +
                          std::to_string(limit) + ")");
        const uint32_t nq = self ? base->n : queries->n;
        DevBuf<uint64_t> keys(size_t(nq) * k);
        DevBuf<uint32_t> selfids;
        if (self) {
            std::vector<uint32_t> iota(nq);
            for (uint32_t i = 0; i < nq; ++i) iota[i] = i;
            selfids.alloc(nq);
            selfids.upload(iota.data(), nq);
        }
        const annk_dataset* qs = self ? base : queries;
        const bool u8 = base->u8 && qs->u8 && qs->ld8 == base->ld8;
        brute_force_device(base, qs->data.p, base->ld, nq, self ? selfids.p : nullptr, k, keys.p,
                           u8 ? qs->data8.p : nullptr, u8 ? qs->norms8.p : nullptr);
        finish_keys(keys, size_t(nq) * k, out_ids, out_dists);
        if (dist_comps) *dist_comps += uint64_t(nq) * (self ? base->n - 1 : base->n);
    });
}

int annk_accuracy_vs_k(const annk_dataset* vs, const uint32_t* graph_ids, uint32_t n, uint32_t k,
                       const uint32_t* k_list, uint32_t n_k, double* out) {
    return abi([&] {
        if (!vs || !graph_ids || !k_list || !out) throw_invalid("accuracy_vs_k: null argument");
        if (n != vs->n) throw_invalid("accuracy_vs_k: graph does not match data");
        if (n_k == 0) throw_invalid("accuracy_vs_k: empty k list");
        uint32_t kmax = 0;
        for (uint32_t q = 0; q < n_k; ++q) kmax = std::max(kmax, k_list[q]);
        if (kmax > vs->n - 1) throw_invalid("accuracy_vs_k: k exceeds n-1");
        if (k == 0) throw_invalid("accuracy_vs_k: empty graph rows");
        // exact self-mode truth at k_max (eval.cpp:139 brute_force_knn)
        DevBuf<uint64_t> keys(size_t(n) * kmax);
        DevBuf<uint32_t> selfids(n);
        {
            std::vector<uint32_t> iota(n);
            for (uint32_t i = 0; i < n; ++i) iota[i] = i;
            selfids.upload(iota.data(), n);
        }
        brute_force_device(vs, vs->data.p, vs->ld, n, selfids.p, kmax, keys.p, vs->u8 ? vs->data8.p : nullptr,
                           vs->u8 ? vs->norms8.p : nullptr);
        DevBuf<uint32_t> truth(size_t(n) * kmax), g(size_t(n) * k), kl(n_k);
        const uint32_t kgrid = uint32_t(std::min<size_t>((size_t(n) * kmax + 255) / 256, 65535));
        LAUNCH(keys_to_ids_kernel, std::max(kgrid, 1u), 256, 0, keys.p, size_t(n) * kmax, truth.p, nullptr);
        keys.release();
        g.upload(graph_ids, size_t(n) * k);
        kl.upload(k_list, n_k);
        DevBuf<unsigned long long> hits(n_k);
        hits.zero();
        uint32_t slots = 64;
        while (slots < 2 * kmax) slots *= 2;
        const size_t sm = size_t(slots) * 8 + size_t(n_k) * 8;
        if (sm > 200 * 1024) throw_invalid("accuracy_vs_k: k_max too large for the device membership kernel");
        CK(cudaFuncSetAttribute(accuracy_hits_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
        LAUNCH(accuracy_hits_kernel, std::min<uint32_t>(n, uint32_t(num_sms()) * 4), 256, sm, g.p, n, k, truth.p,
               kmax, kl.p, n_k, slots, hits.p);
        std::vector<unsigned long long> h(n_k);
        hits.download(h.data(), n_k);
        ssync();
        for (uint32_t q = 0; q < n_k; ++q) out[q] = double(h[q]) / (double(n) * k);
    });
}

int annk_brute_force_rows(const annk_dataset* base, const uint32_t* rows, uint32_t n_rows, uint32_t k,
                          uint32_t* out_ids, float* out_dists) {
    return abi([&] {
        if (!base || (!rows && n_rows)) throw_invalid("brute_force_rows: null argument");
        if (k < 1 || k > base->n - 1) throw_invalid("brute_force_rows: k out of range");
        for (uint32_t i = 0; i < n_rows; ++i)
            if (rows[i] >= base->n) throw_range("brute_force_rows: row id out of range");
        if (n_rows == 0) return;
        DevBuf<uint32_t> drows(n_rows);
        drows.upload(rows, n_rows);
        DevBuf<float> q(size_t(n_rows) * base->ld);
        LAUNCH(gather_rows_kernel, n_rows, 128, 0, base->data.p, base->ld, drows.p, n_rows, q.p);
        DevBuf<uint8_t> q8(base->u8 ? size_t(n_rows) * base->ld8 : 0);
        DevBuf<int32_t> qn(base->u8 ? n_rows : 0);
        if (base->u8)
            LAUNCH(gather_rows_u8_kernel, n_rows, 128, 0, base->data8.p, base->norms8.p, base->ld8, drows.p, n_rows,
                   q8.p, qn.p);
        DevBuf<uint64_t> keys(size_t(n_rows) * k);
        brute_force_device(base, q.p, base->ld, n_rows, drows.p, k, keys.p, base->u8 ? q8.p : nullptr,
                           base->u8 ? qn.p : nullptr);
        finish_keys(keys, size_t(n_rows) * k, out_ids, out_dists);
    });
}

int annk_bf_last_scan(uint64_t* tiles_total, uint64_t* tiles_visited, int* pruned) {
    return abi([&] {
        if (!tiles_total || !tiles_visited || !pruned) throw_invalid("bf_last_scan: null argument");
        brute_force_tc_last_scan(tiles_total, tiles_visited, pruned);
    });
}

}  // extern "C"
