// common.cuh — shared device/host plumbing for the EFANNA B200 kernels.
//
// Conventions used by every kernel in this library:
//  * A neighbour entry is ONE 64-bit key: (float_bits(dist) << 32) | id.
//    dist >= +0 always (a sum of squares starting at +0), so unsigned
//    comparison of keys is exactly the reference's entry_less order
//    (proj/include/annkit/neighbor_pool.hpp:17-20: dist, then id).
//  * Distances are the reference's l2_sq (proj/include/annkit/dataset.hpp:67-74):
//    fp32, index ascending, separate multiply and add (no FMA).  Every kernel
//    computes a pair's distance in ONE thread with __fsub_rn/__fmul_rn/__fadd_rn,
//    so results are bit-identical to the CPU reference.
//  * Rows live in HBM with a padded stride `ld` (multiple of 4 floats, zero
//    padding).  Padding adds (0-0)^2 = +0 at the end of the chain: exact.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>

namespace annk {

enum Status : int {
    kOk = 0,
    kInvalidArgument = 1,
    kOutOfRange = 2,
    kCudaError = 3,
    kOutOfMemory = 4,
    kInternal = 5,
};

struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void throw_invalid(const std::string& m) { throw Error(kInvalidArgument, m); }
[[noreturn]] inline void throw_range(const std::string& m) { throw Error(kOutOfRange, m); }

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
    if (e != cudaSuccess) {
        const int code = e == cudaErrorMemoryAllocation ? kOutOfMemory : kCudaError;
        throw Error(code, std::string(what) + ": " + cudaGetErrorString(e) + " at " + file + ":" +
                              std::to_string(line));
    }
}
#define CK(x) ::annk::cuda_check((x), #x, __FILE__, __LINE__)

// Library-wide stream and launch accounting (bench.py reports gpu_launches).
cudaStream_t stream();
void note_launch();
int num_sms();
int max_smem_optin();
// Optional per-kernel CUDA-event timing on the library stream (annk_profile_*).
void prof_begin(const char* name);
void prof_end();

#define LAUNCH(kernel, grid, block, smem, ...)                                   \
    do {                                                                         \
        ::annk::prof_begin(#kernel);                                             \
        kernel<<<(grid), (block), (smem), ::annk::stream()>>>(__VA_ARGS__);      \
        ::annk::prof_end();                                                      \
        ::annk::note_launch();                                                   \
        CK(cudaGetLastError());                                                  \
    } while (0)

// Device memory through a size-keyed block cache on top of the stream-ordered
// pool: repeated builds reuse the previous state's scratch (GBs at 1M points)
// instead of re-mapping it.  All work runs on one stream, so reuse is ordered.
void* dev_alloc(size_t bytes);
void dev_free(void* p, size_t bytes) noexcept;

// Stream-ordered device buffer.
template <class T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    DevBuf() = default;
    explicit DevBuf(size_t count) { alloc(count); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) { release(); p = o.p; n = o.n; o.p = nullptr; o.n = 0; }
        return *this;
    }
    ~DevBuf() { release(); }
    void alloc(size_t count) {
        release();
        n = count;
        if (count) p = static_cast<T*>(dev_alloc(count * sizeof(T)));
    }
    void release() noexcept {
        if (p) dev_free(p, n * sizeof(T));
        p = nullptr;
        n = 0;
    }
    void zero() {
        if (n) CK(cudaMemsetAsync(p, 0, n * sizeof(T), stream()));
    }
    void fill_bytes(int v) {
        if (n) CK(cudaMemsetAsync(p, v, n * sizeof(T), stream()));
    }
    void upload(const T* host, size_t count) {
        if (count) CK(cudaMemcpyAsync(p, host, count * sizeof(T), cudaMemcpyHostToDevice, stream()));
    }
    void download(T* host, size_t count) const {
        if (count) CK(cudaMemcpyAsync(host, p, count * sizeof(T), cudaMemcpyDeviceToHost, stream()));
    }
};

inline void ssync() { CK(cudaStreamSynchronize(stream())); }

// Device bounds checks for debug builds (make debug): report and trap.
#ifdef ANNK_DEBUG_CHECKS
#define DCHK(c)                                                                              \
    do {                                                                                     \
        if (!(c)) {                                                                          \
            printf("DCHK failed %s:%d block %d thread %d: %s\n", __FILE__, __LINE__,         \
                   int(blockIdx.x), int(threadIdx.x), #c);                                   \
            __trap();                                                                        \
        }                                                                                    \
    } while (0)
#else
#define DCHK(c) \
    do {        \
    } while (0)
#endif

// ------------------------------------------------------------ device utils

constexpr uint32_t kInvalidId = 0xffffffffu;
constexpr uint32_t kLeaf = 0xffffffffu;
constexpr uint64_t kEmptyKey = ~0ull;

__host__ __device__ __forceinline__ uint64_t make_key(float dist, uint32_t id) {
#ifdef __CUDA_ARCH__
    return (uint64_t(__float_as_uint(dist)) << 32) | id;
#else
    uint32_t b;
    memcpy(&b, &dist, 4);
    return (uint64_t(b) << 32) | id;
#endif
}
__host__ __device__ __forceinline__ uint32_t key_id(uint64_t k) { return uint32_t(k); }
__device__ __forceinline__ float key_dist(uint64_t k) { return __uint_as_float(uint32_t(k >> 32)); }

// The reference l2_sq, bit-exact: one thread, index ascending, no contraction.
__device__ __forceinline__ float l2_exact(const float* __restrict__ a, const float* __restrict__ b,
                                          uint32_t dim) {
    float acc = 0.0f;
    uint32_t i = 0;
    if ((reinterpret_cast<uintptr_t>(a) & 15) == 0 && (reinterpret_cast<uintptr_t>(b) & 15) == 0) {
        for (; i + 4 <= dim; i += 4) {
            const float4 x = *reinterpret_cast<const float4*>(a + i);
            const float4 y = *reinterpret_cast<const float4*>(b + i);
            float d;
            d = __fsub_rn(x.x, y.x); acc = __fadd_rn(acc, __fmul_rn(d, d));
            d = __fsub_rn(x.y, y.y); acc = __fadd_rn(acc, __fmul_rn(d, d));
            d = __fsub_rn(x.z, y.z); acc = __fadd_rn(acc, __fmul_rn(d, d));
            d = __fsub_rn(x.w, y.w); acc = __fadd_rn(acc, __fmul_rn(d, d));
        }
    }
    for (; i < dim; ++i) {
        const float d = __fsub_rn(a[i], b[i]);
        acc = __fadd_rn(acc, __fmul_rn(d, d));
    }
    return acc;
}

// Read-only global variant (rows gathered by id).
__device__ __forceinline__ float l2_exact_ldg(const float* __restrict__ a, const float* __restrict__ b,
                                              uint32_t dim_pad4) {
    float acc = 0.0f;
    for (uint32_t i = 0; i < dim_pad4; i += 4) {
        const float4 x = *reinterpret_cast<const float4*>(a + i);
        const float4 y = __ldg(reinterpret_cast<const float4*>(b + i));
        float d;
        d = __fsub_rn(x.x, y.x); acc = __fadd_rn(acc, __fmul_rn(d, d));
        d = __fsub_rn(x.y, y.y); acc = __fadd_rn(acc, __fmul_rn(d, d));
        d = __fsub_rn(x.z, y.z); acc = __fadd_rn(acc, __fmul_rn(d, d));
        d = __fsub_rn(x.w, y.w); acc = __fadd_rn(acc, __fmul_rn(d, d));
    }
    return acc;
}

// The same chain with the row streamed 8 float4 (one 128-byte line) at a time:
// the eight loads are issued before the chain consumes them, so a thread keeps a
// whole line in flight instead of one 16-byte piece (wide rows, one row per lane).
__device__ __forceinline__ float l2_exact_ldg8(const float* __restrict__ a, const float* __restrict__ b,
                                               uint32_t dim_pad4) {
    float acc = 0.0f;
    uint32_t i = 0;
    for (; i + 32 <= dim_pad4; i += 32) {
        float4 y[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) y[u] = __ldg(reinterpret_cast<const float4*>(b + i) + u);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const float4 x = *reinterpret_cast<const float4*>(a + i + 4 * u);
            float d;
            d = __fsub_rn(x.x, y[u].x); acc = __fadd_rn(acc, __fmul_rn(d, d));
            d = __fsub_rn(x.y, y[u].y); acc = __fadd_rn(acc, __fmul_rn(d, d));
            d = __fsub_rn(x.z, y[u].z); acc = __fadd_rn(acc, __fmul_rn(d, d));
            d = __fsub_rn(x.w, y[u].w); acc = __fadd_rn(acc, __fmul_rn(d, d));
        }
    }
    for (; i < dim_pad4; i += 4) {
        const float4 x = *reinterpret_cast<const float4*>(a + i);
        const float4 y = __ldg(reinterpret_cast<const float4*>(b + i));
        float d;
        d = __fsub_rn(x.x, y.x); acc = __fadd_rn(acc, __fmul_rn(d, d));
        d = __fsub_rn(x.y, y.y); acc = __fadd_rn(acc, __fmul_rn(d, d));
        d = __fsub_rn(x.z, y.z); acc = __fadd_rn(acc, __fmul_rn(d, d));
        d = __fsub_rn(x.w, y.w); acc = __fadd_rn(acc, __fmul_rn(d, d));
    }
    return acc;
}

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31; }

// In-place ascending bitonic sort of n (power of two) 64-bit keys in shared
// memory by the whole block.
__device__ inline void block_bitonic_sort(uint64_t* s, uint32_t n) {
    for (uint32_t k = 2; k <= n; k <<= 1) {
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
                const uint32_t ixj = i ^ j;
                if (ixj > i) {
                    const uint64_t a = s[i], b = s[ixj];
                    const bool up = (i & k) == 0;
                    if ((a > b) == up) { s[i] = b; s[ixj] = a; }
                }
            }
            __syncthreads();
        }
    }
}

// Same, by one warp (no block barriers).
__device__ inline void warp_bitonic_sort(uint64_t* s, uint32_t n) {
    const uint32_t lane = lane_id();
    for (uint32_t k = 2; k <= n; k <<= 1) {
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            for (uint32_t i = lane; i < n; i += 32) {
                const uint32_t ixj = i ^ j;
                if (ixj > i) {
                    const uint64_t a = s[i], b = s[ixj];
                    const bool up = (i & k) == 0;
                    if ((a > b) == up) { s[i] = b; s[ixj] = a; }
                }
            }
            __syncwarp();
        }
    }
}
__device__ inline void warp_bitonic_sort_u32(uint32_t* s, uint32_t n) {
    const uint32_t lane = lane_id();
    for (uint32_t k = 2; k <= n; k <<= 1) {
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            for (uint32_t i = lane; i < n; i += 32) {
                const uint32_t ixj = i ^ j;
                if (ixj > i) {
                    const uint32_t a = s[i], b = s[ixj];
                    const bool up = (i & k) == 0;
                    if ((a > b) == up) { s[i] = b; s[ixj] = a; }
                }
            }
            __syncwarp();
        }
    }
}

__device__ __forceinline__ uint64_t shfl_xor_u64(uint64_t v, uint32_t m) {
    const uint32_t lo = __shfl_xor_sync(0xffffffffu, uint32_t(v), m);
    const uint32_t hi = __shfl_xor_sync(0xffffffffu, uint32_t(v >> 32), m);
    return (uint64_t(hi) << 32) | lo;
}

__device__ __forceinline__ uint64_t shfl_idx_u64(uint64_t v, uint32_t src) {
    const uint32_t lo = __shfl_sync(0xffffffffu, uint32_t(v), src);
    const uint32_t hi = __shfl_sync(0xffffffffu, uint32_t(v >> 32), src);
    return (uint64_t(hi) << 32) | lo;
}

// Register-resident ascending bitonic sort of 32*V keys held V per lane in
// element order e = r*32 + lane (no shared memory; cross-lane steps shuffle).
template <int V>
__device__ __forceinline__ void warp_sort_regs(uint64_t (&v)[V]) {
    const uint32_t lane = threadIdx.x & 31;
#pragma unroll
    for (uint32_t k = 2; k <= 32u * V; k <<= 1) {
#pragma unroll
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            if (j >= 32) {
#pragma unroll
                for (int r = 0; r < V; ++r) {
                    const int rp = r ^ int(j / 32);
                    if (rp > r) {
                        const bool up = ((uint32_t(r) * 32 + lane) & k) == 0;
                        const uint64_t a = v[r], b = v[rp];
                        if ((a > b) == up) { v[r] = b; v[rp] = a; }
                    }
                }
            } else {
#pragma unroll
                for (int r = 0; r < V; ++r) {
                    const uint64_t o = shfl_xor_u64(v[r], j);
                    const bool up = ((uint32_t(r) * 32 + lane) & k) == 0;
                    const bool lower = (lane & j) == 0;
                    v[r] = (lower == up) ? (v[r] < o ? v[r] : o) : (v[r] < o ? o : v[r]);
                }
            }
        }
    }
}

// The same network for 32-bit keys.
template <int V>
__device__ __forceinline__ void warp_sort_regs_u32(uint32_t (&v)[V]) {
    const uint32_t lane = threadIdx.x & 31;
#pragma unroll
    for (uint32_t k = 2; k <= 32u * V; k <<= 1) {
#pragma unroll
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            if (j >= 32) {
#pragma unroll
                for (int r = 0; r < V; ++r) {
                    const int rp = r ^ int(j / 32);
                    if (rp > r) {
                        const bool up = ((uint32_t(r) * 32 + lane) & k) == 0;
                        const uint32_t a = v[r], b = v[rp];
                        if ((a > b) == up) { v[r] = b; v[rp] = a; }
                    }
                }
            } else {
#pragma unroll
                for (int r = 0; r < V; ++r) {
                    const uint32_t o = __shfl_xor_sync(0xffffffffu, v[r], j);
                    const bool up = ((uint32_t(r) * 32 + lane) & k) == 0;
                    const bool lower = (lane & j) == 0;
                    v[r] = (lower == up) ? min(v[r], o) : max(v[r], o);
                }
            }
        }
    }
}

__host__ __device__ __forceinline__ uint32_t next_pow2(uint32_t x) {  // saturates at 2^31 (no wrap to 0)
    uint32_t p = 1;
    while (p < x && p < 0x80000000u) p <<= 1;
    return p;
}

// splitmix64 finalizer and seed streams (proj/include/annkit/util.hpp:9-19).
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}
__host__ __device__ __forceinline__ uint64_t substream(uint64_t seed, uint64_t id) {
    return mix64(seed ^ mix64(id));
}

// std::mt19937_64 tempering.
__host__ __device__ __forceinline__ uint64_t mt_temper(uint64_t x) {
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71d67fffeda60000ULL;
    x ^= (x << 37) & 0xfff7eee000000000ULL;
    x ^= x >> 43;
    return x;
}
__host__ __device__ __forceinline__ uint64_t mt_twist(uint64_t cur, uint64_t next, uint64_t far) {
    const uint64_t y = (cur & 0xffffffff80000000ULL) | (next & 0x7fffffffULL);
    return far ^ (y >> 1) ^ ((y & 1) ? 0xb5026f5aa96619e9ULL : 0);
}

}  // namespace annk
