// peaks.cu — measurement only: the dense tcgen05 kind::i8 rate of this GPU, the
// denominator of the exact-kNN tensor roofline (bench.py).  No reference
// counterpart.  One CTA per SM; one thread issues M=128 x N=256 x K=32 u8 MMAs
// back to back on operands already in shared memory (no loads, no epilogue),
// alternating between two TMEM accumulators; the kernel ends when the last
// commit has arrived.
#include "internal.cuh"
#include "tcgen05.cuh"

namespace annk {
namespace {
using namespace tc;

constexpr uint32_t kM = 128, kN = 256, kRowB = 128;  // 128-byte K-major rows (4 K=32 steps)
constexpr uint32_t kIdescPeak = (2u << 4) | ((kN >> 3) << 17) | ((kM >> 4) << 24);
constexpr uint32_t kSmemPeak = 1024 + (kM + kN) * kRowB + 64;

__global__ void __launch_bounds__(64, 1) i8_peak_kernel(uint32_t groups) {
    extern __shared__ __align__(1024) unsigned char raw[];
    unsigned char* base = reinterpret_cast<unsigned char*>((uintptr_t(raw) + 1023) & ~uintptr_t(1023));
    unsigned char* A = base;
    unsigned char* B = base + kM * kRowB;
    uint64_t* bar = reinterpret_cast<uint64_t*>(B + kN * kRowB);
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 1);
    uint32_t x = blockIdx.x * 2654435761u + threadIdx.x * 40503u + 12345u;
    for (uint32_t i = threadIdx.x; i < (kM + kN) * kRowB / 4; i += blockDim.x) {
        x = x * 1664525u + 1013904223u;
        reinterpret_cast<uint32_t*>(base)[i] = x;
    }
    if (threadIdx.x == 0) mbar_init(bar, 1);
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tslot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;
    if (threadIdx.x == 32) {
        const uint32_t sA = smem_u32(A), sB = smem_u32(B);
        for (uint32_t g = 0; g < groups; ++g) {
#pragma unroll
            for (uint32_t kk = 0; kk < kRowB / 32; ++kk)
                mma_i8(tmem + (g & 1) * kN, sdesc_sw128(sA + kk * 32), sdesc_sw128(sB + kk * 32), kIdescPeak, kk);
        }
        tc_commit(bar);
        mbar_wait(bar, 0);
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}

}  // namespace
}  // namespace annk

using namespace annk;

extern "C" int annk_measure_i8_peak(uint32_t groups, double* tera_ops) {
    return abi([&] {
        if (!tera_ops || groups == 0) throw_invalid("measure_i8_peak: bad argument");
        CK(cudaFuncSetAttribute(i8_peak_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kSmemPeak)));
        const uint32_t grid = uint32_t(num_sms());
        cudaEvent_t e0, e1;
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        double best = 0;
        for (int rep = 0; rep < 4; ++rep) {  // the first launch warms up
            CK(cudaEventRecord(e0, stream()));
            LAUNCH(i8_peak_kernel, grid, 64, kSmemPeak, groups);
            CK(cudaEventRecord(e1, stream()));
            CK(cudaEventSynchronize(e1));
            float ms = 0;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            const double ops = 2.0 * kM * kN * kRowB * double(groups) * grid;
            if (rep > 0) best = std::max(best, ops / (ms * 1e-3) / 1e12);
        }
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        *tera_ops = best;
    });
}
