// distance.cu — the reference's distance entry points on the device.
//
// proj/include/annkit/dataset.hpp:67-77: l2_sq(a, b, dim), dist_sq(vs, a, b),
// dist_sq_q(vs, q, b).  Every pair is one thread running the reference's
// sequential fp32 chain (index ascending, separate multiply and add), so the
// results are bit-identical to the CPU library; ids past the set raise
// ANNK_OUT_OF_RANGE as the reference's std::out_of_range (dataset.cpp:218,225).
#include "../../include/annkit_b200.h"
#include "internal.cuh"

namespace annk {
namespace {

// out[j] = l2_sq(row(a[j]) or q, row(b[j])) over padded rows of stride ld.
__global__ void pair_dist_kernel(const float* __restrict__ x, uint32_t ld, uint32_t dim,
                                 const uint32_t* __restrict__ a, const float* __restrict__ q,
                                 const uint32_t* __restrict__ b, uint32_t m, float* __restrict__ out) {
    const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= m) return;
    const float* ra = q ? q : x + size_t(a[j]) * ld;
    out[j] = l2_exact(ra, x + size_t(b[j]) * ld, dim);
}

void check_ids(const uint32_t* ids, uint32_t m, uint32_t n, const char* what) {
    for (uint32_t j = 0; j < m; ++j)
        if (ids[j] >= n) throw_range(std::string(what) + ": id out of range");
}

}  // namespace
}  // namespace annk

using namespace annk;

extern "C" {

int annk_l2_sq(const float* a, const float* b, uint32_t dim, float* out) {
    return abi([&] {
        if (!out || (dim && (!a || !b))) throw_invalid("l2_sq: null argument");
        DevBuf<float> d(size_t(2) * dim + 1);
        DevBuf<uint32_t> ids(2);
        const uint32_t h[2] = {0, 1};
        if (dim) {
            CK(cudaMemcpyAsync(d.p, a, size_t(dim) * 4, cudaMemcpyDefault, stream()));
            CK(cudaMemcpyAsync(d.p + dim, b, size_t(dim) * 4, cudaMemcpyDefault, stream()));
        }
        ids.upload(h, 2);
        LAUNCH(pair_dist_kernel, 1, 32, 0, d.p, dim, dim, ids.p, nullptr, ids.p + 1, 1u, d.p + 2 * size_t(dim));
        CK(cudaMemcpyAsync(out, d.p + 2 * size_t(dim), 4, cudaMemcpyDeviceToHost, stream()));
        ssync();
    });
}

int annk_dist_sq(const annk_dataset* ds, const uint32_t* a, const uint32_t* b, uint32_t m, float* out) {
    return abi([&] {
        if (!ds || (m && (!a || !b || !out))) throw_invalid("dist_sq: null argument");
        check_ids(a, m, ds->n, "dist_sq");
        check_ids(b, m, ds->n, "dist_sq");
        if (m == 0) return;
        DevBuf<uint32_t> ids(size_t(2) * m);
        DevBuf<float> o(m);
        ids.upload(a, m);
        CK(cudaMemcpyAsync(ids.p + m, b, size_t(m) * 4, cudaMemcpyHostToDevice, stream()));
        LAUNCH(pair_dist_kernel, (m + 255) / 256, 256, 0, ds->data.p, ds->ld, ds->dim, ids.p, nullptr, ids.p + m, m,
               o.p);
        o.download(out, m);
        ssync();
    });
}

int annk_dist_sq_q(const annk_dataset* ds, const float* q, uint32_t dim, const uint32_t* b, uint32_t m,
                   float* out) {
    return abi([&] {
        if (!ds || !q || (m && (!b || !out))) throw_invalid("dist_sq_q: null argument");
        if (dim != ds->dim) throw_invalid("dist_sq_q: query dimension differs from the set");
        check_ids(b, m, ds->n, "dist_sq_q");
        if (m == 0) return;
        DevBuf<float> dq(ds->ld);
        DevBuf<uint32_t> ids(m);
        DevBuf<float> o(m);
        dq.zero();
        CK(cudaMemcpyAsync(dq.p, q, size_t(dim) * 4, cudaMemcpyHostToDevice, stream()));
        ids.upload(b, m);
        LAUNCH(pair_dist_kernel, (m + 255) / 256, 256, 0, ds->data.p, ds->ld, ds->dim, nullptr, dq.p, ids.p, m, o.p);
        o.download(out, m);
        ssync();
    });
}

}  // extern "C"
