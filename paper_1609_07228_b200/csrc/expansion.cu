// expansion.cu — the NN-expansion refinement baseline on the device.
//
// Reference: proj/src/graph_build.cpp:164-207 detail::nn_expansion_iteration
// (the paper's comparison strategy).  Per point i: every
// entry of its pool not yet `checked` is marked checked and expanded — each
// id l of that neighbour's pool (as it was when the round started) is offered
// to i's pool unless l == i or i's pool currently holds l; every offer made
// costs one distance.  A point only changes its own pool, so points run in
// parallel (one warp each) and the result is the reference's at any worker
// count; within a point the offers are replayed in the reference's order.
// `checked` lives in bit 1 of a pool slot's flag byte (bit 0: flag_new).
#include "../../include/annkit_b200.h"
#include "internal.cuh"

namespace annk {
namespace {

struct ExpArgs {
    const float* x;
    uint32_t n, ld, dim, P;
    uint64_t* keys;
    uint8_t* flags;
    uint32_t* sizes;
    const uint64_t* snap;        // pools at the start of the round (n x P keys)
    const uint32_t* snap_sizes;
    unsigned long long* comps;
    unsigned long long* changes;
};

__host__ __device__ inline size_t exp_warp_bytes(uint32_t P) {
    return (size_t(P) * 8 + size_t(P) * 4 + size_t(P) + 15) & ~size_t(15);
}

__global__ void expansion_kernel(ExpArgs a) {
    extern __shared__ __align__(16) unsigned char sm[];
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31, lt = (1u << lane) - 1u;
    unsigned char* base = sm + size_t(warp) * exp_warp_bytes(a.P);
    uint64_t* S = reinterpret_cast<uint64_t*>(base);
    uint32_t* ex = reinterpret_cast<uint32_t*>(S + a.P);
    uint8_t* F = reinterpret_cast<uint8_t*>(ex + a.P);
    unsigned long long comps = 0, changes = 0;
    for (uint32_t i = blockIdx.x * (blockDim.x >> 5) + warp; i < a.n; i += gridDim.x * (blockDim.x >> 5)) {
        uint32_t sz = a.sizes[i];
        // graph_build.cpp:183-188: unchecked entries, in pool order, become checked
        uint32_t nexp = 0;
        for (uint32_t j0 = 0; j0 < sz; j0 += 32) {
            const uint32_t j = j0 + lane;
            uint64_t k = 0;
            uint8_t f = 0;
            if (j < sz) {
                k = a.keys[size_t(i) * a.P + j];
                f = a.flags[size_t(i) * a.P + j];
                S[j] = k;
            }
            const bool take = j < sz && !(f & 2);
            const uint32_t b = __ballot_sync(0xffffffffu, take);
            if (take) ex[nexp + __popc(b & lt)] = key_id(k);
            if (j < sz) F[j] = f | 2;
            nexp += __popc(b);
        }
        __syncwarp();
        const float* xi = a.x + size_t(i) * a.ld;
        for (uint32_t e = 0; e < nexp; ++e) {
            const uint32_t jn = ex[e];
            const uint32_t rs = a.snap_sizes[jn];
            const uint64_t* row = a.snap + size_t(jn) * a.P;
            for (uint32_t p0 = 0; p0 < rs; p0 += 32) {
                // the chunk's distances in parallel (one exact chain per lane); the
                // offers are then made one by one in the reference's order
                const uint32_t p = p0 + lane;
                const uint32_t l = p < rs ? key_id(row[p]) : i;
                const float d = p < rs ? l2_exact(xi, a.x + size_t(l) * a.ld, a.dim) : 0.0f;
                const uint32_t cnt = min(32u, rs - p0);
                for (uint32_t s = 0; s < cnt; ++s) {
                    const uint32_t ls = __shfl_sync(0xffffffffu, l, s);
                    const float ds = __shfl_sync(0xffffffffu, d, s);
                    if (ls == i) continue;
                    bool has = false;  // NeighborPool::contains on the current pool
                    for (uint32_t j = lane; j < sz; j += 32) has |= key_id(S[j]) == ls;
                    if (__any_sync(0xffffffffu, has)) continue;
                    ++comps;
                    const uint64_t key = make_key(ds, ls);
                    uint32_t below = 0;
                    for (uint32_t j = lane; j < sz; j += 32) below += S[j] < key ? 1u : 0u;
                    const uint32_t pos = __reduce_add_sync(0xffffffffu, below);
                    if (pos >= a.P) continue;  // a full pool keeps its tail
                    // shift [pos, sz) up by one (the old tail falls off a full pool)
                    const uint32_t top = min(sz, a.P - 1);
                    for (int32_t hi = int32_t(top); hi > int32_t(pos); hi -= 32) {
                        const int32_t q = hi - 32 + int32_t(lane);
                        uint64_t v = 0;
                        uint8_t f = 0;
                        if (q >= int32_t(pos)) {
                            v = S[q];
                            f = F[q];
                        }
                        __syncwarp();
                        if (q >= int32_t(pos)) {
                            S[q + 1] = v;
                            F[q + 1] = f;
                        }
                        __syncwarp();
                    }
                    if (lane == 0) {
                        S[pos] = key;
                        F[pos] = 1;  // flag_new, not checked
                    }
                    __syncwarp();
                    sz = min(sz + 1, a.P);
                    ++changes;
                }
            }
        }
        for (uint32_t j = lane; j < a.P; j += 32) {
            a.keys[size_t(i) * a.P + j] = j < sz ? S[j] : kEmptyKey;
            a.flags[size_t(i) * a.P + j] = j < sz ? F[j] : 0;
        }
        if (lane == 0) a.sizes[i] = sz;
        __syncwarp();
    }
    if (lane == 0) {
        if (comps) atomicAdd(a.comps, comps);
        if (changes) atomicAdd(a.changes, changes);
    }
}

}  // namespace
}  // namespace annk

using namespace annk;

extern "C" {

int annk_nn_expansion_iteration(annk_state* s, const annk_dataset* ds, uint64_t* changes) {
    return abi([&] {
        if (!s || !ds || ds->n != s->n) throw_invalid("nn_expansion_iteration: state/dataset mismatch");
        const uint32_t n = s->n, P = s->P;
        DevBuf<uint64_t> snap(size_t(n) * P);
        DevBuf<uint32_t> snap_sizes(n);
        DevBuf<unsigned long long> ctr(2);
        ctr.zero();
        CK(cudaMemcpyAsync(snap.p, s->keys.p, size_t(n) * P * 8, cudaMemcpyDeviceToDevice, stream()));
        CK(cudaMemcpyAsync(snap_sizes.p, s->sizes.p, size_t(n) * 4, cudaMemcpyDeviceToDevice, stream()));
        ExpArgs a{ds->data.p, n, ds->ld, ds->dim, P, s->keys.p, s->flags.p, s->sizes.p, snap.p, snap_sizes.p,
                  ctr.p, ctr.p + 1};
        uint32_t wpb = 8;
        while (wpb > 1 && exp_warp_bytes(P) * wpb > 96 * 1024) wpb /= 2;
        const size_t smem = exp_warp_bytes(P) * wpb;
        if (smem > size_t(max_smem_optin())) throw_invalid("nn_expansion_iteration: pool_cap too large");
        CK(cudaFuncSetAttribute(expansion_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        int per_sm = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, expansion_kernel, wpb * 32, smem));
        const uint32_t grid =
            std::max(1u, std::min<uint32_t>((n + wpb - 1) / wpb, uint32_t(num_sms()) * std::max(per_sm, 1)));
        LAUNCH(expansion_kernel, grid, wpb * 32, smem, a);
        unsigned long long c[2] = {0, 0};
        ctr.download(c, 2);
        ssync();
        s->dist_comps += c[0];
        s->iteration += 1;
        s->last_changes = c[1];
        if (changes) *changes = c[1];
    });
}

}  // extern "C"
