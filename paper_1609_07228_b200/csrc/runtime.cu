#include <cstdio>
// runtime.cu — library state, error plumbing, dataset handles, host-side
// input generators.
#include <cmath>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/annkit_b200.h"
#include "internal.cuh"

namespace annk {

namespace {
thread_local std::string g_err;
int g_device = 0;
cudaStream_t g_stream = nullptr;
unsigned long long g_launches = 0;
int g_sms = 0, g_smem_optin = 0;

void init_runtime() {
    if (g_stream) return;
    int count = 0;
    CK(cudaGetDeviceCount(&count));
    if (count == 0) throw Error(kCudaError, "no CUDA device");
    CK(cudaSetDevice(g_device));
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, g_device));
    if (prop.major < 10)
        throw Error(kCudaError, std::string("annkit_b200 needs an sm_100 device, found ") + prop.name);
    g_sms = prop.multiProcessorCount;
    g_smem_optin = int(prop.sharedMemPerBlockOptin);
    CK(cudaStreamCreateWithFlags(&g_stream, cudaStreamNonBlocking));
    cudaMemPool_t pool;
    CK(cudaDeviceGetDefaultMemPool(&pool, g_device));
    uint64_t thresh = ~0ull;  // keep freed blocks cached across calls
    CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thresh));
}
}  // namespace

cudaStream_t stream() {
    init_runtime();
    return g_stream;
}
void note_launch() { ++g_launches; }

// ---- size-keyed device block cache (see common.cuh)
namespace {
struct Cached {
    size_t bytes;
    void* p;
};
std::vector<Cached> g_cache;
size_t g_cache_bytes = 0;
constexpr size_t kCacheCap = size_t(48) << 30;
}  // namespace

void* dev_alloc(size_t bytes) {
    for (size_t i = g_cache.size(); i-- > 0;) {
        if (g_cache[i].bytes == bytes) {
            void* p = g_cache[i].p;
            g_cache_bytes -= bytes;
            g_cache.erase(g_cache.begin() + long(i));
            return p;
        }
    }
    void* p = nullptr;
    cudaError_t e = cudaMallocAsync(&p, bytes, stream());
    if (e == cudaErrorMemoryAllocation && !g_cache.empty()) {  // give cached blocks back and retry
        cudaGetLastError();
        for (auto& c : g_cache) cudaFreeAsync(c.p, stream());
        g_cache.clear();
        g_cache_bytes = 0;
        e = cudaMallocAsync(&p, bytes, stream());
    }
    CK(e);
    return p;
}

void dev_free(void* p, size_t bytes) noexcept {
    if (!p) return;
    if (bytes < (size_t(1) << 20)) {  // small blocks: the pool handles them well
        cudaFreeAsync(p, g_stream);
        return;
    }
    g_cache.push_back(Cached{bytes, p});
    g_cache_bytes += bytes;
    while (g_cache_bytes > kCacheCap && !g_cache.empty()) {
        cudaFreeAsync(g_cache.front().p, g_stream);
        g_cache_bytes -= g_cache.front().bytes;
        g_cache.erase(g_cache.begin());
    }
}

// ---- per-kernel CUDA-event profiler (annk_profile_*): events are recorded on
// the library stream around each launch; durations are resolved lazily.
namespace {
struct ProfRec {
    const char* name;
    cudaEvent_t a, b;
};
bool g_prof = false;
std::vector<ProfRec> g_prof_pending;
std::vector<cudaEvent_t> g_prof_free;
struct ProfAgg {
    std::string name;
    uint64_t count = 0;
    double ms = 0.0;
};
std::vector<ProfAgg> g_prof_agg;
cudaEvent_t prof_event() {
    if (!g_prof_free.empty()) {
        cudaEvent_t e = g_prof_free.back();
        g_prof_free.pop_back();
        return e;
    }
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    return e;
}
void prof_resolve() {
    if (g_prof_pending.empty()) return;
    CK(cudaStreamSynchronize(g_stream));
    const bool trace = getenv("ANNK_PROF_TRACE") != nullptr;  // per-launch timeline on stderr
    for (const ProfRec& r : g_prof_pending) {
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, r.a, r.b));
        if (trace) {
            float at = 0.f;
            CK(cudaEventElapsedTime(&at, g_prof_pending.front().a, r.a));
            fprintf(stderr, "[prof] %10.3f ms  %8.3f ms  %s\n", at, ms, r.name);
        }
        ProfAgg* agg = nullptr;
        for (auto& x : g_prof_agg)
            if (x.name == r.name) agg = &x;
        if (!agg) {
            g_prof_agg.push_back(ProfAgg{r.name});
            agg = &g_prof_agg.back();
        }
        agg->count += 1;
        agg->ms += ms;
        g_prof_free.push_back(r.a);
        g_prof_free.push_back(r.b);
    }
    g_prof_pending.clear();
}
}  // namespace

void prof_begin(const char* name) {
    if (!g_prof) return;
    ProfRec r{name, prof_event(), prof_event()};
    CK(cudaEventRecord(r.a, stream()));
    g_prof_pending.push_back(r);
    if (g_prof_pending.size() > 4096) {  // bound the number of live events
        ProfRec last = g_prof_pending.back();
        g_prof_pending.pop_back();
        prof_resolve();
        g_prof_pending.push_back(last);
    }
}
void prof_end() {
    if (!g_prof || g_prof_pending.empty()) return;
    const cudaError_t e = cudaEventRecord(g_prof_pending.back().b, stream());
    if (e != cudaSuccess)
        throw Error(kCudaError, std::string("after kernel ") + g_prof_pending.back().name + ": " +
                                    cudaGetErrorString(e));
}
int num_sms() {
    init_runtime();
    return g_sms;
}
int max_smem_optin() {
    init_runtime();
    return g_smem_optin;
}

void set_error(const std::string& m) { g_err = m; }

}  // namespace annk

using namespace annk;

// Builds the u8 copy + norms; flags any value that is not an integer in [0,255].
__global__ void to_u8_kernel(const float* __restrict__ x, uint32_t n, uint32_t dim, uint32_t ld,
                             uint8_t* __restrict__ x8, uint32_t ld8, int32_t* __restrict__ norms,
                             uint32_t* __restrict__ bad) {
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) / 32, lane = threadIdx.x & 31;
    if (warp >= n) return;
    const float* r = x + size_t(warp) * ld;
    uint8_t* o = x8 + size_t(warp) * ld8;
    int32_t nrm = 0;
    bool ok = true;
    for (uint32_t j = lane; j < ld8; j += 32) {
        const float v = j < dim ? r[j] : 0.0f;
        const bool good = v >= 0.0f && v <= 255.0f && v == floorf(v);
        ok &= good;
        const uint32_t b = good ? uint32_t(v) : 0u;
        o[j] = uint8_t(b);
        nrm += int32_t(b * b);
    }
    for (int s = 16; s > 0; s >>= 1) nrm += __shfl_xor_sync(0xffffffffu, nrm, s);
    if (lane == 0) norms[warp] = nrm;
    if (!__all_sync(0xffffffffu, ok) && lane == 0) atomicOr(bad, 1u);
}

__global__ void finite_kernel(const float* __restrict__ x, size_t count, uint32_t* __restrict__ bad) {
    bool ok = true;
    for (size_t t = blockIdx.x * size_t(blockDim.x) + threadIdx.x; t < count; t += size_t(gridDim.x) * blockDim.x)
        ok &= isfinite(x[t]);
    if (!__all_sync(0xffffffffu, ok) && (threadIdx.x & 31) == 0) atomicOr(bad, 1u);
}

void check_finite(annk_dataset* ds) {
    const size_t count = size_t(ds->n) * ds->ld;
    if (count == 0) return;
    DevBuf<uint32_t> bad(1);
    bad.zero();
    LAUNCH(finite_kernel, uint32_t(std::min<size_t>((count + 255) / 256, 8192)), 256, 0, ds->data.p, count, bad.p);
    uint32_t h = 0;
    bad.download(&h, 1);
    ssync();
    if (h) throw_invalid("dataset_create: non-finite value");
}

void make_u8(annk_dataset* ds) {
    ds->u8 = false;
    if (ds->n == 0 || uint64_t(ds->dim) * 255ull * 255ull >= (1ull << 24)) return;
    ds->ld8 = (ds->dim + 15) & ~15u;
    ds->data8.alloc(size_t(ds->n) * ds->ld8);
    ds->norms8.alloc(ds->n);
    DevBuf<uint32_t> bad(1);
    bad.zero();
    LAUNCH(to_u8_kernel, (ds->n + 7) / 8, 256, 0, ds->data.p, ds->n, ds->dim, ds->ld, ds->data8.p, ds->ld8,
           ds->norms8.p, bad.p);
    uint32_t h = 0;
    bad.download(&h, 1);
    ssync();
    if (h) {
        ds->data8.release();
        ds->norms8.release();
        return;
    }
    ds->u8 = true;
}

// Upload with zero padding to the ld stride.
static void upload_rows(annk_dataset* ds, const float* host) {
    const size_t n = ds->n, dim = ds->dim, ld = ds->ld;
    ds->data.alloc(std::max<size_t>(n * ld, 1));
    if (n == 0) return;
    if (ld == dim) {
        ds->data.upload(host, n * dim);
    } else {
        CK(cudaMemsetAsync(ds->data.p, 0, n * ld * sizeof(float), stream()));
        CK(cudaMemcpy2DAsync(ds->data.p, ld * sizeof(float), host, dim * sizeof(float),
                             dim * sizeof(float), n, cudaMemcpyHostToDevice, stream()));
    }
}

extern "C" {

const char* annk_last_error(void) { return g_err.c_str(); }
const char* annk_version(void) { return "annkit_b200 0.1 (sm_100a)"; }

int annk_set_device(int device) {
    return abi([&] {
        if (g_stream) {
            if (device != g_device) throw_invalid("annk_set_device: device already initialised");
            return;
        }
        g_device = device;
        init_runtime();
    });
}
uint64_t annk_stream(void) {
    uint64_t s = 0;
    abi([&] { s = reinterpret_cast<uint64_t>(stream()); });
    return s;
}
uint64_t annk_launch_count(void) { return g_launches; }

int annk_profile_enable(int on) {
    return abi([&] {
        stream();
        prof_resolve();
        g_prof = on != 0;
    });
}
int annk_profile_reset(void) {
    return abi([&] {
        prof_resolve();
        g_prof_agg.clear();
    });
}
// Writes "name count total_ms\n" lines into buf (NUL-terminated).
int annk_profile_report(char* buf, uint64_t cap) {
    return abi([&] {
        prof_resolve();
        std::string out;
        for (const auto& x : g_prof_agg)
            out += x.name + " " + std::to_string(x.count) + " " + std::to_string(x.ms) + "\n";
        if (cap == 0) return;
        const size_t m = std::min<size_t>(out.size(), cap - 1);
        memcpy(buf, out.data(), m);
        buf[m] = 0;
    });
}
int annk_synchronize(void) {
    return abi([&] { ssync(); });
}

int annk_dataset_create(const float* host, uint32_t n, uint32_t dim, annk_dataset** out) {
    return abi([&] {
        if (!out) throw_invalid("dataset_create: null out");
        if (dim < 1) throw_invalid("dataset_create: dim must be >= 1");
        if (n > 0 && !host) throw_invalid("dataset_create: null data");
        auto* ds = new annk_dataset;
        ds->n = n;
        ds->dim = dim;
        ds->ld = (dim + 3) & ~3u;
        try {
            upload_rows(ds, host);
            check_finite(ds);  // load_fvecs rejects non-finite values (dataset.cpp:123-126)
            const char* off = getenv("ANNK_DISABLE_U8");
            if (!(off && off[0] == '1')) make_u8(ds);
            ssync();
        } catch (...) {
            delete ds;
            throw;
        }
        *out = ds;
    });
}
int annk_dataset_destroy(annk_dataset* ds) {
    return abi([&] { delete ds; });
}
int annk_dataset_info(const annk_dataset* ds, uint32_t* out4) {
    return abi([&] {
        out4[0] = ds->n;
        out4[1] = ds->dim;
        out4[2] = ds->u8 ? 1u : 0u;
        out4[3] = ds->u8 ? ds->ld8 : ds->ld * 4;  // bytes per gathered row
    });
}

int annk_dataset_shape(const annk_dataset* ds, uint32_t* n, uint32_t* dim) {
    return abi([&] {
        *n = ds->n;
        *dim = ds->dim;
    });
}

// dataset.cpp:201-214: std::mt19937_64(seed), top 24 bits * 2^-24.
int annk_gen_synthetic(uint32_t n, uint32_t dim, uint64_t seed, float* out) {
    return abi([&] {
        if (dim < 1) throw_invalid("gen_synthetic: dim must be >= 1");
        uint64_t mt[312];
        mt[0] = seed;
        for (int i = 1; i < 312; ++i) mt[i] = 6364136223846793005ULL * (mt[i - 1] ^ (mt[i - 1] >> 62)) + uint64_t(i);
        int idx = 312;
        for (size_t i = 0; i < size_t(n) * dim; ++i) {
            if (idx == 312) {
                for (int j = 0; j < 312; ++j) mt[j] = mt_twist(mt[j], mt[(j + 1) % 312], mt[(j + 156) % 312]);
                idx = 0;
            }
            out[i] = float(uint32_t(mt_temper(mt[idx++]) >> 40)) * 0x1p-24f;
        }
    });
}

// Seeded Gaussian mixture.  Counter-based so
// any thread split produces the same bytes:
//   u(s, j)   = (mix64(s + j) >> 11) * 2^-53
//   center[c][j] = lo + (hi - lo) * u(substream(seed, 0), c*dim + j)
//   point i of stream sid: ps = substream(substream(seed, sid), i),
//     c = mix64(ps) % n_centers, z_j = sqrt(-2 ln(1-u(ps,1+2j))) cos(2 pi u(ps,2+2j)),
//     v = clip(center[c][j] + sd * z_j), optionally nearbyint.
int annk_gen_mixture(uint32_t n, uint32_t dim, uint32_t n_centers, float center_lo,
                     float center_hi, float sd, float clip_lo, float clip_hi, int round_to_int,
                     uint64_t seed, uint32_t stream_id, float* out) {
    return abi([&] {
        if (dim < 1 || n_centers < 1) throw_invalid("gen_mixture: dim and n_centers must be >= 1");
        auto u = [](uint64_t s, uint64_t j) { return double(mix64(s + j) >> 11) * 0x1p-53; };
        std::vector<double> centers(size_t(n_centers) * dim);
        const uint64_t s0 = substream(seed, 0);
        for (size_t i = 0; i < centers.size(); ++i)
            centers[i] = double(center_lo) + (double(center_hi) - double(center_lo)) * u(s0, i);
        const uint64_t ss = substream(seed, stream_id);
        unsigned hw = std::max(1u, std::thread::hardware_concurrency());
        const uint32_t workers = std::min<uint32_t>(hw, std::max<uint32_t>(1, n / 4096));
        auto work = [&](uint32_t b, uint32_t e) {
            const double two_pi = 6.283185307179586476925286766559;
            for (uint32_t i = b; i < e; ++i) {
                const uint64_t ps = substream(ss, i);
                const uint32_t c = uint32_t(mix64(ps) % n_centers);
                for (uint32_t j = 0; j < dim; ++j) {
                    const double u1 = u(ps, 1 + 2ull * j), u2 = u(ps, 2 + 2ull * j);
                    const double z = std::sqrt(-2.0 * std::log(1.0 - u1)) * std::cos(two_pi * u2);
                    double v = centers[size_t(c) * dim + j] + double(sd) * z;
                    v = std::min(std::max(v, double(clip_lo)), double(clip_hi));
                    if (round_to_int) v = std::nearbyint(v);
                    out[size_t(i) * dim + j] = float(v);
                }
            }
        };
        if (workers <= 1) {
            work(0, n);
        } else {
            std::vector<std::thread> th;
            const uint32_t chunk = (n + workers - 1) / workers;
            for (uint32_t w = 0; w < workers; ++w) {
                const uint32_t b = w * chunk, e = std::min(n, b + chunk);
                if (b < e) th.emplace_back(work, b, e);
            }
            for (auto& t : th) t.join();
        }
    });
}

}  // extern "C"
