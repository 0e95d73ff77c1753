// search.cu — batched tree-seeded graph search (reference: proj/src/search.cpp).
//
// One CTA per query (persistent over the batch).  Per query:
//   1. seeding (search.cpp:121-151): each of the first n_trees threads runs
//      best-bin-first on its tree (kd_forest.cpp:276-305, heap in global
//      scratch); the leaves' points are visited in parallel.  A per-slot
//      visited bitmap (HBM) plays the reference's epoch-stamped visit table;
//      every fresh id costs one exact distance, so dist_comps matches the
//      reference exactly.  Seeds are sorted by (dist, id); the first E form the
//      pool, the rest are kept as the "reserve" (they may re-enter later with
//      their cached distance, search.cpp:56-63,79-82).
//   2. expansion rounds (search.cpp:65-93): the unchecked pool members are
//      snapshotted and marked checked; their graph rows are visited in
//      parallel; every candidate that beats the pool's start-of-round tail is
//      buffered in shared memory and merged (sort, unique, keep P).  The result
//      is top-P of (pool U buffer), i.e. the reference's sort+unique+truncate.
//   3. fallback scan (search.cpp:95-106) when fewer than k_return remain.
#include <algorithm>

#include "../../include/annkit_b200.h"
#include "internal.cuh"

namespace annk {
namespace {

constexpr uint32_t kThreads = 256;
// candidate buffer between merges: 1024 keys at small pools (6 CTAs per SM
// instead of 5 with 2048), 2048 once P >= 700 (below that a buffer that fills
// past P + one batch would merge after every batch)
constexpr uint32_t kBufMin = 1024, kBufMax = 2048;
constexpr uint32_t kU = 4;  // expansion slots per worker thread per batch (atomics in flight)
constexpr size_t kHeapSmem = 12288;  // BBF heaps in shared memory up to this size

struct HeapEnt {
    double cost;
    uint32_t node;
    uint32_t pad;
};
__device__ __forceinline__ bool hless(const HeapEnt& x, const HeapEnt& y) {
    return x.cost != y.cost ? x.cost < y.cost : x.node < y.node;
}

struct SearchArgs {
    const float* x;
    uint32_t n, ld;
    const float* q;
    uint32_t nq;
    const TreeView* trees;
    uint32_t nt, n_node, leaf_cap;
    const uint32_t* graph;
    uint32_t gk;
    uint32_t k_return, P, E, iters;
    int random_init;
    uint32_t rcount;
    uint64_t seed;
    uint32_t seed_cap;   // pow2 >= max seed points
    // per-slot scratch
    uint32_t* bitmap;    // slots x words
    uint32_t words;
    uint32_t* vlist;     // slots x vcap
    uint32_t vcap;
    HeapEnt* heaps;      // slots x 32 x hcap (nullptr: heaps in shared memory)
    uint32_t hcap;
    uint2* leaves;       // slots x 2 x nt x n_node leaf ranges [left, right) of point_index
    uint64_t* mtstate;   // slots x 312 (random init)
    uint64_t* out_keys;  // nq x k_return
    uint64_t* stats;     // nq x 4
    // exact u8 datapath (nullptr: fp32 path)
    const uint8_t* x8;
    const int32_t* norms8;
    uint32_t ld8;
    const uint8_t* q8;
    const int32_t* qnorms8;
    uint32_t gk_magic;  // floor(2^32 / gk): slot -> (expanded point, column) without a hardware divide
    uint32_t* qnext;    // query work counter: CTAs take queries dynamically (query costs vary)
    uint32_t kbuf;      // candidate buffer capacity (kBufMin or kBufMax)
};

struct Smem {
    uint64_t* pool;     // P
    uint8_t* checked;   // P
    uint64_t* seeds;    // seed_cap
    uint64_t* buf;      // kBuf
    uint64_t* tmp;      // P
    uint8_t* tmpc;      // P
    uint32_t* expand;   // P
    uint32_t* scan;     // kThreads/32 + 1
    float* q;           // ld
    uint8_t* q8;        // ld8
    int32_t qnorm;
    uint32_t* ctr;      // [0] pool size, [1] buf count, [2] visited count, [3] seeds, [4] reserve size,
                        // [5] expand count, [6] leaves visited, [7] hops
    uint32_t* hist;     // kHist radix-select bins + 8 scalars
    HeapEnt* heap;      // min(nt, 32) x hcap when the heaps fit kHeapSmem
    uint32_t* lcnt;     // leaves emitted per leaf-range buffer
    uint64_t* rhash;    // 2 x seed_cap: the reserve, open addressing on id, entries (id << 32) | dist bits
};

__device__ __forceinline__ uint32_t rhash_slot(uint32_t id, uint32_t rbits) {
    return (id * 2654435761u) >> (32 - rbits);
}

constexpr uint32_t kHist = 256;
constexpr uint32_t kConsumed = 0xffffffffu;  // reserve entry already offered (low word of an id-major key)

__device__ __forceinline__ uint32_t lower_bound64(const uint64_t* a, uint32_t n, uint64_t v) {
    uint32_t lo = 0, hi = n;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (a[mid] < v) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// Visit id: returns true if fresh (this thread owns its distance).
__device__ __forceinline__ bool mark_visited(const SearchArgs& a, uint32_t slot, Smem& s, uint32_t id) {
    uint32_t* bm = a.bitmap + size_t(slot) * a.words;
    DCHK(id < a.n);
    const uint32_t bit = 1u << (id & 31);
    const uint32_t old = atomicOr(&bm[id >> 5], bit);
    if (old & bit) return false;
    const uint32_t v = atomicAdd(&s.ctr[2], 1u);
    if (v < a.vcap) a.vlist[size_t(slot) * a.vcap + v] = id;
    return true;
}

__device__ __forceinline__ float qdist(const SearchArgs& a, const Smem& s, uint32_t id) {
    DCHK(id < a.n);
    if (a.x8) return l2_u8(s.q8, a.x8 + size_t(id) * a.ld8, a.ld8, s.qnorm, a.norms8[id]);
    return l2_exact_ldg8(s.q, a.x + size_t(id) * a.ld, a.ld);
}

// Worker barrier (named barrier 1 over the W worker threads; the BBF
// producer warp, when present, never joins it).
template <uint32_t W>
__device__ __forceinline__ void wsync() {
    asm volatile("bar.sync 1, %0;" ::"n"(W) : "memory");
}
// Producer/worker hand-off barriers over all kThreads threads; id is
// 2 + b ("ranges of buffer b ready") or 4 + b ("buffer b read").  Immediate
// barrier ids keep the kernel at 6 hardware barriers.
__device__ __forceinline__ void bar_sync(uint32_t id, uint32_t) {
    switch (id) {
        case 2: asm volatile("bar.sync 2, %0;" ::"n"(kThreads) : "memory"); break;
        case 3: asm volatile("bar.sync 3, %0;" ::"n"(kThreads) : "memory"); break;
        case 4: asm volatile("bar.sync 4, %0;" ::"n"(kThreads) : "memory"); break;
        default: asm volatile("bar.sync 5, %0;" ::"n"(kThreads) : "memory"); break;
    }
}
__device__ __forceinline__ void bar_arrive(uint32_t id, uint32_t) {
    switch (id) {
        case 2: asm volatile("bar.arrive 2, %0;" ::"n"(kThreads) : "memory"); break;
        case 3: asm volatile("bar.arrive 3, %0;" ::"n"(kThreads) : "memory"); break;
        case 4: asm volatile("bar.arrive 4, %0;" ::"n"(kThreads) : "memory"); break;
        default: asm volatile("bar.arrive 5, %0;" ::"n"(kThreads) : "memory"); break;
    }
}

// Block exclusive scan of one flag per thread; returns prefix, total in *tot.
template <uint32_t W>
__device__ __forceinline__ uint32_t block_scan(Smem& s, bool f, uint32_t* tot) {
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t b = __ballot_sync(0xffffffffu, f);
    if (lane == 0) s.scan[warp] = __popc(b);
    wsync<W>();
    uint32_t pre = 0, all = 0;
    for (uint32_t w = 0; w < W / 32; ++w) {
        const uint32_t c = s.scan[w];
        if (w < warp) pre += c;
        all += c;
    }
    wsync<W>();
    *tot = all;
    return pre + __popc(b & ((1u << lane) - 1u));
}

template <int V>
__device__ __forceinline__ void warp0_sort(uint64_t* a, uint32_t n) {
    if (threadIdx.x < 32) {
        uint64_t v[V];
#pragma unroll
        for (int r = 0; r < V; ++r) {
            const uint32_t e = uint32_t(r) * 32 + threadIdx.x;
            v[r] = e < n ? a[e] : kEmptyKey;
        }
        warp_sort_regs<V>(v);
#pragma unroll
        for (int r = 0; r < V; ++r) {
            const uint32_t e = uint32_t(r) * 32 + threadIdx.x;
            if (e < n) a[e] = v[r];
        }
    }
}

// Ascending sort of a[0..n); up to 256 keys in warp 0's registers (no block
// barriers inside), larger sets by the block (a must have room for
// next_pow2(n) keys).  Ends with a barrier.
template <uint32_t W>
__device__ void block_sort_keys(uint64_t* a, uint32_t n) {
    if (n <= 32) warp0_sort<1>(a, n);
    else if (n <= 64) warp0_sort<2>(a, n);
    else if (n <= 128) warp0_sort<4>(a, n);
    else if (n <= 256) warp0_sort<8>(a, n);
    else {
        const uint32_t m = next_pow2(n);
        for (uint32_t j = n + threadIdx.x; j < m; j += W) a[j] = kEmptyKey;
        wsync<W>();
        for (uint32_t k = 2; k <= m; k <<= 1) {
            for (uint32_t j = k >> 1; j > 0; j >>= 1) {
                for (uint32_t i = threadIdx.x; i < m; i += W) {
                    const uint32_t ixj = i ^ j;
                    if (ixj > i) {
                        const uint64_t x = a[i], y = a[ixj];
                        if ((x > y) == ((i & k) == 0)) { a[i] = y; a[ixj] = x; }
                    }
                }
                wsync<W>();
            }
        }
    }
    wsync<W>();
}

// Keep the `want` smallest of the c (> want) DISTINCT keys in buf, compacted
// to buf[0..want) in no particular order: MSD radix select over 8-bit digits,
// starting at the highest bit in which the keys differ.  Entry and exit at a
// barrier.
template <uint32_t W>
__device__ void block_select_smallest(Smem& s, uint32_t c, uint32_t want) {
    uint32_t* hist = s.hist;
    const uint32_t tid = threadIdx.x, lane = tid & 31;
    if (tid < 2) hist[kHist + tid] = 0;
    wsync<W>();
    const uint64_t k0 = s.buf[0];
    uint64_t diff = 0;
    for (uint32_t j = tid; j < c; j += W) diff |= s.buf[j] ^ k0;
    const uint32_t dlo = __reduce_or_sync(0xffffffffu, uint32_t(diff));
    const uint32_t dhi = __reduce_or_sync(0xffffffffu, uint32_t(diff >> 32));
    if (lane == 0) {
        if (dlo) atomicOr(&hist[kHist], dlo);
        if (dhi) atomicOr(&hist[kHist + 1], dhi);
    }
    wsync<W>();
    const uint64_t d = (uint64_t(hist[kHist + 1]) << 32) | hist[kHist];
    int shift = d ? ((63 - __clzll(d)) & ~7) : 0;  // byte holding the highest differing bit
    uint64_t prefix = shift + 8 < 64 ? (k0 >> (shift + 8)) << (shift + 8) : 0;
    uint32_t need = want;
    for (;;) {
        for (uint32_t j = tid; j < kHist; j += W) hist[j] = 0;
        wsync<W>();
        const uint32_t hs = uint32_t(shift) + 8;
        for (uint32_t j = tid; j < c; j += W) {
            const uint64_t v = s.buf[j];
            if (hs >= 64 || (v >> hs) == (prefix >> hs)) atomicAdd(&hist[uint32_t(v >> shift) & 255u], 1u);
        }
        wsync<W>();
        if (tid < 32) {  // bucket b with below(b) < need <= below(b) + hist[b]
            uint32_t h[8], sum = 0;
#pragma unroll
            for (int r = 0; r < 8; ++r) { h[r] = hist[lane * 8 + r]; sum += h[r]; }
            uint32_t inc = sum;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= uint32_t(o)) inc += t;
            }
            uint32_t below = inc - sum;
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                if (below < need && need <= below + h[r]) {
                    hist[kHist + 2] = lane * 8 + r;
                    hist[kHist + 3] = below;
                    hist[kHist + 4] = h[r];
                }
                below += h[r];
            }
        }
        wsync<W>();
        const uint32_t b = hist[kHist + 2], below = hist[kHist + 3], inb = hist[kHist + 4];
        prefix |= uint64_t(b) << shift;
        need -= below;
        if (need == inb || shift == 0) break;  // distinct keys: at shift 0 a bucket holds one key
        shift -= 8;
    }
    // keep v iff (v >> shift) <= (prefix >> shift): exactly `want` keys
    uint32_t nu = 0;
    for (uint32_t base = 0; base < c; base += W) {
        const uint32_t j = base + tid;
        uint64_t v = 0;
        bool keep = false;
        if (j < c) {
            v = s.buf[j];
            keep = (v >> shift) <= (prefix >> shift);
        }
        uint32_t tot;
        const uint32_t pos = block_scan<W>(s, keep, &tot);
        if (keep) s.buf[nu + pos] = v;  // nu + pos <= j; block_scan's barriers order reads before writes
        nu += tot;
    }
    DCHK(nu == want);
    wsync<W>();
}

// pool := top-P(pool U buf).  Buffer keys are distinct (fresh visits, and
// reserve entries are consumed on their first offer); a buffer key may equal
// a pool key only in the fallback scan, so pooled keys are dropped here.
// Only the P smallest buffer keys can enter the top-P, so larger buffers are
// cut to those before sorting.
template <uint32_t W>
__device__ void merge_buffer(const SearchArgs& a, Smem& s) {
    wsync<W>();
    uint32_t c = s.ctr[1];
    if (c == 0) return;
    if (c > a.P) {
        block_select_smallest<W>(s, c, a.P);
        c = a.P;
    }
    block_sort_keys<W>(s.buf, c);
    const uint32_t ps = s.ctr[0];
    uint32_t nu = 0;
    for (uint32_t base = 0; base < c; base += W) {
        const uint32_t j = base + threadIdx.x;
        uint64_t v = kEmptyKey;
        bool keep = false;
        if (j < c) {
            v = s.buf[j];
            const uint32_t p = lower_bound64(s.pool, ps, v);
            keep = !(p < ps && s.pool[p] == v);
        }
        uint32_t tot;
        const uint32_t pos = block_scan<W>(s, keep, &tot);
        if (keep) s.buf[nu + pos] = v;
        nu += tot;
    }
    wsync<W>();
    for (uint32_t j = threadIdx.x; j < ps; j += W) {
        const uint32_t r = j + lower_bound64(s.buf, nu, s.pool[j]);
        if (r < a.P) { s.tmp[r] = s.pool[j]; s.tmpc[r] = s.checked[j]; }
    }
    for (uint32_t j = threadIdx.x; j < nu; j += W) {
        const uint32_t r = j + lower_bound64(s.pool, ps, s.buf[j]);
        if (r < a.P) { s.tmp[r] = s.buf[j]; s.tmpc[r] = 0; }
    }
    wsync<W>();
    const uint32_t nps = min(a.P, ps + nu);
    for (uint32_t j = threadIdx.x; j < nps; j += W) {
        s.pool[j] = s.tmp[j];
        s.checked[j] = s.tmpc[j];
    }
    wsync<W>();
    if (threadIdx.x == 0) {
        s.ctr[0] = nps;
        s.ctr[1] = 0;
    }
    wsync<W>();
}

__device__ __forceinline__ uint64_t tail_key(const SearchArgs& a, const Smem& s) {
    return s.ctr[0] == a.P ? s.pool[a.P - 1] : kEmptyKey;
}

__device__ __forceinline__ void push_buf(Smem& s, uint64_t key) {
    const uint32_t slot = atomicAdd(&s.ctr[1], 1u);
    DCHK(slot < kBufMax);
    s.buf[slot] = key;
}

// BBF producer (tree-seeded search): the last warp walks the trees of the
// CTA's NEXT query (kd_forest.cpp:276-305, one lane per tree) while the
// worker warps process the current one.  Leaf ranges go to one of two
// buffers; named barriers 2+b ("ranges of buffer b ready", producer arrives)
// and 4+b ("buffer b read", workers arrive) hand them over.
__device__ void bbf_producer(const SearchArgs& a, Smem& s) {
    const uint32_t lane = threadIdx.x & 31, slot = blockIdx.x;
    HeapEnt* h = a.heaps ? a.heaps + (size_t(slot) * 32 + lane) * a.hcap : s.heap + lane * a.hcap;
    uint32_t k = 0;
    for (;; ++k) {
        const uint32_t b = k & 1;
        if (k >= 2) bar_sync(4 + b, kThreads);
        uint32_t qi = 0;
        if (lane == 0) qi = atomicAdd(a.qnext, 1u);
        qi = __shfl_sync(0xffffffffu, qi, 0);
        if (qi >= a.nq) {  // no queries left: an end marker in buffer b
            if (lane == 0) s.lcnt[2 + b] = 0xffffffffu;
            __threadfence_block();
            __syncwarp();
            bar_arrive(2 + b, kThreads);
            break;
        }
        const float* q = a.q + size_t(qi) * a.ld;
        uint2* leaves = a.leaves + (size_t(slot) * 2 + b) * a.nt * a.n_node;
        uint32_t tot = 0;
        for (uint32_t t = lane; t < a.nt; t += 32) {
            const TreeView tv = a.trees[t];
            uint2* out = leaves + size_t(t) * a.n_node;
            const uint32_t want = min(a.n_node, tv.leaf_count);
            uint32_t hn = 0, cnt = 0;
            uint32_t nd = tv.root;
            double cost = 0.0;
            if (want > 0) {
                for (;;) {
                    KdNodeDev x = tv.nodes[nd];
                    for (; x.split_dim != kLeaf; x = tv.nodes[nd]) {
                        const double diff = double(__ldg(q + x.split_dim)) - double(x.split_val);
                        const HeapEnt v{cost + fabs(diff), diff <= 0.0 ? x.right : x.left, 0};
                        uint32_t i = hn++;
                        while (i > 0) {
                            const uint32_t p = (i - 1) / 2;
                            if (!hless(v, h[p])) break;
                            h[i] = h[p];
                            i = p;
                        }
                        DCHK(i < a.hcap);
                        h[i] = v;
                        nd = diff <= 0.0 ? x.left : x.right;
                    }
                    DCHK(cnt < a.n_node);
                    out[cnt++] = make_uint2(x.left, x.right);
                    if (cnt >= want || hn == 0) break;
                    const HeapEnt top = h[0];
                    const HeapEnt last = h[--hn];
                    uint32_t i = 0;
                    for (;;) {
                        uint32_t c = 2 * i + 1;
                        if (c >= hn) break;
                        if (c + 1 < hn && hless(h[c + 1], h[c])) ++c;
                        if (!hless(h[c], last)) break;
                        h[i] = h[c];
                        i = c;
                    }
                    if (hn) h[i] = last;
                    nd = top.node;
                    cost = top.cost;
                }
            }
            for (uint32_t j = cnt; j < a.n_node; ++j) out[j] = make_uint2(0, 0);
            tot += cnt;
        }
        tot = __reduce_add_sync(0xffffffffu, tot);
        if (lane == 0) {
            s.lcnt[b] = tot;
            s.lcnt[2 + b] = qi;  // the query these ranges belong to
        }
        __threadfence_block();
        __syncwarp();
        bar_arrive(2 + b, kThreads);
    }
    // k = the end marker's production; the workers read productions 0..k-1 and
    // arrived on "buffer read" for each; the production-k step above synced on
    // generation k-2, so generation k-1 is left to match
    if (k >= 1) bar_sync(4 + ((k - 1) & 1), kThreads);
}

template <bool kTree>
__global__ void __launch_bounds__(kThreads, 6) search_kernel(SearchArgs a) {
    constexpr uint32_t W = kTree ? kThreads - 32 : kThreads;  // worker threads
    extern __shared__ __align__(16) unsigned char raw[];
    Smem s;
    {
        unsigned char* p = raw;
        s.heap = reinterpret_cast<HeapEnt*>(p); p += a.heaps ? 0 : size_t(min(a.nt, 32u)) * a.hcap * sizeof(HeapEnt);
        s.q = reinterpret_cast<float*>(p); p += size_t(a.ld) * 4;  // float4 loads need 16 B alignment
        s.q8 = p; p += a.x8 ? a.ld8 : 0;
        s.pool = reinterpret_cast<uint64_t*>(p); p += size_t(a.P) * 8;
        s.tmp = reinterpret_cast<uint64_t*>(p); p += size_t(a.P) * 8;
        s.seeds = reinterpret_cast<uint64_t*>(p); p += size_t(a.seed_cap) * 8;
        s.buf = reinterpret_cast<uint64_t*>(p); p += size_t(a.kbuf) * 8;
        s.rhash = reinterpret_cast<uint64_t*>(p); p += size_t(a.seed_cap) * 16;  // 8-byte entries: before expand
        s.expand = reinterpret_cast<uint32_t*>(p); p += size_t(a.P) * 4;
        s.scan = reinterpret_cast<uint32_t*>(p); p += 64;
        s.ctr = reinterpret_cast<uint32_t*>(p); p += 64;
        s.hist = reinterpret_cast<uint32_t*>(p); p += (kHist + 8) * 4;
        s.lcnt = reinterpret_cast<uint32_t*>(p); p += 16;
        s.checked = p; p += a.P;
        s.tmpc = p;
    }
    const uint32_t slot = blockIdx.x, tid = threadIdx.x;
    if (kTree && tid >= W) {
        bbf_producer(a, s);
        return;
    }
    for (uint32_t k = 0;; ++k) {
        uint32_t qi;
        if (kTree) {
            bar_sync(2 + (k & 1), kThreads);  // production k (this query's leaf ranges, or the end marker)
            qi = s.lcnt[2 + (k & 1)];
        } else {
            if (tid == 0) s.lcnt[2] = atomicAdd(a.qnext, 1u);
            wsync<W>();
            qi = s.lcnt[2];
        }
        if (qi >= a.nq) break;
        for (uint32_t j = tid; j < a.ld; j += W) s.q[j] = a.q[size_t(qi) * a.ld + j];
        if (a.x8) {
            for (uint32_t j = tid; j < a.ld8; j += W) s.q8[j] = a.q8[size_t(qi) * a.ld8 + j];
            s.qnorm = a.qnorms8[qi];
        }
        if (tid < 16) s.ctr[tid] = 0;
        wsync<W>();
        // ------------------------------------------------ seeding
        if (kTree) {
            const uint32_t b = k & 1;
            if (tid == 0) s.ctr[6] = s.lcnt[b];
            // visit every point of every emitted leaf: one thread per (leaf, slot)
            const uint2* leaves = a.leaves + (size_t(slot) * 2 + b) * a.nt * a.n_node;
            const uint32_t items = a.nt * a.n_node * a.leaf_cap;
            for (uint32_t j = tid; j < items; j += W) {
                const uint32_t L = j / a.leaf_cap;
                const uint2 r = leaves[L];
                const uint32_t* pidx = a.trees[L / a.n_node].pidx;
                for (uint32_t p = r.x + (j - L * a.leaf_cap); p < r.y; p += a.leaf_cap) {
                    const uint32_t id = pidx[p];
                    if (mark_visited(a, slot, s, id)) {
                        const uint32_t kk = atomicAdd(&s.ctr[3], 1u);
                        DCHK(kk < a.seed_cap); DCHK(id < a.n);
                        s.seeds[kk] = make_key(qdist(a, s, id), id);
                    }
                }
            }
            bar_arrive(4 + b, kThreads);  // buffer b may be refilled
        } else {
            // search.cpp:156-173: mt19937_64(seed) draws id % n until `want` distinct
            if (tid == 0) {
                uint64_t* mt = a.mtstate + size_t(slot) * 312;
                // 1: per-query substream(seed, qi) (recall_curve, search.cpp:208);
                // 2: the seed as given (a single GraphSearcher::search_random_init call)
                const uint64_t sd = a.random_init == 2 ? a.seed : substream(a.seed, qi);
                mt[0] = sd;
                for (int i = 1; i < 312; ++i) mt[i] = 6364136223846793005ULL * (mt[i - 1] ^ (mt[i - 1] >> 62)) + uint64_t(i);
                int idx = 312;
                const uint32_t want = min(a.rcount == 0 ? a.E : a.rcount, a.n);
                uint32_t have = 0;
                while (have < want) {
                    if (idx == 312) {
                        for (int j = 0; j < 312; ++j) mt[j] = mt_twist(mt[j], mt[(j + 1) % 312], mt[(j + 156) % 312]);
                        idx = 0;
                    }
                    const uint32_t id = uint32_t(mt_temper(mt[idx++]) % a.n);
                    if (!mark_visited(a, slot, s, id)) continue;
                    s.seeds[have++] = id;  // ids first; distances below
                }
                s.ctr[3] = have;
            }
            wsync<W>();
            for (uint32_t j = tid; j < s.ctr[3]; j += W) {
                const uint32_t id = uint32_t(s.seeds[j]);
                s.seeds[j] = make_key(qdist(a, s, id), id);
            }
        }
        wsync<W>();
        const uint32_t ns = s.ctr[3];
        block_sort_keys<W>(s.seeds, ns);
        const uint32_t ps = min(ns, a.E);
        for (uint32_t j = tid; j < ps; j += W) {
            s.pool[j] = s.seeds[j];
            s.checked[j] = 0;
        }
        // reserve: seeds ranked past E, in a hash table on id (load <= 1/2)
        const uint32_t nr = ns - ps;
        const uint32_t rbits = 32 - __clz(max(2 * nr, 2u) - 1);  // table of 2^rbits >= 2 nr slots
        const uint32_t rmask = (1u << rbits) - 1;
        for (uint32_t j = tid; j <= rmask; j += W) s.rhash[j] = kEmptyKey;
        if (tid == 0) s.ctr[0] = ps;
        wsync<W>();
        for (uint32_t j = tid; j < nr; j += W) {
            const uint64_t k = s.seeds[ps + j];
            const uint32_t id = key_id(k);
            const unsigned long long v = (uint64_t(id) << 32) | uint32_t(k >> 32);
            uint32_t h = rhash_slot(id, rbits);
            while (atomicCAS(reinterpret_cast<unsigned long long*>(&s.rhash[h]), kEmptyKey, v) != kEmptyKey)
                h = (h + 1) & rmask;
        }
        wsync<W>();
        // ------------------------------------------------ expansion rounds
        for (uint32_t it = 0; it < a.iters; ++it) {
            const uint32_t pss = s.ctr[0];
            uint32_t ne = 0;
            for (uint32_t base = 0; base < pss; base += W) {
                const uint32_t j = base + tid;
                const bool f = j < pss && !s.checked[j];
                uint32_t tot;
                const uint32_t pos = block_scan<W>(s, f, &tot);
                if (f) {
                    DCHK(ne + pos < a.P);
                    s.expand[ne + pos] = key_id(s.pool[j]);
                    s.checked[j] = 1;
                }
                ne += tot;
            }
            wsync<W>();
            if (ne == 0) break;
            if (tid == 0) s.ctr[7] += ne;
            uint64_t thr = tail_key(a, s);
            const uint32_t slots = ne * a.gk;
            uint32_t* bm = a.bitmap + size_t(slot) * a.words;
            for (uint32_t base = 0; base < slots; base += W * kU) {
                // kU slots per thread: graph reads, then the visited atomics all in flight
                uint32_t nb[kU], old[kU];
#pragma unroll
                for (uint32_t u = 0; u < kU; ++u) {
                    const uint32_t j = base + u * W + tid;
                    nb[u] = kInvalidId;
                    if (j < slots) {
                        uint32_t q = __umulhi(j, a.gk_magic), c = j - q * a.gk;
                        if (c >= a.gk) { ++q; c -= a.gk; }
                        const uint32_t e = s.expand[q];
                        DCHK(e < a.n);
                        nb[u] = a.graph[size_t(e) * a.gk + c];
                    }
                }
                // a plain (L1-cached) read settles most revisits without an L2 atomic: a set
                // bit is always current (bits are only cleared by this CTA's own stores at
                // the end of a query); a clear bit may be stale, so it is set atomically
#pragma unroll
                for (uint32_t u = 0; u < kU; ++u) old[u] = nb[u] != kInvalidId ? bm[nb[u] >> 5] : 0u;
#pragma unroll
                for (uint32_t u = 0; u < kU; ++u)
                    if (nb[u] != kInvalidId && !(old[u] & (1u << (nb[u] & 31))))
                        old[u] = atomicOr(&bm[nb[u] >> 5], 1u << (nb[u] & 31));
#pragma unroll
                for (uint32_t u = 0; u < kU; ++u) {
                    const uint32_t id = nb[u];
                    if (id == kInvalidId) continue;
                    if (!(old[u] & (1u << (id & 31)))) {
                        const uint32_t v = atomicAdd(&s.ctr[2], 1u);
                        if (v < a.vcap) a.vlist[size_t(slot) * a.vcap + v] = id;
                        const uint64_t key = make_key(qdist(a, s, id), id);
                        if (key < thr) push_buf(s, key);
                        continue;
                    }
                    if (nr == 0) continue;
                    // a reserve seed re-enters with its cached distance (search.cpp:79-82).
                    // It is offered once: the pool tail never rises, so a key
                    // the pool rejects (or evicts) can never re-enter it.
                    for (uint32_t h = rhash_slot(id, rbits);; h = (h + 1) & rmask) {
                        const uint64_t e = s.rhash[h];
                        if (e == kEmptyKey) break;
                        if (uint32_t(e >> 32) != id) continue;
                        if (uint32_t(e) != kConsumed) {
                            const uint64_t key = (uint64_t(uint32_t(e)) << 32) | id;
                            if (key < thr) {
                                const unsigned long long mark = (uint64_t(id) << 32) | kConsumed;
                                const uint64_t prev = atomicExch(reinterpret_cast<unsigned long long*>(&s.rhash[h]), mark);
                                if (uint32_t(prev) != kConsumed) push_buf(s, key);
                            }
                        }
                        break;
                    }
                }
                wsync<W>();
                if (s.ctr[1] + W * kU > a.kbuf) {
                    merge_buffer<W>(a, s);
                    thr = tail_key(a, s);
                }
            }
            merge_buffer<W>(a, s);
        }
        // ------------------------------------------------ fallback scan
        wsync<W>();
        if (s.ctr[0] < a.k_return) {
            uint64_t thr = tail_key(a, s);
            for (uint32_t base = 0; base < a.n; base += W) {
                const uint32_t id = base + tid;
                if (id < a.n) {
                    mark_visited(a, slot, s, id);
                    const uint64_t key = make_key(qdist(a, s, id), id);
                    if (key < thr) push_buf(s, key);
                }
                wsync<W>();
                if (s.ctr[1] + W > a.kbuf) {
                    merge_buffer<W>(a, s);
                    thr = tail_key(a, s);
                }
            }
            merge_buffer<W>(a, s);
        }
        wsync<W>();
        // ------------------------------------------------ output + cleanup
        const uint32_t fin = s.ctr[0];
        for (uint32_t j = tid; j < a.k_return; j += W)
            a.out_keys[size_t(qi) * a.k_return + j] = j < fin ? s.pool[j] : kEmptyKey;
        const uint32_t nv = s.ctr[2];
        if (tid == 0) {
            uint64_t* st = a.stats + size_t(qi) * 4;
            st[0] = nv;
            st[1] = s.ctr[6];
            st[2] = s.ctr[7];
            st[3] = ns;
        }
        uint32_t* bm = a.bitmap + size_t(slot) * a.words;
        if (nv <= a.vcap) {
            for (uint32_t j = tid; j < nv; j += W) {
                const uint32_t id = a.vlist[size_t(slot) * a.vcap + j];
                bm[id >> 5] = 0;
            }
        } else {
            for (uint32_t j = tid; j < a.words; j += W) bm[j] = 0;
        }
        wsync<W>();
    }
}

__global__ void keys_split_kernel(const uint64_t* __restrict__ keys, size_t cnt, uint32_t* ids, float* dists) {
    for (size_t t = blockIdx.x * size_t(blockDim.x) + threadIdx.x; t < cnt; t += size_t(gridDim.x) * blockDim.x) {
        const uint64_t k = keys[t];
        ids[t] = k == kEmptyKey ? kInvalidId : key_id(k);
        dists[t] = k == kEmptyKey ? 0.0f : key_dist(k);
    }
}

void check_status(int st) {
    if (st != 0) throw Error(st, annk_last_error());
}

void run_search(annk_searcher* sr, const annk_dataset* qds, const annk_search_params* p, uint32_t* out_ids,
                float* out_dists, uint64_t* stats_out) {
    const annk_dataset* base = sr->base;
    const annk_forest* f = sr->forest;
    // search.cpp:37-45 begin_query validation
    if (p->k_return < 1 || p->k_return > p->pool_size) throw_invalid("search: need 1 <= k_return <= pool_size");
    if (p->expansion > p->pool_size) throw_invalid("search: need expansion <= pool_size");
    if (p->k_return > base->n) throw_invalid("search: k_return exceeds n");
    if (!p->random_init && !f) throw_invalid("search: tree-seeded search needs a forest");
    const uint32_t nq = qds->n;
    if (nq == 0) return;
    uint32_t nt = 0, n_node = 0, leaf_cap = 1, max_depth = 0;
    if (!p->random_init) {
        nt = p->n_trees_used == 0 ? f->n_trees : std::min(p->n_trees_used, f->n_trees);
        // search.cpp:131-133: truncating division, clamped per tree
        n_node = p->pool_size / std::max(1u, f->leaf_cap) / std::max(1u, nt) + 1;
        leaf_cap = f->leaf_cap;
        for (uint32_t t = 0; t < nt; ++t) max_depth = std::max(max_depth, f->trees[t].max_depth);
        if (nt > kThreads) throw_invalid("search: more than 256 trees in use is not supported");
    }
    const uint64_t seed_bound =
        p->random_init ? std::min<uint64_t>(p->random_seed_count ? p->random_seed_count : p->expansion, base->n)
                       : std::min<uint64_t>(uint64_t(nt) * n_node * leaf_cap, base->n);
    const uint32_t seed_cap = next_pow2(uint32_t(std::max<uint64_t>(seed_bound, 1)));
    const uint32_t P = p->pool_size;
    const uint32_t hcap = (n_node + 1) * (max_depth + 1) + 1;
    const size_t heap_bytes = size_t(std::min(nt, 32u)) * hcap * sizeof(HeapEnt);  // one heap per producer lane
    const bool heap_smem = heap_bytes <= kHeapSmem;
    const uint32_t kbuf = P >= 700 ? kBufMax : kBufMin;
    const size_t smem = (heap_smem ? heap_bytes : 0) + size_t(P) * 16 + size_t(seed_cap) * 8 + size_t(kbuf) * 8 +
                        size_t(base->ld) * 4 + size_t(P) * 4 + 128 + (kHist + 8) * 4 + 16 + size_t(seed_cap) * 16 +
                        size_t(P) * 2 + 16 + base->ld8;
    if (smem > size_t(max_smem_optin()))
        throw_invalid("search: pool_size/seed budget exceeds on-chip capacity");
    const auto kern = p->random_init ? search_kernel<false> : search_kernel<true>;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, smem));
    const uint32_t slots = std::min<uint32_t>(nq, uint32_t(num_sms()) * std::max(per_sm, 1));
    const uint32_t words = (base->n + 31) / 32;
    const uint64_t vbound = seed_bound + uint64_t(p->iters) * P * sr->gk;
    const uint32_t vcap = uint32_t(std::min<uint64_t>(vbound, base->n));
    // the visited bitmap lives with the searcher: zeroed once, every query leaves its row clean
    if (sr->bitmap.n < size_t(slots) * words) {
        sr->bitmap.alloc(size_t(slots) * words);
        sr->bitmap.zero();
    }
    DevBuf<uint32_t> vlist(size_t(slots) * std::max(vcap, 1u));
    DevBuf<HeapEnt> heaps(heap_smem || p->random_init ? 0 : size_t(slots) * 32 * hcap);
    DevBuf<uint2> leaves(std::max<size_t>(size_t(slots) * 2 * nt * n_node, 1));
    DevBuf<uint64_t> mt(p->random_init ? size_t(slots) * 312 : 1);
    DevBuf<uint64_t> keys(size_t(nq) * p->k_return), st(size_t(nq) * 4);
    const bool u8 = base->u8 && qds->u8 && base->ld8 == qds->ld8;
    SearchArgs a{base->data.p, base->n, base->ld, qds->data.p, nq, f ? f->views.p : nullptr, nt, n_node, leaf_cap,
                 sr->graph.p, sr->gk, p->k_return, P, p->expansion, p->iters, p->random_init,
                 p->random_seed_count, p->seed, seed_cap, sr->bitmap.p, words, vlist.p, vcap, heaps.p, hcap,
                 leaves.p, mt.p, keys.p, st.p, u8 ? base->data8.p : nullptr, u8 ? base->norms8.p : nullptr,
                 base->ld8, u8 ? qds->data8.p : nullptr, u8 ? qds->norms8.p : nullptr,
                 sr->gk > 1 ? uint32_t((uint64_t(1) << 32) / sr->gk) : 0xffffffffu, nullptr};
    DevBuf<uint32_t> qnext(1);
    qnext.zero();
    a.qnext = qnext.p;
    a.kbuf = kbuf;
    if (p->random_init) LAUNCH(search_kernel<false>, slots, kThreads, smem, a);
    else LAUNCH(search_kernel<true>, slots, kThreads, smem, a);
    const size_t cnt = size_t(nq) * p->k_return;
    DevBuf<uint32_t> di(cnt);
    DevBuf<float> dd(cnt);
    LAUNCH(keys_split_kernel, uint32_t(std::min<size_t>((cnt + 255) / 256, 65535)), 256, 0, keys.p, cnt, di.p, dd.p);
    di.download(out_ids, cnt);
    dd.download(out_dists, cnt);
    if (stats_out) st.download(stats_out, size_t(nq) * 4);
    ssync();
}

}  // namespace
}  // namespace annk

using namespace annk;

extern "C" {

int annk_searcher_create(const annk_dataset* base, const annk_forest* f, const uint32_t* graph_ids,
                         uint32_t graph_n, uint32_t graph_k, annk_searcher** out) {
    return abi([&] {
        if (!base || !out) throw_invalid("searcher: null argument");
        // search.cpp:23-35
        if (graph_n != base->n) throw_invalid("searcher: graph does not match base set");
        for (size_t i = 0; i < size_t(graph_n) * graph_k; ++i)
            if (graph_ids[i] >= base->n) throw_invalid("searcher: graph id out of range");
        if (f && (f->n != base->n || f->dim != base->dim)) throw_invalid("searcher: forest does not match base set");
        auto sr = std::make_unique<annk_searcher>();
        sr->base = base;
        sr->forest = f;
        sr->gn = graph_n;
        sr->gk = graph_k;
        sr->graph.alloc(std::max<size_t>(size_t(graph_n) * graph_k, 1));
        sr->graph.upload(graph_ids, size_t(graph_n) * graph_k);
        if (f) forest_ensure_links(const_cast<annk_forest*>(f));
        ssync();
        *out = sr.release();
    });
}

int annk_searcher_destroy(annk_searcher* s) {
    return abi([&] { delete s; });
}

int annk_search(annk_searcher* s, const float* queries, uint32_t nq, uint32_t dim, const annk_search_params* p,
                uint32_t* out_ids, float* out_dists, uint64_t* stats) {
    return abi([&] {
        if (!s || !p) throw_invalid("search: null argument");
        if (dim != s->base->dim) throw_invalid("search: query length mismatch");
        // a transient query set (uploads and gets the same exactness check as a dataset)
        annk_dataset* qds = nullptr;
        check_status(annk_dataset_create(queries, nq, dim, &qds));
        std::unique_ptr<annk_dataset> hold(qds);
        run_search(s, qds, p, out_ids, out_dists, stats);
    });
}

int annk_search_dataset(annk_searcher* s, const annk_dataset* queries, const annk_search_params* p,
                        uint32_t* out_ids, float* out_dists, uint64_t* stats) {
    return abi([&] {
        if (!s || !p || !queries) throw_invalid("search: null argument");
        if (queries->dim != s->base->dim) throw_invalid("search: query length mismatch");
        run_search(s, queries, p, out_ids, out_dists, stats);
    });
}

}  // extern "C"
