/*
 * annkit_oracle.c — TEST INFRASTRUCTURE ONLY: the CPU oracle.
 *
 * A plain-C restatement of the reference ("annkit", /root/reference/proj)
 * algorithms on the EFANNA hot path, written from the reference's documented
 * behaviour.  It is the checker the GPU parity tests compare against; it is
 * itself pinned against the unmodified reference (oracle/_ref, built by
 * oracle/Makefile) by tests/test_oracle_pin.py on seeded inputs and against
 * the reference's recorded known-answer values (proj/test_output.txt).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg load
 * this library.  The product (paper_1609_07228_b200) never does.
 *
 * Semantics are the reference's single-worker (deterministic) semantics;
 * `workers` only parallelises the per-row independent loops (brute force,
 * init, search) exactly as parallel_for does (proj/include/annkit/parallel.hpp:13-32),
 * which cannot change results.  Floating point: compiled with
 * -ffp-contract=off so l2_sq stays a sequential mul/add chain.
 */
#define _GNU_SOURCE
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#include "oracle_abi.h"

#define INVALID_ID 0xffffffffu
#define LEAF_MARKER 0xffffffffu

static __thread char g_err[512];
static int set_err(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}
const char* ora_last_error(void) { return g_err; }
const char* ora_impl_name(void) { return "oracle-c"; }

static void* xmalloc(size_t n) {
    void* p = malloc(n ? n : 1);
    if (!p) abort();
    return p;
}
static void* xcalloc(size_t n, size_t s) {
    void* p = calloc(n ? n : 1, s ? s : 1);
    if (!p) abort();
    return p;
}
static double now_s(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

/* ---------------------------------------------------------------- RNG ---- */
/* util.hpp:9-19 mix64 (splitmix64 finalizer) and substream. */
uint64_t ora_mix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}
uint64_t ora_substream(uint64_t seed, uint64_t id) { return ora_mix64(seed ^ ora_mix64(id)); }

/* std::mt19937_64 as fixed by the C++ standard [rand.predef]
 * (w=64, n=312, m=156, r=31, a=0xb5026f5aa96619e9, u=29, d=0x5555555555555555,
 *  s=17, b=0x71d67fffeda60000, t=37, c=0xfff7eee000000000, l=43,
 *  f=6364136223846793005). */
typedef struct {
    uint64_t mt[312];
    int idx;
} mt64;
static void mt64_seed(mt64* g, uint64_t seed) {
    g->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
    g->idx = 312;
}
static uint64_t mt64_next(mt64* g) {
    if (g->idx >= 312) {
        const uint64_t UM = 0xffffffff80000000ULL, LM = 0x7fffffffULL;
        for (int i = 0; i < 312; ++i) {
            const uint64_t y = (g->mt[i] & UM) | (g->mt[(i + 1) % 312] & LM);
            g->mt[i] = g->mt[(i + 156) % 312] ^ (y >> 1) ^ ((y & 1) ? 0xb5026f5aa96619e9ULL : 0);
        }
        g->idx = 0;
    }
    uint64_t x = g->mt[g->idx++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71d67fffeda60000ULL;
    x ^= (x << 37) & 0xfff7eee000000000ULL;
    x ^= x >> 43;
    return x;
}
void ora_mt19937_64(uint64_t seed, uint32_t count, uint64_t* out) {
    mt64 g;
    mt64_seed(&g, seed);
    for (uint32_t i = 0; i < count; ++i) out[i] = mt64_next(&g);
}

/* ------------------------------------------------------------ dataset ---- */
typedef struct {
    uint32_t n, dim;
    float* data;
} vset;
static const float* row(const vset* v, uint32_t i) { return v->data + (size_t)i * v->dim; }

void* ora_vs_create(const float* data, uint32_t n, uint32_t dim) {
    vset* v = xmalloc(sizeof *v);
    v->n = n;
    v->dim = dim;
    v->data = xmalloc((size_t)n * dim * sizeof(float));
    memcpy(v->data, data, (size_t)n * dim * sizeof(float));
    return v;
}
void ora_vs_free(void* p) {
    vset* v = p;
    if (!v) return;
    free(v->data);
    free(v);
}

/* dataset.cpp:201-214: top 24 bits of each mt19937_64 draw times 2^-24. */
void ora_gen_synthetic(uint32_t n, uint32_t dim, uint64_t seed, float* out) {
    mt64 g;
    mt64_seed(&g, seed);
    for (size_t i = 0; i < (size_t)n * dim; ++i)
        out[i] = (float)(uint32_t)(mt64_next(&g) >> 40) * 0x1p-24f;
}

/* dataset.hpp:67-74: sequential fp32, index ascending, separate mul and add. */
static float l2(const float* a, const float* b, uint32_t dim) {
    float acc = 0.0f;
    for (uint32_t i = 0; i < dim; ++i) {
        const float d = a[i] - b[i];
        acc += d * d;
    }
    return acc;
}
float ora_l2_sq(const float* a, const float* b, uint32_t dim) { return l2(a, b, dim); }

/* ------------------------------------------------------- parallel for ---- */
/* parallel.hpp:13-32: contiguous chunks, chunk boundaries from (n, workers). */
typedef void (*range_fn)(void* ctx, uint32_t begin, uint32_t end);
typedef struct {
    range_fn fn;
    void* ctx;
    uint32_t b, e;
} pf_job;
static void* pf_tramp(void* p) {
    pf_job* j = p;
    j->fn(j->ctx, j->b, j->e);
    return NULL;
}
static void parallel_for(uint32_t n, uint32_t workers, range_fn fn, void* ctx) {
    if (n == 0) return;
    if (workers <= 1 || n == 1) {
        fn(ctx, 0, n);
        return;
    }
    if (workers > n) workers = n;
    pthread_t* th = xmalloc(sizeof(pthread_t) * workers);
    pf_job* jobs = xmalloc(sizeof(pf_job) * workers);
    const uint32_t chunk = n / workers, rem = n % workers;
    uint32_t b = 0;
    for (uint32_t w = 0; w < workers; ++w) {
        const uint32_t e = b + chunk + (w < rem ? 1 : 0);
        jobs[w] = (pf_job){fn, ctx, b, e};
        pthread_create(&th[w], NULL, pf_tramp, &jobs[w]);
        b = e;
    }
    for (uint32_t w = 0; w < workers; ++w) pthread_join(th[w], NULL);
    free(th);
    free(jobs);
}

/* The BASELINE configs' seeded Gaussian mixture (DESIGN.md "Synthetic
 * inputs"; the reference has no mixture generator).  The same arithmetic as
 * the product's annk_gen_mixture — counter-based streams, so any thread split
 * yields the same bytes — restated here so the CPU baseline and the reference
 * arm can build their inputs without loading the product library:
 *   u(s, j) = (mix64(s + j) >> 11) * 2^-53
 *   center[c][j] = lo + (hi - lo) * u(substream(seed, 0), c*dim + j)
 *   point i of stream sid: ps = substream(substream(seed, sid), i),
 *     c = mix64(ps) % n_centers, z_j = sqrt(-2 ln(1-u(ps,1+2j))) cos(2 pi u(ps,2+2j)),
 *     v = clip(center[c][j] + sd * z_j), optionally nearbyint. */
typedef struct {
    const double* centers;
    uint32_t dim, n_centers;
    uint64_t ss;
    double sd, clo, chi;
    int rnd;
    float* out;
} mix_ctx;
static double mix_u(uint64_t s, uint64_t j) { return (double)(ora_mix64(s + j) >> 11) * 0x1p-53; }
static void mix_range(void* c, uint32_t b, uint32_t e) {
    const mix_ctx* x = c;
    const double two_pi = 6.283185307179586476925286766559;
    for (uint32_t i = b; i < e; ++i) {
        const uint64_t ps = ora_substream(x->ss, i);
        const uint32_t cc = (uint32_t)(ora_mix64(ps) % x->n_centers);
        for (uint32_t j = 0; j < x->dim; ++j) {
            const double u1 = mix_u(ps, 1 + 2ull * j), u2 = mix_u(ps, 2 + 2ull * j);
            const double z = sqrt(-2.0 * log(1.0 - u1)) * cos(two_pi * u2);
            double v = x->centers[(size_t)cc * x->dim + j] + x->sd * z;
            v = v < x->clo ? x->clo : v;
            v = v > x->chi ? x->chi : v;
            if (x->rnd) v = nearbyint(v);
            x->out[(size_t)i * x->dim + j] = (float)v;
        }
    }
}
void ora_gen_mixture(uint32_t n, uint32_t dim, uint32_t n_centers, float center_lo, float center_hi, float sd,
                     float clip_lo, float clip_hi, int round_to_int, uint64_t seed, uint32_t stream_id,
                     uint32_t workers, float* out) {
    double* centers = xmalloc(sizeof(double) * (size_t)n_centers * dim);
    const uint64_t s0 = ora_substream(seed, 0);
    for (size_t i = 0; i < (size_t)n_centers * dim; ++i)
        centers[i] = (double)center_lo + ((double)center_hi - (double)center_lo) * mix_u(s0, i);
    mix_ctx x = {centers, dim, n_centers, ora_substream(seed, stream_id), (double)sd, (double)clip_lo,
                 (double)clip_hi, round_to_int, out};
    parallel_for(n, workers, mix_range, &x);
    free(centers);
}

/* --------------------------------------------------------------- pool ---- */
/* neighbor_pool.hpp:9-69: ascending (dist, id), capacity-bounded, a duplicate
 * id (same id and dist at the insertion slot) keeps the existing entry. */
typedef struct {
    uint32_t id;
    float dist;
    uint8_t flag_new, checked;
} entry;
typedef struct {
    uint32_t cap, size;
    entry* e;
} pool;
static int entry_less(const entry* a, const entry* b) {
    if (a->dist != b->dist) return a->dist < b->dist;
    return a->id < b->id;
}
static void pool_init(pool* p, uint32_t cap) {
    p->cap = cap;
    p->size = 0;
    p->e = xmalloc(sizeof(entry) * (cap + 1));
}
static int pool_insert(pool* p, uint32_t id, float dist, int flag_new) {
    const entry x = {id, dist, (uint8_t)(flag_new ? 1 : 0), 0};
    uint32_t lo = 0, hi = p->size;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) / 2;
        if (entry_less(&p->e[mid], &x))
            lo = mid + 1;
        else
            hi = mid;
    }
    if (lo < p->size && p->e[lo].id == id && p->e[lo].dist == dist) return 0;
    if (lo >= p->cap) return 0;
    memmove(&p->e[lo + 1], &p->e[lo], sizeof(entry) * (p->size - lo));
    p->e[lo] = x;
    if (p->size < p->cap) ++p->size; /* else the former tail fell off */
    return 1;
}
static int pool_contains(const pool* p, uint32_t id) {
    for (uint32_t j = 0; j < p->size; ++j)
        if (p->e[j].id == id) return 1;
    return 0;
}

/* --------------------------------------------------------- brute force --- */
/* eval.cpp:17-61 exact_row / brute_force_knn / brute_force_graph. */
typedef struct {
    const vset *base, *q;
    uint32_t k;
    uint32_t* ids;
    float* dists;
} bf_ctx;
static void bf_range(void* c, uint32_t b, uint32_t e) {
    bf_ctx* x = c;
    const int self = x->q == NULL;
    pool p;
    pool_init(&p, x->k);
    for (uint32_t i = b; i < e; ++i) {
        const float* q = self ? row(x->base, i) : row(x->q, i);
        p.size = 0;
        for (uint32_t j = 0; j < x->base->n; ++j) {
            if (self && j == i) continue;
            pool_insert(&p, j, l2(q, row(x->base, j), x->base->dim), 0);
        }
        for (uint32_t j = 0; j < x->k; ++j) {
            x->ids[(size_t)i * x->k + j] = p.e[j].id;
            if (x->dists) x->dists[(size_t)i * x->k + j] = p.e[j].dist;
        }
    }
    free(p.e);
}
int ora_brute_force(void* base, void* queries, uint32_t k, uint32_t workers, uint32_t* ids,
                    float* dists, uint64_t* dist_comps) {
    const vset* b = base;
    const vset* q = queries;
    if (b->n == 0) return set_err(1, "brute_force_knn: empty base set");
    if (q && q->dim != b->dim) return set_err(1, "brute_force_knn: query dim mismatch");
    const uint32_t limit = q ? b->n : b->n - 1;
    if (k < 1 || k > limit) return set_err(1, "brute_force_knn: k out of range");
    const uint32_t nq = q ? q->n : b->n;
    bf_ctx c = {b, q, k, ids, dists};
    parallel_for(nq, workers, bf_range, &c);
    if (dist_comps) *dist_comps += (uint64_t)nq * (q ? b->n : b->n - 1);
    return 0;
}

/* -------------------------------------------------------------- forest --- */
/* kd_forest.hpp:18-53 node layout; kd_forest.cpp:29-97 TreeBuilder. */
typedef struct {
    uint32_t split_dim;
    float split_val;
    uint32_t left, right, depth;
    uint8_t even;
} node;
typedef struct {
    node* nodes;
    uint32_t n_nodes, cap_nodes, root, leaf_count;
    uint32_t* pidx;
} tree;
typedef struct {
    uint32_t n, dim, leaf_cap, n_trees;
    uint64_t seed;
    tree* trees;
} forest;

typedef struct {
    const vset* vs;
    tree* t;
    uint32_t leaf_cap;
    mt64 rng;
    uint32_t* tmp;
    uint32_t sort_d;
} builder;

static uint32_t push_node(tree* t, node nd) {
    if (t->n_nodes == t->cap_nodes) {
        t->cap_nodes = t->cap_nodes ? t->cap_nodes * 2 : 64;
        t->nodes = realloc(t->nodes, sizeof(node) * t->cap_nodes);
        if (!t->nodes) abort();
    }
    t->nodes[t->n_nodes] = nd;
    return t->n_nodes++;
}

static __thread const vset* g_sort_vs;
static __thread uint32_t g_sort_d;
static int cmp_val_id(const void* pa, const void* pb) {
    const uint32_t a = *(const uint32_t*)pa, b = *(const uint32_t*)pb;
    const float va = row(g_sort_vs, a)[g_sort_d], vb = row(g_sort_vs, b)[g_sort_d];
    if (va != vb) return va < vb ? -1 : 1;
    return a < b ? -1 : (a > b);
}

/* libstdc++ std::midpoint<float> for finite inputs (<numeric>). */
static float midpoint_f(float a, float b) {
    const float aa = fabsf(a), ab = fabsf(b), hi = 3.40282347e38f / 2;
    if (aa <= hi && ab <= hi) return (a + b) / 2;
    if (aa < 1.17549435e-38f * 2) return a + b / 2;
    if (ab < 1.17549435e-38f * 2) return a / 2 + b;
    return a / 2 + b / 2;
}

static uint32_t build_node(builder* B, uint32_t start, uint32_t end, uint32_t depth) {
    tree* t = B->t;
    const uint32_t size = end - start;
    if (size <= B->leaf_cap) {
        node leaf = {LEAF_MARKER, 0.0f, start, end, depth, 0};
        ++t->leaf_count;
        return push_node(t, leaf);
    }
    const uint32_t d = (uint32_t)(mt64_next(&B->rng) % B->vs->dim);
    double sum = 0.0;
    for (uint32_t p = start; p < end; ++p) sum += row(B->vs, t->pidx[p])[d];
    float split = (float)(sum / size);
    /* stable partition by value <= split */
    uint32_t nl = 0, nr = 0;
    for (uint32_t p = start; p < end; ++p) {
        const uint32_t id = t->pidx[p];
        if (row(B->vs, id)[d] <= split)
            t->pidx[start + nl++] = id;
        else
            B->tmp[nr++] = id;
    }
    memcpy(t->pidx + start + nl, B->tmp, sizeof(uint32_t) * nr);
    uint32_t mid = start + nl;
    const uint32_t lmax = nl > nr ? nl : nr, lmin = nl < nr ? nl : nr;
    uint8_t even = 0;
    if (nl == 0 || nr == 0 || lmax > 4u * lmin) {
        g_sort_vs = B->vs;
        g_sort_d = d;
        qsort(t->pidx + start, size, sizeof(uint32_t), cmp_val_id);
        mid = start + size / 2;
        split = midpoint_f(row(B->vs, t->pidx[mid - 1])[d], row(B->vs, t->pidx[mid])[d]);
        even = 1;
    }
    node in = {d, split, 0, 0, depth, even};
    const uint32_t id = push_node(t, in);
    const uint32_t l = build_node(B, start, mid, depth + 1);
    const uint32_t r = build_node(B, mid, end, depth + 1);
    t->nodes[id].left = l;
    t->nodes[id].right = r;
    return id;
}

typedef struct {
    const vset* vs;
    forest* f;
} bfor_ctx;
static void forest_range(void* c, uint32_t b, uint32_t e) {
    bfor_ctx* x = c;
    for (uint32_t t = b; t < e; ++t) {
        builder B;
        B.vs = x->vs;
        B.t = &x->f->trees[t];
        B.leaf_cap = x->f->leaf_cap;
        mt64_seed(&B.rng, ora_substream(x->f->seed, t));
        B.tmp = xmalloc(sizeof(uint32_t) * x->vs->n);
        B.t->pidx = xmalloc(sizeof(uint32_t) * x->vs->n);
        for (uint32_t i = 0; i < x->vs->n; ++i) B.t->pidx[i] = i;
        B.t->root = build_node(&B, 0, x->vs->n, 0);
        free(B.tmp);
    }
}
void* ora_forest_build(void* vsp, uint32_t n_trees, uint32_t leaf_cap, uint64_t seed,
                       uint32_t workers, int* status) {
    const vset* vs = vsp;
    if (vs->n < 1) {
        *status = set_err(1, "build_forest: empty dataset");
        return NULL;
    }
    if (n_trees < 1 || leaf_cap < 1) {
        *status = set_err(1, "build_forest: n_trees and leaf_cap must be >= 1");
        return NULL;
    }
    forest* f = xcalloc(1, sizeof *f);
    f->n = vs->n;
    f->dim = vs->dim;
    f->leaf_cap = leaf_cap;
    f->seed = seed;
    f->n_trees = n_trees;
    f->trees = xcalloc(n_trees, sizeof(tree));
    bfor_ctx c = {vs, f};
    parallel_for(n_trees, workers, forest_range, &c);
    *status = 0;
    return f;
}
void ora_forest_free(void* p) {
    forest* f = p;
    if (!f) return;
    for (uint32_t t = 0; t < f->n_trees; ++t) {
        free(f->trees[t].nodes);
        free(f->trees[t].pidx);
    }
    free(f->trees);
    free(f);
}
uint32_t ora_forest_num_trees(void* f) { return ((forest*)f)->n_trees; }
uint32_t ora_forest_num_nodes(void* f, uint32_t t) { return ((forest*)f)->trees[t].n_nodes; }
void ora_forest_export(void* fp, uint32_t t, uint32_t* split_dim, float* split_val,
                       uint32_t* left, uint32_t* right, uint32_t* depth, uint8_t* even,
                       uint32_t* point_index, uint32_t* root_and_leaves) {
    const forest* f = fp;
    const tree* tr = &f->trees[t];
    for (uint32_t i = 0; i < tr->n_nodes; ++i) {
        split_dim[i] = tr->nodes[i].split_dim;
        split_val[i] = tr->nodes[i].split_val;
        left[i] = tr->nodes[i].left;
        right[i] = tr->nodes[i].right;
        depth[i] = tr->nodes[i].depth;
        even[i] = tr->nodes[i].even;
    }
    memcpy(point_index, tr->pidx, sizeof(uint32_t) * f->n);
    root_and_leaves[0] = tr->root;
    root_and_leaves[1] = tr->leaf_count;
}
void* ora_forest_import(uint32_t n, uint32_t dim, uint32_t leaf_cap, uint64_t seed,
                        uint32_t n_trees, const uint32_t* node_counts, const uint32_t* roots,
                        const uint32_t* split_dim, const float* split_val, const uint32_t* left,
                        const uint32_t* right, const uint32_t* depth, const uint8_t* even,
                        const uint32_t* point_index) {
    forest* f = xcalloc(1, sizeof *f);
    f->n = n;
    f->dim = dim;
    f->leaf_cap = leaf_cap;
    f->seed = seed;
    f->n_trees = n_trees;
    f->trees = xcalloc(n_trees, sizeof(tree));
    size_t off = 0;
    for (uint32_t t = 0; t < n_trees; ++t) {
        tree* tr = &f->trees[t];
        tr->n_nodes = tr->cap_nodes = node_counts[t];
        tr->nodes = xmalloc(sizeof(node) * node_counts[t]);
        tr->root = roots[t];
        tr->leaf_count = 0;
        for (uint32_t i = 0; i < node_counts[t]; ++i) {
            node nd = {split_dim[off + i], split_val[off + i], left[off + i], right[off + i],
                       depth[off + i], even[off + i]};
            tr->nodes[i] = nd;
            tr->leaf_count += nd.split_dim == LEAF_MARKER;
        }
        tr->pidx = xmalloc(sizeof(uint32_t) * n);
        memcpy(tr->pidx, point_index + (size_t)t * n, sizeof(uint32_t) * n);
        off += node_counts[t];
    }
    return f;
}

/* kd_forest.cpp:266-274 */
static uint32_t descend(const tree* t, const float* q, uint32_t nd) {
    while (t->nodes[nd].split_dim != LEAF_MARKER) {
        const node* x = &t->nodes[nd];
        nd = q[x->split_dim] <= x->split_val ? x->left : x->right;
    }
    return nd;
}
int ora_descend_from(void* fp, uint32_t t, const float* q, uint32_t qlen, uint32_t nd,
                     uint32_t* out) {
    const forest* f = fp;
    if (nd >= f->trees[t].n_nodes) return set_err(2, "descend_from: node id out of range");
    if (qlen != f->dim) return set_err(1, "descend_from: query length mismatch");
    *out = descend(&f->trees[t], q, nd);
    return 0;
}

/* kd_forest.cpp:276-305 best-bin-first; min-heap over (double cost, node). */
typedef struct {
    double cost;
    uint32_t node;
} hent;
typedef struct {
    hent* a;
    uint32_t n, cap;
} heap;
static int hless(const hent* x, const hent* y) {
    if (x->cost != y->cost) return x->cost < y->cost;
    return x->node < y->node;
}
static void heap_push(heap* h, hent v) {
    if (h->n == h->cap) {
        h->cap = h->cap ? h->cap * 2 : 64;
        h->a = realloc(h->a, sizeof(hent) * h->cap);
        if (!h->a) abort();
    }
    uint32_t i = h->n++;
    while (i > 0) {
        const uint32_t p = (i - 1) / 2;
        if (!hless(&v, &h->a[p])) break;
        h->a[i] = h->a[p];
        i = p;
    }
    h->a[i] = v;
}
static hent heap_pop(heap* h) {
    const hent top = h->a[0];
    const hent last = h->a[--h->n];
    uint32_t i = 0;
    for (;;) {
        uint32_t c = 2 * i + 1;
        if (c >= h->n) break;
        if (c + 1 < h->n && hless(&h->a[c + 1], &h->a[c])) ++c;
        if (!hless(&h->a[c], &last)) break;
        h->a[i] = h->a[c];
        i = c;
    }
    if (h->n) h->a[i] = last;
    return top;
}
static uint32_t leaves_bbf(const tree* t, const float* q, uint32_t n_leaves, uint32_t* out,
                           heap* h) {
    uint32_t cnt = 0;
    if (n_leaves == 0) return 0;
    if (n_leaves > t->leaf_count) n_leaves = t->leaf_count;
    h->n = 0;
    uint32_t nd = t->root;
    double cost = 0.0;
    for (;;) {
        while (t->nodes[nd].split_dim != LEAF_MARKER) {
            const node* x = &t->nodes[nd];
            const double diff = (double)q[x->split_dim] - (double)x->split_val;
            const uint32_t other = diff <= 0.0 ? x->right : x->left;
            heap_push(h, (hent){cost + fabs(diff), other});
            nd = diff <= 0.0 ? x->left : x->right;
        }
        out[cnt++] = nd;
        if (cnt >= n_leaves || h->n == 0) break;
        const hent top = heap_pop(h);
        nd = top.node;
        cost = top.cost;
    }
    return cnt;
}
int ora_search_leaves(void* fp, uint32_t t, const float* q, uint32_t qlen, uint32_t n_leaves,
                      uint32_t* out, uint32_t* n_out) {
    const forest* f = fp;
    if (qlen != f->dim) return set_err(1, "search_leaves: query length mismatch");
    heap h = {0};
    *n_out = leaves_bbf(&f->trees[t], q, n_leaves, out, &h);
    free(h.a);
    return 0;
}

/* --------------------------------------------------------- refine state -- */
typedef struct {
    uint32_t* a;
    uint32_t n, cap;
} ulist;
static void ul_push(ulist* l, uint32_t v) {
    if (l->n == l->cap) {
        l->cap = l->cap ? l->cap * 2 : 8;
        l->a = realloc(l->a, sizeof(uint32_t) * l->cap);
        if (!l->a) abort();
    }
    l->a[l->n++] = v;
}
static int cmp_u32(const void* a, const void* b) {
    const uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
    return x < y ? -1 : (x > y);
}
static void ul_dedup(ulist* l) {
    if (l->n == 0) return;
    qsort(l->a, l->n, sizeof(uint32_t), cmp_u32);
    uint32_t w = 1;
    for (uint32_t r = 1; r < l->n; ++r)
        if (l->a[r] != l->a[w - 1]) l->a[w++] = l->a[r];
    l->n = w;
}

/* graph_build.hpp:17-30 */
typedef struct {
    uint32_t n, k, pool_cap, sample_cap, iteration;
    uint64_t seed, dist_comps, last_changes;
    pool* pools;
    ulist *g_new, *g_old, *g_rnew, *g_rold;
} rstate;

/* graph_build.cpp:18-35 make_state */
static rstate* make_state(uint32_t n, uint32_t k, uint32_t pool_cap, uint32_t sample_cap,
                          uint64_t seed, int* status) {
    if (n < 2) {
        *status = set_err(1, "graph build: need at least 2 points");
        return NULL;
    }
    if (k < 1) {
        *status = set_err(1, "graph build: k must be >= 1");
        return NULL;
    }
    if (pool_cap < k) {
        *status = set_err(1, "graph build: pool_cap must be >= k");
        return NULL;
    }
    if (sample_cap < 1) {
        *status = set_err(1, "graph build: sample_cap must be >= 1");
        return NULL;
    }
    rstate* s = xcalloc(1, sizeof *s);
    s->n = n;
    s->k = k;
    s->pool_cap = pool_cap;
    s->sample_cap = sample_cap;
    s->seed = seed;
    s->pools = xmalloc(sizeof(pool) * n);
    for (uint32_t i = 0; i < n; ++i) pool_init(&s->pools[i], pool_cap);
    s->g_new = xcalloc(n, sizeof(ulist));
    s->g_old = xcalloc(n, sizeof(ulist));
    s->g_rnew = xcalloc(n, sizeof(ulist));
    s->g_rold = xcalloc(n, sizeof(ulist));
    *status = 0;
    return s;
}
void ora_state_free(void* p) {
    rstate* s = p;
    if (!s) return;
    for (uint32_t i = 0; i < s->n; ++i) {
        free(s->pools[i].e);
        free(s->g_new[i].a);
        free(s->g_old[i].a);
        free(s->g_rnew[i].a);
        free(s->g_rold[i].a);
    }
    free(s->pools);
    free(s->g_new);
    free(s->g_old);
    free(s->g_rnew);
    free(s->g_rold);
    free(s);
}

/* graph_build.cpp:230-292 init_graph */
typedef struct {
    const vset* vs;
    const forest* f;
    rstate* s;
    uint32_t** owner;
    uint32_t** parent;
    uint32_t dep;
    uint64_t* comps; /* per worker chunk start -> accumulate under lock */
    pthread_mutex_t* mu;
} init_ctx;
static void init_range(void* c, uint32_t b, uint32_t e) {
    init_ctx* x = c;
    ulist cand = {0};
    uint64_t comps = 0;
    for (uint32_t i = b; i < e; ++i) {
        cand.n = 0;
        const float* q = row(x->vs, i);
        for (uint32_t t = 0; t < x->f->n_trees; ++t) {
            const tree* tr = &x->f->trees[t];
            const uint32_t leaf = x->owner[t][i];
            for (uint32_t p = tr->nodes[leaf].left; p < tr->nodes[leaf].right; ++p)
                ul_push(&cand, tr->pidx[p]);
            uint32_t nd = leaf;
            for (;;) {
                const uint32_t par = x->parent[t][nd];
                if (par == INVALID_ID || tr->nodes[par].depth < x->dep) break;
                const node* pn = &tr->nodes[par];
                const uint32_t sib = pn->left == nd ? pn->right : pn->left;
                const uint32_t sl = descend(tr, q, sib);
                for (uint32_t p = tr->nodes[sl].left; p < tr->nodes[sl].right; ++p)
                    ul_push(&cand, tr->pidx[p]);
                nd = par;
            }
        }
        ul_dedup(&cand);
        for (uint32_t j = 0; j < cand.n; ++j) {
            const uint32_t c2 = cand.a[j];
            if (c2 == i) continue;
            pool_insert(&x->s->pools[i], c2, l2(q, row(x->vs, c2), x->vs->dim), 1);
            ++comps;
        }
    }
    free(cand.a);
    pthread_mutex_lock(x->mu);
    *x->comps += comps;
    pthread_mutex_unlock(x->mu);
}
void* ora_init_graph(void* vsp, void* fp, uint32_t k, uint32_t conquer_depth, uint32_t pool_cap,
                     uint32_t sample_cap, uint64_t seed, uint32_t workers, int* status) {
    const vset* vs = vsp;
    const forest* f = fp;
    if (f->n != vs->n || f->dim != vs->dim) {
        *status = set_err(1, "init_graph: forest was built over different data");
        return NULL;
    }
    rstate* s = make_state(vs->n, k, pool_cap, sample_cap, seed, status);
    if (!s) return NULL;
    uint32_t** owner = xmalloc(sizeof(uint32_t*) * f->n_trees);
    uint32_t** parent = xmalloc(sizeof(uint32_t*) * f->n_trees);
    for (uint32_t t = 0; t < f->n_trees; ++t) {
        const tree* tr = &f->trees[t];
        owner[t] = xmalloc(sizeof(uint32_t) * vs->n);
        parent[t] = xmalloc(sizeof(uint32_t) * tr->n_nodes);
        for (uint32_t i = 0; i < vs->n; ++i) owner[t][i] = INVALID_ID;
        for (uint32_t i = 0; i < tr->n_nodes; ++i) parent[t][i] = INVALID_ID;
        for (uint32_t id = 0; id < tr->n_nodes; ++id) {
            const node* nd = &tr->nodes[id];
            if (nd->split_dim == LEAF_MARKER) {
                for (uint32_t p = nd->left; p < nd->right; ++p) owner[t][tr->pidx[p]] = id;
            } else {
                parent[t][nd->left] = id;
                parent[t][nd->right] = id;
            }
        }
    }
    uint64_t comps = 0;
    pthread_mutex_t mu = PTHREAD_MUTEX_INITIALIZER;
    init_ctx c = {vs, f, s, owner, parent, conquer_depth, &comps, &mu};
    parallel_for(vs->n, workers, init_range, &c);
    s->dist_comps += comps;
    for (uint32_t t = 0; t < f->n_trees; ++t) {
        free(owner[t]);
        free(parent[t]);
    }
    free(owner);
    free(parent);
    return s;
}

/* graph_build.cpp:294-326 init_random (baseline; not a GPU path) */
void* ora_init_random(void* vsp, uint32_t k, uint32_t pool_cap, uint32_t sample_cap,
                      uint64_t seed, uint32_t workers, int* status) {
    (void)workers;
    const vset* vs = vsp;
    rstate* s = make_state(vs->n, k, pool_cap, sample_cap, seed, status);
    if (!s) return NULL;
    const uint32_t n = vs->n;
    for (uint32_t i = 0; i < n; ++i) {
        const float* ir = row(vs, i);
        const uint32_t want = pool_cap < n - 1 ? pool_cap : n - 1;
        if (want == n - 1) {
            for (uint32_t j = 0; j < n; ++j) {
                if (j == i) continue;
                pool_insert(&s->pools[i], j, l2(ir, row(vs, j), vs->dim), 1);
                ++s->dist_comps;
            }
            continue;
        }
        mt64 g;
        mt64_seed(&g, ora_substream(seed, i));
        uint32_t have = 0;
        while (have < want) {
            const uint32_t j = (uint32_t)(mt64_next(&g) % n);
            if (j == i || pool_contains(&s->pools[i], j)) continue;
            pool_insert(&s->pools[i], j, l2(ir, row(vs, j), vs->dim), 1);
            ++s->dist_comps;
            ++have;
        }
    }
    return s;
}

void* ora_state_import(uint32_t n, uint32_t k, uint32_t pool_cap, uint32_t sample_cap,
                       uint64_t seed, uint32_t iteration, uint64_t dist_comps,
                       const uint32_t* sizes, const uint32_t* ids, const float* dists,
                       const uint8_t* flags) {
    rstate* s = xcalloc(1, sizeof *s);
    s->n = n;
    s->k = k;
    s->pool_cap = pool_cap;
    s->sample_cap = sample_cap;
    s->seed = seed;
    s->iteration = iteration;
    s->dist_comps = dist_comps;
    s->pools = xmalloc(sizeof(pool) * n);
    s->g_new = xcalloc(n, sizeof(ulist));
    s->g_old = xcalloc(n, sizeof(ulist));
    s->g_rnew = xcalloc(n, sizeof(ulist));
    s->g_rold = xcalloc(n, sizeof(ulist));
    for (uint32_t i = 0; i < n; ++i) {
        pool_init(&s->pools[i], pool_cap);
        for (uint32_t j = 0; j < sizes[i]; ++j) {
            const size_t o = (size_t)i * pool_cap + j;
            pool_insert(&s->pools[i], ids[o], dists[o], flags[o] & 1);
        }
        for (uint32_t j = 0; j < sizes[i]; ++j)  /* bit 1: `checked` (nn-expansion) */
            for (uint32_t e = 0; e < s->pools[i].size; ++e)
                if (s->pools[i].e[e].id == ids[(size_t)i * pool_cap + j])
                    s->pools[i].e[e].checked = (flags[(size_t)i * pool_cap + j] >> 1) & 1;
    }
    return s;
}
void ora_state_export(void* p, uint32_t* sizes, uint32_t* ids, float* dists, uint8_t* flags,
                      uint64_t* meta) {
    const rstate* s = p;
    for (uint32_t i = 0; i < s->n; ++i) {
        sizes[i] = s->pools[i].size;
        for (uint32_t j = 0; j < s->pools[i].size; ++j) {
            const size_t o = (size_t)i * s->pool_cap + j;
            ids[o] = s->pools[i].e[j].id;
            dists[o] = s->pools[i].e[j].dist;
            flags[o] = (uint8_t)(s->pools[i].e[j].flag_new | (s->pools[i].e[j].checked << 1));
        }
    }
    meta[0] = s->iteration;
    meta[1] = s->dist_comps;
    meta[2] = s->last_changes;
}
void ora_state_lists(void* p, int which, uint32_t* offsets, uint32_t* data) {
    const rstate* s = p;
    const ulist* L = which == 0 ? s->g_new : which == 1 ? s->g_old : which == 2 ? s->g_rnew : s->g_rold;
    uint32_t o = 0;
    for (uint32_t i = 0; i < s->n; ++i) {
        offsets[i] = o;
        if (data) memcpy(data + o, L[i].a, sizeof(uint32_t) * L[i].n);
        o += L[i].n;
    }
    offsets[s->n] = o;
}

/* graph_build.cpp:59-86 rebuild_sample_lists (serial pool scan). */
void ora_rebuild_sample_lists(void* p) {
    rstate* s = p;
    for (uint32_t i = 0; i < s->n; ++i) s->g_new[i].n = s->g_old[i].n = s->g_rnew[i].n = s->g_rold[i].n = 0;
    for (uint32_t i = 0; i < s->n; ++i) {
        uint32_t taken = 0;
        pool* pl = &s->pools[i];
        for (uint32_t j = 0; j < pl->size; ++j) {
            if (taken >= s->sample_cap) break;
            entry* e = &pl->e[j];
            if (e->flag_new) {
                ul_push(&s->g_new[i], e->id);
                ul_push(&s->g_rnew[e->id], i);
                e->flag_new = 0;
                ++taken;
            } else {
                ul_push(&s->g_old[i], e->id);
                ul_push(&s->g_rold[e->id], i);
            }
        }
    }
}

/* graph_build.cpp:38-48 sample_down: canonical (sorted, unique) content, then
 * a partial Fisher-Yates over the first cap slots. */
static void sample_down(ulist* l, uint32_t cap, uint64_t seed) {
    ul_dedup(l);
    if (l->n <= cap) return;
    mt64 g;
    mt64_seed(&g, seed);
    for (uint32_t i = 0; i < cap; ++i) {
        const uint32_t j = i + (uint32_t)(mt64_next(&g) % (uint64_t)(l->n - i));
        const uint32_t tmp = l->a[i];
        l->a[i] = l->a[j];
        l->a[j] = tmp;
    }
    l->n = cap;
}

/* graph_build.cpp:88-103 union_reverse_lists */
void ora_union_reverse_lists(void* p) {
    rstate* s = p;
    const uint64_t round_seed = ora_substream(s->seed, s->iteration);
    ulist rn = {0}, ro = {0};
    for (uint32_t i = 0; i < s->n; ++i) {
        rn.n = ro.n = 0;
        for (uint32_t j = 0; j < s->g_rnew[i].n; ++j) ul_push(&rn, s->g_rnew[i].a[j]);
        for (uint32_t j = 0; j < s->g_rold[i].n; ++j) ul_push(&ro, s->g_rold[i].a[j]);
        sample_down(&rn, s->sample_cap, ora_substream(round_seed, 2 * (uint64_t)i));
        sample_down(&ro, s->sample_cap, ora_substream(round_seed, 2 * (uint64_t)i + 1));
        for (uint32_t j = 0; j < rn.n; ++j) ul_push(&s->g_new[i], rn.a[j]);
        for (uint32_t j = 0; j < ro.n; ++j) ul_push(&s->g_old[i], ro.a[j]);
        ul_dedup(&s->g_new[i]);
        ul_dedup(&s->g_old[i]);
    }
    free(rn.a);
    free(ro.a);
}

/* ------------------------------------------------------------ shard mode --
 * Test-only restatement of the multi-GPU protocol (include/annkit_b200.h,
 * "shard mode"): the same five steps over a per-rank copy of the state, with
 * the forward rows / thresholds / offers exchanged by the Python driver.  The
 * pools it yields equal ora_nn_descent_iteration's (graph_build.cpp:105-162
 * reads only the snapshot lists, so the join's inserts commute). */
static uint64_t pool_key(const entry* e) {
    uint32_t b;
    memcpy(&b, &e->dist, 4);
    return ((uint64_t)b << 32) | e->id;
}

/* graph_build.cpp:71-85 for i in [lo, hi): forward rows + start tails. */
void ora_shard_sample(void* p, uint32_t lo, uint32_t hi, uint32_t* fnew, uint32_t* cnew, uint32_t* fold,
                      uint32_t* cold, uint64_t* thr) {
    rstate* s = p;
    const uint32_t S = s->sample_cap, P = s->pool_cap;
    for (uint32_t i = lo; i < hi; ++i) {
        uint32_t taken = 0, nold = 0;
        pool* pl = &s->pools[i];
        for (uint32_t j = 0; j < pl->size; ++j) {
            if (taken >= S) break;
            entry* e = &pl->e[j];
            if (e->flag_new) {
                fnew[(size_t)i * S + taken++] = e->id;
                e->flag_new = 0;
            } else {
                fold[(size_t)i * P + nold++] = e->id;
            }
        }
        cnew[i] = taken;
        cold[i] = nold;
        thr[i] = pl->size == P ? pool_key(&pl->e[P - 1]) : ~0ull;
    }
}

/* graph_build.cpp:59-103 from the forward rows of all points: reverse lists in
 * ascending owner order, sample_down, union (every rank computes all points). */
void ora_shard_union(void* p, const uint32_t* fnew, const uint32_t* cnew, const uint32_t* fold,
                     const uint32_t* cold) {
    rstate* s = p;
    const uint32_t S = s->sample_cap, P = s->pool_cap;
    for (uint32_t i = 0; i < s->n; ++i) s->g_new[i].n = s->g_old[i].n = s->g_rnew[i].n = s->g_rold[i].n = 0;
    for (uint32_t i = 0; i < s->n; ++i) {
        for (uint32_t j = 0; j < cnew[i]; ++j) {
            const uint32_t id = fnew[(size_t)i * S + j];
            ul_push(&s->g_new[i], id);
            ul_push(&s->g_rnew[id], i);
        }
        for (uint32_t j = 0; j < cold[i]; ++j) {
            const uint32_t id = fold[(size_t)i * P + j];
            ul_push(&s->g_old[i], id);
            ul_push(&s->g_rold[id], i);
        }
    }
    ora_union_reverse_lists(s);
}

/* Offers produced by the join of the owned points (target, key, source). */
typedef struct {
    uint32_t* tgt;
    uint64_t* key;
    uint32_t* src;
    size_t n, cap;
} offer_list;
static __thread offer_list g_offers;
static void offer_push(uint32_t tgt, uint64_t key, uint32_t src) {
    if (g_offers.n == g_offers.cap) {
        g_offers.cap = g_offers.cap ? g_offers.cap * 2 : 1024;
        g_offers.tgt = realloc(g_offers.tgt, sizeof(uint32_t) * g_offers.cap);
        g_offers.key = realloc(g_offers.key, sizeof(uint64_t) * g_offers.cap);
        g_offers.src = realloc(g_offers.src, sizeof(uint32_t) * g_offers.cap);
        if (!g_offers.tgt || !g_offers.key || !g_offers.src) abort();
    }
    g_offers.tgt[g_offers.n] = tgt;
    g_offers.key[g_offers.n] = key;
    g_offers.src[g_offers.n] = src;
    ++g_offers.n;
}
static uint64_t make_key_f(float d, uint32_t id) {
    uint32_t b;
    memcpy(&b, &d, 4);
    return ((uint64_t)b << 32) | id;
}

/* graph_build.cpp:105-162 join for i in [lo, hi), offers in the reference's
 * sequential order; offers that beat the target's start tail thr[target] are
 * kept (the rest cannot enter its pool at any point of the round).  Returns
 * the distance count; the offers stay in a thread-local list. */
uint64_t ora_shard_join(void* p, void* vsp, uint32_t lo, uint32_t hi, const uint64_t* thr, uint64_t* n_offers) {
    rstate* s = p;
    const vset* vs = vsp;
    g_offers.n = 0;
    uint64_t comps = 0;
    for (uint32_t i = lo; i < hi; ++i) {
        const ulist* nw = &s->g_new[i];
        const ulist* od = &s->g_old[i];
        for (uint32_t a = 0; a < nw->n; ++a) {
            const uint32_t j = nw->a[a];
            const float* jr = row(vs, j);
            for (uint32_t b = a + 1; b < nw->n; ++b) {
                const uint32_t k2 = nw->a[b];
                const float d = l2(jr, row(vs, k2), vs->dim);
                ++comps;
                if (j != k2) {
                    if (make_key_f(d, k2) < thr[j]) offer_push(j, make_key_f(d, k2), i);
                    if (make_key_f(d, j) < thr[k2]) offer_push(k2, make_key_f(d, j), i);
                }
            }
            for (uint32_t b = 0; b < od->n; ++b) {
                const uint32_t l = od->a[b];
                if (l == j) continue;
                const float d = l2(jr, row(vs, l), vs->dim);
                ++comps;
                if (make_key_f(d, l) < thr[j]) offer_push(j, make_key_f(d, l), i);
                if (make_key_f(d, j) < thr[l]) offer_push(l, make_key_f(d, j), i);
            }
        }
    }
    s->dist_comps += comps;
    *n_offers = g_offers.n;
    return comps;
}
void ora_shard_offers_get(uint32_t* tgt, uint64_t* key, uint32_t* src) {
    memcpy(tgt, g_offers.tgt, sizeof(uint32_t) * g_offers.n);
    memcpy(key, g_offers.key, sizeof(uint64_t) * g_offers.n);
    memcpy(src, g_offers.src, sizeof(uint32_t) * g_offers.n);
}

typedef struct {
    uint32_t tgt, src;
    size_t idx;
} offer_ord;
static int offer_ord_cmp(const void* pa, const void* pb) {
    const offer_ord* a = pa;
    const offer_ord* b = pb;
    if (a->tgt != b->tgt) return a->tgt < b->tgt ? -1 : 1;
    if (a->src != b->src) return a->src < b->src ? -1 : 1;
    return a->idx < b->idx ? -1 : (a->idx > b->idx);
}

/* Inserts offers (all for owned targets) into their pools with flag new, per
 * target in the reference's sequential order: source point ascending, and a
 * source's offers in the order given (its pair order).  Returns the accepted
 * inserts — the reference's `changes` contribution. */
uint64_t ora_shard_replay(void* p, const uint32_t* tgt, const uint64_t* key, const uint32_t* src, size_t m) {
    rstate* s = p;
    offer_ord* ord = xmalloc(sizeof(offer_ord) * (m ? m : 1));
    for (size_t r = 0; r < m; ++r) {
        ord[r].tgt = tgt[r];
        ord[r].src = src[r];
        ord[r].idx = r;
    }
    qsort(ord, m, sizeof(offer_ord), offer_ord_cmp);
    uint64_t changes = 0;
    for (size_t q = 0; q < m; ++q) {
        const size_t r = ord[q].idx;
        float d;
        const uint32_t b = (uint32_t)(key[r] >> 32);
        memcpy(&d, &b, 4);
        changes += pool_insert(&s->pools[tgt[r]], (uint32_t)key[r], d, 1);
    }
    free(ord);
    return changes;
}

/* Ends a sharded round (the replayed pieces' changes summed by the caller). */
void ora_shard_finish(void* p, uint64_t changes) {
    rstate* s = p;
    ++s->iteration;
    s->last_changes = changes;
}

/* graph_build.cpp:105-162 nn_descent_iteration, single-worker order. */
uint64_t ora_nn_descent_iteration(void* p, void* vsp, uint32_t workers) {
    (void)workers;
    rstate* s = p;
    const vset* vs = vsp;
    ora_rebuild_sample_lists(s);
    ora_union_reverse_lists(s);
    uint64_t changes = 0, comps = 0;
    for (uint32_t i = 0; i < s->n; ++i) {
        const ulist* nw = &s->g_new[i];
        const ulist* od = &s->g_old[i];
        for (uint32_t a = 0; a < nw->n; ++a) {
            const uint32_t j = nw->a[a];
            const float* jr = row(vs, j);
            for (uint32_t b = a + 1; b < nw->n; ++b) {
                const uint32_t k2 = nw->a[b];
                const float d = l2(jr, row(vs, k2), vs->dim);
                ++comps;
                if (j != k2) {
                    changes += pool_insert(&s->pools[j], k2, d, 1);
                    changes += pool_insert(&s->pools[k2], j, d, 1);
                }
            }
            for (uint32_t b = 0; b < od->n; ++b) {
                const uint32_t l = od->a[b];
                if (l == j) continue;
                const float d = l2(jr, row(vs, l), vs->dim);
                ++comps;
                changes += pool_insert(&s->pools[j], l, d, 1);
                changes += pool_insert(&s->pools[l], j, d, 1);
            }
        }
    }
    s->dist_comps += comps;
    ++s->iteration;
    s->last_changes = changes;
    return changes;
}

/* graph_build.cpp:164-207 nn_expansion_iteration (baseline; not a GPU path). */
uint64_t ora_nn_expansion_iteration(void* p, void* vsp, uint32_t workers) {
    (void)workers;
    rstate* s = p;
    const vset* vs = vsp;
    ulist* rows = xcalloc(s->n, sizeof(ulist));
    for (uint32_t i = 0; i < s->n; ++i)
        for (uint32_t j = 0; j < s->pools[i].size; ++j) ul_push(&rows[i], s->pools[i].e[j].id);
    uint64_t changes = 0, comps = 0;
    ulist te = {0};
    for (uint32_t i = 0; i < s->n; ++i) {
        te.n = 0;
        pool* pl = &s->pools[i];
        for (uint32_t j = 0; j < pl->size; ++j)
            if (!pl->e[j].checked) {
                pl->e[j].checked = 1;
                ul_push(&te, pl->e[j].id);
            }
        const float* ir = row(vs, i);
        for (uint32_t a = 0; a < te.n; ++a) {
            const ulist* r = &rows[te.a[a]];
            for (uint32_t b = 0; b < r->n; ++b) {
                const uint32_t l = r->a[b];
                if (l == i || pool_contains(pl, l)) continue;
                const float d = l2(ir, row(vs, l), vs->dim);
                ++comps;
                changes += pool_insert(pl, l, d, 1);
            }
        }
    }
    for (uint32_t i = 0; i < s->n; ++i) free(rows[i].a);
    free(rows);
    free(te.a);
    s->dist_comps += comps;
    ++s->iteration;
    s->last_changes = changes;
    return changes;
}

/* graph_build.cpp:328-335 */
int ora_refine_nn_descent(void* p, void* vs, uint32_t max_iters, uint32_t workers,
                          double min_change_rate) {
    rstate* s = p;
    const double thr = min_change_rate * (double)s->n * (double)s->pool_cap;
    for (uint32_t it = 0; it < max_iters; ++it) {
        const uint64_t ch = ora_nn_descent_iteration(s, vs, workers);
        if ((double)ch < thr) break;
    }
    return 0;
}

/* graph_build.cpp:346-373 finalize */
int ora_finalize(void* p, void* vsp, uint32_t k, uint32_t* ids, float* dists) {
    rstate* s = p;
    const vset* vs = vsp;
    if (s->n < 2 || s->n - 1 < k) return set_err(1, "finalize: need n-1 >= k");
    if (k > s->pool_cap) return set_err(1, "finalize: k exceeds pool capacity");
    for (uint32_t i = 0; i < s->n; ++i) {
        pool* pl = &s->pools[i];
        if (pl->size < k) {
            for (uint32_t j = 0; j < s->n && pl->size < k; ++j) {
                if (j == i || pool_contains(pl, j)) continue;
                pool_insert(pl, j, l2(row(vs, i), row(vs, j), vs->dim), 0);
                ++s->dist_comps;
            }
        }
        for (uint32_t j = 0; j < k; ++j) {
            ids[(size_t)i * k + j] = pl->e[j].id;
            dists[(size_t)i * k + j] = pl->e[j].dist;
        }
    }
    return 0;
}

/* graph_build.cpp:209-226 pool_topk_accuracy */
double ora_pool_topk_accuracy(void* p, const uint32_t* gt_ids, uint32_t gt_n, uint32_t gt_k) {
    const rstate* s = p;
    double sum = 0.0;
    uint32_t* truth = xmalloc(sizeof(uint32_t) * gt_k);
    for (uint32_t i = 0; i < gt_n; ++i) {
        memcpy(truth, gt_ids + (size_t)i * gt_k, sizeof(uint32_t) * gt_k);
        qsort(truth, gt_k, sizeof(uint32_t), cmp_u32);
        const uint32_t m = s->k < s->pools[i].size ? s->k : s->pools[i].size;
        uint32_t hits = 0;
        for (uint32_t j = 0; j < m; ++j) {
            const uint32_t id = s->pools[i].e[j].id;
            hits += bsearch(&id, truth, gt_k, sizeof(uint32_t), cmp_u32) != NULL;
        }
        sum += (double)hits / (double)gt_k;
    }
    free(truth);
    return sum / gt_n;
}

/* eval.cpp:82-127 recall / graph_accuracy (used for the brute-force strategy log) */
static double graph_accuracy(const uint32_t* g, const uint32_t* gt, uint32_t n, uint32_t k) {
    uint32_t* a = xmalloc(sizeof(uint32_t) * k);
    uint32_t* b = xmalloc(sizeof(uint32_t) * k);
    double sum = 0;
    for (uint32_t i = 0; i < n; ++i) {
        memcpy(a, g + (size_t)i * k, 4 * k);
        memcpy(b, gt + (size_t)i * k, 4 * k);
        qsort(a, k, 4, cmp_u32);
        qsort(b, k, 4, cmp_u32);
        uint32_t x = 0, y = 0, h = 0;
        while (x < k && y < k) {
            if (a[x] < b[y])
                ++x;
            else if (b[y] < a[x])
                ++y;
            else {
                ++h;
                ++x;
                ++y;
            }
        }
        sum += (double)h / k;
    }
    free(a);
    free(b);
    return sum / n;
}

/* graph_build.cpp:395-461 build_graph */
int ora_build_graph(void* vsp, void* fp, uint32_t k, uint32_t conquer_depth, uint32_t pool_cap,
                    uint32_t sample_cap, uint32_t max_iters, int strategy, uint64_t seed,
                    uint32_t workers, double min_change_rate, const uint32_t* gt_ids,
                    uint32_t gt_k, uint32_t* out_ids, float* out_dists, double* log_rows,
                    uint32_t* n_log, double* summary) {
    vset* vs = vsp;
    memset(summary, 0, sizeof(double) * 4);
    *n_log = 0;
    if (strategy == 3) {
        const double t0 = now_s();
        uint64_t comps = 0;
        float* d = out_dists ? out_dists : xmalloc(sizeof(float) * (size_t)vs->n * k);
        int st = ora_brute_force(vs, NULL, k, workers, out_ids, d, &comps);
        if (!out_dists) free(d);
        if (st) return st;
        summary[0] = now_s() - t0;
        summary[2] = (double)comps;
        log_rows[0] = 0;
        log_rows[1] = summary[0];
        log_rows[2] = (double)comps;
        log_rows[3] = 0;
        log_rows[4] = gt_ids ? graph_accuracy(out_ids, gt_ids, vs->n, k) : -1.0;
        *n_log = 1;
        return 0;
    }
    const int tree_init = strategy == 0 || strategy == 4;
    if (tree_init && fp == NULL) return set_err(1, "build_graph: strategy needs a forest");
    int st = 0;
    const double t0 = now_s();
    rstate* s = tree_init ? ora_init_graph(vs, fp, k, conquer_depth, pool_cap, sample_cap, seed, workers, &st)
                          : ora_init_random(vs, k, pool_cap, sample_cap, seed, workers, &st);
    if (!s) return st;
    summary[0] = now_s() - t0;
    double refine = 0.0;
#define LOG_ROW(ch)                                                                 \
    do {                                                                            \
        double* r_ = log_rows + 5 * (*n_log);                                       \
        r_[0] = s->iteration;                                                       \
        r_[1] = summary[0] + refine;                                                \
        r_[2] = (double)s->dist_comps;                                              \
        r_[3] = (double)(ch);                                                       \
        r_[4] = gt_ids ? ora_pool_topk_accuracy(s, gt_ids, vs->n, gt_k) : -1.0;     \
        ++*n_log;                                                                   \
    } while (0)
    LOG_ROW(0);
    const uint32_t iters = strategy == 4 ? 0 : max_iters;
    const double thr = min_change_rate * (double)s->n * (double)s->pool_cap;
    for (uint32_t it = 0; it < iters; ++it) {
        const double t1 = now_s();
        const uint64_t ch = strategy == 2 ? ora_nn_expansion_iteration(s, vs, workers)
                                          : ora_nn_descent_iteration(s, vs, workers);
        refine += now_s() - t1;
        LOG_ROW(ch);
        if ((double)ch < thr) {
            summary[3] = 1.0;
            break;
        }
    }
#undef LOG_ROW
    summary[1] = refine;
    float* d = out_dists ? out_dists : xmalloc(sizeof(float) * (size_t)vs->n * k);
    st = ora_finalize(s, vs, k, out_ids, d);
    if (!out_dists) free(d);
    summary[2] = (double)s->dist_comps;
    ora_state_free(s);
    return st;
}

/* -------------------------------------------------------------- search --- */
/* search.cpp:23-154 GraphSearcher with epoch-stamped visit tables. */
typedef struct {
    uint32_t id;
    float dist;
} cand;
static int cand_cmp(const void* pa, const void* pb) {
    const cand* a = pa;
    const cand* b = pb;
    if (a->dist != b->dist) return a->dist < b->dist ? -1 : 1;
    return a->id < b->id ? -1 : (a->id > b->id);
}
typedef struct {
    const vset *base, *qs;
    const forest* f;
    const uint32_t* gids;
    uint32_t gk;
    uint32_t k_return, pool_size, expansion, iters, n_trees_used, rcount;
    uint64_t seed;
    int random_init;
    uint32_t* out_ids;
    float* out_dists;
    uint64_t* stats;
    double* time_us;
} search_ctx;

typedef struct {
    uint32_t *vstamp, *cstamp, epoch;
    float* vdist;
    cand *c, *buf;
    size_t ncap, bcap;
    uint32_t nc, nb;
    uint64_t comps;
} searcher;

static float s_visit(searcher* S, const search_ctx* x, const float* q, uint32_t id) {
    if (S->vstamp[id] != S->epoch) {
        S->vstamp[id] = S->epoch;
        S->vdist[id] = l2(q, row(x->base, id), x->base->dim);
        ++S->comps;
    }
    return S->vdist[id];
}
static void c_push(cand** a, size_t* cap, uint32_t* n, cand v) {
    if (*n == *cap) {
        *cap = *cap ? *cap * 2 : 256;
        *a = realloc(*a, sizeof(cand) * *cap);
        if (!*a) abort();
    }
    (*a)[(*n)++] = v;
}
static void sort_unique(cand* a, uint32_t* n) {
    qsort(a, *n, sizeof(cand), cand_cmp);
    if (*n == 0) return;
    uint32_t w = 1;
    for (uint32_t r = 1; r < *n; ++r)
        if (a[r].id != a[w - 1].id) a[w++] = a[r];
    *n = w;
}
static void search_range(void* cp, uint32_t b, uint32_t e) {
    const search_ctx* x = cp;
    const uint32_t N = x->base->n;
    searcher S = {0};
    S.vstamp = xcalloc(N, 4);
    S.cstamp = xcalloc(N, 4);
    S.vdist = xcalloc(N, 4);
    heap h = {0};
    uint32_t* leaves = xmalloc(sizeof(uint32_t) * (x->pool_size + 2));
    for (uint32_t qi = b; qi < e; ++qi) {
        const double t0 = now_s();
        const float* q = row(x->qs, qi);
        ++S.epoch;
        S.nc = S.nb = 0;
        S.comps = 0;
        uint32_t leaves_visited = 0, hops = 0, seed_points = 0;
        if (!x->random_init) {
            const uint32_t nt_all = x->f->n_trees;
            const uint32_t nt = x->n_trees_used == 0 ? nt_all : (x->n_trees_used < nt_all ? x->n_trees_used : nt_all);
            const uint32_t lc = x->f->leaf_cap > 1 ? x->f->leaf_cap : 1;
            const uint32_t n_node = x->pool_size / lc / (nt > 1 ? nt : 1) + 1;
            for (uint32_t t = 0; t < nt; ++t) {
                const tree* tr = &x->f->trees[t];
                const uint32_t nl = leaves_bbf(tr, q, n_node, leaves, &h);
                leaves_visited += nl;
                for (uint32_t l = 0; l < nl; ++l) {
                    const node* nd = &tr->nodes[leaves[l]];
                    for (uint32_t p = nd->left; p < nd->right; ++p) {
                        const uint32_t id = tr->pidx[p];
                        const int fresh = S.vstamp[id] != S.epoch;
                        const float d = s_visit(&S, x, q, id);
                        if (fresh) c_push(&S.c, &S.ncap, &S.nc, (cand){id, d});
                    }
                }
            }
        } else {
            /* search.cpp:156-180 */
            uint32_t want = x->rcount == 0 ? x->expansion : x->rcount;
            if (want > N) want = N;
            mt64 g;
            mt64_seed(&g, ora_substream(x->seed, qi));
            uint32_t have = 0;
            while (have < want) {
                const uint32_t id = (uint32_t)(mt64_next(&g) % N);
                if (S.vstamp[id] == S.epoch) continue;
                const float d = s_visit(&S, x, q, id);
                c_push(&S.c, &S.ncap, &S.nc, (cand){id, d});
                ++have;
            }
        }
        seed_points = S.nc;
        qsort(S.c, S.nc, sizeof(cand), cand_cmp);
        if (S.nc > x->expansion) S.nc = x->expansion;
        /* search.cpp:65-119 expand */
        for (uint32_t it = 0; it < x->iters; ++it) {
            S.nb = 0;
            int any = 0;
            for (uint32_t j = 0; j < S.nc; ++j) {
                const uint32_t id = S.c[j].id;
                if (S.cstamp[id] == S.epoch) continue;
                S.cstamp[id] = S.epoch;
                ++hops;
                any = 1;
                for (uint32_t t = 0; t < x->gk; ++t) {
                    const uint32_t nb = x->gids[(size_t)id * x->gk + t];
                    const float d = s_visit(&S, x, q, nb);
                    c_push(&S.buf, &S.bcap, &S.nb, (cand){nb, d});
                }
            }
            if (!any) break;
            for (uint32_t j = 0; j < S.nb; ++j) c_push(&S.c, &S.ncap, &S.nc, S.buf[j]);
            sort_unique(S.c, &S.nc);
            if (S.nc > x->pool_size) S.nc = x->pool_size;
        }
        if (S.nc < x->k_return) {
            for (uint32_t id = 0; id < N; ++id) {
                const float d = s_visit(&S, x, q, id);
                c_push(&S.c, &S.ncap, &S.nc, (cand){id, d});
            }
            sort_unique(S.c, &S.nc);
        }
        const uint32_t out = x->k_return < S.nc ? x->k_return : S.nc;
        for (uint32_t j = 0; j < x->k_return; ++j) {
            x->out_ids[(size_t)qi * x->k_return + j] = j < out ? S.c[j].id : INVALID_ID;
            x->out_dists[(size_t)qi * x->k_return + j] = j < out ? S.c[j].dist : 0.0f;
        }
        x->stats[(size_t)qi * 4 + 0] = S.comps;
        x->stats[(size_t)qi * 4 + 1] = leaves_visited;
        x->stats[(size_t)qi * 4 + 2] = hops;
        x->stats[(size_t)qi * 4 + 3] = seed_points;
        if (x->time_us) x->time_us[qi] = (now_s() - t0) * 1e6;
    }
    free(S.vstamp);
    free(S.cstamp);
    free(S.vdist);
    free(S.c);
    free(S.buf);
    free(h.a);
    free(leaves);
}
int ora_search(void* base, void* fp, const uint32_t* graph_ids, const float* graph_dists,
               uint32_t graph_n, uint32_t graph_k, void* queries, uint32_t k_return,
               uint32_t pool_size, uint32_t expansion, uint32_t iters, uint32_t n_trees_used,
               uint32_t random_seed_count, uint64_t seed, int random_init, uint32_t workers,
               uint32_t* out_ids, float* out_dists, uint64_t* stats, double* time_us) {
    (void)graph_dists;
    const vset* b = base;
    const vset* qs = queries;
    const forest* f = fp;
    if (graph_n != b->n) return set_err(1, "searcher: graph does not match base set");
    for (size_t i = 0; i < (size_t)graph_n * graph_k; ++i)
        if (graph_ids[i] >= b->n) return set_err(1, "searcher: graph id out of range");
    if (f && (f->n != b->n || f->dim != b->dim)) return set_err(1, "searcher: forest does not match base set");
    if (!random_init && !f) return set_err(1, "search: tree-seeded search needs a forest");
    if (qs->dim != b->dim) return set_err(1, "search: query length mismatch");
    if (k_return < 1 || k_return > pool_size) return set_err(1, "search: need 1 <= k_return <= pool_size");
    if (expansion > pool_size) return set_err(1, "search: need expansion <= pool_size");
    if (k_return > b->n) return set_err(1, "search: k_return exceeds n");
    search_ctx c = {b, qs, f, graph_ids, graph_k, k_return, pool_size, expansion, iters,
                    n_trees_used, random_seed_count, seed, random_init, out_ids, out_dists, stats, time_us};
    parallel_for(qs->n, workers, search_range, &c);
    return 0;
}
