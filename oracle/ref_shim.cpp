// ref_shim.cpp — TEST INFRASTRUCTURE ONLY (see oracle_abi.h).
//
// extern "C" wrapper over the UNMODIFIED reference library ("annkit",
// /root/reference/proj).  oracle/Makefile compiles this file together with
// the reference sources where they lie, with the reference's own Release
// flags (-std=c++20 -O3 -DNDEBUG, proj/CMakeLists.txt:3-10,23), into
// oracle/_ref/libannkit_ref.so.  No reference source is copied into the repo.
#include <cstring>
#include <exception>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "annkit/dataset.hpp"
#include "annkit/eval.hpp"
#include "annkit/graph_build.hpp"
#include "annkit/kd_forest.hpp"
#include "annkit/knn_graph.hpp"
#include "annkit/parallel.hpp"
#include "annkit/search.hpp"
#include "annkit/util.hpp"
#include "oracle_abi.h"

using namespace annkit;

namespace {
thread_local std::string g_err;

int fail(const std::exception& e, int code) {
    g_err = e.what();
    return code;
}

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        return fail(e, 1);
    } catch (const std::out_of_range& e) {
        return fail(e, 2);
    } catch (const std::exception& e) {
        return fail(e, 5);
    }
}

VectorSet* V(void* p) { return static_cast<VectorSet*>(p); }
KdForest* F(void* p) { return static_cast<KdForest*>(p); }
RefineState* S(void* p) { return static_cast<RefineState*>(p); }
}  // namespace

extern "C" {

const char* ora_last_error(void) { return g_err.c_str(); }
const char* ora_impl_name(void) { return "reference"; }

void* ora_vs_create(const float* data, uint32_t n, uint32_t dim) {
    auto* vs = new VectorSet;
    vs->n = n;
    vs->dim = dim;
    vs->data.assign(data, data + std::size_t(n) * dim);
    return vs;
}
void ora_vs_free(void* vs) { delete V(vs); }

void ora_gen_synthetic(uint32_t n, uint32_t dim, uint64_t seed, float* out) {
    const VectorSet vs = gen_synthetic(n, dim, seed);
    std::memcpy(out, vs.data.data(), vs.data.size() * sizeof(float));
}
float ora_l2_sq(const float* a, const float* b, uint32_t dim) { return l2_sq(a, b, dim); }
uint64_t ora_mix64(uint64_t x) { return mix64(x); }
uint64_t ora_substream(uint64_t seed, uint64_t id) { return substream(seed, id); }
void ora_mt19937_64(uint64_t seed, uint32_t count, uint64_t* out) {
    std::mt19937_64 rng(seed);
    for (uint32_t i = 0; i < count; ++i) out[i] = rng();
}

int ora_brute_force(void* base, void* queries, uint32_t k, uint32_t workers, uint32_t* ids,
                    float* dists, uint64_t* dist_comps) {
    return guard([&] {
        if (dists && queries == nullptr) {
            const KnnGraph g = brute_force_graph(*V(base), k, workers, dist_comps);
            std::memcpy(ids, g.ids.data(), g.ids.size() * 4);
            std::memcpy(dists, g.dists.data(), g.dists.size() * 4);
            return;
        }
        const GroundTruth gt =
            brute_force_knn(*V(base), queries ? V(queries) : nullptr, k, workers, dist_comps);
        std::memcpy(ids, gt.ids.data(), gt.ids.size() * 4);
        if (dists) {  // query mode with distances: recompute from the ids
            const VectorSet& b = *V(base);
            const VectorSet& q = *V(queries);
            for (uint32_t i = 0; i < gt.n; ++i)
                for (uint32_t j = 0; j < k; ++j)
                    dists[std::size_t(i) * k + j] =
                        l2_sq(q.row_ptr(i), b.row_ptr(gt.ids[std::size_t(i) * k + j]), b.dim);
        }
    });
}

void* ora_forest_build(void* vs, uint32_t n_trees, uint32_t leaf_cap, uint64_t seed,
                       uint32_t workers, int* status) {
    KdForest* out = nullptr;
    *status = guard([&] { out = new KdForest(build_forest(*V(vs), n_trees, leaf_cap, seed, workers)); });
    return out;
}
void ora_forest_free(void* f) { delete F(f); }
uint32_t ora_forest_num_trees(void* f) { return uint32_t(F(f)->trees.size()); }
uint32_t ora_forest_num_nodes(void* f, uint32_t t) { return uint32_t(F(f)->trees[t].nodes.size()); }
void ora_forest_export(void* f, uint32_t t, uint32_t* split_dim, float* split_val,
                       uint32_t* left, uint32_t* right, uint32_t* depth, uint8_t* even,
                       uint32_t* point_index, uint32_t* root_and_leaves) {
    const KdTree& tr = F(f)->trees[t];
    for (std::size_t i = 0; i < tr.nodes.size(); ++i) {
        const KdNode& nd = tr.nodes[i];
        split_dim[i] = nd.split_dim;
        split_val[i] = nd.split_val;
        left[i] = nd.left;
        right[i] = nd.right;
        depth[i] = nd.depth;
        even[i] = nd.even_split ? 1 : 0;
    }
    std::memcpy(point_index, tr.point_index.data(), tr.point_index.size() * 4);
    root_and_leaves[0] = tr.root;
    root_and_leaves[1] = tr.leaf_count;
}
void* ora_forest_import(uint32_t n, uint32_t dim, uint32_t leaf_cap, uint64_t seed,
                        uint32_t n_trees, const uint32_t* node_counts, const uint32_t* roots,
                        const uint32_t* split_dim, const float* split_val, const uint32_t* left,
                        const uint32_t* right, const uint32_t* depth, const uint8_t* even,
                        const uint32_t* point_index) {
    auto* f = new KdForest;
    f->n = n;
    f->dim = dim;
    f->leaf_cap = leaf_cap;
    f->seed = seed;
    f->trees.resize(n_trees);
    std::size_t off = 0;
    for (uint32_t t = 0; t < n_trees; ++t) {
        KdTree& tr = f->trees[t];
        tr.root = roots[t];
        tr.leaf_cap = leaf_cap;
        tr.n = n;
        tr.dim = dim;
        tr.nodes.resize(node_counts[t]);
        tr.leaf_count = 0;
        for (uint32_t i = 0; i < node_counts[t]; ++i) {
            KdNode& nd = tr.nodes[i];
            nd.split_dim = split_dim[off + i];
            nd.split_val = split_val[off + i];
            nd.left = left[off + i];
            nd.right = right[off + i];
            nd.depth = depth[off + i];
            nd.even_split = even[off + i] != 0;
            tr.leaf_count += nd.is_leaf() ? 1 : 0;
        }
        tr.point_index.assign(point_index + std::size_t(t) * n, point_index + std::size_t(t + 1) * n);
        off += node_counts[t];
    }
    return f;
}
int ora_search_leaves(void* f, uint32_t t, const float* q, uint32_t qlen, uint32_t n_leaves,
                      uint32_t* out, uint32_t* n_out) {
    return guard([&] {
        const auto v = search_leaves(F(f)->trees[t], std::span<const float>(q, qlen), n_leaves);
        std::memcpy(out, v.data(), v.size() * 4);
        *n_out = uint32_t(v.size());
    });
}
int ora_descend_from(void* f, uint32_t t, const float* q, uint32_t qlen, uint32_t node,
                     uint32_t* out) {
    return guard([&] { *out = descend_from(F(f)->trees[t], std::span<const float>(q, qlen), node); });
}

void* ora_init_graph(void* vs, void* f, uint32_t k, uint32_t conquer_depth, uint32_t pool_cap,
                     uint32_t sample_cap, uint64_t seed, uint32_t workers, int* status) {
    RefineState* out = nullptr;
    *status = guard([&] {
        out = new RefineState(
            init_graph(*V(vs), *F(f), k, conquer_depth, pool_cap, sample_cap, seed, workers));
    });
    return out;
}
void* ora_init_random(void* vs, uint32_t k, uint32_t pool_cap, uint32_t sample_cap,
                      uint64_t seed, uint32_t workers, int* status) {
    RefineState* out = nullptr;
    *status = guard([&] {
        out = new RefineState(init_random(*V(vs), k, pool_cap, sample_cap, seed, workers));
    });
    return out;
}
void* ora_state_import(uint32_t n, uint32_t k, uint32_t pool_cap, uint32_t sample_cap,
                       uint64_t seed, uint32_t iteration, uint64_t dist_comps,
                       const uint32_t* sizes, const uint32_t* ids, const float* dists,
                       const uint8_t* flags) {
    auto* s = new RefineState;
    s->k = k;
    s->pool_cap = pool_cap;
    s->sample_cap = sample_cap;
    s->seed = seed;
    s->iteration = iteration;
    s->dist_comps = dist_comps;
    s->pools.assign(n, NeighborPool(pool_cap));
    s->g_new.resize(n);
    s->g_old.resize(n);
    s->g_rnew.resize(n);
    s->g_rold.resize(n);
    for (uint32_t i = 0; i < n; ++i)
        for (uint32_t j = 0; j < sizes[i]; ++j) {
            const std::size_t o = std::size_t(i) * pool_cap + j;
            s->pools[i].insert(ids[o], dists[o], (flags[o] & 1) != 0);
        }
    for (uint32_t i = 0; i < n; ++i)  // bit 1: `checked` (nn-expansion)
        for (auto& e : s->pools[i].entries())
            for (uint32_t j = 0; j < sizes[i]; ++j)
                if (ids[std::size_t(i) * pool_cap + j] == e.id) e.checked = (flags[std::size_t(i) * pool_cap + j] >> 1) & 1;
    return s;
}
void ora_state_free(void* s) { delete S(s); }
void ora_state_export(void* sp, uint32_t* sizes, uint32_t* ids, float* dists, uint8_t* flags,
                      uint64_t* meta) {
    RefineState& s = *S(sp);
    for (uint32_t i = 0; i < s.n(); ++i) {
        const auto e = s.pools[i].entries();
        sizes[i] = uint32_t(e.size());
        for (std::size_t j = 0; j < e.size(); ++j) {
            const std::size_t o = std::size_t(i) * s.pool_cap + j;
            ids[o] = e[j].id;
            dists[o] = e[j].dist;
            flags[o] = uint8_t((e[j].flag_new ? 1 : 0) | (e[j].checked ? 2 : 0));
        }
    }
    meta[0] = s.iteration;
    meta[1] = s.dist_comps;
    meta[2] = s.last_changes;
}
void ora_state_lists(void* sp, int which, uint32_t* offsets, uint32_t* data) {
    RefineState& s = *S(sp);
    const auto& L = which == 0 ? s.g_new : which == 1 ? s.g_old : which == 2 ? s.g_rnew : s.g_rold;
    uint32_t o = 0;
    for (uint32_t i = 0; i < s.n(); ++i) {
        offsets[i] = o;
        if (data) std::memcpy(data + o, L[i].data(), L[i].size() * 4);
        o += uint32_t(L[i].size());
    }
    offsets[s.n()] = o;
}
uint64_t ora_nn_descent_iteration(void* s, void* vs, uint32_t workers) {
    return detail::nn_descent_iteration(*S(s), *V(vs), workers);
}
uint64_t ora_nn_expansion_iteration(void* s, void* vs, uint32_t workers) {
    return detail::nn_expansion_iteration(*S(s), *V(vs), workers);
}
void ora_rebuild_sample_lists(void* s) { detail::rebuild_sample_lists(*S(s)); }
void ora_union_reverse_lists(void* s) { detail::union_reverse_lists(*S(s)); }
int ora_refine_nn_descent(void* s, void* vs, uint32_t max_iters, uint32_t workers,
                          double min_change_rate) {
    return guard([&] { refine_nn_descent(*S(s), *V(vs), max_iters, workers, min_change_rate); });
}
int ora_finalize(void* s, void* vs, uint32_t k, uint32_t* ids, float* dists) {
    return guard([&] {
        const KnnGraph g = finalize(*S(s), *V(vs), k);
        std::memcpy(ids, g.ids.data(), g.ids.size() * 4);
        std::memcpy(dists, g.dists.data(), g.dists.size() * 4);
    });
}
double ora_pool_topk_accuracy(void* s, const uint32_t* gt_ids, uint32_t gt_n, uint32_t gt_k) {
    GroundTruth gt;
    gt.n = gt_n;
    gt.k = gt_k;
    gt.ids.assign(gt_ids, gt_ids + std::size_t(gt_n) * gt_k);
    return detail::pool_topk_accuracy(*S(s), gt);
}

int ora_build_graph(void* vs, void* f, uint32_t k, uint32_t conquer_depth, uint32_t pool_cap,
                    uint32_t sample_cap, uint32_t max_iters, int strategy, uint64_t seed,
                    uint32_t workers, double min_change_rate, const uint32_t* gt_ids,
                    uint32_t gt_k, uint32_t* out_ids, float* out_dists, double* log_rows,
                    uint32_t* n_log, double* summary) {
    return guard([&] {
        BuildParams p;
        p.k = k;
        p.conquer_depth = conquer_depth;
        p.pool_cap = pool_cap;
        p.sample_cap = sample_cap;
        p.max_iters = max_iters;
        p.strategy = static_cast<BuildStrategy>(strategy);
        p.seed = seed;
        p.workers = workers;
        p.min_change_rate = min_change_rate;
        GroundTruth gt;
        if (gt_ids) {
            gt.n = V(vs)->n;
            gt.k = gt_k;
            gt.ids.assign(gt_ids, gt_ids + std::size_t(gt.n) * gt_k);
        }
        const BuildResult r = build_graph(*V(vs), F(f), p, gt_ids ? &gt : nullptr);
        std::memcpy(out_ids, r.graph.ids.data(), r.graph.ids.size() * 4);
        if (out_dists && !r.graph.dists.empty())
            std::memcpy(out_dists, r.graph.dists.data(), r.graph.dists.size() * 4);
        *n_log = uint32_t(r.stats.iterations.size());
        for (std::size_t i = 0; i < r.stats.iterations.size(); ++i) {
            const IterationLog& row = r.stats.iterations[i];
            log_rows[i * 5 + 0] = row.iteration;
            log_rows[i * 5 + 1] = row.seconds;
            log_rows[i * 5 + 2] = double(row.dist_comps);
            log_rows[i * 5 + 3] = double(row.changes);
            log_rows[i * 5 + 4] = row.accuracy;
        }
        summary[0] = r.stats.init_seconds;
        summary[1] = r.stats.refine_seconds;
        summary[2] = double(r.stats.dist_comps);
        summary[3] = r.stats.early_stopped ? 1.0 : 0.0;
    });
}

int ora_search(void* base, void* f, const uint32_t* graph_ids, const float* graph_dists,
               uint32_t graph_n, uint32_t graph_k, void* queries, uint32_t k_return,
               uint32_t pool_size, uint32_t expansion, uint32_t iters, uint32_t n_trees_used,
               uint32_t random_seed_count, uint64_t seed, int random_init, uint32_t workers,
               uint32_t* out_ids, float* out_dists, uint64_t* stats, double* time_us) {
    return guard([&] {
        KnnGraph g;
        g.n = graph_n;
        g.k = graph_k;
        g.ids.assign(graph_ids, graph_ids + std::size_t(graph_n) * graph_k);
        if (graph_dists) g.dists.assign(graph_dists, graph_dists + std::size_t(graph_n) * graph_k);
        const VectorSet& qs = *V(queries);
        SearchParams p;
        p.k_return = k_return;
        p.pool_size = pool_size;
        p.expansion = expansion;
        p.iters = iters;
        p.n_trees_used = n_trees_used;
        p.random_seed_count = random_seed_count;
        p.seed = seed;
        GraphSearcher probe(*V(base), F(f), g);  // constructor validation up front
        std::vector<std::string> errs(qs.n);
        std::vector<int> codes(qs.n, 0);
        parallel_for(qs.n, workers, [&](uint32_t begin, uint32_t end) {
            GraphSearcher searcher(*V(base), F(f), g);
            for (uint32_t qi = begin; qi < end; ++qi) {
                SearchParams pq = p;
                pq.seed = substream(p.seed, qi);
                try {
                    StopWatch watch;
                    const SearchResult r = random_init ? searcher.search_random_init(qs.row(qi), pq)
                                                       : searcher.search(qs.row(qi), pq);
                    if (time_us) time_us[qi] = watch.seconds() * 1e6;
                    for (uint32_t j = 0; j < k_return; ++j) {
                        out_ids[std::size_t(qi) * k_return + j] = j < r.ids.size() ? r.ids[j] : 0xffffffffu;
                        out_dists[std::size_t(qi) * k_return + j] = j < r.dists.size() ? r.dists[j] : 0.0f;
                    }
                    stats[qi * 4 + 0] = r.stats.dist_comps;
                    stats[qi * 4 + 1] = r.stats.leaves_visited;
                    stats[qi * 4 + 2] = r.stats.graph_hops;
                    stats[qi * 4 + 3] = r.stats.seed_points;
                } catch (const std::invalid_argument& e) {
                    codes[qi] = 1;
                    errs[qi] = e.what();
                }
            }
        });
        for (uint32_t qi = 0; qi < qs.n; ++qi)
            if (codes[qi]) throw std::invalid_argument(errs[qi]);
    });
}

/* Reference file writers/readers (kd_forest.cpp:307-372, dataset.cpp:96-200,
 * knn_graph.cpp:5-37): byte-compatibility checks for the framework's formats. */
int ora_ref_save_forest(void* f, const char* path) {
    return guard([&] { save_forest(*F(f), path); });
}
void* ora_ref_load_forest(const char* path, int* status) {
    KdForest* out = nullptr;
    *status = guard([&] { out = new KdForest(load_forest(path)); });
    return out;
}
int ora_ref_save_fvecs(void* vs, const char* path) {
    return guard([&] { save_fvecs(*V(vs), path); });
}
int ora_ref_accuracy_vs_k(void* vs, const uint32_t* ids, uint32_t n, uint32_t k, const uint32_t* kl,
                          uint32_t nk, double* out) {
    return guard([&] {
        KnnGraph g;
        g.n = n;
        g.k = k;
        g.ids.assign(ids, ids + size_t(n) * k);
        const auto t = accuracy_vs_k(g, *V(vs), std::span<const uint32_t>(kl, nk), 1);
        for (uint32_t q = 0; q < nk; ++q) out[q] = t[q].second;
    });
}
int ora_ref_save_ivecs(const uint32_t* ids, uint32_t n, uint32_t k, const char* path) {
    return guard([&] {
        GroundTruth gt;
        gt.n = n;
        gt.k = k;
        gt.ids.assign(ids, ids + size_t(n) * k);
        save_ivecs(gt, path);
    });
}

}  // extern "C"
