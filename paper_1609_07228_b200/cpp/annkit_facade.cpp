// annkit_facade.cpp — the C++ host API (include/annkit_b200.hpp) over the
// C-ABI (include/annkit_b200.h).  Host code only: it moves arguments to the
// device handles, calls the C-ABI and maps status codes back to the
// reference's exception types (std::invalid_argument / std::out_of_range).
#include <algorithm>
#include <chrono>
#include <cstring>

#include "annkit_b200.h"
#include "annkit_b200.hpp"

namespace annkit {

struct DeviceDataset {
    annk_dataset* h = nullptr;
    const float* src = nullptr;  // the host array it was uploaded from
    std::uint32_t n = 0, dim = 0;
    ~DeviceDataset() { annk_dataset_destroy(h); }
};
struct DeviceForest {
    annk_forest* h = nullptr;
    ~DeviceForest() { annk_forest_destroy(h); }
};
struct DeviceState {
    annk_state* h = nullptr;
    ~DeviceState() { annk_state_destroy(h); }
};
struct DeviceSearcher {
    annk_searcher* h = nullptr;
    ~DeviceSearcher() { annk_searcher_destroy(h); }
};

namespace {

void check(int st) {
    if (st == ANNK_OK) return;
    const std::string m = annk_last_error();
    if (st == ANNK_INVALID_ARGUMENT) throw std::invalid_argument(m);
    if (st == ANNK_OUT_OF_RANGE) throw std::out_of_range(m);
    throw std::runtime_error(m);
}

// Device copy of a VectorSet (uploaded on first use, re-uploaded if the host
// array was replaced).
annk_dataset* dev(const VectorSet& vs) {
    if (vs.data.size() != std::size_t(vs.n) * vs.dim) throw std::invalid_argument("VectorSet: data size != n*dim");
    if (!vs.device || vs.device->src != vs.data.data() || vs.device->n != vs.n || vs.device->dim != vs.dim) {
        auto d = std::make_shared<DeviceDataset>();
        const float zero = 0.0f;
        check(annk_dataset_create(vs.data.empty() ? &zero : vs.data.data(), vs.n, vs.dim, &d->h));
        d->src = vs.data.data();
        d->n = vs.n;
        d->dim = vs.dim;
        vs.device = std::move(d);
    }
    return vs.device->h;
}

annk_forest* import_trees(const std::vector<KdTree>& trees, std::uint32_t n, std::uint32_t dim,
                          std::uint32_t leaf_cap, std::uint64_t seed) {
    std::vector<std::uint32_t> counts, roots, sd, le, ri, de, pi;
    std::vector<float> sv;
    std::vector<std::uint8_t> ev;
    for (const auto& t : trees) {
        counts.push_back(std::uint32_t(t.nodes.size()));
        roots.push_back(t.root);
        for (const auto& nd : t.nodes) {
            sd.push_back(nd.split_dim);
            sv.push_back(nd.split_val);
            le.push_back(nd.left);
            ri.push_back(nd.right);
            de.push_back(nd.depth);
            ev.push_back(nd.even_split ? 1 : 0);
        }
        pi.insert(pi.end(), t.point_index.begin(), t.point_index.end());
    }
    annk_forest* h = nullptr;
    check(annk_forest_import(n, dim, leaf_cap, seed, std::uint32_t(trees.size()), counts.data(), roots.data(),
                             sd.data(), sv.data(), le.data(), ri.data(), de.data(), ev.data(), pi.data(), &h));
    return h;
}

annk_forest* dev(const KdForest& f) {
    if (!f.device) {
        auto d = std::make_shared<DeviceForest>();
        d->h = import_trees(f.trees, f.n, f.dim, f.leaf_cap, f.seed);
        f.device = std::move(d);
    }
    return f.device->h;
}

annk_state* dev(RefineState& s) {
    if (!s.device) {  // a host-built state (pools only)
        const std::uint32_t n = s.n(), P = s.pool_cap;
        std::vector<std::uint32_t> sizes(n), ids(std::size_t(n) * P);
        std::vector<float> dists(std::size_t(n) * P);
        std::vector<std::uint8_t> flags(std::size_t(n) * P);
        for (std::uint32_t i = 0; i < n; ++i) {
            const auto e = s.pools[i].entries();
            sizes[i] = std::uint32_t(e.size());
            for (std::size_t j = 0; j < e.size(); ++j) {
                ids[std::size_t(i) * P + j] = e[j].id;
                dists[std::size_t(i) * P + j] = e[j].dist;
                flags[std::size_t(i) * P + j] = std::uint8_t((e[j].flag_new ? 1 : 0) | (e[j].checked ? 2 : 0));
            }
        }
        auto d = std::make_shared<DeviceState>();
        check(annk_state_import(n, s.k, P, s.sample_cap, s.seed, s.iteration, s.dist_comps, sizes.data(),
                                ids.data(), dists.data(), flags.data(), &d->h));
        s.device = std::move(d);
    }
    return s.device->h;
}

// Host mirror of a device state: counters, pools and the four adjacency lists.
void refresh(RefineState& s) {
    annk_state* h = s.device->h;
    std::uint64_t m[8];
    check(annk_state_meta(h, m));
    const std::uint32_t n = std::uint32_t(m[0]), P = std::uint32_t(m[2]);
    s.k = std::uint32_t(m[1]);
    s.pool_cap = P;
    s.sample_cap = std::uint32_t(m[3]);
    s.seed = m[4];
    s.iteration = std::uint32_t(m[5]);
    s.dist_comps = m[6];
    s.last_changes = m[7];
    std::vector<std::uint32_t> sizes(n), ids(std::size_t(n) * P);
    std::vector<float> dists(std::size_t(n) * P);
    std::vector<std::uint8_t> flags(std::size_t(n) * P);
    check(annk_state_export(h, sizes.data(), ids.data(), dists.data(), flags.data()));
    s.pools.assign(n, NeighborPool(P));
    for (std::uint32_t i = 0; i < n; ++i) {
        auto& e = s.pools[i].mutable_entries();
        e.resize(sizes[i]);
        for (std::uint32_t j = 0; j < sizes[i]; ++j) {
            const std::size_t c = std::size_t(i) * P + j;
            e[j] = NeighborEntry{ids[c], dists[c], (flags[c] & 1) != 0, (flags[c] & 2) != 0};
        }
    }
    std::vector<std::vector<std::uint32_t>>* lists[4] = {&s.g_new, &s.g_old, &s.g_rnew, &s.g_rold};
    std::vector<std::uint32_t> off(std::size_t(n) + 1);
    for (int w = 0; w < 4; ++w) {
        check(annk_state_lists(h, w, off.data(), nullptr));
        std::vector<std::uint32_t> data(std::max<std::uint32_t>(off[n], 1));
        check(annk_state_lists(h, w, off.data(), data.data()));
        auto& L = *lists[w];
        L.assign(n, {});
        for (std::uint32_t i = 0; i < n; ++i) L[i].assign(data.begin() + off[i], data.begin() + off[i + 1]);
    }
}

RefineState adopt(annk_state* h) {
    RefineState s;
    s.device = std::make_shared<DeviceState>();
    s.device->h = h;
    refresh(s);
    return s;
}

double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }

annk_search_params cparams(const SearchParams& p, int random_init) {
    annk_search_params c{};
    c.k_return = p.k_return;
    c.pool_size = p.pool_size;
    c.expansion = p.expansion;
    c.iters = p.iters;
    c.n_trees_used = p.n_trees_used;
    c.random_seed_count = p.random_seed_count;
    c.seed = p.seed;
    c.random_init = random_init;
    return c;
}

}  // namespace

// --------------------------------------------------------------- dataset

float l2_sq(const float* a, const float* b, std::uint32_t dim) {
    float out = 0.0f;
    check(annk_l2_sq(a, b, dim, &out));
    return out;
}

float dist_sq(const VectorSet& vs, std::uint32_t a, std::uint32_t b) {
    if (a >= vs.n || b >= vs.n) throw std::out_of_range("dist_sq: id out of range");
    float out = 0.0f;
    check(annk_dist_sq(dev(vs), &a, &b, 1, &out));
    return out;
}

float dist_sq_q(const VectorSet& vs, std::span<const float> q, std::uint32_t b) {
    if (b >= vs.n) throw std::out_of_range("dist_sq_q: id out of range");
    if (q.size() != vs.dim) throw std::invalid_argument("dist_sq_q: query dimension differs from the set");
    float out = 0.0f;
    check(annk_dist_sq_q(dev(vs), q.data(), vs.dim, &b, 1, &out));
    return out;
}

GroundTruth graph_to_ground_truth(const KnnGraph& g) {
    GroundTruth gt;
    gt.n = g.n;
    gt.k = g.k;
    gt.ids = g.ids;
    return gt;
}

KnnGraph graph_from_ground_truth(const GroundTruth& gt) {
    KnnGraph g;
    g.n = gt.n;
    g.k = gt.k;
    g.ids = gt.ids;
    return g;
}

VectorSet gen_synthetic(std::uint32_t n, std::uint32_t dim, std::uint64_t seed) {
    VectorSet vs;
    vs.n = n;
    vs.dim = dim;
    vs.data.resize(std::size_t(n) * dim);
    check(annk_gen_synthetic(n, dim, seed, vs.data.data()));
    return vs;
}

// ---------------------------------------------------------------- forest

KdForest build_forest(const VectorSet& vs, std::uint32_t n_trees, std::uint32_t leaf_cap, std::uint64_t seed,
                      std::uint32_t /*workers*/) {
    auto d = std::make_shared<DeviceForest>();
    check(annk_forest_build(dev(vs), n_trees, leaf_cap, seed, &d->h));
    KdForest f;
    f.seed = seed;
    f.n = vs.n;
    f.dim = vs.dim;
    f.leaf_cap = leaf_cap;
    f.trees.resize(n_trees);
    for (std::uint32_t t = 0; t < n_trees; ++t) {
        std::uint32_t info[4];
        check(annk_forest_tree_info(d->h, t, info));
        const std::uint32_t m = info[0];
        std::vector<std::uint32_t> sd(m), le(m), ri(m), de(m);
        std::vector<float> sv(m);
        std::vector<std::uint8_t> ev(m);
        KdTree& tr = f.trees[t];
        tr.point_index.resize(vs.n);
        check(annk_forest_export(d->h, t, sd.data(), sv.data(), le.data(), ri.data(), de.data(), ev.data(),
                                 tr.point_index.data()));
        tr.nodes.resize(m);
        for (std::uint32_t i = 0; i < m; ++i) tr.nodes[i] = KdNode{sd[i], sv[i], le[i], ri[i], de[i], ev[i] != 0};
        tr.root = info[1];
        tr.leaf_count = info[2];
        tr.leaf_cap = leaf_cap;
        tr.n = vs.n;
        tr.dim = vs.dim;
    }
    f.device = std::move(d);
    return f;
}

std::vector<std::uint32_t> search_leaves(const KdTree& tree, std::span<const float> q, std::uint32_t n_leaves) {
    if (q.size() != tree.dim) throw std::invalid_argument("search_leaves: query dim mismatch");
    DeviceForest one;
    one.h = import_trees({tree}, tree.n, tree.dim, tree.leaf_cap, 0);
    std::vector<std::uint32_t> out(std::max<std::uint32_t>(n_leaves, 1)), cnt(1);
    check(annk_search_leaves(one.h, 0, q.data(), 1, tree.dim, n_leaves, out.data(), cnt.data()));
    out.resize(cnt[0]);
    return out;
}

std::uint32_t descend_from(const KdTree& tree, std::span<const float> q, std::uint32_t node) {
    if (q.size() != tree.dim) throw std::invalid_argument("descend_from: query dim mismatch");
    if (node >= tree.nodes.size()) throw std::out_of_range("descend_from: node out of range");
    DeviceForest one;
    one.h = import_trees({tree}, tree.n, tree.dim, tree.leaf_cap, 0);
    std::uint32_t out = 0;
    check(annk_descend_from(one.h, 0, q.data(), 1, tree.dim, &node, &out));
    return out;
}

// ----------------------------------------------------------- graph build

RefineState init_graph(const VectorSet& vs, const KdForest& forest, std::uint32_t k, std::uint32_t conquer_depth,
                       std::uint32_t pool_cap, std::uint32_t sample_cap, std::uint64_t seed, std::uint32_t) {
    annk_state* h = nullptr;
    check(annk_init_graph(dev(vs), dev(forest), k, conquer_depth, pool_cap, sample_cap, seed, &h));
    return adopt(h);
}

RefineState init_random(const VectorSet& vs, std::uint32_t k, std::uint32_t pool_cap, std::uint32_t sample_cap,
                        std::uint64_t seed, std::uint32_t) {
    annk_state* h = nullptr;
    check(annk_init_random(dev(vs), k, pool_cap, sample_cap, seed, &h));
    return adopt(h);
}

void refine_nn_descent(RefineState& state, const VectorSet& vs, std::uint32_t max_iters, std::uint32_t,
                       double min_change_rate) {
    std::uint32_t ran = 0;
    check(annk_refine_nn_descent(dev(state), dev(vs), max_iters, min_change_rate, &ran));
    refresh(state);
}

KnnGraph finalize(RefineState& state, const VectorSet& vs, std::uint32_t k) {
    KnnGraph g;
    g.n = state.n();
    g.k = k;
    g.ids.resize(std::size_t(g.n) * k);
    g.dists.resize(std::size_t(g.n) * k);
    check(annk_finalize(dev(state), dev(vs), k, g.ids.data(), g.dists.data()));
    refresh(state);
    return g;
}

namespace detail {
std::uint64_t nn_descent_iteration(RefineState& state, const VectorSet& vs, std::uint32_t) {
    std::uint64_t ch = 0;
    check(annk_nn_descent_iteration(dev(state), dev(vs), &ch));
    refresh(state);
    return ch;
}
std::uint64_t nn_expansion_iteration(RefineState& state, const VectorSet& vs, std::uint32_t) {
    std::uint64_t ch = 0;
    check(annk_nn_expansion_iteration(dev(state), dev(vs), &ch));
    refresh(state);
    return ch;
}

void rebuild_sample_lists(RefineState& state) {
    check(annk_rebuild_sample_lists(dev(state)));
    refresh(state);
}
void union_reverse_lists(RefineState& state) {
    check(annk_union_reverse_lists(dev(state)));
    refresh(state);
}
double pool_topk_accuracy(const RefineState& state, const GroundTruth& gt) {
    if (!state.device) throw std::invalid_argument("accuracy hook: state has no device copy");
    double acc = 0.0;
    check(annk_pool_topk_accuracy(state.device->h, gt.ids.data(), gt.n, gt.k, nullptr, &acc));
    return acc;
}
}  // namespace detail

BuildResult build_graph(const VectorSet& vs, const KdForest* forest, const BuildParams& p, const GroundTruth* gt) {
    BuildResult out;
    BuildStats& st = out.stats;
    if (p.strategy == BuildStrategy::brute_force) {
        const double t0 = now();
        std::uint64_t comps = 0;
        out.graph = brute_force_graph(vs, p.k, p.workers, &comps);
        st.init_seconds = now() - t0;
        st.dist_comps = comps;
        st.iterations.push_back({0, st.init_seconds, comps, 0, gt ? graph_accuracy(out.graph, *gt) : -1.0});
        return out;
    }
    // graph_build.cpp:415-416: only efanna and init_only start from the forest
    const bool tree_init = p.strategy == BuildStrategy::efanna || p.strategy == BuildStrategy::init_only;
    if (tree_init && !forest) throw std::invalid_argument("build_graph: strategy needs a forest");
    double t0 = now();
    RefineState s = tree_init ? init_graph(vs, *forest, p.k, p.conquer_depth, p.pool_cap, p.sample_cap, p.seed)
                              : init_random(vs, p.k, p.pool_cap, p.sample_cap, p.seed);
    st.init_seconds = now() - t0;
    auto log = [&](std::uint64_t changes) {
        st.iterations.push_back({s.iteration, st.init_seconds + st.refine_seconds, s.dist_comps, changes,
                                 gt ? detail::pool_topk_accuracy(s, *gt) : -1.0});
    };
    log(0);
    const std::uint32_t iters = p.strategy == BuildStrategy::init_only ? 0 : p.max_iters;
    const double threshold = p.min_change_rate * double(vs.n) * double(p.pool_cap);
    bool finalized = false;
    for (std::uint32_t it = 0; it < iters; ++it) {
        t0 = now();
        std::uint64_t ch = 0;
        if (it + 1 == iters && !gt && p.strategy != BuildStrategy::nn_expansion) {
            // the iteration cap makes this the last round: replay and finalize in one
            // call, the finalized rows copied out while the remaining targets replay
            std::uint64_t round_comps = 0;
            KnnGraph& g = out.graph;
            g.n = s.n();
            g.k = p.k;
            g.ids.resize(std::size_t(g.n) * p.k);
            g.dists.resize(std::size_t(g.n) * p.k);
            check(annk_nn_descent_iteration_finalize(s.device->h, dev(vs), p.k, g.ids.data(), g.dists.data(), &ch,
                                                     &round_comps));
            st.refine_seconds += now() - t0;
            refresh(s);
            st.iterations.push_back({s.iteration, st.init_seconds + st.refine_seconds, round_comps, ch, -1.0});
            st.early_stopped = double(ch) < threshold;
            finalized = true;
            break;
        }
        if (p.strategy == BuildStrategy::nn_expansion) check(annk_nn_expansion_iteration(s.device->h, dev(vs), &ch));
        else check(annk_nn_descent_iteration(s.device->h, dev(vs), &ch));
        st.refine_seconds += now() - t0;
        refresh(s);
        log(ch);
        if (double(ch) < threshold) {
            st.early_stopped = true;
            break;
        }
    }
    if (!finalized) out.graph = finalize(s, vs, p.k);
    st.dist_comps = s.dist_comps;
    return out;
}

// ---------------------------------------------------------------- search


GraphSearcher::GraphSearcher(const VectorSet& base, const KdForest* forest, const KnnGraph& graph)
    : base_(base), forest_(forest), graph_(graph), dev_(std::make_shared<DeviceSearcher>()) {
    check(annk_searcher_create(dev(base), forest ? dev(*forest) : nullptr, graph.ids.data(), graph.n, graph.k,
                               &dev_->h));
}

std::vector<SearchResult> GraphSearcher::search_batch(const VectorSet& queries, const SearchParams& p,
                                                      bool random_init) {
    const std::uint32_t nq = queries.n, kr = p.k_return;
    std::vector<std::uint32_t> ids(std::size_t(nq) * kr);
    std::vector<float> d(std::size_t(nq) * kr);
    std::vector<std::uint64_t> stats(std::size_t(nq) * 4);
    const annk_search_params c = cparams(p, random_init ? 1 : 0);
    check(annk_search(dev_->h, queries.data.data(), nq, queries.dim, &c, ids.data(), d.data(), stats.data()));
    std::vector<SearchResult> out(nq);
    for (std::uint32_t q = 0; q < nq; ++q) {
        auto& r = out[q];
        r.ids.assign(ids.begin() + std::size_t(q) * kr, ids.begin() + std::size_t(q + 1) * kr);
        r.dists.assign(d.begin() + std::size_t(q) * kr, d.begin() + std::size_t(q + 1) * kr);
        while (!r.ids.empty() && r.ids.back() == kInvalidId) {  // fewer than k_return found
            r.ids.pop_back();
            r.dists.pop_back();
        }
        r.stats = SearchStats{stats[q * 4], std::uint32_t(stats[q * 4 + 1]), std::uint32_t(stats[q * 4 + 2]),
                              std::uint32_t(stats[q * 4 + 3])};
    }
    return out;
}

namespace {
SearchResult one_query(annk_searcher* h, std::span<const float> q, const annk_search_params& c) {
    std::vector<std::uint32_t> ids(c.k_return);
    std::vector<float> d(c.k_return);
    std::uint64_t stats[4] = {0, 0, 0, 0};
    check(annk_search(h, q.data(), 1, std::uint32_t(q.size()), &c, ids.data(), d.data(), stats));
    SearchResult r;
    r.ids = std::move(ids);
    r.dists = std::move(d);
    while (!r.ids.empty() && r.ids.back() == kInvalidId) {
        r.ids.pop_back();
        r.dists.pop_back();
    }
    r.stats = SearchStats{stats[0], std::uint32_t(stats[1]), std::uint32_t(stats[2]), std::uint32_t(stats[3])};
    return r;
}
}  // namespace

SearchResult GraphSearcher::search(std::span<const float> q, const SearchParams& params) {
    return one_query(dev_->h, q, cparams(params, 0));
}

SearchResult GraphSearcher::search_random_init(std::span<const float> q, const SearchParams& params) {
    return one_query(dev_->h, q, cparams(params, 2));  // mt19937_64(params.seed) as given
}

std::vector<SweepRow> recall_curve(const VectorSet& base, const KdForest* forest, const KnnGraph& graph,
                                   const VectorSet& queries, const GroundTruth& gt, std::span<const SweepPoint> sweep,
                                   const SearchParams& params, bool random_init, std::uint32_t) {
    if (queries.n == 0) throw std::invalid_argument("recall_curve: empty query set");
    if (queries.dim != base.dim) throw std::invalid_argument("recall_curve: query dim mismatch");
    if (gt.n != queries.n) throw std::invalid_argument("recall_curve: ground truth shape");
    if (gt.k < params.k_return) throw std::invalid_argument("recall_curve: ground truth narrower than k_return");
    GraphSearcher s(base, forest, graph);
    std::vector<SweepRow> table;
    for (const auto& pt : sweep) {
        SearchParams p = params;
        p.expansion = pt.expansion;
        p.pool_size = pt.pool_size;
        const double t0 = now();
        const auto rs = s.search_batch(queries, p, random_init);
        const double dt = now() - t0;
        SweepRow row;
        row.expansion = pt.expansion;
        row.pool_size = pt.pool_size;
        row.mean_time_us = dt * 1e6 / queries.n;
        for (std::uint32_t q = 0; q < queries.n; ++q) {
            row.avg_recall += recall(rs[q].ids, gt.row(q).subspan(0, p.k_return));
            row.avg_dist_comps += double(rs[q].stats.dist_comps);
            row.avg_seed_points += double(rs[q].stats.seed_points);
        }
        row.avg_recall /= queries.n;
        row.avg_dist_comps /= queries.n;
        row.avg_seed_points /= queries.n;
        table.push_back(row);
    }
    return table;
}

// ------------------------------------------------------------------ eval

GroundTruth brute_force_knn(const VectorSet& base, const VectorSet* queries, std::uint32_t k, std::uint32_t,
                            std::uint64_t* dist_comps) {
    GroundTruth gt;
    gt.n = queries ? queries->n : base.n;
    gt.k = k;
    gt.ids.resize(std::size_t(gt.n) * k);
    check(annk_brute_force_knn(dev(base), queries ? dev(*queries) : nullptr, k, gt.ids.data(), nullptr, dist_comps));
    return gt;
}

KnnGraph brute_force_graph(const VectorSet& base, std::uint32_t k, std::uint32_t, std::uint64_t* dist_comps) {
    KnnGraph g;
    g.n = base.n;
    g.k = k;
    g.ids.resize(std::size_t(g.n) * k);
    g.dists.resize(std::size_t(g.n) * k);
    check(annk_brute_force_knn(dev(base), nullptr, k, g.ids.data(), g.dists.data(), dist_comps));
    return g;
}

double recall(std::span<const std::uint32_t> result_ids, std::span<const std::uint32_t> gt_row) {
    if (result_ids.size() != gt_row.size()) throw std::invalid_argument("recall: result and truth sizes differ");
    if (gt_row.empty()) throw std::invalid_argument("recall: empty truth row");
    // eval.cpp:82-104: multiset intersection of the sorted rows (a duplicated
    // result id counts once per matching truth entry)
    std::vector<std::uint32_t> a(result_ids.begin(), result_ids.end()), t(gt_row.begin(), gt_row.end());
    std::sort(a.begin(), a.end());
    std::sort(t.begin(), t.end());
    std::size_t hits = 0;
    for (std::size_t i = 0, j = 0; i < a.size() && j < t.size();) {
        if (a[i] < t[j]) ++i;
        else if (t[j] < a[i]) ++j;
        else { ++hits; ++i; ++j; }
    }
    return double(hits) / double(gt_row.size());
}

double graph_accuracy(const KnnGraph& graph, const GroundTruth& gt) {
    if (graph.n != gt.n || graph.k != gt.k) throw std::invalid_argument("graph_accuracy: shape mismatch");
    if (graph.n == 0) throw std::invalid_argument("graph_accuracy: empty graph");
    double sum = 0.0;
    for (std::uint32_t i = 0; i < graph.n; ++i) sum += recall(graph.row(i), gt.row(i));
    return sum / graph.n;
}

std::vector<std::pair<std::uint32_t, double>> accuracy_vs_k(const KnnGraph& graph, const VectorSet& vs,
                                                            std::span<const std::uint32_t> k_list, std::uint32_t) {
    std::vector<double> out(std::max<std::size_t>(k_list.size(), 1));
    check(annk_accuracy_vs_k(dev(vs), graph.ids.data(), graph.n, graph.k, k_list.data(),
                             std::uint32_t(k_list.size()), out.data()));
    std::vector<std::pair<std::uint32_t, double>> table;
    for (std::size_t q = 0; q < k_list.size(); ++q) table.emplace_back(k_list[q], out[q]);
    return table;
}

}  // namespace annkit
