// C++ facade tests (run by tests/test_cpp_facade.py on the GPU box): the
// reference-shaped host API over the device library, pinned on the
// reference's own recorded acceptance answers (proj/test_output.txt:11-13)
// and on its unit-test invariants (tests/test_{kd_forest,graph_build,search}.cpp).
#include <algorithm>
#include <cstdio>
#include <numeric>
#include <stdexcept>

#include "annkit_b200.hpp"

using namespace annkit;

static int g_fail = 0;
#define CHECK(c)                                                              \
    do {                                                                      \
        if (!(c)) {                                                           \
            std::fprintf(stderr, "CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #c); \
            ++g_fail;                                                         \
        }                                                                     \
    } while (0)
template <class E, class F>
static bool throws(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

// eval.cpp:82-104: multiset intersection; a repeated result id counts once per truth match
static void test_recall_duplicates() {
    const std::uint32_t res[3] = {5, 5, 7}, gt[3] = {5, 7, 9};
    CHECK(recall(std::span<const std::uint32_t>(res, 3), std::span<const std::uint32_t>(gt, 3)) == 2.0 / 3.0);
    CHECK(throws<std::invalid_argument>(
        [&] { recall(std::span<const std::uint32_t>(res, 2), std::span<const std::uint32_t>(gt, 3)); }));
}

static void test_forest_invariants() {
    const VectorSet vs = gen_synthetic(3000, 12, 7);
    const KdForest f = build_forest(vs, 3, 8, 7);
    CHECK(f.trees.size() == 3 && f.n == 3000 && f.dim == 12);
    for (const auto& t : f.trees) {
        std::vector<std::uint32_t> p = t.point_index;
        std::sort(p.begin(), p.end());
        for (std::uint32_t i = 0; i < 3000; ++i) CHECK(p[i] == i);
        std::uint32_t leaves = 0, covered = 0;
        for (const auto& nd : t.nodes)
            if (nd.is_leaf()) {
                ++leaves;
                CHECK(nd.right > nd.left && nd.right - nd.left <= 8);
                covered += nd.right - nd.left;
            }
        CHECK(leaves == t.leaf_count && covered == 3000);
        // the first best-bin-first leaf is the pure descent (kd_forest.hpp search_leaves)
        for (std::uint32_t q = 0; q < 20; ++q) {
            const auto leaves_q = search_leaves(t, vs.row(q * 100), 4);
            CHECK(!leaves_q.empty() && leaves_q[0] == descend_from(t, vs.row(q * 100), t.root));
        }
    }
    CHECK(throws<std::out_of_range>([&] { descend_from(f.trees[0], vs.row(0), 1u << 30); }));
}

static void test_refine_state_mirror() {
    const VectorSet vs = gen_synthetic(800, 8, 3);
    const KdForest f = build_forest(vs, 4, 10, 3);
    RefineState s = init_graph(vs, f, 10, 2, 30, 20, 3);
    CHECK(s.n() == 800 && s.pool_cap == 30 && s.iteration == 0 && s.dist_comps > 0);
    for (const auto& pl : s.pools) {
        const auto e = pl.entries();
        for (std::size_t j = 0; j < e.size(); ++j) {
            CHECK(e[j].flag_new);
            if (j) CHECK(e[j - 1].dist < e[j].dist || (e[j - 1].dist == e[j].dist && e[j - 1].id < e[j].id));
        }
    }
    detail::rebuild_sample_lists(s);
    for (std::uint32_t i = 0; i < s.n(); ++i) CHECK(s.g_new[i].size() <= 20);
    detail::union_reverse_lists(s);
    const std::uint64_t before = s.dist_comps;
    refine_nn_descent(s, vs, 3);
    CHECK(s.iteration >= 1 && s.dist_comps > before);
    const KnnGraph g = finalize(s, vs, 10);
    CHECK(g.n == 800 && g.k == 10 && g.has_dists());
    CHECK(throws<std::invalid_argument>([&] { init_graph(vs, f, 10, 2, 5, 20, 3); }));  // pool_cap < k
}

static std::uint64_t crossing(const BuildResult& r) {
    for (const auto& row : r.stats.iterations)
        if (row.accuracy >= 0.90) return row.dist_comps;
    return 0;
}

static void test_acceptance_build() {
    // proj/test_output.txt:11-12 (criteria 2/3): 10k x 128 uniform, 8 trees leaf 10,
    // Dep 6, P = L = 30: efanna crosses 0.90 at 29,454,671 distance computations,
    // random-descent at 37,263,414.
    const VectorSet vs = gen_synthetic(10000, 128, 1);
    const GroundTruth gt = brute_force_knn(vs, nullptr, 10);
    const KdForest f = build_forest(vs, 8, 10, 1);
    BuildParams p;
    p.k = 10;
    p.conquer_depth = 6;
    p.pool_cap = 30;
    p.sample_cap = 30;
    p.max_iters = 14;
    p.seed = 1;
    const std::uint64_t a = crossing(build_graph(vs, &f, p, &gt));
    p.strategy = BuildStrategy::random_descent;
    p.max_iters = 20;
    const std::uint64_t b = crossing(build_graph(vs, nullptr, p, &gt));
    std::printf("acceptance build: efanna %llu (29454671), random-descent %llu (37263414)\n",
                (unsigned long long)a, (unsigned long long)b);
    CHECK(a == 29454671ull);
    CHECK(b == 37263414ull);
}

static void test_acceptance_search() {
    // proj/test_output.txt:13 (criterion 4): 10k x 32 uniform, exact 10-NN graph,
    // 8 trees leaf 10, E = 50, P = 100: recall 0.9440 at 1285 comps/query.
    const VectorSet base = gen_synthetic(10000, 32, 1);
    const VectorSet queries = gen_synthetic(100, 32, 2);
    const GroundTruth qgt = brute_force_knn(base, &queries, 10);
    const KnnGraph graph = brute_force_graph(base, 10);
    const KdForest f = build_forest(base, 8, 10, 1);
    SearchParams sp;
    sp.k_return = 10;
    const SweepPoint pt{50, 100};
    const auto rows = recall_curve(base, &f, graph, queries, qgt, std::span<const SweepPoint>(&pt, 1), sp);
    char rec[32], comps[32];
    std::snprintf(rec, sizeof rec, "%.4f", rows[0].avg_recall);
    std::snprintf(comps, sizeof comps, "%.0f", rows[0].avg_dist_comps);
    std::printf("acceptance search: recall %s (0.9440) at %s comps/query (1285)\n", rec, comps);
    CHECK(std::string(rec) == "0.9440");
    CHECK(std::string(comps) == "1285");
    // single-query search equals the batch row
    GraphSearcher s(base, &f, graph);
    SearchParams one = sp;
    one.expansion = 50;
    one.pool_size = 100;
    const SearchResult r0 = s.search(queries.row(0), one);
    const auto rb = s.search_batch(queries, one);
    CHECK(r0.ids == rb[0].ids && r0.stats.dist_comps == rb[0].stats.dist_comps);
    SearchParams bad = sp;
    bad.pool_size = 5;
    CHECK(throws<std::invalid_argument>([&] { s.search(queries.row(0), bad); }));
}

int main() {
    test_recall_duplicates();
    test_forest_invariants();
    test_refine_state_mirror();
    test_acceptance_search();
    test_acceptance_build();
    std::printf(g_fail ? "FAILED (%d)\n" : "all facade tests passed\n", g_fail);
    return g_fail ? 1 : 0;
}
