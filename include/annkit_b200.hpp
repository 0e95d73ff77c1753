// annkit_b200.hpp — the C++ host API of the B200 framework.
//
// Source-compatible with the reference library's hot-path API (namespace
// annkit, proj/include/annkit/{dataset,kd_forest,neighbor_pool,graph_build,
// knn_graph,search,eval}.hpp): same type names and fields, same function
// names, signatures and exceptions, so a caller of the CPU library can switch
// by changing the include and the link line.  Every entry point runs on the
// device through the C-ABI in annkit_b200.h (libannkit_facade.so links
// libannkit_b200.so); results are bit-identical to the reference at
// workers = 1.  `workers` arguments are accepted and ignored.
//
// Device residency: VectorSet, KdForest and RefineState carry a shared
// handle to their device copy (uploaded on first use; the reference declares
// these immutable after construction, and so does this API).  RefineState's
// host fields (pools, g_new, g_old, g_rnew, g_rold, counters) are refreshed
// after every call that changes the device state, which is what the
// reference's unit tests inspect; that copy costs O(n * pool_cap) per call.
#pragma once

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <memory>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

namespace annkit {

constexpr std::uint32_t kInvalidId = 0xffffffffu;
constexpr std::uint32_t kLeafMarker = 0xffffffffu;

struct DeviceDataset;  // opaque device copies (annk_dataset / annk_forest / annk_state)
struct DeviceForest;
struct DeviceState;

// ---------------------------------------------------------------- util.hpp
// util.hpp:9-31: seed streams and the wall-clock timer the reference's callers use.
inline std::uint64_t mix64(std::uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}
inline std::uint64_t substream(std::uint64_t seed, std::uint64_t id) { return mix64(seed ^ mix64(id)); }
class StopWatch {
  public:
    StopWatch() : t0_(std::chrono::steady_clock::now()) {}
    double seconds() const { return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0_).count(); }
    void restart() { t0_ = std::chrono::steady_clock::now(); }

  private:
    std::chrono::steady_clock::time_point t0_;
};

// ------------------------------------------------------------ dataset.hpp
struct VectorSet {
    std::uint32_t n = 0;
    std::uint32_t dim = 0;
    std::vector<float> data;  // row-major n x dim
    mutable std::shared_ptr<DeviceDataset> device;  // set on first device use

    std::span<const float> row(std::uint32_t i) const { return {data.data() + std::size_t(i) * dim, dim}; }
    const float* row_ptr(std::uint32_t i) const { return data.data() + std::size_t(i) * dim; }
};

struct GroundTruth {
    std::uint32_t n = 0;
    std::uint32_t k = 0;
    std::vector<std::uint32_t> ids;  // n x k

    std::span<const std::uint32_t> row(std::uint32_t i) const { return {ids.data() + std::size_t(i) * k, k}; }
    // dataset.cpp:78-95: ids < base_n and no duplicate within a row (data_error otherwise)
    void validate_against(std::uint32_t base_n) const;
};

// dataset.hpp:15-24 error classes of the file readers
struct format_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct data_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// dataset.hpp:67-77 distances, computed on the device with the reference's
// sequential fp32 chain (bit-identical); ids past the set throw std::out_of_range.
float l2_sq(const float* a, const float* b, std::uint32_t dim);
float dist_sq(const VectorSet& vs, std::uint32_t a, std::uint32_t b);
float dist_sq_q(const VectorSet& vs, std::span<const float> q, std::uint32_t b);

// dataset.cpp:201-214 (same bytes as the reference's generator).
VectorSet gen_synthetic(std::uint32_t n, std::uint32_t dim, std::uint64_t seed);

// dataset.cpp:96-200 fvecs / ivecs: per record an int32 dimension then that
// many little-endian float32 / int32 values (annkit_io.cpp).
VectorSet load_fvecs(const std::string& path);
void save_fvecs(const VectorSet& vs, const std::string& path);
GroundTruth load_ivecs(const std::string& path);
void save_ivecs(const GroundTruth& gt, const std::string& path);

// ---------------------------------------------------------- kd_forest.hpp
struct KdNode {
    std::uint32_t split_dim = kLeafMarker;
    float split_val = 0.0f;
    std::uint32_t left = 0;   // internal: left child; leaf: first slot of its point_index range
    std::uint32_t right = 0;  // internal: right child; leaf: one past its last slot
    std::uint32_t depth = 0;
    bool even_split = false;

    bool is_leaf() const { return split_dim == kLeafMarker; }
};

struct KdTree {
    std::vector<KdNode> nodes;
    std::uint32_t root = 0;
    std::uint32_t leaf_cap = 0;
    std::uint32_t n = 0;
    std::uint32_t dim = 0;
    std::vector<std::uint32_t> point_index;
    std::uint32_t leaf_count = 0;

    std::span<const std::uint32_t> leaf_points(std::uint32_t node) const {
        return {point_index.data() + nodes[node].left, nodes[node].right - nodes[node].left};
    }
};

struct KdForest {
    std::vector<KdTree> trees;
    std::uint64_t seed = 0;
    std::uint32_t n = 0;
    std::uint32_t dim = 0;
    std::uint32_t leaf_cap = 0;
    mutable std::shared_ptr<DeviceForest> device;  // the device forest (built or imported)
};

KdForest build_forest(const VectorSet& vs, std::uint32_t n_trees, std::uint32_t leaf_cap, std::uint64_t seed,
                      std::uint32_t workers = 1);
std::vector<std::uint32_t> search_leaves(const KdTree& tree, std::span<const float> q, std::uint32_t n_leaves);
// kd_forest.cpp:307-372 AKF1 persistence (load validates every tree as kd_forest.cpp:175-241)
void save_forest(const KdForest& forest, const std::string& path);
KdForest load_forest(const std::string& path);
std::uint32_t descend_from(const KdTree& tree, std::span<const float> q, std::uint32_t node);

// ------------------------------------------------------ neighbor_pool.hpp
struct NeighborEntry {
    std::uint32_t id;
    float dist;
    bool flag_new;
    bool checked;
};

// Host view of one device pool (ascending (dist, id)).
class NeighborPool {
  public:
    NeighborPool() = default;
    explicit NeighborPool(std::uint32_t capacity) : capacity_(capacity) {}
    std::span<const NeighborEntry> entries() const { return entries_; }
    std::uint32_t size() const { return std::uint32_t(entries_.size()); }
    std::uint32_t capacity() const { return capacity_; }
    bool contains(std::uint32_t id) const {
        for (const auto& e : entries_)
            if (e.id == id) return true;
        return false;
    }
    // neighbor_pool.hpp:35-53 semantics for host-built pools (a caller's own
    // start state, uploaded on the next device call): the pool stays sorted by
    // (dist, id); a duplicate (same id and dist at the insertion slot) and
    // anything not better than a full pool's worst entry are rejected.
    bool insert(std::uint32_t id, float dist, bool flag_new) {
        const NeighborEntry e{id, dist, flag_new, false};
        auto less = [](const NeighborEntry& x, const NeighborEntry& y) {
            return x.dist != y.dist ? x.dist < y.dist : x.id < y.id;
        };
        const auto it = std::lower_bound(entries_.begin(), entries_.end(), e, less);
        const std::size_t pos = std::size_t(it - entries_.begin());
        if (it != entries_.end() && it->id == id && it->dist == dist) return false;
        if (pos >= capacity_) return false;
        entries_.insert(it, e);
        if (entries_.size() > capacity_) entries_.pop_back();
        return true;
    }
    std::span<NeighborEntry> entries() { return entries_; }
    std::vector<NeighborEntry>& mutable_entries() { return entries_; }

  private:
    std::vector<NeighborEntry> entries_;
    std::uint32_t capacity_ = 0;
};

// -------------------------------------------------------- knn_graph.hpp
struct KnnGraph {
    std::uint32_t n = 0;
    std::uint32_t k = 0;
    std::vector<std::uint32_t> ids;  // n x k, rows ascending by (dist, id)
    std::vector<float> dists;

    std::span<const std::uint32_t> row(std::uint32_t i) const { return {ids.data() + std::size_t(i) * k, k}; }
    std::span<const float> row_dists(std::uint32_t i) const { return {dists.data() + std::size_t(i) * k, k}; }
    bool has_dists() const { return !dists.empty(); }
};

// knn_graph.cpp:5-37: ids as ivecs, distances (optional) as a companion fvecs
void save_graph(const KnnGraph& graph, const std::string& ids_path,
                const std::optional<std::string>& dists_path = std::nullopt);
KnnGraph load_graph(const std::string& ids_path, const std::optional<std::string>& dists_path = std::nullopt);
// knn_graph.hpp:36-38: the id rows as ground truth and back (shape-preserving copies)
GroundTruth graph_to_ground_truth(const KnnGraph& g);
KnnGraph graph_from_ground_truth(const GroundTruth& gt);

// ------------------------------------------------------ graph_build.hpp
struct RefineState {
    std::uint32_t k = 0;
    std::uint32_t pool_cap = 0;
    std::uint32_t sample_cap = 0;
    std::uint64_t seed = 0;
    std::uint32_t iteration = 0;
    std::uint64_t dist_comps = 0;
    std::uint64_t last_changes = 0;  // accepted inserts of the last round, the reference's sequential count

    std::vector<NeighborPool> pools;
    std::vector<std::vector<std::uint32_t>> g_new, g_old, g_rnew, g_rold;
    std::shared_ptr<DeviceState> device;

    std::uint32_t n() const { return std::uint32_t(pools.size()); }
};

RefineState init_graph(const VectorSet& vs, const KdForest& forest, std::uint32_t k, std::uint32_t conquer_depth,
                       std::uint32_t pool_cap, std::uint32_t sample_cap, std::uint64_t seed,
                       std::uint32_t workers = 1);
RefineState init_random(const VectorSet& vs, std::uint32_t k, std::uint32_t pool_cap, std::uint32_t sample_cap,
                        std::uint64_t seed, std::uint32_t workers = 1);
void refine_nn_descent(RefineState& state, const VectorSet& vs, std::uint32_t max_iters, std::uint32_t workers = 1,
                       double min_change_rate = 0.001);
KnnGraph finalize(RefineState& state, const VectorSet& vs, std::uint32_t k);

enum class BuildStrategy { efanna, random_descent, nn_expansion, brute_force, init_only };
const char* to_string(BuildStrategy s);                  // graph_build.cpp:375-384
BuildStrategy strategy_from_string(const std::string& s);  // :386-393

struct BuildParams {
    std::uint32_t k = 10;
    std::uint32_t conquer_depth = 4;
    std::uint32_t pool_cap = 30;
    std::uint32_t sample_cap = 20;
    std::uint32_t max_iters = 8;
    BuildStrategy strategy = BuildStrategy::efanna;
    std::uint64_t seed = 1;
    std::uint32_t workers = 1;
    double min_change_rate = 0.001;
};

struct IterationLog {
    std::uint32_t iteration = 0;
    double seconds = 0.0;
    std::uint64_t dist_comps = 0;
    std::uint64_t changes = 0;
    double accuracy = -1.0;
};

struct BuildStats {
    double init_seconds = 0.0;
    double refine_seconds = 0.0;
    std::uint64_t dist_comps = 0;
    bool early_stopped = false;
    std::vector<IterationLog> iterations;

    double total_seconds() const { return init_seconds + refine_seconds; }
};

struct BuildResult {
    KnnGraph graph;
    BuildStats stats;
};

// Device strategies: efanna, random_descent, init_only, brute_force
// (all five strategies run on the device; nn_expansion / random_descent start
// from init_random, as graph_build.cpp:415-425).
BuildResult build_graph(const VectorSet& vs, const KdForest* forest, const BuildParams& params,
                        const GroundTruth* gt = nullptr);

namespace detail {
std::uint64_t nn_descent_iteration(RefineState& state, const VectorSet& vs, std::uint32_t workers);
std::uint64_t nn_expansion_iteration(RefineState& state, const VectorSet& vs, std::uint32_t workers);
void rebuild_sample_lists(RefineState& state);
void union_reverse_lists(RefineState& state);
double pool_topk_accuracy(const RefineState& state, const GroundTruth& gt);
}  // namespace detail

// ----------------------------------------------------------- search.hpp
struct SearchParams {
    std::uint32_t k_return = 10;
    std::uint32_t pool_size = 100;
    std::uint32_t expansion = 100;
    std::uint32_t iters = 4;
    std::uint32_t n_trees_used = 0;
    std::uint32_t random_seed_count = 0;
    std::uint64_t seed = 1;
};

struct SearchStats {
    std::uint64_t dist_comps = 0;
    std::uint32_t leaves_visited = 0;
    std::uint32_t graph_hops = 0;
    std::uint32_t seed_points = 0;
};

struct SearchResult {
    std::vector<std::uint32_t> ids;
    std::vector<float> dists;
    SearchStats stats;
};

struct DeviceSearcher;

// Keeps references to base / forest / graph like the reference (the caller
// keeps them alive); the device searcher holds its own graph copy.
class GraphSearcher {
  public:
    GraphSearcher(const VectorSet& base, const KdForest* forest, const KnnGraph& graph);
    SearchResult search(std::span<const float> q, const SearchParams& params);
    SearchResult search_random_init(std::span<const float> q, const SearchParams& params);
    // Batch form (the device path's natural shape): nq queries, row-major.
    std::vector<SearchResult> search_batch(const VectorSet& queries, const SearchParams& params,
                                           bool random_init = false);

  private:
    const VectorSet& base_;
    const KdForest* forest_;
    const KnnGraph& graph_;
    std::shared_ptr<DeviceSearcher> dev_;
};

struct SweepPoint {
    std::uint32_t expansion = 0;
    std::uint32_t pool_size = 0;
};

struct SweepRow {
    std::uint32_t expansion = 0;
    std::uint32_t pool_size = 0;
    double mean_time_us = 0.0;
    double avg_recall = 0.0;
    double avg_dist_comps = 0.0;
    double avg_seed_points = 0.0;
};

std::vector<SweepRow> recall_curve(const VectorSet& base, const KdForest* forest, const KnnGraph& graph,
                                   const VectorSet& queries, const GroundTruth& gt, std::span<const SweepPoint> sweep,
                                   const SearchParams& params, bool random_init = false, std::uint32_t workers = 1);

// ------------------------------------------------------------- eval.hpp
GroundTruth brute_force_knn(const VectorSet& base, const VectorSet* queries, std::uint32_t k,
                            std::uint32_t workers = 1, std::uint64_t* dist_comps = nullptr);
KnnGraph brute_force_graph(const VectorSet& base, std::uint32_t k, std::uint32_t workers = 1,
                           std::uint64_t* dist_comps = nullptr);
double recall(std::span<const std::uint32_t> result_ids, std::span<const std::uint32_t> gt_row);
double graph_accuracy(const KnnGraph& graph, const GroundTruth& gt);
struct EvalReport {  // eval.hpp
    std::string metric;
    double value = 0.0;
    double seconds = 0.0;
    std::vector<double> breakdown;  // per row
};
EvalReport graph_accuracy_report(const KnnGraph& graph, const GroundTruth& gt);  // eval.cpp:106-123
std::vector<std::pair<std::uint32_t, double>> accuracy_vs_k(const KnnGraph& graph, const VectorSet& vs,
                                                            std::span<const std::uint32_t> k_list,
                                                            std::uint32_t workers = 1);

}  // namespace annkit
