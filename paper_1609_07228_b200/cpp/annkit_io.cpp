// annkit_io.cpp — the reference's on-disk formats for the C++ host API
// (SURVEY §8(f) row 1): fvecs / ivecs datasets (dataset.cpp:96-200), AKF1
// forests (kd_forest.cpp:307-372, validated like kd_forest.cpp:175-241) and
// graphs as ivecs + companion fvecs (knn_graph.cpp:5-37).  Host byte layout
// only; arrays reach the device through the facade's handles.  Same layouts
// and checks as paper_1609_07228_b200/formats.py.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <fstream>
#include <iterator>

#include "annkit_b200.hpp"

namespace annkit {

namespace {

constexpr char kMagic[4] = {'A', 'K', 'F', '1'};
constexpr std::uint32_t kVersion = 1;

std::vector<unsigned char> read_file(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw format_error("cannot open file for reading: " + path);
    return std::vector<unsigned char>(std::istreambuf_iterator<char>(in), std::istreambuf_iterator<char>());
}

std::ofstream open_binary(const std::string& path) {
    std::ofstream out(path, std::ios::binary | std::ios::trunc);
    if (!out) throw std::runtime_error("cannot open file for writing: " + path);
    return out;
}

template <class T>
void put(std::ofstream& out, const T& v) {
    out.write(reinterpret_cast<const char*>(&v), sizeof(T));
}

// Records of one int32 dimension followed by `dim` 4-byte values: returns
// (n, dim, payload words row-major).  A record cut short reports the byte at
// which its first missing value starts (dataset.cpp:96-133 reports offsets).
void read_records(const std::string& path, std::uint32_t& n, std::uint32_t& dim, std::vector<std::uint32_t>& body) {
    const std::vector<unsigned char> raw = read_file(path);
    const std::size_t words = raw.size() / 4;  // whole 4-byte values present
    auto word = [&](std::size_t i) {
        std::int32_t v;
        std::memcpy(&v, raw.data() + 4 * i, 4);
        return v;
    };
    n = dim = 0;
    body.clear();
    std::size_t at = 0;  // word offset of the current record
    for (std::uint32_t rec = 0;; ++rec) {
        if (at == words) {
            if (raw.size() % 4)
                throw format_error("truncated record " + std::to_string(rec) + " at byte " +
                                   std::to_string(4 * at) + " in " + path);
            break;
        }
        const std::int32_t d = word(at);
        if (d < 1)
            throw format_error("record " + std::to_string(rec) + " at byte " + std::to_string(4 * at) +
                               " declares dimension " + std::to_string(d) + " in " + path);
        if (rec == 0) dim = std::uint32_t(d);
        if (std::uint32_t(d) != dim)
            throw format_error("record " + std::to_string(rec) + " has dimension " + std::to_string(d) +
                               ", expected " + std::to_string(dim) + " in " + path);
        if (at + 1 + dim > words)  // the first value that is not all there
            throw format_error("truncated record " + std::to_string(rec) + " at byte " +
                               std::to_string(4 * words) + " in " + path);
        body.insert(body.end(), reinterpret_cast<const std::uint32_t*>(raw.data() + 4 * (at + 1)),
                    reinterpret_cast<const std::uint32_t*>(raw.data() + 4 * (at + 1 + dim)));
        at += 1 + dim;
        n = rec + 1;
    }
}

}  // namespace

VectorSet load_fvecs(const std::string& path) {
    VectorSet vs;
    std::vector<std::uint32_t> body;
    read_records(path, vs.n, vs.dim, body);
    vs.data.resize(body.size());
    std::memcpy(vs.data.data(), body.data(), body.size() * 4);
    for (std::size_t t = 0; t < vs.data.size(); ++t)
        if (!std::isfinite(vs.data[t]))
            throw data_error("non-finite value in record " + std::to_string(t / vs.dim) + " component " +
                             std::to_string(t % vs.dim) + " in " + path);
    return vs;
}

void save_fvecs(const VectorSet& vs, const std::string& path) {
    auto out = open_binary(path);
    const std::int32_t d = std::int32_t(vs.dim);
    for (std::uint32_t i = 0; i < vs.n; ++i) {
        put(out, d);
        out.write(reinterpret_cast<const char*>(vs.row_ptr(i)), std::streamsize(vs.dim) * 4);
    }
    if (!out) throw std::runtime_error("write failed: " + path);
}

GroundTruth load_ivecs(const std::string& path) {
    GroundTruth gt;
    read_records(path, gt.n, gt.k, gt.ids);
    for (std::size_t t = 0; t < gt.ids.size(); ++t)
        if (gt.ids[t] > 0x7fffffffu)
            throw data_error("negative id in record " + std::to_string(t / gt.k) + " component " +
                             std::to_string(t % gt.k) + " in " + path);
    return gt;
}

void save_ivecs(const GroundTruth& gt, const std::string& path) {
    for (const auto id : gt.ids)
        if (id > 0x7fffffffu) throw data_error("id " + std::to_string(id) + " does not fit an int32 payload");
    auto out = open_binary(path);
    const std::int32_t k = std::int32_t(gt.k);
    for (std::uint32_t i = 0; i < gt.n; ++i) {
        put(out, k);
        out.write(reinterpret_cast<const char*>(gt.ids.data() + std::size_t(i) * gt.k), std::streamsize(gt.k) * 4);
    }
    if (!out) throw std::runtime_error("write failed: " + path);
}

// dataset.cpp:78-95 contract: every id < base_n and no id twice in a row
// (data_error naming the row otherwise).
void GroundTruth::validate_against(std::uint32_t base_n) const {
    std::vector<std::uint32_t> sorted;
    for (std::uint32_t i = 0; i < n; ++i) {
        const auto r = row(i);
        const auto bad = std::find_if(r.begin(), r.end(), [&](std::uint32_t id) { return id >= base_n; });
        if (bad != r.end())
            throw data_error("row " + std::to_string(i) + " holds id " + std::to_string(*bad) +
                             " outside base set of size " + std::to_string(base_n));
        sorted.assign(r.begin(), r.end());
        std::sort(sorted.begin(), sorted.end());
        const auto dup = std::adjacent_find(sorted.begin(), sorted.end());
        if (dup != sorted.end())
            throw data_error("row " + std::to_string(i) + " holds duplicate id " + std::to_string(*dup));
    }
}

// ------------------------------------------------------------------ graph

void save_graph(const KnnGraph& graph, const std::string& ids_path, const std::optional<std::string>& dists_path) {
    GroundTruth g;
    g.n = graph.n;
    g.k = graph.k;
    g.ids = graph.ids;
    save_ivecs(g, ids_path);
    if (dists_path) {
        if (!graph.has_dists()) throw std::invalid_argument("save_graph: graph has no distances");
        VectorSet d;
        d.n = graph.n;
        d.dim = graph.k;
        d.data = graph.dists;
        save_fvecs(d, *dists_path);
    }
}

KnnGraph load_graph(const std::string& ids_path, const std::optional<std::string>& dists_path) {
    GroundTruth g = load_ivecs(ids_path);
    KnnGraph out;
    out.n = g.n;
    out.k = g.k;
    out.ids = std::move(g.ids);
    if (dists_path) {
        VectorSet d = load_fvecs(*dists_path);
        if (d.n != out.n || d.dim != out.k)
            throw format_error("distance file " + *dists_path + " has shape " + std::to_string(d.n) + "x" +
                               std::to_string(d.dim) + ", graph is " + std::to_string(out.n) + "x" + std::to_string(out.k));
        out.dists = std::move(d.data);
    }
    return out;
}

// ----------------------------------------------------------------- forest

void save_forest(const KdForest& forest, const std::string& path) {
    auto out = open_binary(path);
    out.write(kMagic, 4);
    put(out, kVersion);
    put(out, forest.n);
    put(out, forest.dim);
    put(out, std::uint32_t(forest.trees.size()));
    put(out, forest.leaf_cap);
    put(out, forest.seed);
    for (const KdTree& t : forest.trees) {
        put(out, std::uint32_t(t.nodes.size()));
        put(out, t.root);
        for (const KdNode& nd : t.nodes) {  // packed 21-byte node
            put(out, nd.split_dim);
            put(out, nd.split_val);
            put(out, nd.left);
            put(out, nd.right);
            put(out, nd.depth);
            put(out, std::uint8_t(nd.even_split ? 1 : 0));
        }
        out.write(reinterpret_cast<const char*>(t.point_index.data()), std::streamsize(t.point_index.size()) * 4);
    }
    if (!out) throw std::runtime_error("write failed: " + path);
}

namespace {

// kd_forest.cpp:175-241 validate_tree: same conditions and error class.
void validate_tree(const KdTree& t, std::uint32_t n, std::uint32_t dim, std::uint32_t leaf_cap) {
    const std::uint32_t m = std::uint32_t(t.nodes.size());
    if (m == 0 || t.root >= m) throw format_error("forest file: bad tree root");
    if (t.point_index.size() != n) throw format_error("forest file: point_index size mismatch");
    std::vector<std::uint8_t> seen(n, 0);
    for (const auto p : t.point_index) {
        if (p >= n) throw format_error("forest file: point id out of range");
        if (seen[p]++) throw format_error("forest file: point_index is not a permutation");
    }
    if (t.nodes[t.root].depth != 0) throw format_error("forest file: root depth not 0");
    std::uint32_t max_depth = 16;
    for (std::uint32_t mm = n; mm > 1; mm /= 2) max_depth += 4;
    std::vector<std::uint32_t> refs(m, 0);
    for (const KdNode& nd : t.nodes) {
        if (nd.is_leaf()) continue;
        if (nd.left >= m || nd.right >= m) throw format_error("forest file: child id out of range");
        ++refs[nd.left];
        ++refs[nd.right];
    }
    for (std::uint32_t i = 0; i < m; ++i) {
        const std::uint32_t expect = i == t.root ? 0 : 1;
        if (refs[i] > expect) throw format_error("forest file: malformed tree topology");
    }
    for (std::uint32_t i = 0; i < m; ++i) {
        const std::uint32_t expect = i == t.root ? 0 : 1;
        if (refs[i] < expect) throw format_error("forest file: unreachable nodes present");
    }
    for (const KdNode& nd : t.nodes)
        if (nd.depth > max_depth) throw format_error("forest file: implausible tree depth");
    for (const KdNode& nd : t.nodes)
        if (!nd.is_leaf() && nd.split_dim >= dim) throw format_error("forest file: split dimension out of range");
    for (const KdNode& nd : t.nodes)
        if (!nd.is_leaf() && (t.nodes[nd.left].depth != nd.depth + 1 || t.nodes[nd.right].depth != nd.depth + 1))
            throw format_error("forest file: child depth mismatch");
    for (const KdNode& nd : t.nodes)
        if (nd.is_leaf() && (nd.left >= nd.right || nd.right > n || nd.right - nd.left > leaf_cap))
            throw format_error("forest file: leaf range violates 1..leaf_cap");
    // ranges bottom-up: a left subtree's range must end where its sibling's begins
    std::vector<std::int64_t> lo(m, -1), hi(m, -1);
    std::vector<std::uint32_t> order(m);
    for (std::uint32_t i = 0; i < m; ++i) order[i] = i;
    std::stable_sort(order.begin(), order.end(),
                     [&](std::uint32_t a, std::uint32_t b) { return t.nodes[a].depth > t.nodes[b].depth; });
    for (const std::uint32_t i : order) {
        const KdNode& nd = t.nodes[i];
        if (nd.is_leaf()) {
            lo[i] = nd.left;
            hi[i] = nd.right;
            continue;
        }
        if (hi[nd.left] != lo[nd.right]) throw format_error("forest file: left subtree does not precede right subtree");
        lo[i] = lo[nd.left];
        hi[i] = hi[nd.right];
    }
    if (lo[t.root] != 0 || hi[t.root] != std::int64_t(n)) throw format_error("forest file: leaf ranges do not cover all points");
}

}  // namespace

KdForest load_forest(const std::string& path) {
    const std::vector<unsigned char> blob = read_file(path);
    std::size_t off = 0;
    auto take = [&](void* dst, std::size_t bytes) {
        if (off + bytes > blob.size()) throw format_error("unexpected end of file in " + path);
        std::memcpy(dst, blob.data() + off, bytes);
        off += bytes;
    };
    char magic[4];
    take(magic, 4);
    if (std::memcmp(magic, kMagic, 4) != 0) throw format_error("not a forest file: " + path);
    std::uint32_t hdr[5];
    take(hdr, sizeof(hdr));
    if (hdr[0] != kVersion) throw format_error("unsupported forest version in " + path);
    KdForest f;
    f.n = hdr[1];
    f.dim = hdr[2];
    const std::uint32_t n_trees = hdr[3];
    f.leaf_cap = hdr[4];
    take(&f.seed, 8);
    if (f.n < 1 || f.dim < 1 || n_trees < 1 || f.leaf_cap < 1) throw format_error("forest file: degenerate header in " + path);
    f.trees.resize(n_trees);
    for (KdTree& t : f.trees) {
        std::uint32_t count, root;
        take(&count, 4);
        take(&root, 4);
        if (count == 0 || count > 2 * f.n) throw format_error("forest file: implausible node count in " + path);
        t.nodes.resize(count);
        std::uint32_t leaves = 0;
        for (KdNode& nd : t.nodes) {
            std::uint8_t even;
            take(&nd.split_dim, 4);
            take(&nd.split_val, 4);
            take(&nd.left, 4);
            take(&nd.right, 4);
            take(&nd.depth, 4);
            take(&even, 1);
            nd.even_split = even != 0;
            leaves += nd.is_leaf();
        }
        t.point_index.resize(f.n);
        take(t.point_index.data(), std::size_t(f.n) * 4);
        t.root = root;
        t.leaf_cap = f.leaf_cap;
        t.n = f.n;
        t.dim = f.dim;
        t.leaf_count = leaves;
        validate_tree(t, f.n, f.dim, f.leaf_cap);
    }
    if (off != blob.size()) throw format_error("forest file: trailing bytes in " + path);
    return f;
}

// ------------------------------------------------------- names and scoring

const char* to_string(BuildStrategy s) {
    switch (s) {
        case BuildStrategy::efanna: return "efanna";
        case BuildStrategy::random_descent: return "random-descent";
        case BuildStrategy::nn_expansion: return "nn-expansion";
        case BuildStrategy::brute_force: return "brute-force";
        case BuildStrategy::init_only: return "init-only";
    }
    return "unknown";
}

BuildStrategy strategy_from_string(const std::string& s) {
    if (s == "efanna") return BuildStrategy::efanna;
    if (s == "random-descent") return BuildStrategy::random_descent;
    if (s == "nn-expansion") return BuildStrategy::nn_expansion;
    if (s == "brute-force") return BuildStrategy::brute_force;
    if (s == "init-only") return BuildStrategy::init_only;
    throw std::invalid_argument("unknown build strategy: " + s);
}

EvalReport graph_accuracy_report(const KnnGraph& graph, const GroundTruth& gt) {
    if (graph.n != gt.n || graph.k != gt.k) throw std::invalid_argument("graph_accuracy: graph and truth shapes differ");
    if (graph.n == 0) throw std::invalid_argument("graph_accuracy: empty graph");
    const auto t0 = std::chrono::steady_clock::now();
    EvalReport r;
    r.metric = "graph_accuracy";
    r.breakdown.resize(graph.n);
    double sum = 0.0;
    for (std::uint32_t i = 0; i < graph.n; ++i) {
        r.breakdown[i] = recall(graph.row(i), gt.row(i));
        sum += r.breakdown[i];
    }
    r.value = sum / graph.n;
    r.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return r;
}

}  // namespace annkit
