// annkit_cli.cpp — the `annkit` command line over the B200 host API
// (SURVEY §8(f) row 2).  Same subcommands, flags, defaults, artifacts and CSV
// layout as the reference CLI (proj/tools/main.cpp:399-493): convert,
// build-trees, gt, build-graph, search, eval.  Every artifact (AKF1 forest,
// ivecs/fvecs ground truth, graph, search results) is byte-identical to the
// reference's for the same inputs and seeds; CSV rows are identical except the
// timing columns.  Differences: `--workers` is accepted and ignored (the
// device decides the parallelism), search runs each sweep point as one device
// batch, so `time_us` / `mean_time_us` are the batch wall time divided by the
// query count, and `--config` files are not supported.
#include <chrono>
#include <cstdlib>
#include <fstream>
#include <functional>
#include <iomanip>
#include <iostream>
#include <map>
#include <optional>
#include <sstream>
#include <string>
#include <vector>

#include "annkit_b200.hpp"

namespace {

using namespace annkit;

struct UsageError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

using ConfigEcho = std::vector<std::pair<std::string, std::string>>;

double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// Every CSV starts with the resolved configuration (main.cpp:30-34 layout).
void write_header(std::ostream& out, const std::string& command, const ConfigEcho& config) {
    out << "# annkit " << command << "\n";
    for (const auto& [key, value] : config) out << "# " << key << "=" << value << "\n";
}

std::ofstream open_out(const std::string& path) {
    std::ofstream out(path);
    if (!out) throw std::runtime_error("cannot open output file: " + path);
    out << std::setprecision(10);
    return out;
}

// ---------------------------------------------------------------- options

struct Option {
    std::function<void(const std::string&)> set;
    bool flag = false, required = false, seen = false;
};

template <class T>
std::function<void(const std::string&)> num(T& dst, const std::string& name) {
    return [&dst, name](const std::string& v) {
        std::istringstream in(v);
        T x{};
        if (!(in >> x) || !in.eof()) throw UsageError(name + ": invalid value '" + v + "'");
        dst = x;
    };
}
std::function<void(const std::string&)> str(std::string& dst) {
    return [&dst](const std::string& v) { dst = v; };
}

void parse(const std::string& cmd, std::map<std::string, Option>& opts, int argc, char** argv) {
    for (int i = 2; i < argc; ++i) {
        std::string a = argv[i], val;
        bool has_val = false;
        if (const auto eq = a.find('='); a.rfind("--", 0) == 0 && eq != std::string::npos) {
            val = a.substr(eq + 1);
            a = a.substr(0, eq);
            has_val = true;
        }
        auto it = opts.find(a);
        if (it == opts.end()) throw UsageError(cmd + ": unknown option " + a);
        Option& o = it->second;
        if (o.flag) {
            if (has_val) throw UsageError(a + " takes no value");
            o.set("1");
        } else {
            if (!has_val) {
                if (i + 1 >= argc) throw UsageError(a + " needs a value");
                val = argv[++i];
            }
            o.set(val);
        }
        o.seen = true;
    }
    for (const auto& [name, o] : opts)
        if (o.required && !o.seen) throw UsageError(cmd + ": " + name + " is required");
}

std::vector<SweepPoint> parse_sweep(const std::string& s) {
    std::vector<SweepPoint> sweep;
    std::istringstream in(s);
    std::string part;
    while (std::getline(in, part, ',')) {
        SweepPoint p;
        char c = 0;
        std::istringstream pin(part);
        if (!(pin >> p.expansion >> c >> p.pool_size) || c != ':') throw UsageError("--sweep expects E:P[,E:P...]");
        sweep.push_back(p);
    }
    if (sweep.empty()) throw UsageError("--sweep expects E:P[,E:P...]");
    return sweep;
}

GroundTruth slice_k(const GroundTruth& gt, std::uint32_t k) {
    GroundTruth cut;
    cut.n = gt.n;
    cut.k = k;
    cut.ids.reserve(std::size_t(gt.n) * k);
    for (std::uint32_t i = 0; i < gt.n; ++i) {
        const auto row = gt.row(i);
        cut.ids.insert(cut.ids.end(), row.begin(), row.begin() + k);
    }
    return cut;
}

void truncate(VectorSet& vs, std::uint32_t limit) {
    if (limit && limit < vs.n) {
        vs.n = limit;
        vs.data.resize(std::size_t(limit) * vs.dim);
    }
}

// ------------------------------------------------------------ subcommands

int cmd_convert(int argc, char** argv) {
    std::string in_path, synthetic, out_path;
    std::uint32_t limit = 0;
    std::map<std::string, Option> o{{"--in", {str(in_path)}},
                                    {"--synthetic", {str(synthetic)}},
                                    {"--out", {str(out_path), false, true}},
                                    {"--limit", {num(limit, "--limit")}}};
    parse("convert", o, argc, argv);
    if (in_path.empty() == synthetic.empty()) throw UsageError("convert needs exactly one of --in / --synthetic");
    if (!synthetic.empty()) {
        std::uint32_t n = 0, dim = 0;
        std::uint64_t seed = 0;
        char c1 = 0, c2 = 0;
        std::istringstream in(synthetic);
        if (!(in >> n >> c1 >> dim >> c2 >> seed) || c1 != ':' || c2 != ':')
            throw UsageError("--synthetic expects N:DIM:SEED");
        VectorSet vs = gen_synthetic(n, dim, seed);
        truncate(vs, limit);
        save_fvecs(vs, out_path);
        std::cout << "wrote " << vs.n << "x" << vs.dim << " vectors to " << out_path << "\n";
        return 0;
    }
    if (in_path.size() >= 6 && in_path.compare(in_path.size() - 6, 6, ".ivecs") == 0) {
        GroundTruth gt = load_ivecs(in_path);
        if (limit && limit < gt.n) {
            gt.n = limit;
            gt.ids.resize(std::size_t(limit) * gt.k);
        }
        save_ivecs(gt, out_path);
        std::cout << "wrote " << gt.n << "x" << gt.k << " id rows to " << out_path << "\n";
    } else {
        VectorSet vs = load_fvecs(in_path);
        truncate(vs, limit);
        save_fvecs(vs, out_path);
        std::cout << "wrote " << vs.n << "x" << vs.dim << " vectors to " << out_path << "\n";
    }
    return 0;
}

int cmd_build_trees(int argc, char** argv) {
    std::string base_path, out_path;
    std::uint32_t trees = 8, leaf_cap = 10, workers = 1;
    std::uint64_t seed = 1;
    std::map<std::string, Option> o{{"--base", {str(base_path), false, true}},
                                    {"--trees", {num(trees, "--trees")}},
                                    {"--leaf-cap", {num(leaf_cap, "--leaf-cap")}},
                                    {"--seed", {num(seed, "--seed"), false, true}},
                                    {"--workers", {num(workers, "--workers")}},
                                    {"--out", {str(out_path), false, true}}};
    parse("build-trees", o, argc, argv);
    const VectorSet base = load_fvecs(base_path);
    const double t0 = now_s();
    const KdForest forest = build_forest(base, trees, leaf_cap, seed, workers);
    const double seconds = now_s() - t0;
    save_forest(forest, out_path);
    std::cout << "tree build: n=" << base.n << " dim=" << base.dim << " trees=" << trees << " leaf_cap=" << leaf_cap
              << " seed=" << seed << "\n";
    std::cout << "tree build time: " << std::setprecision(6) << seconds << " s\n";
    std::cout << "forest written to " << out_path << "\n";
    return 0;
}

int cmd_gt(int argc, char** argv) {
    std::string base_path, queries_path, out_path, dists_path;
    std::uint32_t k = 10, workers = 1;
    std::map<std::string, Option> o{{"--base", {str(base_path), false, true}},
                                    {"--queries", {str(queries_path)}},
                                    {"--k", {num(k, "--k")}},
                                    {"--out", {str(out_path), false, true}},
                                    {"--out-dists", {str(dists_path)}},
                                    {"--workers", {num(workers, "--workers")}}};
    parse("gt", o, argc, argv);
    const VectorSet base = load_fvecs(base_path);
    std::optional<VectorSet> queries;
    if (!queries_path.empty()) queries = load_fvecs(queries_path);
    const double t0 = now_s();
    std::uint64_t comps = 0;
    if (dists_path.empty()) {
        save_ivecs(brute_force_knn(base, queries ? &*queries : nullptr, k, workers, &comps), out_path);
    } else if (!queries) {
        save_graph(brute_force_graph(base, k, workers, &comps), out_path, dists_path);
    } else {
        throw UsageError("--out-dists is only available in self mode");
    }
    std::cout << "ground truth: k=" << k << " mode=" << (queries ? "query" : "self") << " dist_comps=" << comps << "\n";
    std::cout << "oracle time: " << std::setprecision(6) << now_s() - t0 << " s\n";
    std::cout << "ground truth written to " << out_path << "\n";
    return 0;
}

int cmd_build_graph(int argc, char** argv) {
    std::string base_path, forest_path, gt_path, out_path, dists_path, log_path, strategy = "efanna";
    BuildParams p;
    std::map<std::string, Option> o{{"--base", {str(base_path), false, true}},
                                    {"--forest", {str(forest_path)}},
                                    {"--gt", {str(gt_path)}},
                                    {"--k", {num(p.k, "--k")}},
                                    {"--dep", {num(p.conquer_depth, "--dep")}},
                                    {"--pool", {num(p.pool_cap, "--pool")}},
                                    {"--sample", {num(p.sample_cap, "--sample")}},
                                    {"--iters", {num(p.max_iters, "--iters")}},
                                    {"--min-change-rate", {num(p.min_change_rate, "--min-change-rate")}},
                                    {"--strategy", {str(strategy)}},
                                    {"--seed", {num(p.seed, "--seed"), false, true}},
                                    {"--workers", {num(p.workers, "--workers")}},
                                    {"--out", {str(out_path), false, true}},
                                    {"--out-dists", {str(dists_path)}},
                                    {"--log", {str(log_path)}}};
    parse("build-graph", o, argc, argv);
    p.strategy = strategy_from_string(strategy);
    const VectorSet base = load_fvecs(base_path);
    std::optional<KdForest> forest;
    if (!forest_path.empty()) {
        forest = load_forest(forest_path);
        if (forest->n != base.n || forest->dim != base.dim) throw std::runtime_error("forest file does not match the base set");
    }
    std::optional<GroundTruth> gt;
    if (!gt_path.empty()) {
        gt = load_ivecs(gt_path);
        gt->validate_against(base.n);
        if (gt->n != base.n || gt->k < p.k) throw std::runtime_error("ground truth shape does not cover the build");
        if (gt->k > p.k) gt = slice_k(*gt, p.k);
    }
    const BuildResult result = build_graph(base, forest ? &*forest : nullptr, p, gt ? &*gt : nullptr);
    save_graph(result.graph, out_path, dists_path.empty() ? std::nullopt : std::optional<std::string>(dists_path));
    const ConfigEcho echo = {
        {"base", base_path},
        {"forest", forest_path},
        {"strategy", to_string(p.strategy)},
        {"k", std::to_string(p.k)},
        {"conquer_depth", std::to_string(p.conquer_depth)},
        {"pool_cap", std::to_string(p.pool_cap)},
        {"sample_cap", std::to_string(p.sample_cap)},
        {"max_iters", std::to_string(p.max_iters)},
        {"min_change_rate", std::to_string(p.min_change_rate)},
        {"seed", std::to_string(p.seed)},
        {"workers", std::to_string(p.workers)},
        {"n", std::to_string(base.n)},
        {"dim", std::to_string(base.dim)},
    };
    std::ostringstream csv;
    csv << std::setprecision(10);
    write_header(csv, "build-graph", echo);
    csv << "iteration,seconds,dist_comps,changes,accuracy\n";
    for (const auto& row : result.stats.iterations) {
        csv << row.iteration << "," << row.seconds << "," << row.dist_comps << "," << row.changes << ",";
        if (row.accuracy >= 0.0) csv << row.accuracy;
        csv << "\n";
    }
    if (!log_path.empty()) open_out(log_path) << csv.str();
    std::cout << csv.str();
    std::cout << "graph build time: " << std::setprecision(6) << result.stats.total_seconds() << " s (init "
              << result.stats.init_seconds << " s, refine " << result.stats.refine_seconds
              << " s), dist_comps=" << result.stats.dist_comps << (result.stats.early_stopped ? ", early-stopped" : "")
              << "\n";
    std::cout << "graph written to " << out_path << "\n";
    return 0;
}

int cmd_search(int argc, char** argv) {
    std::string base_path, queries_path, forest_path, graph_path, gt_path, sweep_str, out_path, csv_path, pq_path,
        random_flag;
    SearchParams params;
    std::uint32_t workers = 1;
    std::map<std::string, Option> o{{"--base", {str(base_path), false, true}},
                                    {"--queries", {str(queries_path), false, true}},
                                    {"--forest", {str(forest_path)}},
                                    {"--graph", {str(graph_path), false, true}},
                                    {"--gt", {str(gt_path)}},
                                    {"--k", {num(params.k_return, "--k")}},
                                    {"--iters", {num(params.iters, "--iters")}},
                                    {"--trees-used", {num(params.n_trees_used, "--trees-used")}},
                                    {"--seed-count", {num(params.random_seed_count, "--seed-count")}},
                                    {"--random-init", {str(random_flag), true}},
                                    {"--workers", {num(workers, "--workers")}},
                                    {"--seed", {num(params.seed, "--seed"), false, true}},
                                    {"--sweep", {str(sweep_str), false, true}},
                                    {"--out", {str(out_path)}},
                                    {"--csv", {str(csv_path)}},
                                    {"--per-query", {str(pq_path)}}};
    parse("search", o, argc, argv);
    const bool random_init = !random_flag.empty();
    const VectorSet base = load_fvecs(base_path);
    const VectorSet queries = load_fvecs(queries_path);
    if (queries.n == 0) throw std::runtime_error("empty query set");
    if (queries.dim != base.dim) throw std::runtime_error("query dim does not match base");
    std::optional<KdForest> forest;
    if (!forest_path.empty()) forest = load_forest(forest_path);
    if (!random_init && !forest) throw UsageError("tree-seeded search needs --forest (or pass --random-init)");
    const KnnGraph graph = load_graph(graph_path);
    std::optional<GroundTruth> gt;
    if (!gt_path.empty()) {
        gt = load_ivecs(gt_path);
        gt->validate_against(base.n);
        if (gt->n != queries.n || gt->k < params.k_return)
            throw std::runtime_error("ground truth does not cover the queries at k_return");
    }
    const std::vector<SweepPoint> sweep = parse_sweep(sweep_str);
    const ConfigEcho echo = {
        {"base", base_path},
        {"queries", queries_path},
        {"forest", forest_path},
        {"graph", graph_path},
        {"k_return", std::to_string(params.k_return)},
        {"iters", std::to_string(params.iters)},
        {"n_trees_used", std::to_string(params.n_trees_used)},
        {"random_init", random_init ? "1" : "0"},
        {"seed", std::to_string(params.seed)},
        {"workers", std::to_string(workers)},
        {"sweep", sweep_str},
        {"n", std::to_string(base.n)},
        {"dim", std::to_string(base.dim)},
        {"n_queries", std::to_string(queries.n)},
    };
    std::ostringstream sweep_csv, pq_csv;
    sweep_csv << std::setprecision(10);
    pq_csv << std::setprecision(10);
    write_header(sweep_csv, "search", echo);
    sweep_csv << "expansion,pool_size,mean_time_us,avg_dist_comps,avg_seed_points,avg_recall\n";
    write_header(pq_csv, "search (per query, last sweep point)", echo);
    pq_csv << "query,time_us,dist_comps,recall\n";

    GroundTruth results;  // last sweep point's ids, one row per query
    GraphSearcher searcher(base, forest ? &*forest : nullptr, graph);
    for (std::size_t si = 0; si < sweep.size(); ++si) {
        SearchParams p = params;
        p.expansion = sweep[si].expansion;
        p.pool_size = sweep[si].pool_size;
        const bool last = si + 1 == sweep.size();
        // per-query seed substream(seed, qi) as the reference CLI (main.cpp:291-292)
        const double t0 = now_s();
        const std::vector<SearchResult> rs = searcher.search_batch(queries, p, random_init);
        const double per_query_us = (now_s() - t0) * 1e6 / queries.n;
        if (last) {
            results.n = queries.n;
            results.k = params.k_return;
            results.ids.assign(std::size_t(queries.n) * params.k_return, 0);
        }
        double sum_recall = 0.0, sum_comps = 0.0, sum_seeds = 0.0, sum_time = 0.0;
        for (std::uint32_t qi = 0; qi < queries.n; ++qi) {
            const SearchResult& r = rs[qi];
            const double rec = gt ? recall(r.ids, gt->row(qi).subspan(0, params.k_return)) : -1.0;
            sum_time += per_query_us;
            sum_comps += double(r.stats.dist_comps);
            sum_seeds += double(r.stats.seed_points);
            if (gt) sum_recall += rec;
            if (last) {
                std::copy(r.ids.begin(), r.ids.end(), results.ids.begin() + std::size_t(qi) * params.k_return);
                pq_csv << qi << "," << per_query_us << "," << r.stats.dist_comps << ",";
                if (gt) pq_csv << rec;
                pq_csv << "\n";
            }
        }
        sweep_csv << p.expansion << "," << p.pool_size << "," << sum_time / queries.n << "," << sum_comps / queries.n
                  << "," << sum_seeds / queries.n << ",";
        if (gt) sweep_csv << sum_recall / queries.n;
        sweep_csv << "\n";
    }
    if (!out_path.empty()) save_ivecs(results, out_path);
    if (!csv_path.empty()) open_out(csv_path) << sweep_csv.str();
    if (!pq_path.empty()) open_out(pq_path) << pq_csv.str();
    std::cout << sweep_csv.str();
    if (!out_path.empty()) std::cout << "results written to " << out_path << "\n";
    return 0;
}

int cmd_eval(int argc, char** argv) {
    std::string graph_path, results_path, gt_path, base_path, k_list_str, csv_path;
    std::uint32_t workers = 1;
    std::map<std::string, Option> o{{"--graph", {str(graph_path)}},   {"--results", {str(results_path)}},
                                    {"--gt", {str(gt_path)}},         {"--base", {str(base_path)}},
                                    {"--k-list", {str(k_list_str)}},  {"--workers", {num(workers, "--workers")}},
                                    {"--csv", {str(csv_path)}}};
    parse("eval", o, argc, argv);
    std::ostringstream csv;
    csv << std::setprecision(10);
    if (!k_list_str.empty()) {
        if (graph_path.empty() || base_path.empty()) throw UsageError("--k-list needs --graph and --base");
        const KnnGraph graph = load_graph(graph_path);
        const VectorSet base = load_fvecs(base_path);
        std::vector<std::uint32_t> k_list;
        std::istringstream in(k_list_str);
        std::string part;
        while (std::getline(in, part, ',')) k_list.push_back(std::uint32_t(std::stoul(part)));
        const auto table = accuracy_vs_k(graph, base, k_list, workers);
        write_header(csv, "eval (accuracy vs k)", {{"graph", graph_path}, {"base", base_path}, {"k_list", k_list_str}});
        csv << "k,accuracy\n";
        for (const auto& [k, acc] : table) csv << k << "," << acc << "\n";
    } else if (!graph_path.empty()) {
        if (gt_path.empty()) throw UsageError("graph accuracy needs --gt");
        const KnnGraph graph = load_graph(graph_path);
        GroundTruth gt = load_ivecs(gt_path);
        if (gt.k > graph.k) gt = slice_k(gt, graph.k);
        const EvalReport report = graph_accuracy_report(graph, gt);
        write_header(csv, "eval (graph accuracy)", {{"graph", graph_path}, {"gt", gt_path}});
        csv << "metric,value\n";
        csv << report.metric << "," << report.value << "\n";
    } else if (!results_path.empty()) {
        if (gt_path.empty()) throw UsageError("recall needs --gt");
        const GroundTruth results = load_ivecs(results_path);
        const GroundTruth gt = load_ivecs(gt_path);
        if (gt.n != results.n || gt.k < results.k) throw std::runtime_error("ground truth does not cover the results");
        double sum = 0.0;
        for (std::uint32_t i = 0; i < results.n; ++i) sum += recall(results.row(i), gt.row(i).subspan(0, results.k));
        write_header(csv, "eval (search recall)", {{"results", results_path}, {"gt", gt_path}});
        csv << "metric,value\n";
        csv << "avg_recall," << sum / results.n << "\n";
    } else {
        throw UsageError("eval needs --graph, --results, or --k-list");
    }
    if (!csv_path.empty()) open_out(csv_path) << csv.str();
    std::cout << csv.str();
    return 0;
}

const char* kUsage =
    "annkit (B200) - in-memory approximate nearest neighbor toolkit\n"
    "usage: annkit <convert|build-trees|gt|build-graph|search|eval> [--option value ...]\n";

}  // namespace

int main(int argc, char** argv) {
    const std::map<std::string, int (*)(int, char**)> cmds = {
        {"convert", cmd_convert}, {"build-trees", cmd_build_trees}, {"gt", cmd_gt},
        {"build-graph", cmd_build_graph}, {"search", cmd_search}, {"eval", cmd_eval}};
    if (argc < 2 || std::string(argv[1]) == "--help" || std::string(argv[1]) == "-h") {
        std::cout << kUsage;
        return argc < 2 ? 2 : 0;
    }
    const auto it = cmds.find(argv[1]);
    if (it == cmds.end()) {
        std::cerr << "error: unknown subcommand " << argv[1] << "\n" << kUsage;
        return 2;
    }
    try {
        return it->second(argc, argv);
    } catch (const UsageError& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 2;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    }
}
