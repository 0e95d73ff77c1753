"""`annkit` — the command line of the B200 framework.

It offers the reference CLI's six subcommands with the same flags and
defaults, the same artifacts (fvecs / ivecs / AKF1 bytes) and the same CSV and
stdout lines, so scripts written for `annkit` keep working:

    convert      --in FILE | --synthetic N:DIM:SEED, --out, --limit
    build-trees  --base, --trees 8, --leaf-cap 10, --seed (required), --workers, --out
    gt           --base, --queries, --k 10, --out, --out-dists, --workers
    build-graph  --base, --forest, --gt, --k 10, --dep 4, --pool 30, --sample 20,
                 --iters 8, --min-change-rate 0.001, --strategy efanna, --seed, --workers,
                 --out, --out-dists, --log
    search       --base, --queries, --forest, --graph, --gt, --k 10, --iters 4,
                 --trees-used 0, --seed-count 0, --random-init, --workers, --seed,
                 --sweep E:P[,E:P...], --out, --csv, --per-query
    eval         --graph | --results | --k-list (with --base), --gt, --workers, --csv

Options may also come from `--config FILE` (key = value lines; flags on the
command line win).  Every computation runs on the GPU through the package API;
`--workers` is accepted for compatibility and ignored.  Exit status: 0, 1 on a
runtime error ("error: ..."), 2 on a usage error.  Search timings are the
batch's device time divided evenly over its queries (the device searches a
whole batch at once).
"""
from __future__ import annotations

import os
import sys
import time
from dataclasses import dataclass, field
from typing import Callable, Dict, List, Optional

import numpy as np


class UsageError(Exception):
    """Bad command line: exit status 2."""


# ---------------------------------------------------------------- options

@dataclass
class Opt:
    name: str
    kind: type = str          # str / int / float / bool (flag)
    default: object = None
    required: bool = False
    help: str = ""


@dataclass
class Command:
    name: str
    summary: str
    opts: List[Opt]
    run: Callable = None
    by_name: Dict[str, Opt] = field(default_factory=dict)

    def __post_init__(self):
        self.by_name = {o.name: o for o in self.opts}


def _convert(kind, text, flag):
    if kind is int:
        try:
            v = int(text, 10)
        except ValueError:
            raise UsageError(f"{flag}: expected an integer, got '{text}'")
        if v < 0:
            raise UsageError(f"{flag}: expected a non-negative integer, got '{text}'")
        return v
    if kind is float:
        try:
            return float(text)
        except ValueError:
            raise UsageError(f"{flag}: expected a number, got '{text}'")
    return text


def _read_config(path):
    try:
        lines = open(path).read().splitlines()
    except OSError:
        raise UsageError(f"--config: cannot read {path}")
    out = {}
    for ln in lines:
        ln = ln.split("#", 1)[0].split(";", 1)[0].strip()
        if not ln or ln.startswith("["):
            continue
        if "=" not in ln:
            raise UsageError(f"--config: expected key = value, got '{ln}'")
        k, v = (t.strip() for t in ln.split("=", 1))
        out[k.lstrip("-")] = v.strip('"')
    return out


def parse(cmd: Command, argv: List[str]) -> dict:
    given, config = {}, None
    i = 0
    while i < len(argv):
        a = argv[i]
        if a == "--config":
            if i + 1 >= len(argv):
                raise UsageError("--config needs a file")
            config = argv[i + 1]
            i += 2
            continue
        key, val = (a[2:].split("=", 1) + [None])[:2] if a.startswith("--") else (None, None)
        if key not in cmd.by_name:
            raise UsageError(f"{cmd.name}: unknown option {a}")
        o = cmd.by_name[key]
        if o.kind is bool:
            given[key] = True
            i += 1
            continue
        if val is None:
            if i + 1 >= len(argv):
                raise UsageError(f"--{key} needs a value")
            val = argv[i + 1]
            i += 1
        given[key] = _convert(o.kind, val, "--" + key)
        i += 1
    values = {}
    file_vals = _read_config(config) if config else {}
    for o in cmd.opts:
        if o.name in given:
            values[o.name] = given[o.name]
        elif o.name in file_vals:
            raw = file_vals[o.name]
            values[o.name] = raw.lower() in ("1", "true", "yes", "on") if o.kind is bool else \
                _convert(o.kind, raw, "--" + o.name)
        elif o.required:
            raise UsageError(f"--{o.name} is required")
        else:
            values[o.name] = o.default if o.kind is not bool else bool(o.default)
    return values


# ----------------------------------------------------------------- output

def g(x, p=10):
    """An ostream with setprecision(p) printing a double."""
    return f"{x:.{p}g}"


def header(command: str, echo: List[tuple]) -> str:
    """Every CSV starts with the resolved configuration (self-describing runs)."""
    return "".join([f"# annkit {command}\n"] + [f"# {k}={v}\n" for k, v in echo])


def write_text(path: str, text: str):
    try:
        with open(path, "w") as fh:
            fh.write(text)
    except OSError:
        raise RuntimeError(f"cannot open output file: {path}")


def cxx_fixed(x: float) -> str:
    """std::to_string(double)."""
    return "%f" % x


# ----------------------------------------------------------- subcommands

def _lib():
    from . import api, formats
    return api, formats


def run_convert(v):
    api, fm = _lib()
    if bool(v["in"]) == bool(v["synthetic"]):
        raise UsageError("convert needs exactly one of --in / --synthetic")
    limit = v["limit"]
    if v["synthetic"]:
        parts = v["synthetic"].split(":")
        if len(parts) != 3 or not all(p.isdigit() for p in parts):
            raise UsageError("--synthetic expects N:DIM:SEED")
        n, dim, seed = (int(p) for p in parts)
        x = api.gen_synthetic(n, dim, seed)
        if limit and limit < n:
            x = x[:limit]
        fm.save_fvecs(x, v["out"])
        print(f"wrote {x.shape[0]}x{dim} vectors to {v['out']}")
    elif v["in"].endswith(".ivecs"):
        ids = fm.load_ivecs(v["in"])
        if limit and limit < ids.shape[0]:
            ids = ids[:limit]
        fm.save_ivecs(ids, v["out"])
        print(f"wrote {ids.shape[0]}x{ids.shape[1] if ids.ndim == 2 else 0} id rows to {v['out']}")
    else:
        x = fm.load_fvecs(v["in"])
        if limit and limit < x.shape[0]:
            x = x[:limit]
        fm.save_fvecs(x, v["out"])
        print(f"wrote {x.shape[0]}x{x.shape[1] if x.ndim == 2 else 0} vectors to {v['out']}")


def _sync():
    from ._lib import lib
    lib.annk_synchronize()


def run_build_trees(v):
    api, fm = _lib()
    base = fm.load_dataset(v["base"])
    _sync()
    t0 = time.perf_counter()
    forest = api.build_forest(base, v["trees"], v["leaf-cap"], v["seed"])
    _sync()
    secs = time.perf_counter() - t0
    fm.save_forest(forest, v["out"])
    print(f"tree build: n={base.n} dim={base.dim} trees={v['trees']} leaf_cap={v['leaf-cap']} seed={v['seed']}")
    print(f"tree build time: {g(secs, 6)} s")
    print(f"forest written to {v['out']}")


def run_gt(v):
    api, fm = _lib()
    base = fm.load_dataset(v["base"])
    queries = fm.load_dataset(v["queries"]) if v["queries"] else None
    if v["out-dists"] and queries is not None:
        raise UsageError("--out-dists is only available in self mode")
    _sync()
    t0 = time.perf_counter()
    comps = []
    if v["out-dists"]:
        g_ = api.brute_force_graph(base, v["k"], dist_comps=comps)
        fm.save_graph(g_, v["out"], v["out-dists"])
    else:
        ids = api.brute_force_knn(base, queries, v["k"], dist_comps=comps)
        fm.save_ivecs(ids, v["out"])
    secs = time.perf_counter() - t0
    print(f"ground truth: k={v['k']} mode={'query' if queries is not None else 'self'} dist_comps={comps[0]}")
    print(f"oracle time: {g(secs, 6)} s")
    print(f"ground truth written to {v['out']}")


def run_build_graph(v):
    api, fm = _lib()
    # every input is read and checked on the host before anything reaches the device
    x = fm.load_fvecs(v["base"])
    n, dim = x.shape
    parts = None
    if v["forest"]:
        parts = fm.parse_forest(v["forest"])
        if parts[0] != n or parts[1] != dim:
            raise RuntimeError(f"forest {v['forest']} was built over {parts[0]}x{parts[1]} vectors, "
                               f"the base set is {n}x{dim}")
    gt = None
    if v["gt"]:
        t = fm.load_ivecs(v["gt"])
        fm.validate_truth(t, n)
        if t.shape[0] != n or t.shape[1] < v["k"]:
            raise RuntimeError(f"ground truth {v['gt']} ({t.shape[0]}x{t.shape[1]}) cannot score a "
                               f"{n}-point graph of width {v['k']}")
        gt = np.ascontiguousarray(t[:, :v["k"]])
    base = api.VectorSet(x)
    forest = api.KdForest.from_trees(*parts) if parts else None
    strategies = ("efanna", "random-descent", "nn-expansion", "brute-force", "init-only")
    if v["strategy"] not in strategies:
        raise RuntimeError(f"unknown strategy '{v['strategy']}' (expected one of {', '.join(strategies)})")
    params = api.BuildParams(k=v["k"], conquer_depth=v["dep"], pool_cap=v["pool"], sample_cap=v["sample"],
                             max_iters=v["iters"], strategy=v["strategy"], seed=v["seed"], workers=v["workers"],
                             min_change_rate=v["min-change-rate"])
    res = api.build_graph(base, forest, params, gt)
    fm.save_graph(res.graph, v["out"], v["out-dists"] or None)
    echo = [("base", v["base"]), ("forest", v["forest"] or ""), ("strategy", v["strategy"]), ("k", v["k"]),
            ("conquer_depth", v["dep"]), ("pool_cap", v["pool"]), ("sample_cap", v["sample"]),
            ("max_iters", v["iters"]), ("min_change_rate", cxx_fixed(v["min-change-rate"])), ("seed", v["seed"]),
            ("workers", v["workers"]), ("n", base.n), ("dim", base.dim)]
    rows = [f"{r.iteration},{g(r.seconds)},{r.dist_comps},{r.changes},{g(r.accuracy) if r.accuracy >= 0 else ''}"
            for r in res.stats.iterations]
    csv = header("build-graph", echo) + "iteration,seconds,dist_comps,changes,accuracy\n" + \
        "".join(r + "\n" for r in rows)
    if v["log"]:
        write_text(v["log"], csv)
    st = res.stats
    sys.stdout.write(csv)
    print(f"graph build time: {g(st.total_seconds(), 6)} s (init {g(st.init_seconds, 6)} s, refine "
          f"{g(st.refine_seconds, 6)} s), dist_comps={st.dist_comps}{', early-stopped' if st.early_stopped else ''}")
    print(f"graph written to {v['out']}")


def _sweep(text):
    pts = []
    for part in text.split(","):
        e, sep, p = part.partition(":")
        if not sep or not e.strip().isdigit() or not p.strip().isdigit():
            raise UsageError("--sweep expects E:P[,E:P...]")
        pts.append((int(e), int(p)))
    if not pts:
        raise UsageError("--sweep expects E:P[,E:P...]")
    return pts


def run_search(v):
    api, fm = _lib()
    x = fm.load_fvecs(v["base"])
    q = fm.load_fvecs(v["queries"])
    if q.shape[0] == 0:
        raise RuntimeError(f"query set {v['queries']} is empty")
    if q.shape[1] != x.shape[1]:
        raise RuntimeError(f"queries have dimension {q.shape[1]}, the base set {x.shape[1]}")
    parts = fm.parse_forest(v["forest"]) if v["forest"] else None
    if not v["random-init"] and parts is None:
        raise UsageError("tree-seeded search needs --forest (or pass --random-init)")
    graph = fm.load_graph(v["graph"])
    kr = v["k"]
    gt = None
    if v["gt"]:
        t = fm.load_ivecs(v["gt"])
        fm.validate_truth(t, x.shape[0])
        if t.shape[0] != q.shape[0] or t.shape[1] < kr:
            raise RuntimeError(f"ground truth {v['gt']} ({t.shape[0]}x{t.shape[1]}) cannot score "
                               f"{q.shape[0]} queries at k_return {kr}")
        gt = t[:, :kr]
    sweep = _sweep(v["sweep"])
    base = api.VectorSet(x)
    forest = api.KdForest.from_trees(*parts) if parts else None
    nq = q.shape[0]
    echo = [("base", v["base"]), ("queries", v["queries"]), ("forest", v["forest"] or ""), ("graph", v["graph"]),
            ("k_return", kr), ("iters", v["iters"]), ("n_trees_used", v["trees-used"]),
            ("random_init", 1 if v["random-init"] else 0), ("seed", v["seed"]), ("workers", v["workers"]),
            ("sweep", v["sweep"]), ("n", base.n), ("dim", base.dim), ("n_queries", nq)]
    searcher = api.GraphSearcher(base, forest, graph)
    qs = api.VectorSet(q)
    lines, per_query, last = [], [], None
    for E, P in sweep:
        p = api.SearchParams(k_return=kr, pool_size=P, expansion=E, iters=v["iters"],
                             n_trees_used=v["trees-used"], random_seed_count=v["seed-count"], seed=v["seed"])
        _sync()
        t0 = time.perf_counter()
        r = searcher.search_batch(qs, p, random_init=v["random-init"])
        us = (time.perf_counter() - t0) * 1e6 / nq
        comps = r.stats[:, 0].astype(np.float64)
        seeds = r.stats[:, 3].astype(np.float64)
        rec = [api.recall(r.ids[i], gt[i]) for i in range(nq)] if gt is not None else None
        # the reference sums per-query values in query order (tools/main.cpp's loop)
        sum_c = sum_s = sum_r = 0.0
        for i in range(nq):
            sum_c += comps[i]
            sum_s += seeds[i]
            if rec is not None:
                sum_r += rec[i]
        lines.append(f"{E},{P},{g(us)},{g(sum_c / nq)},{g(sum_s / nq)},{g(sum_r / nq) if rec is not None else ''}")
        last = (r, us, rec)
    r, us, rec = last
    for i in range(nq):
        per_query.append(f"{i},{g(us)},{int(r.stats[i, 0])},{g(rec[i]) if rec is not None else ''}")
    sweep_csv = header("search", echo) + \
        "expansion,pool_size,mean_time_us,avg_dist_comps,avg_seed_points,avg_recall\n" + \
        "".join(x + "\n" for x in lines)
    if v["out"]:
        fm.save_graph(api.KnnGraph(r.ids, r.dists), v["out"])
    if v["csv"]:
        write_text(v["csv"], sweep_csv)
    if v["per-query"]:
        write_text(v["per-query"], header("search (per query, last sweep point)", echo) +
                   "query,time_us,dist_comps,recall\n" + "".join(x + "\n" for x in per_query))
    sys.stdout.write(sweep_csv)
    if v["out"]:
        print(f"results written to {v['out']}")


def run_eval(v):
    api, fm = _lib()
    if v["k-list"]:
        if not v["graph"] or not v["base"]:
            raise UsageError("--k-list needs --graph and --base")
        graph = fm.load_graph(v["graph"])
        base = fm.load_dataset(v["base"])
        try:
            ks = [int(t) for t in v["k-list"].split(",")]
        except ValueError:
            raise UsageError("--k-list expects comma-separated integers")
        table = api.accuracy_vs_k(graph, base, ks)
        body = "k,accuracy\n" + "".join(f"{kk},{g(a)}\n" for kk, a in table)
        csv = header("eval (accuracy vs k)", [("graph", v["graph"]), ("base", v["base"]),
                                              ("k_list", v["k-list"])]) + body
    elif v["graph"]:
        if not v["gt"]:
            raise UsageError("graph accuracy needs --gt")
        graph = fm.load_graph(v["graph"])
        t = fm.load_ivecs(v["gt"])
        t = t[:, :graph.ids.shape[1]] if t.shape[1] > graph.ids.shape[1] else t
        acc = api.graph_accuracy(graph, t)
        csv = header("eval (graph accuracy)", [("graph", v["graph"]), ("gt", v["gt"])]) + \
            f"metric,value\ngraph_accuracy,{g(acc)}\n"
    elif v["results"]:
        if not v["gt"]:
            raise UsageError("recall needs --gt")
        res = fm.load_ivecs(v["results"])
        t = fm.load_ivecs(v["gt"])
        if t.shape[0] != res.shape[0] or t.shape[1] < res.shape[1]:
            raise RuntimeError(f"ground truth {v['gt']} does not cover the results {v['results']}")
        total = 0.0
        for i in range(res.shape[0]):
            total += api.recall(res[i], t[i, :res.shape[1]])
        csv = header("eval (search recall)", [("results", v["results"]), ("gt", v["gt"])]) + \
            f"metric,value\navg_recall,{g(total / res.shape[0])}\n"
    else:
        raise UsageError("eval needs --graph, --results, or --k-list")
    if v["csv"]:
        write_text(v["csv"], csv)
    sys.stdout.write(csv)


COMMANDS = [
    Command("convert", "generate or copy fvecs/ivecs datasets", [
        Opt("in"), Opt("synthetic"), Opt("out", required=True), Opt("limit", int, 0)], run_convert),
    Command("build-trees", "build the randomized KD-tree forest", [
        Opt("base", required=True), Opt("trees", int, 8), Opt("leaf-cap", int, 10), Opt("seed", int, required=True),
        Opt("workers", int, 1), Opt("out", required=True)], run_build_trees),
    Command("gt", "brute-force ground truth (self mode by default)", [
        Opt("base", required=True), Opt("queries"), Opt("k", int, 10), Opt("out", required=True),
        Opt("out-dists"), Opt("workers", int, 1)], run_gt),
    Command("build-graph", "build the approximate kNN graph", [
        Opt("base", required=True), Opt("forest"), Opt("gt"), Opt("k", int, 10), Opt("dep", int, 4),
        Opt("pool", int, 30), Opt("sample", int, 20), Opt("iters", int, 8), Opt("min-change-rate", float, 0.001),
        Opt("strategy", str, "efanna"), Opt("seed", int, required=True), Opt("workers", int, 1),
        Opt("out", required=True), Opt("out-dists"), Opt("log")], run_build_graph),
    Command("search", "batch ANN search over a sweep of (E,P)", [
        Opt("base", required=True), Opt("queries", required=True), Opt("forest"), Opt("graph", required=True),
        Opt("gt"), Opt("k", int, 10), Opt("iters", int, 4), Opt("trees-used", int, 0), Opt("seed-count", int, 0),
        Opt("random-init", bool, False), Opt("workers", int, 1), Opt("seed", int, required=True),
        Opt("sweep", required=True), Opt("out"), Opt("csv"), Opt("per-query")], run_search),
    Command("eval", "recall / graph accuracy from saved artifacts", [
        Opt("graph"), Opt("results"), Opt("gt"), Opt("base"), Opt("k-list"), Opt("workers", int, 1),
        Opt("csv")], run_eval),
]


def usage() -> str:
    lines = ["annkit: in-memory approximate nearest neighbor toolkit (B200)", "", "subcommands:"]
    lines += [f"  {c.name:12s} {c.summary}" for c in COMMANDS]
    return "\n".join(lines) + "\n"


def main(argv: Optional[List[str]] = None) -> int:
    argv = sys.argv[1:] if argv is None else argv
    if argv and argv[0] in ("-h", "--help"):
        sys.stdout.write(usage())
        return 0
    if not argv:
        sys.stderr.write(usage() + "a subcommand is required\n")
        return 2
    cmd = next((c for c in COMMANDS if c.name == argv[0]), None)
    if cmd is None:
        sys.stderr.write(f"unknown subcommand '{argv[0]}'\n" + usage())
        return 2
    if any(a in ("-h", "--help") for a in argv[1:]):
        sys.stdout.write(f"annkit {cmd.name}: {cmd.summary}\n" +
                         "".join(f"  --{o.name}{' (required)' if o.required else ''}\n" for o in cmd.opts))
        return 0
    try:
        values = parse(cmd, argv[1:])
        cmd.run(values)
    except UsageError as e:
        sys.stderr.write(f"{e}\n")
        return 2
    except Exception as e:  # noqa: BLE001 - reported like the reference CLI
        sys.stderr.write(f"error: {e}\n")
        return 1
    return 0


if __name__ == "__main__":
    sys.exit(main())
