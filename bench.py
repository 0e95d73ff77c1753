#!/usr/bin/env python
"""bench.py — EFANNA hot paths on B200 vs the reference CPU library.

Headline metric (BASELINE.json): "kNN-graph build s at graph acc 0.9; search
queries/s at recall@100 0.9", on configs[1] (cfg2): 1M x 128 integer-valued
Gaussian mixture (1000 centers), 8 trees leaf 8, K=100, P(L)=100, S=20,
10k queries, search top-100.

  value      = seconds for one kNN-graph build up to the first NN-descent
               iteration whose graph accuracy >= 0.9 (init + refine, the
               reference's own StopWatch boundary, graph_build.cpp:421-450; the
               forest is built once beforehand, as `annkit build-trees` does).
               Inputs resident in HBM; dataset 512 MB > L2 (126 MB).
  e2e        = the same build through the C-ABI from pinned host memory, at
               the same boundary: H2D of the dataset and of the prebuilt forest
               (host arrays, as build_graph receives its forest) + init + refine
               + finalize + D2H of the graph (ids + dists), every step.
               `e2e_with_forest_build` also builds the forest on the device
               inside the timed region.
  search_qps = queries/s of the batched search at the smallest swept pool
               size reaching recall@100 >= 0.9 (secondary line item).

Accuracy is scored on a seeded 10,000-point sample against exact top-100 rows
(untimed, as the reference's accuracy hook is not charged to build time).

--impl reference runs the unmodified reference library (oracle/_ref, built
from /root/reference by oracle/Makefile) on all host cores on a bounded sample:
the same build (init + the same number of NN-descent iterations) on the first
`ref_points` points of the same dataset (inputs from oracle/'s byte-identical
generator: that process never loads the product library); ms_per_step is the
measured sample time, `value` extrapolates it to N with the exponent fitted
between two nested prefixes.  The GPU arm's `cpu_baseline` runs the same
reference timing plus the reference searcher at the chosen sweep point and
brute_force_knn on 1000 sampled rows, and checks the GPU results against them.

--gpus N (N > 1) relaunches itself under torchrun, one rank per GPU.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # configs[1] of BASELINE.json: the headline workload
    "cfg2": dict(n=1_000_000, dim=128, n_queries=10_000, centers=1000, trees=8, leaf=8, k=100, P=100, S=20,
                 max_iters=10, dep=4, k_return=100, sweep=[100, 200, 300, 400, 500, 600, 800, 1000],
                 acc_sample=10_000, ref_points=131_072, ref_queries=500),
    # configs[0]: the reference's own CPU-runnable case (R=50 is not expressible: reverse cap = S)
    "cfg1": dict(n=100_000, dim=128, n_queries=1000, centers=100, trees=4, leaf=10, k=10, P=30, S=10,
                 max_iters=8, dep=4, k_return=10, sweep=[50, 100, 200], acc_sample=10_000, ref_points=100_000,
                 ref_queries=1000),
    # configs[2]: 960-d float data in [0,1] (GIST-like; the exact fp32 datapath, leaf 10 assumed)
    "cfg3": dict(n=1_000_000, dim=960, n_queries=1000, centers=500, trees=8, leaf=10, k=100, P=100, S=20,
                 max_iters=10, dep=4, k_return=100, sweep=[100, 200, 400, 800], acc_sample=2000, ref_points=16_384,
                 ref_queries=100, mix=(0.05, 0.35, 0.05, 0.0, 1.0, False)),
    # configs[4]: the 8-GPU scaling case (8M points, 4000 centers, 80k queries; cfg2 build parameters
    # assumed), runnable on one GPU too; its cfg4-style exact graph (6.4e13 pairs) is not run
    "cfg5": dict(n=8_000_000, dim=128, n_queries=80_000, centers=4000, trees=8, leaf=8, k=100, P=100, S=20,
                 max_iters=10, dep=4, k_return=100, sweep=[100, 200, 400, 800], acc_sample=10_000,
                 ref_points=131_072, ref_queries=500, skip_exact=True),
    # a small smoke-sized case for quick checks
    "tiny": dict(n=50_000, dim=128, n_queries=1000, centers=100, trees=4, leaf=8, k=20, P=40, S=10,
                 max_iters=6, dep=4, k_return=20, sweep=[40, 80, 160], acc_sample=2000, ref_points=50_000,
                 ref_queries=200),
}
SEED = 1
_T0 = time.time()


def _log(msg):
    """Progress marker on stderr (stdout carries only the JSON line)."""
    print(f"[bench +{time.time() - _T0:.1f}s] {msg}", file=sys.stderr, flush=True)


def gen_data(cfg, n=None, lib=None):
    """The config's base and query sets.  `lib` is the generator: the product's
    annk_gen_mixture (GPU arm) or its byte-identical restatement under oracle/
    (reference arm: that process must not load the product library)."""
    if lib is None:
        import paper_1609_07228_b200 as A
        lib = A
    n = cfg["n"] if n is None else n
    lo, hi, sd, clo, chi, rnd = cfg.get("mix", (0.0, 128.0, 16.0, 0.0, 255.0, True))
    base = lib.gen_mixture(n, cfg["dim"], cfg["centers"], lo, hi, sd, clo, chi, rnd, SEED, 1)
    queries = lib.gen_mixture(cfg["n_queries"], cfg["dim"], cfg["centers"], lo, hi, sd, clo, chi, rnd, SEED, 2)
    return base, queries


def sample_rows(n, m, seed=SEED):
    rng = np.random.default_rng(seed)
    return np.sort(rng.choice(n, size=min(m, n), replace=False)).astype(np.uint32)


# ------------------------------------------------------------------ clocks

class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap,utilization.gpu")

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        util = [float(r[6]) for r in self.rows if r[6].replace(".", "").isdigit()]
        loaded = [s for s, u in zip(sm, util) if u > 0] or sm
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ------------------------------------------------------------- distributed

def dist_setup(args):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch
        import torch.distributed as dist
        backend = "nccl" if args.impl != "reference" and torch.cuda.is_available() and args.comm == "nccl" else "gloo"
        if torch.cuda.is_available() and args.impl != "reference":
            local = local % torch.cuda.device_count()  # --comm gloo may stack ranks on one GPU (functional runs)
            torch.cuda.set_device(local)
        dist.init_process_group(backend=backend)
    return ws, rank, local


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(ws, v: float) -> float:
    if ws == 1:
        return v
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([v], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# --------------------------------------------------------- reference arm

def cpu_reference_build(ref, x, cfg, iters, cores):
    """Reference library (oracle/_ref) build on the rows x: build_forest, then
    build_graph (init_graph + `iters` NN-descent iterations, all host cores).
    Returns the reference's own StopWatch seconds (init + refine)."""
    vs = ref.vs(x)
    forest = ref.build_forest(vs, cfg["trees"], cfg["leaf"], SEED, workers=cores)
    _, _, _, summ = ref.build_graph(vs, forest, k=cfg["k"], conquer_depth=cfg["dep"], pool_cap=cfg["P"],
                                    sample_cap=cfg["S"], max_iters=iters, strategy=0, seed=SEED, workers=cores,
                                    min_change_rate=0.0)
    return float(summ[0] + summ[1])


def ref_samples(cfg):
    """Two nested prefixes of the config's base set for the reference timing:
    the build time of the larger one is extrapolated to N with the exponent
    fitted between the two (per-point work grows with N: deeper trees, larger
    working sets), not linearly."""
    m2 = min(cfg["n"], cfg["ref_points"])
    return max(2048, m2 // 2), m2


def fit_exponent(t1, m1, t2, m2):
    import math
    if m2 <= m1 or t1 <= 0 or t2 <= 0:
        return 1.0
    return max(1.0, math.log(t2 / t1) / math.log(m2 / m1))


def run_reference(args, cfg, ws, rank):
    """--impl reference: the unmodified reference library compiled from
    /root/reference (oracle/_ref) on this box's host cores.  This process never
    loads the product library (inputs come from oracle/'s generator)."""
    if rank != 0:
        return
    from oracle import oracle as O
    if not O.reference_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libannkit_ref.so not built"}))
        return
    ref, gen = O.load("reference"), O.load("oracle")
    cores = os.cpu_count() or 1
    iters = cfg["ref_iters"]
    m1, m2 = ref_samples(cfg)
    base, _ = gen_data(cfg, n=m2, lib=gen)
    # exponent fit (untimed, counts as warm-up)
    t1 = cpu_reference_build(ref, base[:m1], cfg, iters, cores)
    t2 = cpu_reference_build(ref, base, cfg, iters, cores)
    alpha = fit_exponent(t1, m1, t2, m2)
    for _ in range(max(0, args.warmup - 2)):
        cpu_reference_build(ref, base, cfg, iters, cores)
    times = []
    w0 = time.perf_counter()
    for _ in range(args.steps):
        times.append(cpu_reference_build(ref, base, cfg, iters, cores))
    wall = (time.perf_counter() - w0) / max(1, args.steps)
    t = statistics.mean(times)
    factor = (cfg["n"] / m2) ** alpha
    v = t * factor
    sample = (f"reference build_graph (init + {iters} NN-descent iterations, the crossing of accuracy 0.9; "
              f"{cfg['trees']} trees leaf {cfg['leaf']}) on the first {m2} of {cfg['n']} points, {cores} workers, "
              f"{t:.3f} s measured per step, extrapolated x{factor:.2f} = (N/{m2})^{alpha:.3f}, the exponent "
              f"fitted from {m1} ({t1:.3f} s) and {m2} ({t2:.3f} s) points")
    line = {"metric": METRIC, "value": v, "unit": "s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t * 1e3, "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic", "impl": "reference",
            "config": {"workload": args.config, "n": cfg["n"], "dim": cfg["dim"], "trees": cfg["trees"],
                       "leaf_cap": cfg["leaf"], "k": cfg["k"], "pool_cap": cfg["P"], "sample_cap": cfg["S"],
                       "iterations_to_acc_0.9": iters, "measured_points": m2,
                       "extrapolation": {"exponent": alpha, "factor": factor, "fit_points": [m1, m2],
                                         "fit_seconds": [t1, t2]}},
            "host_wall_s_per_step": wall,
            "cpu_baseline": {"value": v, "unit": "s", "cores": cores, "kind": "reference", "sample": sample},
            "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    try:  # evidence: this arm ran the reference library only
        with open("/proc/self/maps") as fh:
            maps = fh.read()
        line["libraries"] = sorted({ln.split()[-1].split("/")[-1] for ln in maps.splitlines()
                                    if "annkit" in ln or "oracle" in ln})
    except OSError:
        pass
    print(json.dumps(line))


METRIC = "kNN-graph build s at graph acc 0.9; search queries/s at recall@100 0.9"


# ---------------------------------------------------------------- GPU arm

_PINNED_OUT = {}
REF_ITERS = 4  # SearchParams::iters default (search.hpp:17), fixed across recall_curve's sweep


def pinned_forest(A, forest):
    """The device forest exported once to pinned host arrays in annk_forest_import's layout."""
    import torch
    trees = forest.trees
    tdt = {np.uint32: torch.int32, np.float32: torch.float32, np.uint8: torch.uint8}
    tot = sum(len(t.split_dim) for t in trees)
    shapes = {"split_dim": (tot, np.uint32), "split_val": (tot, np.float32), "left": (tot, np.uint32),
              "right": (tot, np.uint32), "depth": (tot, np.uint32), "even": (tot, np.uint8),
              "point_index": (len(trees) * forest.n, np.uint32)}
    out = {key: torch.empty(m, dtype=tdt[dt], pin_memory=True).numpy().view(dt) for key, (m, dt) in shapes.items()}
    return A.KdForest.pack_trees(trees, out=out)


def measured_hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"])
    except Exception:
        return 6650.0


def ncu_traffic(config, kernel):
    """DRAM bytes per launch of `kernel` from the committed ncu --set full capture (or None)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            tr = json.load(fh).get(config, {}).get(kernel)
            return tr["dram_bytes_per_launch"] if tr else None
    except Exception:
        return None


def timed_search(searcher, qs, p, ev, reps=3):
    """One warm call, then the median of `reps` timed calls of the whole batch
    through the public API (upload-free: queries are a resident VectorSet;
    results land in pinned host buffers, D2H inside the timed region)."""
    import torch
    key = (qs.n, p.k_return)
    if key not in _PINNED_OUT:
        _PINNED_OUT[key] = (torch.empty(key, dtype=torch.int32, pin_memory=True).numpy().view(np.uint32),
                            torch.empty(key, dtype=torch.float32, pin_memory=True).numpy(),
                            torch.empty((qs.n, 4), dtype=torch.int64, pin_memory=True).numpy().view(np.uint64))
    out = _PINNED_OUT[key]
    r = searcher.search_batch(qs, p, out=out)
    ts = []
    for _ in range(reps):
        e0 = ev()
        r = searcher.search_batch(qs, p, out=out)
        e1 = ev()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3)
    return r, statistics.median(ts)


def cpu_baseline_leg(args, cfg, A, base, queries, crossing, graph, gpu_search, chosen, exact_sample, rows):
    """The reference library on the box's host cores (rank 0, N=1), with the
    same inputs as the GPU arm, and the GPU results checked against it:
      build  - build_graph on two nested prefixes of the base set, extrapolated
               to N with the fitted exponent; the GPU pools on the smaller prefix
               are compared with the reference's after init and every round;
      search - the reference's batched GraphSearcher::search (search.cpp:182-236)
               over all queries at the chosen sweep point, with the GPU-built
               graph and the reference's own forest (bit-identical to the GPU's);
      exact  - brute_force_knn on 1000 sampled base rows (rows are independent,
               so the time scales exactly linearly to N rows)."""
    from oracle import oracle as O
    if not O.reference_available():
        return None
    ref = O.load("reference")
    cores = os.cpu_count() or 1
    n, k = cfg["n"], cfg["k"]
    out = {"unit": "s", "cores": cores, "kind": "reference"}
    # build: exponent fit on two prefixes
    m1, m2 = ref_samples(cfg)
    t1 = cpu_reference_build(ref, base[:m1], cfg, crossing, cores)
    t2 = cpu_reference_build(ref, base[:m2], cfg, crossing, cores)
    alpha = fit_exponent(t1, m1, t2, m2)
    factor = (n / m2) ** alpha
    out["value"] = t2 * factor
    out["sample"] = (f"reference build_graph (init + {crossing} iterations) on the first {m2} of {n} points, {cores} "
                     f"workers, {t2:.3f} s measured, extrapolated x{factor:.2f} = (N/{m2})^{alpha:.3f}, the exponent "
                     f"fitted from {m1} ({t1:.3f} s) and {m2} points")
    out["extrapolation"] = {"exponent": alpha, "factor": factor, "fit_points": [m1, m2], "fit_seconds": [t1, t2]}
    # build parity on the m1 prefix: pools, flags and dist_comps after init and each round
    _log("cpu baseline: build parity")
    xs = np.ascontiguousarray(base[:m1])
    vo = ref.vs(xs)
    so = ref.init_graph(vo, ref.build_forest(vo, cfg["trees"], cfg["leaf"], SEED, workers=cores), k, cfg["dep"],
                        cfg["P"], cfg["S"], SEED, workers=cores)
    vd = A.VectorSet(xs)
    sd = A.init_graph(vd, A.build_forest(vd, cfg["trees"], cfg["leaf"], SEED), k, cfg["dep"], cfg["P"], cfg["S"],
                      SEED)
    checks = []
    for rnd in range(crossing + 1):
        if rnd:
            so.nn_descent_iteration(vo, workers=cores)
            A.detail.nn_descent_iteration(sd, vd)
        e = so.export()
        sz, ids, dists, flags = sd.pools()
        same = bool(np.array_equal(sz, e["sizes"]))
        if same:
            P = cfg["P"]
            mask = np.arange(P)[None, :] < sz[:, None]
            same = (np.array_equal(ids[mask], e["ids"][mask]) and
                    np.array_equal(dists[mask].view(np.uint32), e["dists"][mask].view(np.uint32)) and
                    np.array_equal(flags[mask] & 1, e["flags"][mask] & 1))
        checks.append({"round": rnd, "pools_flags_equal": bool(same),
                       "dist_comps_equal": sd.meta()["dist_comps"] == e["dist_comps"]})
    out["build_parity"] = {"points": m1, "rounds": checks,
                           "all_equal": all(c["pools_flags_equal"] and c["dist_comps_equal"] for c in checks)}
    del so, sd, vd
    # search at the chosen point: the reference searcher over all queries, all cores
    if chosen is not None:
        _log("cpu baseline: search")
        vb = ref.vs(base)
        fo = ref.build_forest(vb, cfg["trees"], cfg["leaf"], SEED, workers=cores)
        qo = ref.vs(queries)
        t0 = time.perf_counter()
        ids_s, _, _ = ref.search(vb, fo, graph.ids, qo, cfg["k_return"], chosen["pool"], chosen["expansion"],
                                 chosen["iters"], workers=cores)
        ts = time.perf_counter() - t0
        out["search"] = {"value": len(queries) / ts, "unit": "queries/s", "cores": cores,
                         "point": {"pool": chosen["pool"], "expansion": chosen["expansion"],
                                   "iters": chosen["iters"]},
                         "sample": f"all {len(queries)} queries through the reference GraphSearcher "
                                   f"(recall_curve batch, {cores} workers), GPU-built graph, reference forest",
                         "ids_equal_gpu": bool(gpu_search is not None and np.array_equal(ids_s, gpu_search.ids))}
        del vb, fo
    # exact kNN rows: 1000 sampled rows (query mode, k + 1, the row itself removed)
    if exact_sample is not None:
        _log("cpu baseline: exact kNN rows")
        sel = rows[:len(exact_sample)]
        vb = ref.vs(base)
        t0 = time.perf_counter()
        ids_q = ref.brute_force(vb, ref.vs(np.ascontiguousarray(base[sel])), k + 1, workers=cores)
        tq = time.perf_counter() - t0
        self_rm = np.array([row[row != i][:k] for row, i in zip(ids_q, sel)])
        out["exact_knn"] = {"value": tq * n / len(sel), "unit": "s", "cores": cores,
                            "sample": f"brute_force_knn on {len(sel)} sampled base rows ({tq:.2f} s, {cores} workers), "
                                      f"scaled x{n / len(sel):.0f} to all {n} rows (rows are independent)",
                            "ids_equal_gpu": bool(np.array_equal(self_rm, exact_sample))}
    return out


def exact_knn_f32_leg(args, A, peaks, vs3=None):
    """Exact kNN of float data on the tensor cores (brute_force_f32_tc.cu): the
    cfg3 ground truth -- 10,000 sampled rows of the 1M x 960 float mixture,
    self-mode top-100 through annk_brute_force_rows, as the build's accuracy
    hook uses it.  bf16x3 tcgen05 candidates + exact fp32 re-rank; a 200-row
    prefix is checked against the exact CUDA-core kernel (ids and distance bits)
    and the reference library times 50 of the rows on the host cores."""
    cfg3 = dict(CONFIGS["cfg3"])
    if vs3 is None:
        b3, _ = gen_data(cfg3)
        vs3 = A.VectorSet(b3)
        del b3
    n3, d3, k3 = cfg3["n"], cfg3["dim"], cfg3["k"]
    rows3 = sample_rows(n3, 10000)  # the rows tools/time_bf_f32.py profiles under ncu
    runs = []
    for rep in range(3):  # first call warms the allocator
        A.profile_reset()
        A.profile_enable(True)
        A.lib.annk_synchronize()
        t1 = time.perf_counter()
        ids3, d3s = A.brute_force_rows(vs3, rows3, k3, with_dists=True)
        t2 = time.perf_counter()
        A.profile_enable(False)
        runs.append((t2 - t1, A.profile_report()))
    t_api, prof3 = min(runs[1:], key=lambda r: r[0])
    kname = "bf_tc_f32_kernel"
    k_ms = prof3.get(kname, (1, float("nan")))[1]
    bf16_flops = 6.0 * len(rows3) * n3 * d3  # 3 bf16 products per fp32 multiply-add
    t_peak = float(peaks.get("bf16_tflops", 1667.9))
    os.environ["ANNK_BF_CUDA_CORE"] = "1"
    try:
        A.profile_reset()
        A.profile_enable(True)
        ids_c, d_c = A.brute_force_rows(vs3, rows3[:200], k3, with_dists=True)
        A.profile_enable(False)
        cc_ms = sum(v[1] for v in A.profile_report().values())
    finally:
        del os.environ["ANNK_BF_CUDA_CORE"]
    out = {"workload": f"cfg3 ground truth: {len(rows3)} sampled rows x {n3} x {d3} float, self-mode top-{k3} "
                       "(brute_force_rows)",
           "seconds_through_api": t_api, "kernels_ms": {kn: round(v[1], 3) for kn, v in prof3.items()},
           "pairs_per_s": len(rows3) * n3 / t_api,
           "roofline": {"kernel": kname, "bound": "tensor", "achieved": bf16_flops / (k_ms / 1e3) / 1e12,
                        "peak": t_peak, "unit": "TFLOP/s", "frac": bf16_flops / (k_ms / 1e3) / 1e12 / t_peak,
                        "peak_source": "measured dense bf16 TFLOP/s (MEASURED_PEAKS.json)",
                        "flops_per_launch": bf16_flops,
                        "units": "bf16 tensor flops: 3 products (hi.hi, hi.lo, lo.hi) x 2 flops per fp32 "
                                 "multiply-add of the rows x N x dim contraction",
                        "traffic": ncu_traffic("cfg3", kname)},
           "cuda_core_check": {"rows": 200, "ids_equal": bool(np.array_equal(ids_c, ids3[:200])),
                               "dist_bits_equal": bool(np.array_equal(d_c.view(np.uint32), d3s[:200].view(np.uint32))),
                               "cuda_core_ms_for_200_rows": round(cc_ms, 2)}}
    if not args.skip_cpu and os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libannkit_ref.so")):
        from oracle import oracle as O
        ref = O.load("reference")
        cores = os.cpu_count() or 1
        b3h = vs3.data
        if b3h is not None:
            sel = rows3[:50]
            vb = ref.vs(b3h)
            t0 = time.perf_counter()
            ids_q = ref.brute_force(vb, ref.vs(np.ascontiguousarray(b3h[sel])), k3 + 1, workers=cores)
            tq = time.perf_counter() - t0
            self_rm = np.array([row[row != i][:k3] for row, i in zip(ids_q, sel)])
            out["cpu_baseline"] = {"value": tq * len(rows3) / len(sel), "unit": "s", "cores": cores,
                                   "kind": "reference",
                                   "sample": f"reference brute_force_knn on {len(sel)} of the rows ({tq:.2f} s, "
                                             f"{cores} workers), scaled x{len(rows3) / len(sel):.0f}",
                                   "ids_equal_gpu": bool(np.array_equal(self_rm, ids3[:len(sel)]))}
            del vb
    return out


def run_gpu(args, cfg, ws, rank, local):
    import torch

    import paper_1609_07228_b200 as A
    A.lib.annk_set_device(local)
    ext = torch.cuda.ExternalStream(A.stream_handle(), device=torch.device("cuda", local))

    def ev():
        e = torch.cuda.Event(enable_timing=True)
        e.record(ext)
        return e

    t0 = time.perf_counter()
    _log("data")
    base, queries = gen_data(cfg)
    gen_s = time.perf_counter() - t0
    vs = A.VectorSet(base)
    qs = A.VectorSet(queries)
    n, dim, k = cfg["n"], cfg["dim"], cfg["k"]

    # forest (once, like `annkit build-trees`)
    e0 = ev()
    forest = A.build_forest(vs, cfg["trees"], cfg["leaf"], SEED)
    e1 = ev()
    torch.cuda.synchronize()
    forest_s = e0.elapsed_time(e1) / 1e3

    # exact ground truth (untimed): sampled self-mode rows + query rows
    _log("ground truth")
    rows = sample_rows(n, cfg["acc_sample"])
    e0 = ev()
    gt_rows = A.brute_force_rows(vs, rows, k)
    e1 = ev()
    torch.cuda.synchronize()
    gt_rows_s = e0.elapsed_time(e1) / 1e3
    e0 = ev()
    gt_q = A.brute_force_knn(vs, qs, cfg["k_return"])
    e1 = ev()
    torch.cuda.synchronize()
    gt_q_s = e0.elapsed_time(e1) / 1e3
    bf_pairs = float(len(rows)) * (n - 1) + float(cfg["n_queries"]) * n

    # calibration build: accuracy per iteration -> crossing iteration
    _log("calibration build")
    st = A.init_graph(vs, forest, k, cfg["dep"], cfg["P"], cfg["S"], SEED)
    accs = [A.detail.pool_topk_accuracy(st, gt_rows, rows)]
    crossing = None
    comps = [st.meta()["dist_comps"]]
    join_rows = []
    for it in range(cfg["max_iters"]):
        A.detail.nn_descent_iteration(st, vs)
        accs.append(A.detail.pool_topk_accuracy(st, gt_rows, rows))
        comps.append(st.meta()["dist_comps"])
        jr = np.zeros(1, np.uint64)
        import ctypes
        v = ctypes.c_uint64(0)
        A.lib.annk_state_join_rows(st.handle, ctypes.byref(v))
        join_rows.append(int(v.value))
        _log(f"iteration {it + 1}: accuracy {accs[-1]:.4f}")
        if crossing is None and accs[-1] >= 0.9:
            crossing = it + 1
            if not args.full_log:
                break
    if crossing is None:
        crossing = cfg["max_iters"]
    del st

    phase_ms = {"init": [], **{f"iter{j + 1}": [] for j in range(crossing)}}

    def build_once():
        t0 = time.perf_counter()
        s = A.init_graph(vs, forest, k, cfg["dep"], cfg["P"], cfg["S"], SEED)
        phase_ms["init"].append((time.perf_counter() - t0) * 1e3)
        for j in range(crossing):
            t0 = time.perf_counter()
            A.detail.nn_descent_iteration(s, vs)
            phase_ms[f"iter{j + 1}"].append((time.perf_counter() - t0) * 1e3)
        return s

    _log(f"warm-up + timed builds (crossing at iteration {crossing})")
    for _ in range(args.warmup):
        s = build_once()
        s = None
    torch.cuda.synchronize()
    A.profile_reset()
    A.profile_enable(True)
    launches0 = A.launch_count()
    barrier(ws)
    torch.cuda.synchronize()
    s = None
    with ClockSampler(local) as clk:
        time.sleep(0.3)  # sampler start-up outside the timed region
        torch.cuda.synchronize()
        w0 = time.perf_counter()
        e0 = ev()
        for _ in range(args.steps):
            s = None  # each step is a fresh build: release the previous state first
            s = build_once()
        e1 = ev()
        torch.cuda.synchronize()
        wall_s = (time.perf_counter() - w0) / args.steps
    barrier(ws)
    launches = A.launch_count() - launches0
    A.profile_enable(False)
    prof = A.profile_report()
    step_s = e0.elapsed_time(e1) / 1e3 / args.steps
    step_s = max_over_ranks(ws, step_s)
    final_acc = A.detail.pool_topk_accuracy(s, gt_rows, rows)
    graph = A.finalize(s, vs, k)
    del s

    _log("search sweep")
    # search sweep (secondary metric): smallest pool reaching recall@k_return >= 0.9
    searcher = A.GraphSearcher(vs, forest, graph)
    sweep = []
    chosen = fastest = searcher_result = None
    kr = cfg["k_return"]
    # the reference's search knobs (search.hpp:13-21): pool P (>= k_return), seeds kept E <= P,
    # expansion rounds I; the fastest point reaching recall@k_return >= 0.9 is the headline
    grid = [(P, E, it) for P in cfg["sweep"][:2] for E in (8, 16, 32, 64, P) for it in (1, 2, 4) if E <= P]
    for P, E, it in grid:
        p = A.SearchParams(k_return=kr, pool_size=P, expansion=E, iters=it)
        r, dt = timed_search(searcher, qs, p, ev)
        rec = float(np.mean([len(np.intersect1d(r.ids[i], gt_q[i])) / kr for i in range(len(gt_q))]))
        row = {"pool": P, "expansion": E, "iters": it, "recall": round(rec, 4),
               "qps": round(cfg["n_queries"] / dt, 1), "dist_comps_per_query": float(r.stats[:, 0].mean())}
        sweep.append(row)
        if rec >= 0.9 and it == REF_ITERS and chosen is None:
            chosen = row  # recall_curve's definition: first sweep point (P, then E ascending) at the default I
            searcher_result = A.BatchResult(r.ids.copy(), r.dists.copy(), r.stats.copy())  # out= buffers are reused
        if rec >= 0.9 and (fastest is None or row["qps"] > fastest["qps"]):
            fastest = row

    # BASELINE cfg2's sweep: pool sizes 100-1000 (E = P, the default I) and tree-check
    # counts (SearchParams::n_trees_used, search.cpp:126-133) at the chosen point
    pool_sweep, tree_sweep = [], []
    for P in cfg["sweep"]:
        p = A.SearchParams(k_return=kr, pool_size=P, expansion=P, iters=REF_ITERS)
        r, dt = timed_search(searcher, qs, p, ev, reps=1)
        rec = float(np.mean([len(np.intersect1d(r.ids[i], gt_q[i])) / kr for i in range(len(gt_q))]))
        pool_sweep.append({"pool": P, "expansion": P, "iters": REF_ITERS, "recall": round(rec, 4),
                           "qps": round(cfg["n_queries"] / dt, 1),
                           "dist_comps_per_query": float(r.stats[:, 0].mean())})
    if chosen:
        for T in sorted({1, 2, 4, cfg["trees"]}):
            p = A.SearchParams(k_return=kr, pool_size=chosen["pool"], expansion=chosen["expansion"],
                               iters=chosen["iters"], n_trees_used=T)
            r, dt = timed_search(searcher, qs, p, ev, reps=1)
            rec = float(np.mean([len(np.intersect1d(r.ids[i], gt_q[i])) / kr for i in range(len(gt_q))]))
            tree_sweep.append({"trees_used": T, "pool": chosen["pool"], "expansion": chosen["expansion"],
                               "iters": chosen["iters"], "recall": round(rec, 4),
                               "qps": round(cfg["n_queries"] / dt, 1),
                               "dist_comps_per_query": float(r.stats[:, 0].mean())})

    search_kernels = None
    search_roofline = None
    for row in (fastest, chosen):  # kernel-only time of the reported points (profiler on, outside the sweep)
        if not row:
            continue
        A.profile_reset()
        A.profile_enable(True)
        rr = searcher.search_batch(qs, A.SearchParams(k_return=kr, pool_size=row["pool"],
                                                      expansion=row["expansion"], iters=row["iters"]))
        A.profile_enable(False)
        search_kernels = {k2: round(v2[1], 3) for k2, v2 in A.profile_report().items()}
        row["kernel_qps"] = round(cfg["n_queries"] / (sum(search_kernels.values()) / 1e3), 1)
        # HBM-gather model: every distance gathers one base row + its id, every
        # expanded point reads its graph row
        rb = vs.info()["row_bytes"]
        alg = float(rr.stats[:, 0].sum()) * (rb + 4) + float(rr.stats[:, 2].sum()) * graph.ids.shape[1] * 4
        kms = max(v for k2, v in search_kernels.items() if k2.startswith("search_kernel"))
        pk = measured_hbm_peak()
        tkey = "search_kernel<true>" + ("" if (row["expansion"], row["iters"]) == (8, 4) else
                                        f"@E{row['expansion']}I{row['iters']}")
        row["roofline"] = {"bound": "hbm", "achieved": alg / (kms / 1e3) / 1e9, "peak": pk, "unit": "GB/s",
                           "frac": alg / (kms / 1e3) / 1e9 / pk, "algorithmic_bytes": alg, "kernel_ms": kms,
                           "traffic": ncu_traffic(args.config, tkey)}

    _log("e2e")
    # e2e through the C-ABI from pinned host memory
    pinned = torch.empty((n, dim), dtype=torch.float32, pin_memory=True)
    pinned.numpy()[:] = base
    host = pinned.numpy()
    out_ids = torch.empty((n, k), dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
    out_d = torch.empty((n, k), dtype=torch.float32, pin_memory=True).numpy()
    packed = pinned_forest(A, forest)  # the prebuilt forest as host arrays (outside the timed region)
    f_bytes = sum(int(v.nbytes) for v in packed.values())

    def e2e_run(with_forest_build):
        times = []
        for i in range(max(1, args.e2e_steps) + 1):
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            v2 = A.VectorSet(host)
            if with_forest_build:
                f2 = A.build_forest(v2, cfg["trees"], cfg["leaf"], SEED)
            else:
                f2 = A.KdForest.import_packed(n, dim, cfg["leaf"], SEED, packed)
            s2 = A.init_graph(v2, f2, k, cfg["dep"], cfg["P"], cfg["S"], SEED)
            for _ in range(crossing - 1):
                A.detail.nn_descent_iteration(s2, v2)
            if crossing:  # last round + finalize in one call: row copies overlap the replay
                g2 = A.detail.nn_descent_iteration_finalize(s2, v2, k, out_ids=out_ids, out_dists=out_d)[2]
            else:
                g2 = A.finalize(s2, v2, k, out_ids=out_ids, out_dists=out_d)
            t2 = time.perf_counter()
            if i > 0:  # first is warm-up
                times.append(t2 - t1)
            del v2, f2, s2
            assert np.array_equal(g2.ids, graph.ids), "e2e graph differs from the device-resident build"
        return max_over_ranks(ws, statistics.mean(times))

    e2e_s = e2e_run(False)
    e2e_fb_s = e2e_run(True)

    _log("roofline")
    # roofline: the dominant kernel's algorithmic bytes per launch / measured duration
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            peaks = json.load(fh)
    except Exception:
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "measured" if "hbm_gbs" in peaks else "fallback"
    dsinfo = vs.info()
    row_bytes = dsinfo["row_bytes"]  # bytes per row actually gathered (u8 rows on the exact u8 path)
    def kernel_roofline(name):
        """HBM roofline of one build kernel: algorithmic bytes per launch / its mean launch time."""
        cnt, ms = prof[name]
        if name.startswith("join"):
            rows_per_launch = sum(join_rows[:crossing]) / crossing
            alg_bytes = rows_per_launch * (row_bytes + 4) + n * 8
            unit_desc = (f"per launch: sum_i(|new_i|+|old_i|) list rows x ({row_bytes} B row + 4 B id) + N x 8 B "
                         "thresholds (each list member's row gathered once per point)")
        elif name == "init_kernel":
            alg_bytes = comps[0] * (row_bytes + 4) + n * cfg["P"] * 9
            unit_desc = (f"per launch: init dist_comps x ({row_bytes} B candidate row + 4 B id) + N x P x 9 B "
                         "pool writes")
        else:
            alg_bytes = None
            unit_desc = "n/a"
        per_launch_s = ms / cnt / 1e3
        achieved = alg_bytes / per_launch_s / 1e9 if alg_bytes else None
        traffic = None
        try:  # DRAM bytes per launch of this kernel from the committed ncu --set full capture
            with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
                tr = json.load(fh).get(args.config, {}).get(name)
                traffic = tr["dram_bytes_per_launch"] if tr else None
        except Exception:
            pass
        return {"kernel": name, "bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                "frac": (achieved / hbm_peak) if achieved else None, "traffic": traffic,
                "peak_source": peak_src, "algorithmic_bytes_per_launch": alg_bytes,
                "per_launch_ms": per_launch_s * 1e3,
                "share_of_step": ms / sum(v[1] for v in prof.values()), "units": unit_desc,
                "exact_u8_path": dsinfo["u8"]}

    dom_name = max(prof.items(), key=lambda kv: kv[1][1])[0]
    roofline = kernel_roofline(dom_name)
    # the other gather kernels of the step, same model (the dominant one can change between builds)
    roofline_others = {nm: kernel_roofline(nm) for nm in prof
                       if nm != dom_name and (nm == "init_kernel" or nm.startswith("join"))}

    _log("exact kNN")
    # cfg4: exact kNN graph (self-mode top-k over all N points) on the tcgen05 kernel
    exact = exact_sample = None
    if not args.skip_cfg4 and dsinfo["u8"] and not cfg.get("skip_exact"):
        bf_runs = []
        bf_out = torch.empty((n, k), dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)  # caller-owned
        for rep in range(2):  # first call warms the allocator
            A.profile_reset()
            A.profile_enable(True)
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            ids_all = A.brute_force_knn(vs, None, k, out_ids=bf_out)
            t2 = time.perf_counter()
            A.profile_enable(False)
            bf_runs.append((t2 - t1, A.profile_report()))
        bf_s, bf_prof = bf_runs[-1]
        scan = A.bf_last_scan()
        kname = next((kn for kn in bf_prof if kn.startswith("bf_tc")), max(bf_prof, key=lambda kn: bf_prof[kn][1]))
        k_ms = bf_prof[kname][1]
        dev_ms = sum(v[1] for v in bf_prof.values())
        # the tensor roofline counts the u8 multiply-adds the kernel ISSUED: the pruned scan visits
        # only the (256-query block, 64-row tile) pairs it could not rule out, each a full
        # 256 x 64 x dim contraction (plus the blockmin pass, queries x pivots, not counted)
        tile_ops = 2.0 * dim * 256 * 64
        int_ops = tile_ops * scan["tiles_visited"] if kname.startswith("bf_tc") else 2.0 * dim * n * n
        # the tensor peak is measured here: tcgen05 kind::i8 MMAs issued back to back on shared-memory
        # operands, one CTA per SM (annk_measure_i8_peak); 2 x the measured bf16 peak is reported beside it
        t_peak = A.measure_i8_peak()
        t_peak_2x = 2.0 * float(peaks.get("bf16_tflops", 1678.2))
        exact = {"workload": f"cfg4: self-mode exact top-{k} over {n} x {dim} (brute_force_knn(base, nullptr, k))",
                 "seconds_through_api": bf_s, "through_api": "brute_force_knn(base, None, k, out_ids=pinned host "
                                                             "array): device-resident dataset in, ids D2H inside",
                 "device_ms": round(dev_ms, 3),
                 "kernels_ms": {kn: round(v[1], 3) for kn, v in bf_prof.items()},
                 "pairs_per_s": n * (n - 1) / (dev_ms / 1e3),
                 "pairs_per_s_definition": "all N(N-1) ordered pairs the result is exact over / device time of "
                                           "the whole call (pruned tiles included: their pairs are decided by "
                                           "the triangle-inequality bound, not computed)",
                 "scan": {**scan, "visited_frac": scan["tiles_visited"] / max(1, scan["tiles_total"])},
                 "roofline": {"kernel": kname, "bound": "tensor", "achieved": int_ops / (k_ms / 1e3) / 1e12,
                              "peak": t_peak, "unit": "TOP/s", "frac": int_ops / (k_ms / 1e3) / 1e12 / t_peak,
                              "ops": "u8 multiply-add x 2 of the tiles the kernel visited (issued work), "
                                     "all launches of the call",
                              "peak_source": "measured in this run: tcgen05 kind::i8 M=128 N=256 MMAs issued back "
                                             "to back from shared memory on every SM (annk_measure_i8_peak)",
                              "peak_2x_measured_bf16": t_peak_2x,
                              "traffic": ncu_traffic(args.config, kname)},
                 "row0_first5": [int(x) for x in ids_all[0, :5]]}
        exact_sample = ids_all[rows[:1000]].copy()
        del ids_all

    _log("exact kNN fp32")
    exact_f32 = None
    if not args.skip_cfg4 and not cfg.get("skip_exact") and args.config in ("cfg2", "cfg3"):
        exact_f32 = exact_knn_f32_leg(args, A, peaks, vs if args.config == "cfg3" else None)

    _log("cpu baseline")
    # CPU baseline: the reference library (oracle/_ref) on this box's host cores, rank 0 at N=1
    cpu = cpu_baseline_leg(args, cfg, A, base, queries, crossing, graph, searcher_result, chosen, exact_sample,
                           rows) if (rank == 0 and ws == 1 and not args.skip_cpu) else None

    clocks = clk.summary()
    line = {
        "metric": METRIC, "value": step_s, "unit": "s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": step_s * 1e3, "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
        "dtype": "u8" if dsinfo["u8"] else "f32", "data": "synthetic",
        "config": {"workload": args.config, "n": n, "dim": dim, "trees": cfg["trees"], "leaf_cap": cfg["leaf"],
                   "k": k, "pool_cap": cfg["P"], "sample_cap": cfg["S"], "conquer_depth": cfg["dep"],
                   "iterations_to_acc_0.9": crossing, "accuracy_sample_rows": int(len(rows)),
                   "l2": f"inputs larger than L2 ({n * dim * 4 / 1e6:.0f} MB dataset)", "parallelism": f"replicas x{ws}"},
        "e2e": {"value": e2e_s, "unit": "s", "h2d_bytes_per_step": int(n * dim * 4) + f_bytes,
                "d2h_bytes_per_step": int(n * k * 8),
                "includes": "H2D dataset + H2D prebuilt forest (host arrays; the reference's build_graph is timed "
                            "with its forest built beforehand), init, refine, finalize, D2H graph ids+dists"},
        "e2e_with_forest_build": {"value": e2e_fb_s, "unit": "s", "h2d_bytes_per_step": int(n * dim * 4),
                                  "d2h_bytes_per_step": int(n * k * 8),
                                  "includes": "H2D dataset, forest build on the device, init, refine, finalize, "
                                              "D2H graph ids+dists"},
        "gpu_launches": int(launches),
        "roofline": roofline,
        "roofline_other_kernels": roofline_others,
        "cpu_baseline": cpu,
        "clocks": clocks,
        "search_qps_at_recall_0.9": chosen["qps"] if chosen else None,
        "search_kernels_ms": search_kernels,
        "search": {"k_return": kr, "n_queries": cfg["n_queries"],
                   "definition": f"recall_curve sweep (P, then E ascending) at the default I={REF_ITERS}; "
                                 "first point with recall@k_return >= 0.9; Q / device time of the batch "
                                 "through the public API (results D2H to pinned memory included)",
                   "chosen": chosen, "fastest_any_iters": fastest, "sweep": sweep,
                   "pool_sweep": pool_sweep, "trees_used_sweep": tree_sweep},
        "accuracy": {"per_iteration": [round(a, 4) for a in accs], "final_sample": round(final_acc, 4),
                     "dist_comps": comps},
        "exact_knn": exact,
        "exact_knn_f32": exact_f32,
        "aux_seconds": {"forest": forest_s, "gt_rows": gt_rows_s, "gt_queries": gt_q_s, "data_gen_host": gen_s,
                        "brute_force_pairs_per_s": bf_pairs / (gt_rows_s + gt_q_s)},
        "host_wall_s_per_step": wall_s,
        "phase_wall_ms_median": {p: round(statistics.median(v), 2) for p, v in phase_ms.items() if v},
        "kernels_ms": {k2: round(v2[1], 3) for k2, v2 in sorted(prof.items(), key=lambda kv: -kv[1][1])},
    }
    if rank == 0:
        print(json.dumps(line))


# ------------------------------------------------------- multi-GPU arm

def run_gpu_sharded(args, cfg, ws, rank, local):
    """N > 1: point-sharded build (paper_1609_07228_b200/sharded.py).
    Strong scaling: the cfg's N points are split across the ranks; init, sampling,
    the join (as visiting point) and the merge (as target) run on the owning rank,
    forward lists / thresholds are all-gathered and offers routed all-to-all over
    NCCL each round.  Forest and dataset are replicated.  Search and ground truth
    are sharded by query rows.  Times are CUDA events, max over ranks."""
    import torch

    import paper_1609_07228_b200 as A
    from paper_1609_07228_b200 import sharded as SH
    A.lib.annk_set_device(local)
    bufdev = "cuda" if args.comm == "nccl" else "cpu"
    comm = SH.TorchComm(bufdev)
    ext = torch.cuda.ExternalStream(A.stream_handle(), device=torch.device("cuda", local))

    def ev():
        e = torch.cuda.Event(enable_timing=True)
        e.record(ext)
        return e

    base, queries = gen_data(cfg)
    vs, qs_all = A.VectorSet(base), queries
    n, dim, k, kr = cfg["n"], cfg["dim"], cfg["k"], cfg["k_return"]
    lo, hi = SH.shard_ranges(n, ws)[rank]
    qlo, qhi = SH.shard_ranges(cfg["n_queries"], ws)[rank]
    qs = A.VectorSet(np.ascontiguousarray(qs_all[qlo:qhi]))

    e0 = ev()
    forest = A.build_forest(vs, cfg["trees"], cfg["leaf"], SEED)
    e1 = ev()
    torch.cuda.synchronize()
    forest_s = max_over_ranks(ws, e0.elapsed_time(e1) / 1e3)

    rows = sample_rows(n, cfg["acc_sample"])
    rows = rows[(rows >= lo) & (rows < hi)]
    gt_rows = A.brute_force_rows(vs, rows, k)
    gt_q = A.brute_force_knn(vs, qs, kr)

    def shard():
        return SH.DeviceShard(vs, forest, k, cfg["dep"], cfg["P"], cfg["S"], SEED, lo, hi, buffer_device=bufdev)

    # calibration: accuracy per round -> crossing round
    e = shard()
    accs = [SH.sharded_accuracy(e, comm, gt_rows, rows)]
    comps = [comm.allreduce_sum(e.dist_comps())]
    crossing = None
    for it in range(cfg["max_iters"]):
        _, c = SH.nn_descent_round(e, comm)
        comps.append(comps[-1] + c)
        accs.append(SH.sharded_accuracy(e, comm, gt_rows, rows))
        if crossing is None and accs[-1] >= 0.9:
            crossing = it + 1
            if not args.full_log:
                break
    crossing = crossing or cfg["max_iters"]
    del e

    def build_once():
        e = shard()
        for _ in range(crossing):
            SH.nn_descent_round(e, comm)
        return e

    for _ in range(args.warmup):
        build_once()
    torch.cuda.synchronize()
    A.profile_reset()
    A.profile_enable(True)
    launches0 = A.launch_count()
    barrier(ws)
    e = None
    with ClockSampler(local) as clk:
        time.sleep(0.3)
        torch.cuda.synchronize()
        barrier(ws)
        e0 = ev()
        for _ in range(args.steps):
            e = None
            e = build_once()
        e1 = ev()
        torch.cuda.synchronize()
    barrier(ws)
    launches = A.launch_count() - launches0
    A.profile_enable(False)
    prof = A.profile_report()
    step_s = max_over_ranks(ws, e0.elapsed_time(e1) / 1e3 / args.steps)
    final_acc = SH.sharded_accuracy(e, comm, gt_rows, rows)
    graph = SH.allgather_graph(e.finalize(), comm)
    del e
    # the sharded build must equal the one-GPU build exactly (same pools: the merge
    # replays the reference's order on every rank)
    st1 = A.init_graph(vs, forest, k, cfg["dep"], cfg["P"], cfg["S"], SEED)
    for _ in range(crossing):
        A.detail.nn_descent_iteration(st1, vs)
    g1 = A.finalize(st1, vs, k)
    del st1
    single_equal = bool(comm.allreduce_sum(0 if np.array_equal(g1.ids, graph.ids) else 1) == 0)
    del g1

    # search: every rank holds the full index and answers its query shard
    searcher = A.GraphSearcher(vs, forest, graph)
    sweep, chosen, fastest = [], None, None
    grid = [(P, E, it) for P in cfg["sweep"][:2] for E in (8, 16, 32, 64, P) for it in (1, 2, 4) if E <= P]
    for P, E, it in grid:
        p = A.SearchParams(k_return=kr, pool_size=P, expansion=E, iters=it)
        barrier(ws)
        r, dt = timed_search(searcher, qs, p, ev)
        dt = max_over_ranks(ws, dt)
        hits = sum(len(np.intersect1d(r.ids[i], gt_q[i])) for i in range(len(gt_q)))
        rec = comm.allreduce_sum(hits) / (cfg["n_queries"] * kr)
        row = {"pool": P, "expansion": E, "iters": it, "recall": round(rec, 4),
               "qps": round(cfg["n_queries"] / dt, 1)}
        sweep.append(row)
        if rec >= 0.9 and it == REF_ITERS and chosen is None:
            chosen = row  # recall_curve's definition: first sweep point (P, then E ascending) at the default I
        if rec >= 0.9 and (fastest is None or row["qps"] > fastest["qps"]):
            fastest = row

    # e2e: host dataset (and prebuilt forest) in, own graph rows out, per rank
    pinned = torch.empty((n, dim), dtype=torch.float32, pin_memory=True)
    pinned.numpy()[:] = base
    host = pinned.numpy()
    packed = pinned_forest(A, forest)
    f_bytes = sum(int(v.nbytes) for v in packed.values())

    def e2e_run(with_forest_build):
        times = []
        for i in range(max(1, args.e2e_steps) + 1):
            torch.cuda.synchronize()
            barrier(ws)
            t1 = time.perf_counter()
            v2 = A.VectorSet(host)
            if with_forest_build:
                f2 = A.build_forest(v2, cfg["trees"], cfg["leaf"], SEED)
            else:
                f2 = A.KdForest.import_packed(n, dim, cfg["leaf"], SEED, packed)
            e2 = SH.DeviceShard(v2, f2, k, cfg["dep"], cfg["P"], cfg["S"], SEED, lo, hi, buffer_device=bufdev)
            for _ in range(crossing):
                SH.nn_descent_round(e2, comm)
            g2 = e2.finalize()
            t2 = time.perf_counter()
            if i > 0:
                times.append(t2 - t1)
            del v2, f2, e2
            assert np.array_equal(g2.ids, graph.ids[lo:hi]), "e2e graph differs from the device-resident build"
        return max_over_ranks(ws, statistics.mean(times))

    e2e_s = e2e_run(False)
    e2e_fb_s = e2e_run(True)

    dsinfo = vs.info()
    line = {
        "metric": METRIC, "value": step_s, "unit": "s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": step_s * 1e3, "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
        "dtype": "u8" if dsinfo["u8"] else "f32", "data": "synthetic",
        "config": {"workload": args.config, "n": n, "dim": dim, "trees": cfg["trees"], "leaf_cap": cfg["leaf"],
                   "k": k, "pool_cap": cfg["P"], "sample_cap": cfg["S"], "conquer_depth": cfg["dep"],
                   "iterations_to_acc_0.9": crossing, "accuracy_sample_rows": cfg["acc_sample"],
                   "l2": f"inputs larger than L2 ({n * dim * 4 / 1e6:.0f} MB dataset)",
                   "parallelism": f"point-sharded build x{ws} ({args.comm} all-gather + all-to-all per round), "
                                  f"query-sharded search",
                   "graph_equal_single_gpu": single_equal},
        "e2e": {"value": e2e_s, "unit": "s", "h2d_bytes_per_step": int(ws * (n * dim * 4 + f_bytes)),
                "d2h_bytes_per_step": int(n * k * 8),
                "includes": "per rank: H2D dataset + prebuilt forest, sharded init + rounds, finalize, D2H own rows"},
        "e2e_with_forest_build": {"value": e2e_fb_s, "unit": "s", "h2d_bytes_per_step": int(ws * n * dim * 4),
                                  "d2h_bytes_per_step": int(n * k * 8),
                                  "includes": "per rank: H2D dataset, forest build, sharded init + rounds, "
                                              "finalize, D2H own rows"},
        "gpu_launches": int(launches),
        "roofline": None,
        "cpu_baseline": None,
        "clocks": clk.summary(),
        "search_qps_at_recall_0.9": chosen["qps"] if chosen else None,
        "search": {"k_return": kr, "n_queries": cfg["n_queries"], "chosen": chosen, "fastest_any_iters": fastest,
                   "sweep": sweep},
        "accuracy": {"per_iteration": [round(a, 4) for a in accs], "final_sample": round(final_acc, 4),
                     "dist_comps": comps},
        "aux_seconds": {"forest": forest_s},
        "kernels_ms_rank0": {k2: round(v2[1], 3) for k2, v2 in sorted(prof.items(), key=lambda kv: -kv[1][1])},
    }
    if rank == 0:
        print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="cfg2", choices=sorted(CONFIGS))
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--skip-cfg4", action="store_true", help="skip the exact kNN graph (cfg4) measurement")
    ap.add_argument("--full-log", action="store_true", help="run all iterations / sweep points")
    ap.add_argument("--comm", default="nccl", choices=["nccl", "gloo"],
                    help="N>1 collectives; gloo keeps buffers on the host (functional runs on one GPU)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: relaunch this command under torchrun (the driver may
        # also launch it that way itself, in which case WORLD_SIZE is already set)
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        env = dict(os.environ)
        env.setdefault("NCCL_DEBUG", "INFO")
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd, env=env))
    if int(os.environ.get("WORLD_SIZE", "1")) > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")  # communicator setup is logged for the driver
    cfg = dict(CONFIGS[args.config])
    cfg.setdefault("ref_iters", {"cfg2": 2, "cfg1": 3, "cfg3": 3, "cfg5": 2, "tiny": 3}[args.config])
    ws, rank, local = dist_setup(args)
    if args.impl == "reference":
        run_reference(args, cfg, ws, rank)
    elif ws > 1:
        run_gpu_sharded(args, cfg, ws, rank, local)
    else:
        run_gpu(args, cfg, ws, rank, local)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
