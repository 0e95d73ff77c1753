"""Times one build at a bench config, optionally at reduced N: forest, init and
each NN-descent round (CUDA-event kernel totals from the library profiler)."""
import argparse
import sys
import time

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_1609_07228_b200 as A  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg3")
ap.add_argument("--n", type=int, default=0)
ap.add_argument("--iters", type=int, default=2)
args = ap.parse_args()
cfg = dict(bench.CONFIGS[args.config])
if args.n:
    cfg["n"] = args.n
base, _ = bench.gen_data(cfg)
vs = A.VectorSet(base)
print("dataset", vs.info(), flush=True)
t0 = time.perf_counter()
f = A.build_forest(vs, cfg["trees"], cfg["leaf"], bench.SEED)
A.lib.annk_synchronize()
print(f"forest {time.perf_counter() - t0:.3f} s", flush=True)
A.profile_reset()
A.profile_enable(True)
t0 = time.perf_counter()
s = A.init_graph(vs, f, cfg["k"], cfg["dep"], cfg["P"], cfg["S"], bench.SEED)
print(f"init {time.perf_counter() - t0:.3f} s  {A.profile_report()}", flush=True)
for it in range(args.iters):
    A.profile_reset()
    t0 = time.perf_counter()
    A.detail.nn_descent_iteration(s, vs)
    rep = A.profile_report()
    print(f"iter {it + 1} {time.perf_counter() - t0:.3f} s  " +
          str({k: round(v[1], 1) for k, v in sorted(rep.items(), key=lambda kv: -kv[1][1])[:5]}), flush=True)
