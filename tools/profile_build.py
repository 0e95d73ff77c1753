"""One cfg-shaped build (forest, init, N NN-descent rounds, search batch) for
ncu captures: `ncu -k regex:<kernel> ... python tools/profile_build.py`."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_1609_07228_b200 as A  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg2")
ap.add_argument("--iters", type=int, default=2)
ap.add_argument("--search", action="store_true")
ap.add_argument("--n", type=int, default=0)
ap.add_argument("--search-e", type=int, default=8)
ap.add_argument("--search-iters", type=int, default=4)
args = ap.parse_args()
cfg = dict(bench.CONFIGS[args.config])
if args.n:
    cfg["n"] = args.n
base, queries = bench.gen_data(cfg)
vs = A.VectorSet(base)
f = A.build_forest(vs, cfg["trees"], cfg["leaf"], bench.SEED)
s = A.init_graph(vs, f, cfg["k"], cfg["dep"], cfg["P"], cfg["S"], bench.SEED)
for _ in range(args.iters):
    A.detail.nn_descent_iteration(s, vs)
if args.search:
    g = A.finalize(s, vs, cfg["k"])
    r = A.GraphSearcher(vs, f, g).search_batch(queries, A.SearchParams(cfg["k_return"], cfg["P"], args.search_e,
                                                                      args.search_iters))  # bench's headline point
print("profile_build done", A.launch_count())
