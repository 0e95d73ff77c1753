"""Per-launch timeline of one cfg build after warm-up builds (ANNK_PROF_TRACE):
python tools/timeline.py [--config cfg2] [--iters 2] [--warm 2]"""
import argparse
import os
import sys

os.environ.setdefault("ANNK_PROF_TRACE", "1")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_1609_07228_b200 as A  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg2")
ap.add_argument("--iters", type=int, default=2)
ap.add_argument("--warm", type=int, default=2)
args = ap.parse_args()
cfg = dict(bench.CONFIGS[args.config])
base, _ = bench.gen_data(cfg)
vs = A.VectorSet(base)
f = A.build_forest(vs, cfg["trees"], cfg["leaf"], bench.SEED)


def build():
    s = A.init_graph(vs, f, cfg["k"], cfg["dep"], cfg["P"], cfg["S"], bench.SEED)
    for _ in range(args.iters):
        A.detail.nn_descent_iteration(s, vs)
    return s


for _ in range(args.warm):
    build()
A.profile_reset()
A.profile_enable(True)
print("---- traced build", file=sys.stderr)
s = build()
A.profile_report()
A.profile_enable(False)
