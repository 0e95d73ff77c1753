"""Times build_forest at a bench config (CUDA events on the library stream)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1609_07228_b200 as A  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg2"]
base, _ = bench.gen_data(cfg)
vs = A.VectorSet(base)
for rep in range(3):
    A.lib.annk_synchronize()
    t0 = time.perf_counter()
    f = A.build_forest(vs, cfg["trees"], cfg["leaf"], bench.SEED)
    t1 = time.perf_counter()
    print(f"forest {cfg['trees']} trees: {t1 - t0:.3f} s, nodes/tree {f.tree_info(0)['num_nodes']}", flush=True)
