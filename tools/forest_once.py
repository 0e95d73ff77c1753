"""One build_forest at a bench config (for ncu captures of forest_build_kernel)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1609_07228_b200 as A  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg2"]
base, _ = bench.gen_data(cfg)
vs = A.VectorSet(base)
f = A.build_forest(vs, cfg["trees"], cfg["leaf"], bench.SEED)
A.lib.annk_synchronize()
print("nodes/tree", f.tree_info(0)["num_nodes"])
