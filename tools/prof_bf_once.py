"""One exact kNN (self-mode top-100) on a cfg2-distributed subset: for ncu captures."""
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_1609_07228_b200 as A  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000000
base, _ = bench.gen_data(dict(bench.CONFIGS["cfg2"]), n)
vs = A.VectorSet(base)
A.brute_force_knn(vs, None, 100)
A.lib.annk_synchronize()
