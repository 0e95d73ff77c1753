import sys, time
sys.path.insert(0, ".")
import numpy as np
import bench
import paper_1609_07228_b200 as A
cfg = dict(bench.CONFIGS["cfg5"])
n = int(sys.argv[1]); nq = int(sys.argv[2])
cfg["n"] = n
base, queries = bench.gen_data(cfg)
vs = A.VectorSet(base)
rows = bench.sample_rows(n, nq)
print("start", flush=True)
t0 = time.time(); g = A.brute_force_rows(vs, rows, 100); A.lib.annk_synchronize(); print("rows", time.time() - t0, flush=True)
if len(sys.argv) > 3:
    qs = A.VectorSet(queries[: int(sys.argv[3])])
    t0 = time.time(); g = A.brute_force_knn(vs, qs, 100); A.lib.annk_synchronize(); print("queries", time.time() - t0, flush=True)
