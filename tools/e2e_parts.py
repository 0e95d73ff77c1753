"""Wall time of each public-API call on bench.py's e2e path (cfg2): dataset
upload, forest import, init + rounds, finalize + D2H."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1609_07228_b200 as A  # noqa: E402

cfg = bench.CONFIGS["cfg2"]
base, _ = bench.gen_data(cfg)
n, dim, k = cfg["n"], cfg["dim"], cfg["k"]
vs = A.VectorSet(base)
forest = A.build_forest(vs, cfg["trees"], cfg["leaf"], bench.SEED)
packed = bench.pinned_forest(A, forest)
pinned = torch.empty((n, dim), dtype=torch.float32, pin_memory=True)
pinned.numpy()[:] = base
host = pinned.numpy()
out_ids = torch.empty((n, k), dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
out_d = torch.empty((n, k), dtype=torch.float32, pin_memory=True).numpy()
for rep in range(6):
    t = [time.perf_counter()]
    v2 = A.VectorSet(host); A.lib.annk_synchronize(); t.append(time.perf_counter())
    f2 = A.KdForest.import_packed(n, dim, cfg["leaf"], bench.SEED, packed); A.lib.annk_synchronize(); t.append(time.perf_counter())
    s2 = A.init_graph(v2, f2, k, cfg["dep"], cfg["P"], cfg["S"], bench.SEED)
    fused = rep >= 3
    A.detail.nn_descent_iteration(s2, v2)
    if not fused:
        A.detail.nn_descent_iteration(s2, v2)
    A.lib.annk_synchronize(); t.append(time.perf_counter())
    if fused:
        A.detail.nn_descent_iteration_finalize(s2, v2, k, out_ids=out_ids, out_dists=out_d)
    else:
        A.finalize(s2, v2, k, out_ids=out_ids, out_dists=out_d)
    t.append(time.perf_counter())
    d = np.diff(t) * 1e3
    what = "init+1 round" if fused else "init+2 rounds"
    last = "last round+finalize+D2H (fused)" if fused else "finalize+D2H"
    print(f"dataset {d[0]:.1f} ms  forest import {d[1]:.1f} ms  {what} {d[2]:.1f} ms  {last} {d[3]:.1f} ms  "
          f"total {sum(d):.1f} ms", flush=True)
    del v2, f2, s2
