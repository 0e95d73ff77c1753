"""Times exact kNN (self-mode top-k over n points and query-mode) on the device."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_1609_07228_b200 as A  # noqa: E402

cfg = bench.CONFIGS["cfg2"]
base, queries = bench.gen_data(cfg)
vs = A.VectorSet(base)
qs = A.VectorSet(queries)
for rep in range(2):
    A.lib.annk_synchronize()
    t0 = time.perf_counter()
    A.brute_force_knn(vs, qs, 100)
    t1 = time.perf_counter()
    print(f"query-mode 10k x 1M top-100: {t1 - t0:.3f} s, {1e4 * 1e6 / (t1 - t0) / 1e9:.1f} G pairs/s", flush=True)
if len(sys.argv) > 1:
    t0 = time.perf_counter()
    ids = A.brute_force_knn(vs, None, 100)
    t1 = time.perf_counter()
    print(f"self-mode 1M x 1M top-100 (cfg4): {t1 - t0:.3f} s, {1e12 / (t1 - t0) / 1e9:.1f} G pairs/s", flush=True)
