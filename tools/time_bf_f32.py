"""Times the fp32 exact-kNN path at cfg3 shapes (1M x 960 float mixture):
brute_force_rows over a 10k-row sample and brute_force_knn for the 1k
queries, on tcgen05 (bf16x3 + exact re-rank) and, for a smaller sample, on the
exact CUDA-core kernel; per-kernel CUDA-event times from annk_profile."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_1609_07228_b200 as A  # noqa: E402

cfg = dict(bench.CONFIGS["cfg3"])
if len(sys.argv) > 1:
    cfg["n"] = int(sys.argv[1])
base, queries = bench.gen_data(cfg)
vs = A.VectorSet(base)
qs = A.VectorSet(queries)
rng = np.random.default_rng(1)
rows = np.sort(rng.choice(cfg["n"], 10000, replace=False)).astype(np.uint32)


def timed(label, fn, pairs):
    A.profile_enable(True)
    A.profile_reset()
    A.lib.annk_synchronize()
    t0 = time.perf_counter()
    r = fn()
    t1 = time.perf_counter()
    rep = A.profile_report()
    A.profile_enable(False)
    print(f"{label}: {t1 - t0:.4f} s, {pairs / (t1 - t0) / 1e9:.1f} G pairs/s", flush=True)
    for name, (cnt, ms) in sorted(rep.items(), key=lambda kv: -kv[1][1]):
        print(f"    {name:28s} {cnt:4d} {ms:9.3f} ms")
    return r


for rep in range(2):
    r_tc = timed("tc rows 10k x 1M top-100", lambda: A.brute_force_rows(vs, rows, 100, with_dists=True),
                 1e4 * cfg["n"])
timed("tc queries 1k x 1M top-100", lambda: A.brute_force_knn(vs, qs, 100, with_dists=True), 1e3 * cfg["n"])
os.environ["ANNK_BF_CUDA_CORE"] = "1"
sub = rows[:1000]
r_cc = timed("cuda-core rows 1k x 1M top-100", lambda: A.brute_force_rows(vs, sub, 100, with_dists=True),
             1e3 * cfg["n"])
del os.environ["ANNK_BF_CUDA_CORE"]
assert np.array_equal(r_tc[0][:1000], r_cc[0]) and np.array_equal(r_tc[1][:1000].view(np.uint32),
                                                                   r_cc[1].view(np.uint32)), "tc != cuda-core"
print("tc == cuda-core on the first 1000 rows")
