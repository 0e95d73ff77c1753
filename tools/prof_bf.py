"""Exact kNN on a cfg2-distributed subset, for ncu captures of the tcgen05 kernel."""
import sys
import time

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_1609_07228_b200 as A  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200000
cfg = dict(bench.CONFIGS["cfg2"])
base, _ = bench.gen_data(cfg, n)
vs = A.VectorSet(base)
for rep in range(2):
    A.lib.annk_synchronize()
    t0 = time.perf_counter()
    A.brute_force_knn(vs, None, 100)
    A.lib.annk_synchronize()
    t1 = time.perf_counter()
    print(f"self-mode {n} x {n} top-100: {t1 - t0:.4f} s, {n * n / (t1 - t0) / 1e9:.1f} G pairs/s", flush=True)
A.profile_enable(True)
A.profile_reset()
A.brute_force_knn(vs, None, 100)
A.lib.annk_synchronize()
print({k: round(v, 2) if isinstance(v, float) else v for k, v in A.profile_report().items()}, flush=True)
