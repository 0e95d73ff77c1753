"""Times the search at given (P, E, I) points at a bench config: kernel time per
batch from annk_profile (median of 5) and recall@k_return.
python tools/search_point.py [cfg] P:E:I [P:E:I ...]"""
import statistics
import sys

import numpy as np

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_1609_07228_b200 as A  # noqa: E402

cfg = dict(bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg2"])
pts = [tuple(int(v) for v in p.split(":")) for p in (sys.argv[2:] or ["100:8:4", "100:16:1"])]
base, queries = bench.gen_data(cfg)
vs, qs = A.VectorSet(base), A.VectorSet(queries)
f = A.build_forest(vs, cfg["trees"], cfg["leaf"], bench.SEED)
s = A.init_graph(vs, f, cfg["k"], cfg["dep"], cfg["P"], cfg["S"], bench.SEED)
for _ in range(2):
    A.detail.nn_descent_iteration(s, vs)
g = A.finalize(s, vs, cfg["k"])
kr = cfg["k_return"]
gt = A.brute_force_knn(vs, qs, kr)
sr = A.GraphSearcher(vs, f, g)
for P, E, I in pts:
    p = A.SearchParams(k_return=kr, pool_size=P, expansion=E, iters=I)
    ms = []
    for rep in range(6):
        A.profile_reset()
        A.profile_enable(True)
        r = sr.search_batch(qs, p)
        A.profile_enable(False)
        prof = A.profile_report()
        if rep:
            ms.append(sum(v[1] for k, v in prof.items() if k.startswith("search_kernel")))
    rec = float(np.mean([len(np.intersect1d(r.ids[i], gt[i])) / kr for i in range(len(gt))]))
    km = statistics.median(ms)
    print(f"P={P} E={E} I={I}: kernel {km:.3f} ms = {len(gt) / km * 1e3 / 1e6:.2f} M QPS, recall {rec:.4f}, "
          f"dist_comps/q {float(r.stats[:, 0].mean()):.0f}", flush=True)
