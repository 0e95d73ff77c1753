"""Sweeps search parameters at a bench config: recall@k_return and QPS for
(pool, expansion, trees used, rounds); prints the fastest point with recall >= 0.9."""
import itertools
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_1609_07228_b200 as A  # noqa: E402

cfg = dict(bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg2"])
base, queries = bench.gen_data(cfg)
vs, qs = A.VectorSet(base), A.VectorSet(queries)
f = A.build_forest(vs, cfg["trees"], cfg["leaf"], bench.SEED)
s = A.init_graph(vs, f, cfg["k"], cfg["dep"], cfg["P"], cfg["S"], bench.SEED)
for _ in range(2):
    A.detail.nn_descent_iteration(s, vs)
g = A.finalize(s, vs, cfg["k"])
gt = A.brute_force_knn(vs, qs, cfg["k_return"])
sr = A.GraphSearcher(vs, f, g)
kr = cfg["k_return"]
rows = []
for P, E, T, it in itertools.product([kr], [8, 16, 32, 64, kr], [1, 2, 4, cfg["trees"]], [1, 2, 3, 4]):
    if E > P:
        continue
    p = A.SearchParams(k_return=kr, pool_size=P, expansion=E, iters=it, n_trees_used=T)
    sr.search_batch(qs, p)
    A.lib.annk_synchronize()
    t0 = time.perf_counter()
    r = sr.search_batch(qs, p)
    A.lib.annk_synchronize()
    dt = time.perf_counter() - t0
    rec = float(np.mean([len(np.intersect1d(r.ids[i], gt[i])) / kr for i in range(len(gt))]))
    rows.append((len(gt) / dt, rec, P, E, T, it, float(r.stats[:, 0].mean())))
for q, rec, P, E, T, it, dc in sorted(rows, key=lambda r: -r[0])[:25]:
    print(f"qps {q:12.0f} recall {rec:.4f}  P={P} E={E} trees={T} iters={it} dist_comps/q={dc:.0f}")
ok = [r for r in rows if r[1] >= 0.9]
print("best at recall>=0.9:", max(ok, key=lambda r: r[0]) if ok else None)
