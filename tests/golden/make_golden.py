"""Generates tests/golden/golden_small.npz from the UNMODIFIED reference
library (oracle/_ref, compiled from /root/reference by oracle/Makefile).
Run here (where /root/reference exists): python tests/golden/make_golden.py"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402

ref = O.load("reference")
n, dim, seed, trees, leaf, k, dep, P, S, iters = 600, 12, 42, 3, 10, 8, 2, 24, 12, 4
x = ref.gen_synthetic(n, dim, seed)
q = ref.gen_synthetic(25, dim, seed + 1)
vs = ref.vs(x)
f = ref.build_forest(vs, trees, leaf, seed)
out = dict(n=n, dim=dim, seed=seed, trees=trees, leaf=leaf, k=k, dep=dep, P=P, S=S, iters=iters, base=x, queries=q)
for t in range(trees):
    tr = f.tree(t)
    out[f"t{t}_point_index"] = tr.point_index
    out[f"t{t}_split_dim"] = tr.split_dim
    out[f"t{t}_split_val"] = tr.split_val
s = ref.init_graph(vs, f, k, dep, P, S, seed)
for _ in range(iters):
    s.nn_descent_iteration(vs)
e = s.export()
out.update(pool_ids=e["ids"], pool_sizes=e["sizes"], dist_comps=e["dist_comps"])
g = ref.brute_force(vs, None, k, workers=4)
out["exact_ids"] = g
ids, d, st = ref.search(vs, f, g, ref.vs(q), k, 40, 20, 4)
out.update(search_ids=ids, search_stats=st)
np.savez_compressed(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden_small.npz"), **out)
print("wrote golden_small.npz")
