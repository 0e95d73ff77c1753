import os, sys
sys.path.insert(0, ".")
import numpy as np
import paper_1609_07228_b200 as A
from tests.helpers import ora
rng = np.random.default_rng(5)
x = rng.integers(0, 256, size=(1500, 128)).astype(np.float32)
x[100:400] = x[7]
o = ora()
ids_o, d_o, _ = o.brute_force(o.vs(x), None, 70, workers=8, with_dists=True)
for mode in ("0", "1"):
    os.environ["ANNK_BF_CELLS"] = mode
    ids, d = A.brute_force_knn(x, None, 70, with_dists=True)
    bad = np.where((ids != ids_o).any(axis=1))[0]
    print("mode", mode, "bad rows", len(bad), bad[:20])
    if len(bad):
        r = bad[0]
        print(ids[r][-10:], ids_o[r][-10:], d[r][-5:], d_o[r][-5:])
