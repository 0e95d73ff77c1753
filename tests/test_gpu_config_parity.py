"""GPU parity at the BASELINE configs' own parameters:

* cfg1 in full — 100k x 128 integer mixture, 4 trees leaf 10, K=10, P=30,
  S=10 (R = S: the reference has no separate reverse cap), Dep 4, 8 rounds at
  the reference's DEFAULT min_change_rate (0.001): the build log (iterations
  run, dist_comps and `changes` per round — so the early stop fires at the same
  round) and the final graph equal the CPU oracle's single-worker build, and
  search (top-10, P=50) equals the oracle's on all 1000 queries;
* cfg4 — exact top-100 rows of the 1M x 128 self-mode kNN graph for a seeded
  1000-row sample against the reference library compiled from /root/reference
  (oracle/_ref, the reference's own brute_force_knn);
* cfg2-shaped search — K=100 graph rows with pool sizes 100, 400 and 1000
  (the shared-memory budget paths of the search kernel).
"""
import os

import numpy as np
import pytest

import paper_1609_07228_b200 as A
from oracle import oracle as O
from tests.helpers import mixture, ora

pytestmark = pytest.mark.gpu
CORES = os.cpu_count() or 1


def test_cfg1_full_build_default_early_stop_and_search():
    o = ora()
    n, dim, seed = 100_000, 128, 1
    x = mixture(n, dim, 100, seed)
    q = mixture(1000, dim, 100, seed, stream=2)
    vo = o.vs(x)
    fo = o.build_forest(vo, 4, 10, seed, workers=CORES)
    ids_o, _, log_o, _ = o.build_graph(vo, fo, k=10, conquer_depth=4, pool_cap=30, sample_cap=10, max_iters=8,
                                       strategy=0, seed=seed, workers=1, min_change_rate=0.001)
    fd = A.build_forest(x, 4, 10, seed)
    res = A.build_graph(x, fd, A.BuildParams(k=10, conquer_depth=4, pool_cap=30, sample_cap=10, max_iters=8,
                                             seed=seed, min_change_rate=0.001))
    its = res.stats.iterations
    assert len(its) == len(log_o), "the early stop fires at a different round"
    for row, ro in zip(its, log_o):
        assert row.iteration == int(ro[0])
        assert row.dist_comps == int(ro[2]), f"dist_comps, round {row.iteration}"
        assert row.changes == int(ro[3]), f"changes, round {row.iteration}"
    np.testing.assert_array_equal(res.graph.ids, ids_o)
    # search top-10 with pool 50 over all 1000 queries (cfg1's search setting)
    r = A.GraphSearcher(x, fd, res.graph).search_batch(q, A.SearchParams(10, 50, 50, 4))
    ids_s, d_s, st_s = o.search(vo, fo, ids_o, o.vs(q), 10, 50, 50, 4, workers=CORES)
    np.testing.assert_array_equal(r.ids, ids_s)
    np.testing.assert_array_equal(r.dists.view(np.uint32), d_s.view(np.uint32))
    np.testing.assert_array_equal(r.stats, st_s)


@pytest.mark.skipif(not O.reference_available(), reason="oracle/_ref not built")
def test_cfg4_exact_rows_sample_vs_reference():
    n, dim, k = 1_000_000, 128, 100
    x = mixture(n, dim, 1000, 1)
    rows = np.sort(np.random.default_rng(1).choice(n, 1000, replace=False)).astype(np.uint32)
    ids_d = A.brute_force_rows(x, rows, k)
    ref = O.load("reference")
    ids_q = ref.brute_force(ref.vs(x), ref.vs(np.ascontiguousarray(x[rows])), k + 1, workers=CORES)
    # query mode returns the row itself first (distance 0; no duplicate points here):
    # dropping it gives the self-mode row (eval.cpp:17-29 skips i)
    expect = np.array([r[r != i][:k] for r, i in zip(ids_q, rows)])
    np.testing.assert_array_equal(ids_d, expect)


@pytest.mark.parametrize("P,E", [(100, 8), (400, 32), (1000, 100)])
def test_search_k100_graph_large_pools(P, E):
    o = ora()
    x = mixture(20_000, 128, 100, 3)
    q = mixture(300, 128, 100, 3, stream=2)
    vo = o.vs(x)
    fo = o.build_forest(vo, 8, 8, 3, workers=CORES)
    fd = A.build_forest(x, 8, 8, 3)
    g = A.brute_force_graph(x, 100)
    r = A.GraphSearcher(x, fd, g).search_batch(q, A.SearchParams(100, P, E, 4))
    ids_o, d_o, st_o = o.search(vo, fo, g.ids, o.vs(q), 100, P, E, 4, workers=CORES)
    np.testing.assert_array_equal(r.ids, ids_o)
    np.testing.assert_array_equal(r.dists.view(np.uint32), d_o.view(np.uint32))
    np.testing.assert_array_equal(r.stats, st_o)


def _masked_equal(a, b, sizes, what):
    m = np.arange(a.shape[1])[None, :] < sizes[:, None]
    bad = np.nonzero((np.where(m, a, 0) != np.where(m, b, 0)).any(axis=1))[0]
    assert bad.size == 0, f"{what}: {bad.size} rows differ, first {bad[:5]}"


def test_cfg2_full_size_forest_init_vs_reference_and_round_properties():
    """BASELINE cfg2 at its full size (1M x 128 integer mixture, 8 trees leaf 8, K = P = 100,
    S = 20): the forest and the initial graph (pools, flags, dist_comps) bit-identical to the
    reference run on all host cores (both are independent of the worker count), then two
    NN-descent rounds checked through size-independent properties of the finalized graph."""
    o = O.load("reference") if O.reference_available() else ora()
    n, dim, seed = 1_000_000, 128, 1
    x = mixture(n, dim, 1000, seed)
    vo = o.vs(x)
    fo = o.build_forest(vo, 8, 8, seed, workers=CORES)
    fd = A.build_forest(x, 8, 8, seed)
    for t in range(8):
        td, to = fd.tree(t), fo.tree(t)
        assert td.n_nodes == to.n_nodes and td.leaf_count == to.leaf_count
        np.testing.assert_array_equal(td.split_dim, to.split_dim)
        np.testing.assert_array_equal(td.split_val.view(np.uint32), to.split_val.view(np.uint32))
        np.testing.assert_array_equal(td.left, to.left)
        np.testing.assert_array_equal(td.right, to.right)
        np.testing.assert_array_equal(td.point_index, to.point_index)
    so = o.init_graph(vo, fo, 100, 4, 100, 20, seed, workers=CORES)
    sd = A.init_graph(x, fd, 100, 4, 100, 20, seed)
    s, ids, d, f = sd.pools()
    e = so.export()
    np.testing.assert_array_equal(s, e["sizes"])
    _masked_equal(ids, e["ids"], s, "init pool ids")
    _masked_equal(d.view(np.uint32), e["dists"].view(np.uint32), s, "init pool dists")
    _masked_equal(f, e["flags"], s, "init pool flags")
    assert sd.meta()["dist_comps"] == e["dist_comps"]
    del so, e, ids, d, f
    for _ in range(2):
        A.detail.nn_descent_iteration(sd, x)
    g = A.finalize(sd, x, 100)
    gd = g.dists
    assert (g.ids != np.arange(n, dtype=np.uint32)[:, None]).all(), "a point is its own neighbour"
    key = (gd.view(np.uint32).astype(np.uint64) << np.uint64(32)) | g.ids.astype(np.uint64)
    assert (key[:, 1:] > key[:, :-1]).all(), "rows are not strictly ascending in (dist, id)"
    srt = np.sort(g.ids, axis=1)
    assert (srt[:, 1:] != srt[:, :-1]).all(), "duplicate neighbour ids in a row"
    rows = np.random.default_rng(5).choice(n, 2000, replace=False)
    diff = x[rows].astype(np.int64)[:, None, :] - x[g.ids[rows]].astype(np.int64)
    np.testing.assert_array_equal((diff * diff).sum(axis=2).astype(np.float32).view(np.uint32),
                                  gd[rows].view(np.uint32))
    truth = A.brute_force_rows(x, rows.astype(np.uint32), 100)
    hits = sum(len(np.intersect1d(g.ids[r], truth[j])) for j, r in enumerate(rows))
    assert hits / (len(rows) * 100) >= 0.9, "cfg2 reaches graph accuracy 0.9 after two rounds"
