"""GPU parity: every hot-path entry point through the C-ABI vs the CPU oracle
(our C restatement, itself pinned to the reference in test_oracle_pin.py) on
identical seeded inputs.  Integer/index results must be bit-exact; distances
are compared bit-for-bit too, because the device computes the reference's
sequential fp32 l2_sq (tolerance 0)."""
import numpy as np
import pytest

import paper_1609_07228_b200 as A
from tests.helpers import assert_pools_equal, assert_trees_equal, mixture, ora

pytestmark = pytest.mark.gpu


# ------------------------------------------------------------ brute force

@pytest.mark.parametrize("n,dim,k,seed", [(2000, 8, 10, 12), (3000, 32, 100, 3), (700, 960, 20, 5)])
def test_brute_force_self_and_query(n, dim, k, seed):
    o = ora()
    x = A.gen_synthetic(n, dim, seed)
    q = A.gen_synthetic(57, dim, seed + 1)
    vo, qo = o.vs(x), o.vs(q)
    ids_o, d_o, c_o = o.brute_force(vo, None, k, workers=8, with_dists=True)
    comps = []
    ids, d = A.brute_force_knn(x, None, k, dist_comps=comps, with_dists=True)
    np.testing.assert_array_equal(ids, ids_o)
    np.testing.assert_array_equal(d.view(np.uint32), d_o.view(np.uint32))
    assert comps[0] == c_o == n * (n - 1)
    ids_q = A.brute_force_knn(x, q, k)
    np.testing.assert_array_equal(ids_q, o.brute_force(vo, qo, k, workers=8))


def test_brute_force_integer_mixture_ties():
    # integer-valued clustered data has many exact distance ties: order by id
    o = ora()
    x = mixture(4000, 128, 20, 7)
    ids = A.brute_force_knn(x, None, 50)
    np.testing.assert_array_equal(ids, o.brute_force(o.vs(x), None, 50, workers=8))


def test_brute_force_edge_cases():
    vs = np.array([[0.0], [1.0], [3.0]], np.float32)  # test_eval.cpp:10-21
    np.testing.assert_array_equal(A.brute_force_knn(vs, None, 1)[:, 0], [1, 0, 1])
    base = A.gen_synthetic(40, 6, 4)  # test_eval.cpp:23-33
    ids, d = A.brute_force_knn(base, base[17:18], 3, with_dists=True)
    assert ids[0, 0] == 17 and d[0, 0] == 0.0
    small = A.gen_synthetic(5, 2, 1)  # test_eval.cpp:51-58
    with pytest.raises(A.InvalidArgument):
        A.brute_force_knn(small, None, 5)
    A.brute_force_knn(small, None, 4)
    q = A.gen_synthetic(2, 2, 2)
    A.brute_force_knn(small, q, 5)
    with pytest.raises(A.InvalidArgument):
        A.brute_force_knn(small, q, 6)
    # k beyond the tiled path (large-k route) still exact
    x = A.gen_synthetic(900, 5, 9)
    o = ora()
    np.testing.assert_array_equal(A.brute_force_knn(x, None, 899), o.brute_force(o.vs(x), None, 899, workers=8))


def test_brute_force_rows_sample():
    x = mixture(5000, 128, 30, 11)
    rows = np.array([0, 17, 4999, 2500, 33], np.uint32)
    full = A.brute_force_knn(x, None, 20)
    np.testing.assert_array_equal(A.brute_force_rows(x, rows, 20), full[rows])


# ----------------------------------------------------------------- forest

@pytest.mark.parametrize("n,dim,trees,leaf,seed", [
    (10000, 128, 8, 10, 1),    # test_kd_forest.cpp:71-76 shape
    (500, 12, 4, 10, 1234),    # test_kd_forest.cpp:78-96
    (2000, 8, 2, 10, 55),
    (1, 4, 3, 10, 5), (7, 4, 2, 10, 5), (300, 6, 2, 5, 4),
    (20000, 32, 4, 8, 3),
])
def test_forest_bit_identical(n, dim, trees, leaf, seed):
    o = ora()
    x = A.gen_synthetic(n, dim, seed)
    fo = o.build_forest(o.vs(x), trees, leaf, seed)
    fd = A.build_forest(x, trees, leaf, seed)
    for t in range(trees):
        assert_trees_equal(fd.tree(t), fo.tree(t))


def test_forest_integer_mixture_with_duplicates():
    # clipped integer data: many equal values -> degenerate splits (even_split fallback)
    o = ora()
    x = mixture(30000, 128, 50, 2)
    x[:2000] = x[0]  # a block of exact duplicates
    fo = o.build_forest(o.vs(x), 4, 8, 9)
    fd = A.build_forest(x, 4, 8, 9)
    evens = 0
    for t in range(4):
        td = fd.tree(t)
        assert_trees_equal(td, fo.tree(t))
        evens += int(td.even_split.sum())
    assert evens > 0


@pytest.mark.parametrize("n,dim,trees,leaf,dups", [
    (12000, 960, 2, 8, 0),    # wide rows: staged tiles of 152 points
    (5000, 2500, 1, 8, 0),    # rows too wide to stage: warp path gathers
    (20000, 64, 2, 100, 0),   # leaf_cap above the tile floor
    (24000, 32, 2, 8, 9000),  # duplicate block > kWarpSubtree: block-path even split
])
def test_forest_integer_mixture_shapes(n, dim, trees, leaf, dups):
    o = ora()
    x = mixture(n, dim, 30, 6)
    if dups:
        x[:dups] = x[1]
    fo = o.build_forest(o.vs(x), trees, leaf, 21)
    fd = A.build_forest(x, trees, leaf, 21)
    for t in range(trees):
        assert_trees_equal(fd.tree(t), fo.tree(t))


def test_forest_float_mixture_inexact_sums():
    # [0,1] clipped Gaussian floats (cfg3-like) exercise the serial-sum fallback
    o = ora()
    x = mixture(6000, 96, 20, 4, lo=0.05, hi=0.35, sd=0.05, clip=(0.0, 1.0), rnd=False)
    x[::7, 3] = np.float32(1e-12)  # tiny magnitudes force inexact partial sums
    fo = o.build_forest(o.vs(x), 3, 10, 1)
    fd = A.build_forest(x, 3, 10, 1)
    for t in range(3):
        assert_trees_equal(fd.tree(t), fo.tree(t))


def test_search_leaves_and_descend():
    o = ora()
    x = A.gen_synthetic(1000, 8, 17)
    q = A.gen_synthetic(20, 8, 18)
    fo = o.build_forest(o.vs(x), 2, 10, 99)
    fd = A.build_forest(x, 2, 10, 99)
    for t in range(2):
        for nl in (1, 4, 17, 10000):
            got = fd.search_leaves(t, q, nl)
            for i in range(len(q)):
                np.testing.assert_array_equal(got[i], fo.search_leaves(t, q[i], nl))
        tr = fd.tree(t)
        rng = np.random.default_rng(5)
        starts = rng.integers(0, tr.n_nodes, size=len(q)).astype(np.uint32)
        out = fd.descend_from(t, q, starts)
        for i in range(len(q)):
            assert out[i] == fo.descend_from(t, q[i], int(starts[i]))


# --------------------------------------------------------- init + refine

def _pair(x, trees, leaf, seed, k, dep, P, S):
    o = ora()
    vo = o.vs(x)
    fo = o.build_forest(vo, trees, leaf, seed)
    so = o.init_graph(vo, fo, k, dep, P, S, seed)
    fd = A.build_forest(x, trees, leaf, seed)
    sd = A.init_graph(x, fd, k, dep, P, S, seed)
    return o, vo, so, sd


@pytest.mark.parametrize("n,dim,trees,leaf,k,dep,P,S,seed,iters", [
    (2000, 32, 4, 10, 10, 4, 30, 20, 1, 8),     # test_graph_build.cpp:152-192
    (500, 8, 4, 10, 10, 2, 30, 20, 23, 3),      # :194-212
    (3000, 128, 8, 8, 20, 4, 40, 10, 7, 4),
    (150, 4, 2, 4, 5, 0, 20, 20, 3, 6),         # small sets / Dep 0
])
def test_init_and_nn_descent_bit_exact(n, dim, trees, leaf, k, dep, P, S, seed, iters):
    x = A.gen_synthetic(n, dim, seed)
    o, vo, so, sd = _pair(x, trees, leaf, seed, k, dep, P, S)
    e = assert_pools_equal(sd, so)
    assert sd.meta()["dist_comps"] == e["dist_comps"]
    for it in range(iters):
        co = so.nn_descent_iteration(vo)
        cd = A.detail.nn_descent_iteration(sd, x)
        assert cd == co, f"changes, iteration {it}"  # the reference's sequential accepted inserts
        e = assert_pools_equal(sd, so)
        m = sd.meta()
        assert m["dist_comps"] == e["dist_comps"], f"iteration {it}"
        assert m["iteration"] == e["iteration"]
        assert m["last_changes"] == co
        for which in range(4):
            dl, ol = sd.lists(which), so.lists(which)
            for i in range(n):
                np.testing.assert_array_equal(dl[i], ol[i], err_msg=f"list {which} row {i} iter {it}")


@pytest.mark.parametrize("n,dim,trees,leaf,P,seed", [
    (1500, 960, 8, 10, 100, 4),   # cfg3-shaped wide rows (batched row loads)
    (1001, 50, 4, 10, 30, 8),     # dim not a multiple of 32 (load-batch tail)
])
def test_wide_fp32_init_bit_exact(n, dim, trees, leaf, P, seed):
    x = A.gen_synthetic(n, dim, seed)
    o, vo, so, sd = _pair(x, trees, leaf, seed, 10, 4, P, 10)
    e = assert_pools_equal(sd, so)
    assert sd.meta()["dist_comps"] == e["dist_comps"]


@pytest.mark.parametrize("integer", [True, False])
def test_piecewise_join_round_bit_exact(integer, monkeypatch):
    # a round whose offers exceed one join launch (very large N) is joined in
    # ascending source ranges, each piece's offers replayed before the next: pools,
    # flags, dist_comps and changes must still equal the oracle's (forced here by a
    # tiny offer limit)
    x = mixture(6000, 128, 30, 5) if integer else A.gen_synthetic(6000, 24, 5)
    o, vo, so, sd = _pair(x, 4, 10, 5, 10, 4, 30, 10)
    monkeypatch.setenv("ANNK_JOIN_MAX_OFFERS", "20000")
    for it in range(3):
        co = so.nn_descent_iteration(vo)
        assert A.detail.nn_descent_iteration(sd, x) == co, f"changes, iteration {it}"
        e = assert_pools_equal(sd, so)
        assert sd.meta()["dist_comps"] == e["dist_comps"], f"iteration {it}"


def test_integer_mixture_refine_and_finalize():
    x = mixture(20000, 128, 40, 3)
    o, vo, so, sd = _pair(x, 4, 10, 3, 10, 4, 30, 10)
    for _ in range(3):
        assert A.detail.nn_descent_iteration(sd, x) == so.nn_descent_iteration(vo)
    assert_pools_equal(sd, so)
    ids_o, d_o = so.finalize(vo, 10)
    g = A.finalize(sd, x, 10)
    np.testing.assert_array_equal(g.ids, ids_o)
    np.testing.assert_array_equal(g.dists.view(np.uint32), d_o.view(np.uint32))
    gt = A.brute_force_knn(x, None, 10)
    assert abs(A.detail.pool_topk_accuracy(sd, gt) - so.pool_topk_accuracy(gt)) == 0.0


def test_rebuild_and_union_separately():
    x = A.gen_synthetic(500, 8, 23)
    o, vo, so, sd = _pair(x, 4, 10, 23, 10, 2, 30, 20)
    for _ in range(2):
        so.nn_descent_iteration(vo)
        A.detail.nn_descent_iteration(sd, x)
    so.rebuild_sample_lists()
    A.detail.rebuild_sample_lists(sd)
    for which in range(4):
        dl, ol = sd.lists(which), so.lists(which)
        for i in range(500):
            np.testing.assert_array_equal(dl[i], ol[i])
    m = sd.meta()
    for i, (a, b) in enumerate(zip(sd.g_new, sd.g_old)):
        assert len(a) <= m["sample_cap"] and len(a) + len(b) <= m["pool_cap"]
    so.union_reverse_lists()
    A.detail.union_reverse_lists(sd)
    for which in (0, 1):
        dl, ol = sd.lists(which), so.lists(which)
        for i in range(500):
            np.testing.assert_array_equal(dl[i], ol[i])
    assert_pools_equal(sd, so)


def test_exact_old_state_is_fixed_point():
    # test_graph_build.cpp:121-137
    x = A.gen_synthetic(120, 6, 19)
    gt, d = A.brute_force_knn(x, None, 10, with_dists=True)
    sd = A.RefineState.from_pools(120, 10, 10, 10, 1, np.full(120, 10, np.uint32), gt, d,
                                  np.zeros((120, 10), np.uint8))
    before = sd.pools()[1].copy()
    assert A.detail.nn_descent_iteration(sd, x) == 0
    assert sd.meta()["dist_comps"] == 0
    np.testing.assert_array_equal(sd.pools()[1], before)


def test_two_point_fixed_point_and_errors():
    x = A.gen_synthetic(2, 3, 2)  # test_graph_build.cpp:139-150
    f = A.build_forest(x, 1, 4, 2)
    s = A.init_graph(x, f, 1, 0, 1, 5, 2)
    _, ids, _, _ = s.pools()
    assert ids[0, 0] == 1 and ids[1, 0] == 0
    assert A.detail.nn_descent_iteration(s, x) == 0
    y = A.gen_synthetic(300, 8, 51)
    fy = A.build_forest(y, 4, 10, 51)
    sy = A.init_graph(y, fy, 10, 4, 10, 10, 51)
    with pytest.raises(A.InvalidArgument):
        A.finalize(sy, y, 11)
    with pytest.raises(A.InvalidArgument):
        A.init_graph(y, fy, 10, 4, 5, 10, 51)  # pool_cap < k


# ----------------------------------------------------------------- search

@pytest.mark.parametrize("P,E,I,ntu", [(100, 50, 4, 0), (60, 30, 0, 0), (200, 200, 4, 2), (20, 20, 64, 0),
                                       (300, 10, 8, 0)])
def test_search_bit_exact(P, E, I, ntu):
    o = ora()
    x = A.gen_synthetic(2000, 16, 21)
    q = A.gen_synthetic(50, 16, 22)
    vo = o.vs(x)
    fo = o.build_forest(vo, 8, 10, 21)
    fd = A.build_forest(x, 8, 10, 21)
    g = A.brute_force_graph(x, 10)
    ids_o, d_o, st_o = o.search(vo, fo, g.ids, o.vs(q), 10, P, E, I, ntu)
    r = A.GraphSearcher(x, fd, g).search_batch(q, A.SearchParams(10, P, E, I, ntu))
    np.testing.assert_array_equal(r.ids, ids_o)
    np.testing.assert_array_equal(r.dists.view(np.uint32), d_o.view(np.uint32))
    np.testing.assert_array_equal(r.stats, st_o)


def test_search_random_init_and_fallback():
    o = ora()
    x = A.gen_synthetic(600, 8, 33)
    q = A.gen_synthetic(8, 8, 34)
    vo = o.vs(x)
    g = A.brute_force_graph(x, 10)
    for P, E, I in [(600, 600, 4), (12, 12, 0), (100, 50, 4)]:
        ids_o, d_o, st_o = o.search(vo, None, g.ids, o.vs(q), 10 if P >= 10 else P, P, E, I, random_init=True,
                                    seed=4242)
        r = A.GraphSearcher(x, None, g).search_batch(q, A.SearchParams(10 if P >= 10 else P, P, E, I, seed=4242),
                                                     random_init=True)
        np.testing.assert_array_equal(r.ids, ids_o)
        np.testing.assert_array_equal(r.stats, st_o)
    # disconnected graph -> fallback scan (search.cpp:95-106)
    gbad = np.zeros((600, 2), np.uint32)
    f = A.build_forest(x, 1, 600, 3)
    fo = o.build_forest(vo, 1, 600, 3)
    ids_o, d_o, st_o = o.search(vo, fo, gbad, o.vs(q), 5, 5, 0, 2)
    r = A.GraphSearcher(x, f, gbad).search_batch(q, A.SearchParams(5, 5, 0, 2))
    np.testing.assert_array_equal(r.ids, ids_o)
    np.testing.assert_array_equal(r.stats, st_o)


def test_search_validation():
    x = A.gen_synthetic(50, 4, 66)
    f = A.build_forest(x, 8, 10, 66)
    g = A.brute_force_graph(x, 5)
    s = A.GraphSearcher(x, f, g)
    q = A.gen_synthetic(2, 4, 67)
    for p in (A.SearchParams(k_return=0), A.SearchParams(k_return=20, pool_size=10),
              A.SearchParams(k_return=5, pool_size=10, expansion=11)):
        with pytest.raises(A.InvalidArgument):
            s.search_batch(q, p)
    s.search_batch(q, A.SearchParams(k_return=5, pool_size=10, expansion=10))
    with pytest.raises(A.InvalidArgument):
        s.search(np.zeros(3, np.float32), A.SearchParams(5, 10, 10))
    with pytest.raises(A.InvalidArgument):
        A.GraphSearcher(A.gen_synthetic(10, 4, 1), None, g)


# ------------------------------------------------------ exact u8 datapath

@pytest.mark.parametrize("u8", [True, False])
def test_integer_data_both_datapaths_bit_exact(u8, monkeypatch):
    """Integer-valued data runs the exact u8/dp4a datapath by default; forcing
    the fp32 path (ANNK_DISABLE_U8=1) must give the very same bits, and both must
    equal the oracle (pools, lists, dist_comps, brute force, search)."""
    if not u8:
        monkeypatch.setenv("ANNK_DISABLE_U8", "1")
    o = ora()
    x = mixture(6000, 128, 30, 5)
    q = mixture(80, 128, 30, 5, stream=2)
    vo = o.vs(x)
    ids_o, d_o, _ = o.brute_force(vo, None, 30, workers=8, with_dists=True)
    ids, d = A.brute_force_knn(x, None, 30, with_dists=True)
    np.testing.assert_array_equal(ids, ids_o)
    np.testing.assert_array_equal(d.view(np.uint32), d_o.view(np.uint32))
    np.testing.assert_array_equal(A.brute_force_knn(x, q, 30), o.brute_force(vo, o.vs(q), 30, workers=8))
    rows = np.array([5, 77, 5999], np.uint32)
    np.testing.assert_array_equal(A.brute_force_rows(x, rows, 30), ids_o[rows])
    o2, vo2, so, sd = _pair(x, 4, 8, 5, 20, 4, 40, 10)
    for _ in range(3):
        assert A.detail.nn_descent_iteration(sd, x) == so.nn_descent_iteration(vo2)
        e = assert_pools_equal(sd, so)
        assert sd.meta()["dist_comps"] == e["dist_comps"]
    g = A.finalize(sd, x, 20)
    f = A.build_forest(x, 4, 8, 5)
    fo = o.build_forest(vo, 4, 8, 5)
    r = A.GraphSearcher(x, f, g).search_batch(q, A.SearchParams(20, 60, 40, 4))
    ids_s, d_s, st_s = o.search(vo, fo, g.ids, o.vs(q), 20, 60, 40, 4)
    np.testing.assert_array_equal(r.ids, ids_s)
    np.testing.assert_array_equal(r.dists.view(np.uint32), d_s.view(np.uint32))
    np.testing.assert_array_equal(r.stats, st_s)


def test_dataset_rejects_non_finite():
    x = A.gen_synthetic(100, 5, 1)
    x[37, 2] = np.nan
    with pytest.raises(A.InvalidArgument):
        A.VectorSet(x)
    x[37, 2] = np.inf
    with pytest.raises(A.InvalidArgument):
        A.VectorSet(x)


# ------------------------------------------------- init_random (random-descent)

@pytest.mark.parametrize("n,dim,k,P,S,seed,integer", [
    (2000, 16, 10, 30, 10, 5, False),
    (60, 8, 5, 80, 10, 2, False),        # pool_cap >= n-1: every other point
    (3000, 128, 10, 40, 10, 7, True),    # u8 datapath
    (500, 12, 10, 30, 20, 1234, False),
])
def test_init_random_bit_exact(n, dim, k, P, S, seed, integer):
    o = ora()
    x = mixture(n, dim, 20, seed) if integer else A.gen_synthetic(n, dim, seed)
    so = o.init_random(o.vs(x), k, P, S, seed)
    sd = A.init_random(x, k, P, S, seed)
    e = assert_pools_equal(sd, so)
    assert sd.meta()["dist_comps"] == e["dist_comps"]
    vo = o.vs(x)
    for _ in range(2):  # random-descent = init_random + NN-descent rounds
        assert A.detail.nn_descent_iteration(sd, x) == so.nn_descent_iteration(vo)
        e = assert_pools_equal(sd, so)
        assert sd.meta()["dist_comps"] == e["dist_comps"]


@pytest.mark.parametrize("n,dim,k,nq", [(5000, 128, 100, 300), (3000, 40, 10, 77), (700, 16, 128, 0), (2100, 100, 7, 0)])
def test_brute_force_tensor_core_path_matches_dp4a_and_oracle(n, dim, k, nq):
    import os
    x = mixture(n, dim, 25, 8)
    q = mixture(nq, dim, 25, 8, stream=2) if nq else None
    ids_mma, d_mma = A.brute_force_knn(x, q, k, with_dists=True)
    os.environ["ANNK_BF_DP4A"] = "1"
    try:
        ids_cc, d_cc = A.brute_force_knn(x, q, k, with_dists=True)
    finally:
        del os.environ["ANNK_BF_DP4A"]
    np.testing.assert_array_equal(ids_mma, ids_cc)
    np.testing.assert_array_equal(d_mma.view(np.uint32), d_cc.view(np.uint32))
    o = ora()
    ids_o = o.brute_force(o.vs(x), o.vs(q) if nq else None, k)
    np.testing.assert_array_equal(ids_mma, ids_o)


@pytest.mark.parametrize("dim", [960, 1000])
def test_wide_fp32_rows_join_bit_exact(dim):
    # wide float rows (cfg3 shape; 1000 = a partial last 64-float chunk): the join streams
    # the rows from L2 (join_kernel<kModeWide>)
    o = ora()
    x = mixture(1500, dim, 12, 3, lo=0.05, hi=0.35, sd=0.05, clip=(0.0, 1.0), rnd=False)
    vo = o.vs(x)
    fo = o.build_forest(vo, 3, 10, 3)
    so = o.init_graph(vo, fo, 10, 4, 30, 10, 3)
    fd = A.build_forest(x, 3, 10, 3)
    sd = A.init_graph(x, fd, 10, 4, 30, 10, 3)
    assert_pools_equal(sd, so)
    for _ in range(3):
        assert A.detail.nn_descent_iteration(sd, x) == so.nn_descent_iteration(vo)
        e = assert_pools_equal(sd, so)
        assert sd.meta()["dist_comps"] == e["dist_comps"]


@pytest.mark.parametrize("n,dim,trees,integer,dups", [
    (100000, 8, 2, False, 0),      # fp32 path: nodes > 32k points are split by the whole CTA cluster
    (80000, 32, 2, True, 0),       # u8 path
    (90000, 16, 1, True, 40000),   # a 40k duplicate block: degenerate split of a cluster node
])
def test_forest_cluster_split_bit_identical(n, dim, trees, integer, dups):
    o = ora()
    x = mixture(n, dim, 40, 5) if integer else A.gen_synthetic(n, dim, 5)
    if dups:
        x[:dups] = x[7]
    fo = o.build_forest(o.vs(x), trees, 8, 13)
    fd = A.build_forest(x, trees, 8, 13)
    for t in range(trees):
        assert_trees_equal(fd.tree(t), fo.tree(t))


@pytest.mark.gpu
def test_forest_import_roundtrip_reference_trees_and_validation():
    # annk_forest_import (the AKF1 load path, kd_forest.cpp:332-372): export -> import is the
    # identity, a forest built by the CPU reference drives the device init bit-exactly, and
    # malformed trees are rejected with InvalidArgument
    o = ora()
    n, dim, trees, leaf, seed = 3000, 32, 4, 8, 4
    x = A.gen_synthetic(n, dim, seed)
    fd = A.build_forest(x, trees, leaf, seed)
    fi = A.KdForest.from_trees(n, dim, leaf, seed, fd.trees)
    for t in range(trees):
        a, b = fd.tree(t), fi.tree(t)
        assert (a.root, a.leaf_count, a.max_depth) == (b.root, b.leaf_count, b.max_depth)
        for f in ("split_dim", "left", "right", "depth", "even_split", "point_index"):
            np.testing.assert_array_equal(getattr(a, f), getattr(b, f), err_msg=f)
        np.testing.assert_array_equal(a.split_val.view(np.uint32), b.split_val.view(np.uint32))
    vo = o.vs(x)
    fo = o.build_forest(vo, trees, leaf, seed)
    fref = A.KdForest.from_trees(n, dim, leaf, seed, [fo.tree(t) for t in range(trees)])
    so = o.init_graph(vo, fo, 10, 4, 30, 20, seed)
    sd = A.init_graph(x, fref, 10, 4, 30, 20, seed)
    e = assert_pools_equal(sd, so)
    assert sd.meta()["dist_comps"] == e["dist_comps"]

    packed = A.KdForest.pack_trees(fd.trees)
    m0 = int(packed["node_counts"][0])
    internal = int(np.nonzero(packed["split_dim"][:m0] != 0xffffffff)[0][0])
    leafi = int(np.nonzero(packed["split_dim"][:m0] == 0xffffffff)[0][0])

    def bad(key, idx, val, match):
        p = {k: v.copy() for k, v in packed.items()}
        p[key][idx] = val
        with pytest.raises(A.InvalidArgument, match=match):
            A.KdForest.import_packed(n, dim, leaf, seed, p)

    bad("split_dim", internal, dim, "split dimension")
    bad("left", internal, m0 + 3, "child id")
    bad("right", leafi, n + 1, "leaf range")
    bad("roots", 0, m0, "bad root")
    bad("node_counts", 0, 0, "node count")


@pytest.mark.parametrize("n,dim,k,P,seed,integer", [(2000, 16, 10, 30, 5, False), (3000, 128, 10, 40, 7, True)])
def test_nn_expansion_iteration_bit_exact(n, dim, k, P, seed, integer):
    # graph_build.cpp:164-207 (the NN-expansion baseline): pools, flags (flag_new and
    # `checked`), changes and dist_comps per round equal the oracle's
    o = ora()
    x = mixture(n, dim, 20, seed) if integer else A.gen_synthetic(n, dim, seed)
    vo = o.vs(x)
    so = o.init_random(vo, k, P, 10, seed)
    sd = A.init_random(x, k, P, 10, seed)
    for it in range(3):
        co = so.nn_expansion_iteration(vo)
        assert A.detail.nn_expansion_iteration(sd, x) == co, f"changes, round {it}"
        e = assert_pools_equal(sd, so)
        assert sd.meta()["dist_comps"] == e["dist_comps"], f"round {it}"
    # a descent round after expansion keeps the `checked` bits (mixed use of one state)
    assert A.detail.nn_descent_iteration(sd, x) == so.nn_descent_iteration(vo)
    assert_pools_equal(sd, so)


def test_distance_entry_points():
    # dataset.hpp:67-77 on the device: bit-exact to the reference's sequential chain
    o = ora()
    x = A.gen_synthetic(300, 37, 3)
    q = A.gen_synthetic(1, 37, 4)[0]
    a = np.arange(300, dtype=np.uint32)
    b = (a * 7 + 3) % 300
    d = A.dist_sq(x, a, b)
    for i in (0, 17, 299):
        assert d[i] == o.l2_sq(x[a[i]], x[b[i]])
        assert A.l2_sq(x[a[i]], x[b[i]]) == d[i]
    dq = A.dist_sq_q(x, q, a)
    assert all(dq[i] == o.l2_sq(q, x[i]) for i in (0, 5, 299))
    assert A.dist_sq(x, 5, 9) == A.dist_sq(x, 9, 5)  # symmetric (test_dataset.cpp:211)
    with pytest.raises(A.OutOfRange):
        A.dist_sq(x, 0, 300)
    with pytest.raises(A.OutOfRange):
        A.dist_sq_q(x, q, 300)


@pytest.mark.gpu
def test_hub_reverse_lists_bit_exact():
    """Two hubs (the centres of shells of 9000 and 1000 points in 64 dimensions: each is its
    shell's nearest neighbour) give reverse lists of every size class of the device's list
    sort: registers (<= 256 ids), one CTA in shared memory (<= 8192) and the segmented-sort
    fallback (the 9000-point hub), in the new and in the old lists."""
    rng = np.random.default_rng(3)
    dim = 64

    def shell(c, r, m):
        u = rng.normal(size=(m, dim))
        u /= np.linalg.norm(u, axis=1, keepdims=True)
        return c + r * u

    c0, c1 = np.full(dim, 100.0), np.full(dim, -100.0)
    x = np.vstack([c0[None], c1[None], shell(c0, 10.0, 9000), shell(c1, 10.0, 1000),
                   rng.normal(size=(398, dim)) * 5]).astype(np.float32)
    n = len(x)
    o, vo, so, sd = _pair(x, 4, 10, 7, 10, 2, 40, 40)
    longest = 0
    for it in range(4):
        co = so.nn_descent_iteration(vo)
        cd = A.detail.nn_descent_iteration(sd, x)
        assert cd == co, f"changes, iteration {it}"
        for which in range(4):
            dl, ol = sd.lists(which), so.lists(which)
            for i in range(n):
                np.testing.assert_array_equal(dl[i], ol[i], err_msg=f"list {which} row {i} iter {it}")
            if which >= 2:
                longest = max(longest, max(len(a) for a in ol))
        assert_pools_equal(sd, so)
    assert longest > 8192, "the data no longer produces a hub list beyond the shared-memory sort"


@pytest.mark.gpu
def test_brute_force_caller_owned_outputs():
    x = A.gen_synthetic(700, 12, 9)
    ids, d = A.brute_force_knn(x, None, 7, with_dists=True)
    oi, od = np.full((700, 7), 0xffffffff, np.uint32), np.zeros((700, 7), np.float32)
    ri, rd = A.brute_force_knn(x, None, 7, out_ids=oi, out_dists=od)
    assert ri is oi and rd is od
    np.testing.assert_array_equal(oi, ids)
    np.testing.assert_array_equal(od.view(np.uint32), d.view(np.uint32))
    with pytest.raises(A.InvalidArgument):
        A.brute_force_knn(x, None, 7, out_ids=np.zeros((700, 6), np.uint32))
    with pytest.raises(A.InvalidArgument):
        A.brute_force_knn(x, None, 7, out_ids=np.zeros((700, 7), np.int64))


@pytest.mark.parametrize("n,integer,pieces", [(70000, True, False), (70000, False, False), (6000, True, True)])
def test_last_round_fused_with_finalize_bit_exact(n, integer, pieces, monkeypatch):
    # nn_descent_iteration_finalize (chunked replay overlapped with the row copies) must
    # leave the oracle's changes, dist_comps, pools and graph rows -- also through its
    # piecewise-round fallback and through build_graph's last round
    x = mixture(n, 128, 40, 11) if integer else A.gen_synthetic(n, 24, 11)
    o, vo, so, sd = _pair(x, 4, 10, 5, 10, 4, 30, 10)
    if pieces:
        monkeypatch.setenv("ANNK_JOIN_MAX_OFFERS", "20000")
    assert A.detail.nn_descent_iteration(sd, x) == so.nn_descent_iteration(vo)
    co = so.nn_descent_iteration(vo)
    comps_o = so.export()["dist_comps"]  # after the round, before finalize fills sparse pools
    ch, comps, g = A.detail.nn_descent_iteration_finalize(sd, x, 10)
    assert ch == co and comps == comps_o
    ids_o, d_o = so.finalize(vo, 10)
    np.testing.assert_array_equal(g.ids, ids_o)
    np.testing.assert_array_equal(g.dists.view(np.uint32), d_o.view(np.uint32))
    e = assert_pools_equal(sd, so)
    assert sd.meta()["dist_comps"] == e["dist_comps"]
    if not pieces:
        f = A.build_forest(x, 4, 10, 5)
        r = A.build_graph(x, f, A.BuildParams(k=10, conquer_depth=4, pool_cap=30, sample_cap=10, max_iters=2,
                                              seed=5))
        np.testing.assert_array_equal(r.graph.ids, ids_o)
        np.testing.assert_array_equal(r.graph.dists.view(np.uint32), d_o.view(np.uint32))
        assert r.stats.iterations[-1].changes == co and r.stats.iterations[-1].dist_comps == comps
        assert r.stats.dist_comps == e["dist_comps"]
