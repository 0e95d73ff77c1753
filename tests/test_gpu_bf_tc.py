"""GPU parity of the tcgen05 exact-kNN kernel (brute_force_tc.cu) against the C
oracle (eval.cpp:17-80 restated) and against the mma.sync kernel it replaces.
Integer-valued d=128 data takes the exact u8 datapath; ids and distances must
be bit-identical, ties broken by id (neighbor_pool.hpp:17-20)."""
import os

import numpy as np
import pytest

import paper_1609_07228_b200 as A
from tests.helpers import mixture, ora

pytestmark = pytest.mark.gpu


def _bf(x, q, k, with_dists=False):
    A.profile_enable(True)
    A.profile_reset()
    r = A.brute_force_knn(x, q, k, with_dists=with_dists)
    names = A.profile_report()
    A.profile_enable(False)
    return r, names


def _mma_sync(x, q, k):
    os.environ["ANNK_BF_MMA_SYNC"] = "1"
    try:
        return A.brute_force_knn(x, q, k, with_dists=True)
    finally:
        del os.environ["ANNK_BF_MMA_SYNC"]


@pytest.mark.parametrize("n,k,seed", [(3000, 100, 1), (1000, 1, 2), (2049, 128, 3), (300, 10, 4), (130, 129 - 2, 5),
                                      (50, 5, 6), (64, 63, 7), (65, 64, 8)])
def test_tc_self_mode_matches_oracle(n, k, seed):
    o = ora()
    x = mixture(n, 128, 12, seed)
    (ids, d), names = _bf(x, None, k, with_dists=True)
    assert any("bf_tc_u8_kernel" in s for s in names), names
    ids_o, d_o, _ = o.brute_force(o.vs(x), None, k, workers=8, with_dists=True)
    np.testing.assert_array_equal(ids, ids_o)
    np.testing.assert_array_equal(d.view(np.uint32), d_o.view(np.uint32))
    ids_m, d_m = _mma_sync(x, None, k)
    np.testing.assert_array_equal(ids, ids_m)


@pytest.mark.parametrize("nq,k", [(57, 100), (256, 10), (300, 64), (1, 5)])
def test_tc_query_mode_split_base(nq, k):
    # few query blocks -> the base range is split over CTAs and merged
    o = ora()
    x = mixture(20000, 128, 40, 9)
    q = mixture(nq, 128, 40, 9, stream=2)
    (ids, d), names = _bf(x, q, k, with_dists=True)
    assert any("bf_tc_u8_kernel" in s for s in names), names
    ids_o, d_o, _ = o.brute_force(o.vs(x), o.vs(q), k, workers=8, with_dists=True)
    np.testing.assert_array_equal(ids, ids_o)
    np.testing.assert_array_equal(d.view(np.uint32), d_o.view(np.uint32))


def test_tc_duplicates_and_extremes():
    # exact duplicates (distance 0 ties ordered by id) and the value extremes 0 / 255
    rng = np.random.default_rng(5)
    x = rng.integers(0, 256, size=(1500, 128)).astype(np.float32)
    x[100:160] = x[7]
    x[200] = 255.0
    x[201] = 0.0
    (ids, d), _ = _bf(x, None, 70, with_dists=True)
    o = ora()
    ids_o, d_o, _ = o.brute_force(o.vs(x), None, 70, workers=8, with_dists=True)
    np.testing.assert_array_equal(ids, ids_o)
    np.testing.assert_array_equal(d.view(np.uint32), d_o.view(np.uint32))


def test_tc_large_self_mode_vs_mma_sync():
    # 50k x 50k top-100: many buffer flushes and several work items per CTA;
    # the mma.sync kernel (itself pinned to the oracle above) is the checker
    x = mixture(50000, 128, 100, 13)
    (ids, d), _ = _bf(x, None, 100, with_dists=True)
    ids_m, d_m = _mma_sync(x, None, 100)
    np.testing.assert_array_equal(ids, ids_m)
    np.testing.assert_array_equal(d.view(np.uint32), d_m.view(np.uint32))
    rows = np.array([0, 1, 4097, 49999, 31337], np.uint32)
    o = ora()
    ids_o = o.brute_force(o.vs(x), o.vs(x[rows]), 101, workers=8)
    for r, i in enumerate(rows):
        np.testing.assert_array_equal(ids[i], [j for j in ids_o[r] if j != i][:100])


def test_tc_rows_subset_shard_mode():
    # brute_force_rows (the sharded ground truth): self exclusion by the row's own id
    x = mixture(7000, 128, 30, 21)
    rows = np.array([0, 1, 63, 64, 6999, 4097, 12, 5000], np.uint32)
    full = A.brute_force_knn(x, None, 100)
    np.testing.assert_array_equal(A.brute_force_rows(x, rows, 100), full[rows])


def _cells(mode):
    class _Ctx:
        def __enter__(self):
            os.environ["ANNK_BF_CELLS"] = mode

        def __exit__(self, *a):
            del os.environ["ANNK_BF_CELLS"]
    return _Ctx()


@pytest.mark.parametrize("n,k,seed", [(3000, 100, 1), (2049, 128, 3), (1000, 10, 4), (777, 1, 5)])
def test_tc_pruned_scan_small_matches_oracle(n, k, seed):
    # the pruned scan (rows and queries grouped by nearest pivot, home tiles first, cells beyond
    # every threshold of a query block dropped) forced at small sizes: same ids and distance bits
    o = ora()
    x = mixture(n, 128, 12, seed)
    with _cells("1"):
        (ids, d), names = _bf(x, None, k, with_dists=True)
    assert any("gather_cells_kernel" in s for s in names), names
    ids_o, d_o, _ = o.brute_force(o.vs(x), None, k, workers=8, with_dists=True)
    np.testing.assert_array_equal(ids, ids_o)
    np.testing.assert_array_equal(d.view(np.uint32), d_o.view(np.uint32))
    # separate query set (its own cell order) and a row subset (self exclusion by original id)
    q = mixture(333, 128, 12, seed, stream=2)
    with _cells("1"):
        idq, dq = A.brute_force_knn(x, q, k, with_dists=True)
        rows = np.array([0, 1, 63, 64, n - 1, n // 2], np.uint32)
        sub = A.brute_force_rows(x, rows, k)
    idq_o, dq_o, _ = o.brute_force(o.vs(x), o.vs(q), k, workers=8, with_dists=True)
    np.testing.assert_array_equal(idq, idq_o)
    np.testing.assert_array_equal(dq.view(np.uint32), dq_o.view(np.uint32))
    np.testing.assert_array_equal(sub, ids[rows])


def test_tc_pruned_scan_duplicates():
    rng = np.random.default_rng(5)
    x = rng.integers(0, 256, size=(1500, 128)).astype(np.float32)
    x[100:400] = x[7]   # more ties at distance 0 than k: ordered by original id
    with _cells("1"):
        ids, d = A.brute_force_knn(x, None, 70, with_dists=True)
    o = ora()
    ids_o, d_o, _ = o.brute_force(o.vs(x), None, 70, workers=8, with_dists=True)
    np.testing.assert_array_equal(ids, ids_o)
    np.testing.assert_array_equal(d.view(np.uint32), d_o.view(np.uint32))


def test_tc_pruned_scan_equals_plain_scan_large():
    # 50k x 50k takes the pruned scan by default; the plain scan is the checker
    x = mixture(50000, 128, 100, 13)
    (ids, d), names = _bf(x, None, 100, with_dists=True)
    assert any("gather_cells_kernel" in s for s in names), names
    with _cells("0"):
        (ids0, d0), names0 = _bf(x, None, 100, with_dists=True)
    assert not any("gather_cells_kernel" in s for s in names0), names0
    np.testing.assert_array_equal(ids, ids0)
    np.testing.assert_array_equal(d.view(np.uint32), d0.view(np.uint32))
    q = mixture(40000, 128, 100, 13, stream=2)
    idq = A.brute_force_knn(x, q, 100)
    with _cells("0"):
        idq0 = A.brute_force_knn(x, q, 100)
    np.testing.assert_array_equal(idq, idq0)


def test_tc_pruned_scan_uniform_rows():
    # no cluster structure: nothing can be pruned, every cell is visited after the home tiles
    rng = np.random.default_rng(11)
    x = rng.integers(0, 256, size=(4000, 128)).astype(np.float32)
    q = rng.integers(0, 256, size=(500, 128)).astype(np.float32)
    o = ora()
    with _cells("1"):
        ids, d = A.brute_force_knn(x, None, 50, with_dists=True)
        idq = A.brute_force_knn(x, q, 50)
    ids_o, d_o, _ = o.brute_force(o.vs(x), None, 50, workers=8, with_dists=True)
    np.testing.assert_array_equal(ids, ids_o)
    np.testing.assert_array_equal(d.view(np.uint32), d_o.view(np.uint32))
    np.testing.assert_array_equal(idq, o.brute_force(o.vs(x), o.vs(q), 50, workers=8))
