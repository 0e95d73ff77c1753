"""GPU parity of the fp32 exact-kNN path on the tensor cores
(brute_force_f32_tc.cu: bf16x3 tcgen05 candidates under a certified error
bound, then an exact re-rank with the reference's sequential fp32 chain)
against the C oracle (eval.cpp:17-80 restated).  Ids AND distances must be
bit-identical, ties broken by id (neighbor_pool.hpp:17-20)."""
import os

import numpy as np
import pytest

import paper_1609_07228_b200 as A
from tests.helpers import mixture, ora

pytestmark = pytest.mark.gpu


def _bf(x, q, k, rows=None):
    A.profile_enable(True)
    A.profile_reset()
    if rows is None:
        r = A.brute_force_knn(x, q, k, with_dists=True)
    else:
        r = A.brute_force_rows(x, rows, k, with_dists=True)
    names = A.profile_report()
    A.profile_enable(False)
    return r, names


def _fmix(n, dim, centers, seed, stream=1):
    # cfg3's distribution: centres uniform in [0.05, 0.35]^d, sd 0.05, clipped to [0, 1], not rounded
    return mixture(n, dim, centers, seed, stream=stream, lo=0.05, hi=0.35, sd=0.05, clip=(0.0, 1.0), rnd=False)


def _check(x, q, k, ids, d):
    o = ora()
    ids_o, d_o, _ = o.brute_force(o.vs(x), None if q is None else o.vs(q), k, workers=8, with_dists=True)
    np.testing.assert_array_equal(ids, ids_o)
    np.testing.assert_array_equal(d.view(np.uint32), d_o.view(np.uint32))


def _ran(names, kernel):
    return any(kernel in s for s in names)


@pytest.mark.parametrize("n,dim,k,seed", [(3000, 128, 100, 1), (2000, 960, 100, 2), (1000, 33, 10, 3),
                                          (600, 100, 128, 4), (300, 64, 1, 5), (257, 200, 50, 6), (40, 8, 39, 7)])
def test_f32_tc_self_mode_matches_oracle(n, dim, k, seed):
    x = _fmix(n, dim, 10, seed)
    (ids, d), names = _bf(x, None, k)
    assert _ran(names, "bf_tc_f32_kernel") and _ran(names, "rerank_kernel"), names
    _check(x, None, k, ids, d)


@pytest.mark.parametrize("nq,k", [(57, 100), (1, 5), (300, 64), (129, 128)])
def test_f32_tc_query_mode_split_base(nq, k):
    # few query blocks -> the base range is split over CTAs; lists of all slices re-ranked together
    x = _fmix(20000, 960, 40, 9)
    q = _fmix(nq, 960, 40, 9, stream=2)
    (ids, d), names = _bf(x, q, k)
    assert _ran(names, "bf_tc_f32_kernel"), names
    _check(x, q, k, ids, d)


def test_f32_tc_uniform_and_signed_values():
    # the reference's uniform fixtures and signed values of mixed magnitude
    rng = np.random.default_rng(11)
    x = rng.uniform(0.0, 1.0, size=(4000, 128)).astype(np.float32)
    (ids, d), _ = _bf(x, None, 20)
    _check(x, None, 20, ids, d)
    y = (rng.standard_normal((3000, 50)) * np.exp2(rng.integers(-6, 7, size=(3000, 1)))).astype(np.float32)
    q = (rng.standard_normal((200, 50)) * 4).astype(np.float32)
    (ids, d), names = _bf(y, q, 30)
    assert _ran(names, "bf_tc_f32_kernel"), names
    _check(y, q, 30, ids, d)


def test_f32_tc_near_ties_fall_back_exactly():
    # 1200 identical rows plus 200 tiny perturbations of them: queries near them
    # see more rows inside the error margin than a list (or the re-rank buffer)
    # holds -> flagged and recomputed by the exact CUDA-core kernel; the result
    # is still bit-identical
    rng = np.random.default_rng(3)
    x = rng.uniform(0.0, 1.0, size=(4000, 64)).astype(np.float32)
    x[1000:2200] = x[5]
    x[2200:2400] = x[5] + rng.uniform(-1e-6, 1e-6, size=(200, 64)).astype(np.float32)
    (ids, d), names = _bf(x, None, 100)
    assert _ran(names, "bf_tc_f32_kernel") and _ran(names, "bf_tile_kernel"), names
    _check(x, None, 100, ids, d)


def test_f32_tc_rows_subset_and_cuda_core_agree():
    # brute_force_rows (accuracy sampling, sharded ground truth) and the forced
    # CUDA-core kernel give the same answer
    x = _fmix(9000, 256, 25, 21)
    rows = np.array([0, 1, 127, 128, 8999, 4097, 12, 5000], np.uint32)
    (ids, d), names = _bf(x, None, 100, rows=rows)
    assert _ran(names, "bf_tc_f32_kernel"), names
    os.environ["ANNK_BF_CUDA_CORE"] = "1"
    try:
        (ids_c, d_c), names_c = _bf(x, None, 100, rows=rows)
    finally:
        del os.environ["ANNK_BF_CUDA_CORE"]
    assert not _ran(names_c, "bf_tc_f32_kernel"), names_c
    np.testing.assert_array_equal(ids, ids_c)
    np.testing.assert_array_equal(d.view(np.uint32), d_c.view(np.uint32))
    o = ora()
    ids_o = o.brute_force(o.vs(x), o.vs(x[rows]), 101, workers=8)
    for r, i in enumerate(rows):
        np.testing.assert_array_equal(ids[r], [j for j in ids_o[r] if j != i][:100])


def test_f32_tc_huge_norms_take_exact_kernel():
    # norms beyond the certified range (|b|^2 >= 1e30) go to the exact CUDA-core kernel
    x = (_fmix(500, 32, 5, 4) * 1e16).astype(np.float32)
    q = x[:10].copy()
    (ids, d), names = _bf(x, q, 5)
    assert not _ran(names, "bf_tc_f32_kernel") and _ran(names, "bf_tile_kernel"), names
    _check(x, q, 5, ids, d)
