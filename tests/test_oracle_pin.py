"""Pins the CPU oracle (our C restatement) before it is trusted as the GPU
checker: against the unmodified reference library run here (oracle/_ref),
against the reference's recorded known-answer values (proj/test_output.txt,
reproduced bit-for-bit in the survey container) and against the golden
fixtures committed under tests/golden/ (generated from the reference by
tests/golden/make_golden.py).  CPU only."""
import os

import numpy as np
import pytest

from oracle import oracle as O

HAVE_REF = O.reference_available()
needs_ref = pytest.mark.skipif(not HAVE_REF, reason="oracle/_ref not built")
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def ora():
    return O.load("oracle")


@pytest.fixture(scope="module")
def ref():
    return O.load("reference")


def test_rng_known_answers(ora):
    # [rand.predef]: the 10000th output of a default-seeded mt19937_64
    assert int(ora.mt19937_64(5489, 10000)[-1]) == 9981545732273789042
    assert ora.substream(1, 0) == 627405149472732430
    assert ora.mix64(0) == 16294208416658607535


def test_l2_is_sequential_fp32(ora):
    a = np.array([0, 0], np.float32)
    b = np.array([3, 4], np.float32)
    assert ora.l2_sq(a, b) == 25.0  # test_dataset.cpp:198-202
    x = ora.gen_synthetic(50, 37, 3)
    for i in range(0, 50, 7):
        acc = np.float32(0)
        for t in range(37):
            d = np.float32(x[i, t] - x[0, t])
            acc = np.float32(acc + np.float32(d * d))
        assert ora.l2_sq(x[i], x[0]) == acc
        assert ora.l2_sq(x[i], x[0]) == ora.l2_sq(x[0], x[i])


@needs_ref
def test_gen_synthetic_matches(ora, ref):
    assert np.array_equal(ora.gen_synthetic(300, 7, 11), ref.gen_synthetic(300, 7, 11))


@needs_ref
@pytest.mark.parametrize("n,dim,k", [(2000, 8, 10), (500, 33, 40)])
def test_brute_force_matches_reference(ora, ref, n, dim, k):
    x = ora.gen_synthetic(n, dim, 12)
    q = ora.gen_synthetic(50, dim, 13)
    a = ora.brute_force(ora.vs(x), None, k, workers=8, with_dists=True)
    b = ref.brute_force(ref.vs(x), None, k, workers=8, with_dists=True)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and a[2] == b[2]
    assert np.array_equal(ora.brute_force(ora.vs(x), ora.vs(q), k), ref.brute_force(ref.vs(x), ref.vs(q), k))


@needs_ref
@pytest.mark.parametrize("n,dim,trees,leaf,seed", [(10000, 128, 8, 10, 1), (500, 12, 4, 10, 1234), (1, 4, 3, 10, 5),
                                                   (300, 6, 2, 5, 4)])
def test_forest_matches_reference(ora, ref, n, dim, trees, leaf, seed):
    x = ora.gen_synthetic(n, dim, seed)
    fa = ora.build_forest(ora.vs(x), trees, leaf, seed, workers=4)
    fb = ref.build_forest(ref.vs(x), trees, leaf, seed, workers=4)
    for t in range(trees):
        A, B = fa.tree(t), fb.tree(t)
        for f in ("split_dim", "left", "right", "depth", "even", "point_index"):
            assert np.array_equal(getattr(A, f), getattr(B, f)), f
        assert np.array_equal(A.split_val.view(np.uint32), B.split_val.view(np.uint32))
        assert (A.root, A.leaf_count) == (B.root, B.leaf_count)


@needs_ref
def test_forest_degenerate_splits_match(ora, ref):
    x = np.round(ora.gen_synthetic(3000, 16, 3) * 4).astype(np.float32)  # heavy ties -> fallback sorts
    x[:400] = x[0]
    fa = ora.build_forest(ora.vs(x), 3, 8, 7)
    fb = ref.build_forest(ref.vs(x), 3, 8, 7)
    assert sum(int(fa.tree(t).even.sum()) for t in range(3)) > 0
    for t in range(3):
        assert np.array_equal(fa.tree(t).point_index, fb.tree(t).point_index)
        assert np.array_equal(fa.tree(t).split_val.view(np.uint32), fb.tree(t).split_val.view(np.uint32))


@needs_ref
def test_init_and_descent_match_reference(ora, ref):
    x = ora.gen_synthetic(2000, 32, 1)
    va, vb = ora.vs(x), ref.vs(x)
    fa, fb = ora.build_forest(va, 4, 10, 1), ref.build_forest(vb, 4, 10, 1)
    sa, sb = ora.init_graph(va, fa, 10, 4, 30, 20, 1), ref.init_graph(vb, fb, 10, 4, 30, 20, 1, workers=3)
    gt = ref.brute_force(vb, None, 10, workers=8)
    for it in range(6):
        ea, eb = sa.export(), sb.export()
        for key in ("sizes", "ids", "dists", "flags"):
            assert np.array_equal(ea[key], eb[key]), (it, key)
        assert ea["dist_comps"] == eb["dist_comps"]
        assert sa.pool_topk_accuracy(gt) == sb.pool_topk_accuracy(gt)
        ca, cb = sa.nn_descent_iteration(va), sb.nn_descent_iteration(vb, workers=1)
        assert ca == cb  # single-worker changes are deterministic
        for w in range(4):
            assert all(np.array_equal(p, q) for p, q in zip(sa.lists(w), sb.lists(w)))


@needs_ref
def test_search_matches_reference(ora, ref):
    x = ora.gen_synthetic(2000, 16, 21)
    q = ora.gen_synthetic(40, 16, 22)
    va, vb = ora.vs(x), ref.vs(x)
    fa, fb = ora.build_forest(va, 8, 10, 21), ref.build_forest(vb, 8, 10, 21)
    g = ref.brute_force(vb, None, 10, workers=8)
    for P, E, I, ntu in [(100, 50, 4, 0), (60, 30, 0, 0), (200, 200, 4, 3), (12, 12, 0, 0)]:
        kr = min(10, P)
        a = ora.search(va, fa, g, ora.vs(q), kr, P, E, I, ntu)
        b = ref.search(vb, fb, g, ref.vs(q), kr, P, E, I, ntu, workers=3)
        for u, v in zip(a, b):
            assert np.array_equal(u, v)
        a = ora.search(va, None, g, ora.vs(q), kr, P, E, I, random_init=True, seed=7)
        b = ref.search(vb, None, g, ref.vs(q), kr, P, E, I, random_init=True, seed=7)
        for u, v in zip(a, b):
            assert np.array_equal(u, v)


@needs_ref
def test_build_graph_logs_match(ora, ref):
    x = ora.gen_synthetic(500, 8, 61)
    va, vb = ora.vs(x), ref.vs(x)
    fa, fb = ora.build_forest(va, 4, 10, 61), ref.build_forest(vb, 4, 10, 61)
    gt = ref.brute_force(vb, None, 10, workers=4)
    for strategy in (0, 1, 2, 3, 4):
        ia, _, la, sa = ora.build_graph(va, fa, 10, 2, 30, 20, 6, strategy, 61, 1, 0.001, gt)
        ib, _, lb, sb = ref.build_graph(vb, fb, 10, 2, 30, 20, 6, strategy, 61, 1, 0.001, gt)
        assert np.array_equal(ia, ib), strategy
        assert np.array_equal(la[:, [0, 2, 3, 4]], lb[:, [0, 2, 3, 4]]), strategy
        assert sa[2] == sb[2] and sa[3] == sb[3]


def test_acceptance_known_answers_search(ora):
    """proj/test_output.txt:13 (criterion 4): 10k x 32 uniform, exact 10-NN graph,
    8 trees leaf 10, E=50 P=100, 100 queries: recall 0.9440 at 1285 comps/query."""
    base = ora.gen_synthetic(10000, 32, 1)
    queries = ora.gen_synthetic(100, 32, 2)
    vb, vq = ora.vs(base), ora.vs(queries)
    qgt = ora.brute_force(vb, vq, 10, workers=8)
    graph = ora.brute_force(vb, None, 10, workers=8)
    forest = ora.build_forest(vb, 8, 10, 1)
    ids, _, stats = ora.search(vb, forest, graph, vq, 10, 100, 50, 4, workers=8)
    rec = np.mean([len(np.intersect1d(ids[i], qgt[i])) / 10 for i in range(100)])
    assert f"{rec:.4f}" == "0.9440"
    assert f"{stats[:, 0].mean():.0f}" == "1285"
    # criterion 5 sweep, tree-seeded side: [P=50: 0.851] [P=200: 0.970] [P=600: 0.996]
    for P, want in ((50, "0.851"), (200, "0.970"), (600, "0.996")):
        ids, _, _ = ora.search(vb, forest, graph, vq, 10, P, 50, 4, workers=8)
        rec = np.mean([len(np.intersect1d(ids[i], qgt[i])) / 10 for i in range(100)])
        assert f"{rec:.3f}" == want, P


@pytest.mark.slow
def test_acceptance_known_answers_build(ora):
    """proj/test_output.txt:11-12 (criteria 2/3): 10k x 128 uniform, efanna
    (8 trees leaf 10, Dep 6, P=L=30) reaches 0.90 at 29,454,671 distance comps;
    random-descent at 37,263,414."""
    base = ora.gen_synthetic(10000, 128, 1)
    vb = ora.vs(base)
    gt = ora.brute_force(vb, None, 10, workers=8)
    forest = ora.build_forest(vb, 8, 10, 1, workers=8)

    def crossing(log):
        for row in log:
            if row[4] >= 0.90:
                return int(row[2])
        return None

    _, _, log, _ = ora.build_graph(vb, forest, 10, 6, 30, 30, 14, 0, 1, 8, 0.001, gt)
    assert crossing(log) == 29454671
    _, _, log, _ = ora.build_graph(vb, None, 10, 6, 30, 30, 20, 1, 1, 8, 0.001, gt)
    assert crossing(log) == 37263414


def test_golden_fixtures(ora):
    """Fixtures produced by the reference (tests/golden/make_golden.py)."""
    z = np.load(os.path.join(GOLDEN, "golden_small.npz"))
    x = ora.gen_synthetic(int(z["n"]), int(z["dim"]), int(z["seed"]))
    assert np.array_equal(x, z["base"])
    vs = ora.vs(x)
    f = ora.build_forest(vs, int(z["trees"]), int(z["leaf"]), int(z["seed"]))
    for t in range(int(z["trees"])):
        tr = f.tree(t)
        assert np.array_equal(tr.point_index, z[f"t{t}_point_index"])
        assert np.array_equal(tr.split_dim, z[f"t{t}_split_dim"])
        assert np.array_equal(tr.split_val.view(np.uint32), z[f"t{t}_split_val"].view(np.uint32))
    s = ora.init_graph(vs, f, int(z["k"]), int(z["dep"]), int(z["P"]), int(z["S"]), int(z["seed"]))
    for it in range(int(z["iters"])):
        s.nn_descent_iteration(vs)
    e = s.export()
    assert np.array_equal(e["ids"], z["pool_ids"]) and np.array_equal(e["sizes"], z["pool_sizes"])
    assert e["dist_comps"] == int(z["dist_comps"])
    g = ora.brute_force(vs, None, int(z["k"]), workers=4)
    assert np.array_equal(g, z["exact_ids"])
    ids, d, st = ora.search(vs, f, g, ora.vs(z["queries"]), int(z["k"]), 40, 20, 4)
    assert np.array_equal(ids, z["search_ids"]) and np.array_equal(st, z["search_stats"])


@pytest.mark.parametrize("args", [
    (5000, 128, 100, 0.0, 128.0, 16.0, 0.0, 255.0, True, 1, 1),     # cfg1/2/5 mixture, base stream
    (700, 128, 1000, 0.0, 128.0, 16.0, 0.0, 255.0, True, 1, 2),     # query stream
    (900, 960, 500, 0.05, 0.35, 0.05, 0.0, 1.0, False, 1, 1),       # cfg3 mixture
    (333, 13, 7, -3.0, 5.0, 2.5, -1.0, 4.0, False, 9, 3),
])
def test_oracle_mixture_generator_is_byte_identical(args):
    # the reference arm and the CPU baseline build their inputs with oracle/'s
    # restatement of annk_gen_mixture (that process never loads the product);
    # both must produce the same bytes, for any thread split
    import paper_1609_07228_b200 as A
    o = O.load("oracle")
    a = A.gen_mixture(*args)
    for w in (1, 3, 8):
        b = o.gen_mixture(*args, workers=w)
        np.testing.assert_array_equal(a.view(np.uint32), b.view(np.uint32))
