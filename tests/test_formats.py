"""Reference file formats: fvecs/ivecs, AKF1 forests and
graph files, byte-compatible with the reference's own writers
(dataset.cpp:96-200, kd_forest.cpp:307-372, knn_graph.cpp:5-37) and validated
like its readers."""
import os
import tempfile

import numpy as np
import pytest

from oracle import oracle as O
from paper_1609_07228_b200 import formats as F
from tests.helpers import ora

needs_ref = pytest.mark.skipif(not O.reference_available(), reason="oracle/_ref not built")


@pytest.fixture
def tmp():
    with tempfile.TemporaryDirectory() as d:
        yield d


def _bytes(p):
    with open(p, "rb") as fh:
        return fh.read()


def test_fvecs_ivecs_roundtrip(tmp):
    x = ora().gen_synthetic(37, 5, 3)
    F.save_fvecs(x, os.path.join(tmp, "a.fvecs"))
    np.testing.assert_array_equal(F.load_fvecs(os.path.join(tmp, "a.fvecs")), x)
    ids = np.arange(37 * 4, dtype=np.uint32).reshape(37, 4)
    F.save_ivecs(ids, os.path.join(tmp, "a.ivecs"))
    np.testing.assert_array_equal(F.load_ivecs(os.path.join(tmp, "a.ivecs")), ids)
    g = F.load_graph(os.path.join(tmp, "a.ivecs"))
    assert g.dists is None and g.ids.shape == (37, 4)


@needs_ref
def test_fvecs_ivecs_bytes_match_reference(tmp):
    r = O.load("reference")
    x = r.gen_synthetic(50, 7, 11)
    r.ref_save_fvecs(r.vs(x), os.path.join(tmp, "ref.fvecs"))
    F.save_fvecs(x, os.path.join(tmp, "ours.fvecs"))
    assert _bytes(os.path.join(tmp, "ref.fvecs")) == _bytes(os.path.join(tmp, "ours.fvecs"))
    ids = (np.arange(50 * 6, dtype=np.uint32) * 7919 % 1000).reshape(50, 6)
    r.ref_save_ivecs(ids, os.path.join(tmp, "ref.ivecs"))
    F.save_ivecs(ids, os.path.join(tmp, "ours.ivecs"))
    assert _bytes(os.path.join(tmp, "ref.ivecs")) == _bytes(os.path.join(tmp, "ours.ivecs"))


def test_vecs_format_errors(tmp):
    p = os.path.join(tmp, "bad.fvecs")
    np.array([0], "<i4").tofile(p)
    with pytest.raises(F.FormatError, match="declares dimension"):
        F.load_fvecs(p)
    np.array([2, 0, 0, 3, 0, 0, 0], "<i4").tofile(p)
    with pytest.raises(F.FormatError, match="expected 2"):
        F.load_fvecs(p)
    np.array([2, 0, 0, 2, 0], "<i4").tofile(p)
    with pytest.raises(F.FormatError, match="truncated"):
        F.load_fvecs(p)
    v = np.array([2, 0, 0], "<i4")
    v[2] = np.array([np.inf], "<f4").view("<i4")[0]
    v.tofile(p)
    with pytest.raises(F.DataError, match="non-finite"):
        F.load_fvecs(p)
    np.array([2, 1, -5], "<i4").tofile(p)
    with pytest.raises(F.DataError, match="negative id"):
        F.load_ivecs(p)
    with pytest.raises(F.DataError, match="int32"):
        F.save_ivecs(np.array([[0x80000000]], np.uint32), p)
    F.save_fvecs(np.zeros((3, 2), np.float32), p)
    F.save_fvecs(np.zeros((3, 3), np.float32), p + "2")
    F.save_ivecs(np.zeros((3, 2), np.uint32), p + "3")
    with pytest.raises(F.FormatError, match="has shape"):
        F.load_graph(p + "3", p + "2")


@needs_ref
@pytest.mark.parametrize("n,dim,trees,leaf,seed", [(3000, 16, 3, 8, 4), (500, 12, 4, 10, 1234), (7, 4, 2, 10, 5)])
def test_forest_file_matches_reference(tmp, n, dim, trees, leaf, seed):
    r = O.load("reference")
    x = r.gen_synthetic(n, dim, seed)
    fr = r.build_forest(r.vs(x), trees, leaf, seed)
    r.ref_save_forest(fr, os.path.join(tmp, "ref.akf"))
    F.save_forest(fr, os.path.join(tmp, "ours.akf"))
    assert _bytes(os.path.join(tmp, "ref.akf")) == _bytes(os.path.join(tmp, "ours.akf"))
    n2, dim2, leaf2, seed2, ts = F.parse_forest(os.path.join(tmp, "ref.akf"))
    assert (n2, dim2, leaf2, seed2) == (n, dim, leaf, seed)
    for t in range(trees):
        e = fr.tree(t)
        np.testing.assert_array_equal(ts[t].split_dim, e.split_dim)
        np.testing.assert_array_equal(ts[t].split_val.view(np.uint32), e.split_val.view(np.uint32))
        np.testing.assert_array_equal(ts[t].left, e.left)
        np.testing.assert_array_equal(ts[t].right, e.right)
        np.testing.assert_array_equal(ts[t].point_index, e.point_index)
        assert ts[t].root == e.root


def test_forest_file_validation(tmp):
    o = ora()
    x = o.gen_synthetic(300, 6, 2)
    fo = o.build_forest(o.vs(x), 2, 5, 2)
    good = os.path.join(tmp, "f.akf")
    F.save_forest(fo, good)
    F.parse_forest(good)
    blob = bytearray(_bytes(good))

    def bad(mut, match):
        b = bytearray(blob)
        mut(b)
        p = os.path.join(tmp, "bad.akf")
        with open(p, "wb") as fh:
            fh.write(b)
        with pytest.raises(F.FormatError, match=match):
            F.parse_forest(p)

    bad(lambda b: b.__setitem__(slice(0, 4), b"XKF1"), "not a forest file")
    bad(lambda b: b.__setitem__(slice(4, 8), np.array([2], "<u4").tobytes()), "unsupported forest version")
    bad(lambda b: b.extend(b"\0"), "trailing bytes")
    bad(lambda b: b.__delitem__(slice(len(b) - 2, len(b))), "unexpected end of file")
    t0 = 32  # first tree: node_count, root, nodes...
    m = int(np.frombuffer(bytes(blob[t0:t0 + 4]), "<u4")[0])
    pi0 = t0 + 8 + 21 * m
    bad(lambda b: b.__setitem__(slice(pi0, pi0 + 4), b.__getitem__(slice(pi0 + 4, pi0 + 8))), "not a permutation")
    node1 = t0 + 8 + 21 * 1  # node 1's depth field -> 7
    bad(lambda b: b.__setitem__(slice(node1 + 16, node1 + 20), np.array([7], "<u4").tobytes()),
        "depth mismatch")
    node0 = t0 + 8  # root split_dim -> dim
    bad(lambda b: b.__setitem__(slice(node0, node0 + 4), np.array([6], "<u4").tobytes()),
        "split dimension out of range")


@pytest.mark.gpu
def test_device_forest_and_graph_files(tmp):
    import paper_1609_07228_b200 as A
    x = A.gen_synthetic(4000, 32, 9)
    f = A.build_forest(x, 4, 8, 9)
    p = os.path.join(tmp, "dev.akf")
    F.save_forest(f, p)
    f2 = F.load_forest(p)
    for t in range(4):
        a, b = f.tree(t), f2.tree(t)
        np.testing.assert_array_equal(a.split_dim, b.split_dim)
        np.testing.assert_array_equal(a.point_index, b.point_index)
    if O.reference_available():  # the reference's reader accepts the GPU-built file
        r = O.load("reference")
        fr = r.ref_load_forest(p, 4000, 32, 8, 9)
        np.testing.assert_array_equal(fr.tree(0).split_dim, f.tree(0).split_dim)
    g = A.finalize(A.init_graph(x, f, 10, 4, 20, 10, 9), A.VectorSet(x), 10)
    F.save_graph(g, os.path.join(tmp, "g.ivecs"), os.path.join(tmp, "g.fvecs"))
    g2 = F.load_graph(os.path.join(tmp, "g.ivecs"), os.path.join(tmp, "g.fvecs"))
    np.testing.assert_array_equal(g2.ids, g.ids)
    np.testing.assert_array_equal(g2.dists.view(np.uint32), g.dists.view(np.uint32))
