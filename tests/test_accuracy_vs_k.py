"""accuracy_vs_k (eval.cpp:129-155): exact truth at max k'
plus set membership, on the device, against the reference and a numpy check
over the oracle's exact rows."""
import numpy as np
import pytest

from oracle import oracle as O
from tests.helpers import mixture, ora


def _numpy_acc(graph, truth, k_list):
    out = []
    for kp in k_list:
        hits = sum(np.isin(graph[i], truth[i, :kp]).sum() for i in range(graph.shape[0]))
        out.append(hits / graph.size)
    return out


@pytest.mark.skipif(not O.reference_available(), reason="oracle/_ref not built")
def test_reference_accuracy_vs_k_matches_numpy_restatement():
    r, o = O.load("reference"), ora()
    x = o.gen_synthetic(400, 8, 3)
    vs = o.vs(x)
    graph = np.ascontiguousarray(o.brute_force(vs, None, 20)[:, ::-1][:, :10])  # any n x k rows
    truth = o.brute_force(vs, None, 40)
    k_list = [1, 5, 10, 40]
    np.testing.assert_allclose(r.ref_accuracy_vs_k(r.vs(x), graph, k_list), _numpy_acc(graph, truth, k_list),
                               rtol=0, atol=1e-15)


@pytest.mark.gpu
@pytest.mark.parametrize("integer", [False, True])
def test_device_accuracy_vs_k(integer):
    import paper_1609_07228_b200 as A
    o = ora()
    x = mixture(3000, 32, 20, 4) if integer else A.gen_synthetic(3000, 32, 4)
    f = A.build_forest(x, 4, 8, 4)
    g = A.finalize(A.init_graph(x, f, 10, 4, 20, 10, 4), A.VectorSet(x), 10)
    k_list = [1, 10, 50, 200]
    dev = [a for _, a in A.accuracy_vs_k(g, x, k_list)]
    truth = o.brute_force(o.vs(x), None, 200)
    np.testing.assert_array_equal(dev, _numpy_acc(g.ids, truth, k_list))
    if O.reference_available():
        r = O.load("reference")
        np.testing.assert_array_equal(dev, r.ref_accuracy_vs_k(r.vs(x), g.ids, k_list))
    with pytest.raises(A.InvalidArgument):
        A.accuracy_vs_k(g, x, [])
    with pytest.raises(A.InvalidArgument):
        A.accuracy_vs_k(g, x, [3000])
