"""Shared fixtures/helpers for the parity tests (test infrastructure)."""
import numpy as np

from oracle import oracle as O


def ora():
    return O.load("oracle")


def ref():
    return O.load("reference")


def mixture(n, dim, centers, seed, stream=1, lo=0.0, hi=128.0, sd=16.0, clip=(0.0, 255.0), rnd=True):
    import paper_1609_07228_b200 as A
    return A.gen_mixture(n, dim, centers, lo, hi, sd, clip[0], clip[1], rnd, seed, stream)


def assert_trees_equal(dev_tree, ora_tree):
    assert dev_tree.n_nodes == ora_tree.n_nodes
    assert dev_tree.root == ora_tree.root
    assert dev_tree.leaf_count == ora_tree.leaf_count
    np.testing.assert_array_equal(dev_tree.split_dim, ora_tree.split_dim)
    np.testing.assert_array_equal(dev_tree.split_val.view(np.uint32), ora_tree.split_val.view(np.uint32))
    np.testing.assert_array_equal(dev_tree.left, ora_tree.left)
    np.testing.assert_array_equal(dev_tree.right, ora_tree.right)
    np.testing.assert_array_equal(dev_tree.depth, ora_tree.depth)
    np.testing.assert_array_equal(dev_tree.even_split, ora_tree.even)
    np.testing.assert_array_equal(dev_tree.point_index, ora_tree.point_index)


def assert_pools_equal(dev_state, ora_state):
    s, ids, d, f = dev_state.pools()
    e = ora_state.export()
    np.testing.assert_array_equal(s, e["sizes"])
    for i in range(len(s)):
        m = int(s[i])
        np.testing.assert_array_equal(ids[i, :m], e["ids"][i, :m], err_msg=f"ids row {i}")
        np.testing.assert_array_equal(d[i, :m].view(np.uint32), e["dists"][i, :m].view(np.uint32),
                                      err_msg=f"dists row {i}")
        np.testing.assert_array_equal(f[i, :m], e["flags"][i, :m], err_msg=f"flags row {i}")
    return e
