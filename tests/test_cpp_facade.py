"""The C++ host API (include/annkit_b200.hpp, libannkit_facade.so): the
reference's annkit:: entry points over the C-ABI.  CPU: the library exports
the reference-named symbols; GPU: tests/cpp/test_facade.cpp (acceptance known
answers + unit-test invariants through the C++ API)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1609_07228_b200", "libannkit_facade.so")
BIN = os.path.join(ROOT, "tests", "cpp", "test_facade")

API = ["annkit::build_forest(", "annkit::search_leaves(", "annkit::descend_from(", "annkit::init_graph(",
       "annkit::init_random(", "annkit::refine_nn_descent(", "annkit::finalize(", "annkit::build_graph(",
       "annkit::detail::nn_descent_iteration(", "annkit::detail::rebuild_sample_lists(",
       "annkit::detail::union_reverse_lists(", "annkit::detail::pool_topk_accuracy(",
       "annkit::GraphSearcher::GraphSearcher(", "annkit::GraphSearcher::search(",
       "annkit::GraphSearcher::search_random_init(", "annkit::recall_curve(", "annkit::brute_force_knn(",
       "annkit::brute_force_graph(", "annkit::recall(", "annkit::graph_accuracy(", "annkit::accuracy_vs_k(",
       "annkit::gen_synthetic("]


def test_facade_exports_reference_api():
    out = subprocess.run(["nm", "-DC", "--defined-only", LIB], capture_output=True, text=True, check=True).stdout
    missing = [f for f in API if f not in out]
    assert not missing, missing


@pytest.mark.gpu
def test_facade_program():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
