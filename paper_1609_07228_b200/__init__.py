"""EFANNA hot paths (kNN-graph construction, batched search, exact kNN) on
NVIDIA B200 (sm_100a), behind the reference library's host API.

The compute path is libannkit_b200.so (hand-written CUDA, C-ABI in
include/annkit_b200.h); this package is the reference-shaped host mirror.
"""
from ._lib import AnnkError, InvalidArgument, OutOfRange, lib  # noqa: F401
from .api import (  # noqa: F401
    BatchResult, BuildParams, BuildResult, BuildStats, GraphSearcher, IterationLog, KdForest, KdTree, KnnGraph,
    RefineState, SearchParams, SearchResult, SearchStats, SweepPoint, SweepRow, VectorSet, accuracy_vs_k,
    brute_force_graph,
    brute_force_knn, brute_force_rows, build_forest, build_graph, descend_from, detail, finalize, gen_mixture,
    state_stats,
    gen_synthetic, graph_accuracy, init_graph, init_random, recall, recall_curve, refine_nn_descent, search_leaves,
    l2_sq, dist_sq, dist_sq_q, bf_last_scan, measure_i8_peak,
)

__version__ = "0.1.0"


def launch_count() -> int:
    """Kernels launched by libannkit_b200.so since load."""
    return int(lib.annk_launch_count())


def stream_handle() -> int:
    """The library's cudaStream_t (for CUDA-event timing on the launching stream)."""
    return int(lib.annk_stream())


def profile_enable(on: bool = True) -> None:
    """Per-kernel CUDA-event timing on the library stream."""
    from ._lib import check
    check(lib.annk_profile_enable(int(on)))


def profile_reset() -> None:
    from ._lib import check
    check(lib.annk_profile_reset())


def profile_report() -> dict:
    """{kernel_name: (launches, total_ms)} accumulated since the last reset."""
    import ctypes

    from ._lib import check
    buf = ctypes.create_string_buffer(1 << 16)
    check(lib.annk_profile_report(buf, len(buf)))
    out = {}
    for line in buf.value.decode().splitlines():
        name, cnt, ms = line.rsplit(" ", 2)
        out[name] = (int(cnt), float(ms))
    return out
