"""ctypes binding of the C-ABI in include/annkit_b200.h.

The shared library is built in-tree (``make`` or ``__graft_entry__.build()``)
and loaded from this package directory.  There is no fallback: if the library
is missing, importing the package fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ANNK_LIB") or os.path.join(HERE, "libannkit_b200.so")

ANNK_OK = 0
ANNK_INVALID_ARGUMENT = 1
ANNK_OUT_OF_RANGE = 2
ANNK_CUDA_ERROR = 3
ANNK_OUT_OF_MEMORY = 4
ANNK_INTERNAL = 5

# annk_state_rows buffers (include/annkit_b200.h)
ANNK_ROWS_FNEW, ANNK_ROWS_CNEW, ANNK_ROWS_FOLD, ANNK_ROWS_COLD, ANNK_ROWS_THR = range(5)


class AnnkError(RuntimeError):
    """CUDA / internal failure."""


class InvalidArgument(ValueError):
    """Mirrors the reference's std::invalid_argument."""


class OutOfRange(IndexError):
    """Mirrors the reference's std::out_of_range."""


class SearchParamsC(C.Structure):
    _fields_ = [
        ("k_return", C.c_uint32),
        ("pool_size", C.c_uint32),
        ("expansion", C.c_uint32),
        ("iters", C.c_uint32),
        ("n_trees_used", C.c_uint32),
        ("random_seed_count", C.c_uint32),
        ("seed", C.c_uint64),
        ("random_init", C.c_int32),
    ]


_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C")
_f32p = np.ctypeslib.ndpointer(np.float32, flags="C")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C")
_vp = C.c_void_p
_pp = C.POINTER(C.c_void_p)
_u32 = C.c_uint32
_u64 = C.c_uint64

# name -> argtypes (all return int status unless listed in _RESTYPES)
_SIGS = {
    "annk_set_device": [C.c_int],
    "annk_synchronize": [],
    "annk_profile_enable": [C.c_int],
    "annk_profile_reset": [],
    "annk_profile_report": [C.c_char_p, _u64],
    "annk_dataset_create": [_f32p, _u32, _u32, _pp],
    "annk_dataset_destroy": [_vp],
    "annk_dataset_shape": [_vp, C.POINTER(_u32), C.POINTER(_u32)],
    "annk_dataset_info": [_vp, _u32p],
    "annk_gen_synthetic": [_u32, _u32, _u64, _f32p],
    "annk_gen_mixture": [_u32, _u32, _u32, C.c_float, C.c_float, C.c_float, C.c_float, C.c_float, C.c_int,
                         _u64, _u32, _f32p],
    "annk_brute_force_knn": [_vp, _vp, _u32, _u32p, _vp, C.POINTER(_u64)],
    "annk_brute_force_rows": [_vp, _u32p, _u32, _u32, _u32p, _vp],
    "annk_measure_i8_peak": [_u32, C.POINTER(C.c_double)],
    "annk_bf_last_scan": [C.POINTER(_u64), C.POINTER(_u64), C.POINTER(C.c_int)],
    "annk_accuracy_vs_k": [_vp, _u32p, _u32, _u32, _u32p, _u32, np.ctypeslib.ndpointer(np.float64, flags="C")],
    "annk_forest_build": [_vp, _u32, _u32, _u64, _pp],
    "annk_forest_destroy": [_vp],
    "annk_forest_info": [_vp, _u32p, C.POINTER(_u64)],
    "annk_forest_tree_info": [_vp, _u32, _u32p],
    "annk_forest_export": [_vp, _u32, _u32p, _f32p, _u32p, _u32p, _u32p, _u8p, _u32p],
    "annk_forest_import": [_u32, _u32, _u32, _u64, _u32, _u32p, _u32p, _u32p, _f32p, _u32p, _u32p, _u32p,
                           _u8p, _u32p, _pp],
    "annk_search_leaves": [_vp, _u32, _f32p, _u32, _u32, _u32, _u32p, _u32p],
    "annk_descend_from": [_vp, _u32, _f32p, _u32, _u32, _u32p, _u32p],
    "annk_init_graph": [_vp, _vp, _u32, _u32, _u32, _u32, _u64, _pp],
    "annk_state_import": [_u32, _u32, _u32, _u32, _u64, _u32, _u64, _u32p, _u32p, _f32p, _u8p, _pp],
    "annk_state_destroy": [_vp],
    "annk_state_meta": [_vp, _u64p],
    "annk_state_export": [_vp, _u32p, _u32p, _f32p, _u8p],
    "annk_state_lists": [_vp, C.c_int, _u32p, _vp],
    "annk_nn_descent_iteration": [_vp, _vp, C.POINTER(_u64)],
    "annk_l2_sq": [_vp, _vp, _u32, C.POINTER(C.c_float)],
    "annk_dist_sq": [_vp, _vp, _vp, _u32, _vp],
    "annk_dist_sq_q": [_vp, _vp, _u32, _vp, _u32, _vp],
    "annk_nn_expansion_iteration": [_vp, _vp, C.POINTER(_u64)],
    "annk_rebuild_sample_lists": [_vp],
    "annk_union_reverse_lists": [_vp],
    "annk_refine_nn_descent": [_vp, _vp, _u32, C.c_double, C.POINTER(_u32)],
    "annk_finalize": [_vp, _vp, _u32, _u32p, _f32p],
    "annk_nn_descent_iteration_finalize": [_vp, _vp, _u32, _u32p, _f32p, C.POINTER(_u64), C.POINTER(_u64)],
    "annk_pool_topk_accuracy": [_vp, _u32p, _u32, _u32, _vp, C.POINTER(C.c_double)],
    "annk_state_join_rows": [_vp, C.POINTER(_u64)],
    "annk_state_stats": [_vp, _u64p],
    "annk_init_graph_shard": [_vp, _vp, _u32, _u32, _u32, _u32, _u64, _u32, _u32, _pp],
    "annk_init_random": [_vp, _u32, _u32, _u32, _u64, _pp],
    "annk_state_set_shard": [_vp, _u32, _u32],
    "annk_state_rows": [_vp, C.c_int, C.c_int, _u32, _u32, _vp],
    "annk_shard_sample": [_vp],
    "annk_shard_union": [_vp],
    "annk_shard_join": [_vp, _vp, C.POINTER(_u64)],
    "annk_shard_offers_count": [_vp, _u32, _u32, C.POINTER(_u64)],
    "annk_shard_join_range": [_vp, _vp, _u32, _u32, C.POINTER(_u64), C.POINTER(_u64), C.POINTER(_u32)],
    "annk_shard_offers_pack": [_vp, _u32, _u32, _vp, _vp, _vp],
    "annk_shard_offers_add": [_vp, _u32, _u32, _vp, _vp, _vp],
    "annk_shard_merge": [_vp, C.POINTER(_u64)],
    "annk_shard_merge_piece": [_vp, C.POINTER(_u64)],
    "annk_shard_finish_round": [_vp, C.POINTER(_u64)],
    "annk_searcher_create": [_vp, _vp, _u32p, _u32, _u32, _pp],
    "annk_searcher_destroy": [_vp],
    "annk_search": [_vp, _f32p, _u32, _u32, C.POINTER(SearchParamsC), _u32p, _f32p, _vp],
    "annk_search_dataset": [_vp, _vp, C.POINTER(SearchParamsC), _u32p, _f32p, _vp],
}
_RESTYPES = {
    "annk_last_error": C.c_char_p,
    "annk_version": C.c_char_p,
    "annk_stream": C.c_uint64,
    "annk_launch_count": C.c_uint64,
}

# Every symbol the header declares (checked by tests/test_abi.py).
EXPORTED = sorted(list(_SIGS) + list(_RESTYPES))


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `make` (or __graft_entry__.build()); "
            "this package has no CPU fallback")
    lib = C.CDLL(LIB_PATH)
    for name, args in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = C.c_int
    for name, rt in _RESTYPES.items():
        fn = getattr(lib, name)
        fn.restype = rt
        fn.argtypes = []
    return lib


lib = _load()


def check(status: int) -> None:
    if status == ANNK_OK:
        return
    msg = lib.annk_last_error().decode(errors="replace")
    if status == ANNK_INVALID_ARGUMENT:
        raise InvalidArgument(msg)
    if status == ANNK_OUT_OF_RANGE:
        raise OutOfRange(msg)
    if status == ANNK_OUT_OF_MEMORY:
        raise MemoryError(msg)
    raise AnnkError(f"[{status}] {msg}")


def ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)
