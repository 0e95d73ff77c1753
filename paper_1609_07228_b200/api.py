"""Reference-shaped host API over the B200 C-ABI.

Mirrors the reference library's public surface (namespace ``annkit``,
proj/include/annkit/*.hpp) for the EFANNA hot paths — same names, argument
meaning and error behaviour — so callers and tests read like the reference's
own:

  =====================================  ========================================
  this module                            reference
  =====================================  ========================================
  VectorSet                              dataset.hpp:28-37
  gen_synthetic                          dataset.cpp:201-214
  brute_force_knn / brute_force_graph    eval.cpp:33-80
  build_forest / KdForest / KdTree       kd_forest.cpp:245-264, kd_forest.hpp:18-53
  search_leaves / descend_from           kd_forest.cpp:266-305
  init_graph / RefineState               graph_build.cpp:230-292, graph_build.hpp:17-30
  detail.nn_descent_iteration etc.       graph_build.cpp:59-162, :209-226
  refine_nn_descent / finalize           graph_build.cpp:328-373
  build_graph / BuildParams / ...        graph_build.cpp:395-461, graph_build.hpp:76-115
  GraphSearcher / SearchParams           search.cpp:23-154, search.hpp:13-76
  recall_curve / SweepPoint / SweepRow   search.cpp:182-236, search.hpp:78-98
  recall / graph_accuracy                eval.cpp:82-127
  =====================================  ========================================

std::invalid_argument surfaces as ``InvalidArgument`` (a ValueError) and
std::out_of_range as ``OutOfRange`` (an IndexError).  The ``workers``
arguments of the reference are accepted and ignored: the device path is
deterministic and equals the reference's single-worker results.
"""
from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from ._lib import InvalidArgument, OutOfRange, SearchParamsC, check, lib, ptr

LEAF_MARKER = 0xFFFFFFFF
INVALID_ID = 0xFFFFFFFF


# --------------------------------------------------------------- datasets

class VectorSet:
    """Device-resident dense row-major fp32 vector set (dataset.hpp:28-37)."""

    def __init__(self, data: np.ndarray):
        x = np.ascontiguousarray(data, dtype=np.float32)
        if x.ndim != 2:
            raise InvalidArgument("VectorSet: expected an n x dim array")
        self.data = x
        self.n, self.dim = int(x.shape[0]), int(x.shape[1])
        h = C.c_void_p()
        check(lib.annk_dataset_create(x if x.size else np.zeros(1, np.float32), self.n, max(self.dim, 0),
                                      C.byref(h)))
        self._h = h

    @property
    def handle(self):
        return self._h

    def info(self) -> dict:
        """n, dim, whether the exact u8 datapath is active, bytes per gathered row."""
        out = np.zeros(4, np.uint32)
        check(lib.annk_dataset_info(self._h, out))
        return dict(n=int(out[0]), dim=int(out[1]), u8=bool(out[2]), row_bytes=int(out[3]))

    def row(self, i: int) -> np.ndarray:
        return self.data[i]

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib.annk_dataset_destroy(h)
            self._h = None


def gen_synthetic(n: int, dim: int, seed: int) -> np.ndarray:
    """dataset.cpp:201-214: uniform [0,1) from mt19937_64, same bytes as the reference."""
    out = np.empty((n, dim), np.float32)
    check(lib.annk_gen_synthetic(n, dim, seed, out))
    return out


def gen_mixture(n: int, dim: int, n_centers: int, center_lo: float, center_hi: float, sd: float,
                clip_lo: float, clip_hi: float, round_to_int: bool, seed: int, stream_id: int) -> np.ndarray:
    """Seeded Gaussian mixture used for the BASELINE configs."""
    out = np.empty((n, dim), np.float32)
    check(lib.annk_gen_mixture(n, dim, n_centers, center_lo, center_hi, sd, clip_lo, clip_hi,
                               int(bool(round_to_int)), seed, stream_id, out))
    return out


def l2_sq(a, b) -> float:
    """dataset.hpp:67-74 l2_sq of two vectors, on the device (sequential fp32 chain)."""
    a = np.ascontiguousarray(a, np.float32).ravel()
    b = np.ascontiguousarray(b, np.float32).ravel()
    if a.size != b.size:
        raise InvalidArgument("l2_sq: vectors of different dimension")
    out = C.c_float(0.0)
    check(lib.annk_l2_sq(a.ctypes.data_as(C.c_void_p), b.ctypes.data_as(C.c_void_p), a.size, C.byref(out)))
    return float(out.value)


def dist_sq(vs, a, b):
    """dataset.cpp:216-222 dist_sq(vs, a, b); a and b may be equal-length id arrays
    (one device launch for all pairs).  Ids past the set raise OutOfRange."""
    v = _as_vs(vs)
    aa = np.ascontiguousarray(np.atleast_1d(a), np.uint32)
    bb = np.ascontiguousarray(np.atleast_1d(b), np.uint32)
    if aa.shape != bb.shape:
        raise InvalidArgument("dist_sq: id arrays of different length")
    out = np.empty(aa.size, np.float32)
    check(lib.annk_dist_sq(v.handle, aa.ctypes.data_as(C.c_void_p), bb.ctypes.data_as(C.c_void_p), aa.size,
                           out.ctypes.data_as(C.c_void_p)))
    return float(out[0]) if np.isscalar(a) and np.isscalar(b) else out


def dist_sq_q(vs, q, b):
    """dataset.cpp:224-233 dist_sq_q(vs, q, b) for one id or an id array."""
    v = _as_vs(vs)
    qq = np.ascontiguousarray(q, np.float32).ravel()
    bb = np.ascontiguousarray(np.atleast_1d(b), np.uint32)
    out = np.empty(bb.size, np.float32)
    check(lib.annk_dist_sq_q(v.handle, qq.ctypes.data_as(C.c_void_p), qq.size, bb.ctypes.data_as(C.c_void_p),
                             bb.size, out.ctypes.data_as(C.c_void_p)))
    return float(out[0]) if np.isscalar(b) else out


def _as_vs(x) -> VectorSet:
    return x if isinstance(x, VectorSet) else VectorSet(x)


# --------------------------------------------------------------- exact kNN

@dataclass
class KnnGraph:
    """knn_graph.hpp:16-29: n rows of k ids sorted by (dist, id), plus dists."""
    ids: np.ndarray
    dists: Optional[np.ndarray] = None

    @property
    def n(self):
        return int(self.ids.shape[0])

    @property
    def k(self):
        return int(self.ids.shape[1])

    def row(self, i):
        return self.ids[i]


def brute_force_knn(base, queries=None, k: int = 10, workers: int = 1, dist_comps: Optional[list] = None,
                    with_dists: bool = False, out_ids: Optional[np.ndarray] = None,
                    out_dists: Optional[np.ndarray] = None):
    """eval.cpp:33-61.  queries=None selects self mode.  Returns ids (nq x k) as a
    GroundTruth array (plus dists when with_dists).  out_ids / out_dists: caller-owned
    C-contiguous (nq x k) uint32 / float32 arrays to fill (e.g. pinned memory, which the
    device-to-host copy then reaches at full PCIe rate) instead of fresh ones."""
    b = _as_vs(base)
    q = None if queries is None else _as_vs(queries)
    nq = b.n if q is None else q.n
    for arr, dt, nm in ((out_ids, np.uint32, "out_ids"), (out_dists, np.float32, "out_dists")):
        if arr is not None and (arr.dtype != dt or arr.shape != (nq, k) or not arr.flags["C_CONTIGUOUS"]):
            raise InvalidArgument(f"brute_force_knn: {nm} must be a C-contiguous ({nq}, {k}) {np.dtype(dt).name} array")
    if out_dists is not None:
        with_dists = True
    ids = out_ids if out_ids is not None and k > 0 else (
        np.empty((nq, k), np.uint32) if k > 0 else np.empty((nq, 0), np.uint32))
    dists = out_dists if out_dists is not None else (
        np.empty((nq, k), np.float32) if with_dists and k > 0 else None)
    comps = C.c_uint64(0)
    check(lib.annk_brute_force_knn(b.handle, q.handle if q else None, k, ids if k > 0 else np.empty(1, np.uint32),
                                   ptr(dists), C.byref(comps)))
    if dist_comps is not None:
        dist_comps.append(int(comps.value))
    return (ids, dists) if with_dists else ids


def brute_force_graph(base, k: int, workers: int = 1, dist_comps: Optional[list] = None) -> KnnGraph:
    """eval.cpp:63-80."""
    b = _as_vs(base)
    if b.n == 0:
        raise InvalidArgument("brute_force_graph: empty base set")
    if k < 1 or k > b.n - 1:
        raise InvalidArgument("brute_force_graph: k out of range")
    ids, d = brute_force_knn(b, None, k, dist_comps=dist_comps, with_dists=True)
    return KnnGraph(ids, d)


def brute_force_rows(base, rows: np.ndarray, k: int, with_dists: bool = False):
    """Self-mode exact rows for a subset of base points (accuracy sampling)."""
    b = _as_vs(base)
    rows = np.ascontiguousarray(rows, np.uint32)
    ids = np.empty((len(rows), k), np.uint32)
    d = np.empty((len(rows), k), np.float32) if with_dists else None
    check(lib.annk_brute_force_rows(b.handle, rows, len(rows), k, ids, ptr(d)))
    return (ids, d) if with_dists else ids


def measure_i8_peak(groups: int = 20000) -> float:
    """Measurement only: dense tcgen05 kind::i8 tera-ops/s of this GPU (MMA issue on
    shared-memory operands, no loads, no epilogue)."""
    import ctypes as C
    out = C.c_double(0.0)
    check(lib.annk_measure_i8_peak(groups, C.byref(out)))
    return out.value


def bf_last_scan() -> dict:
    """Measurement only: (query block, base tile) pairs of the last exact-kNN run on
    the tcgen05 u8 kernel, and how many of them its MMA passes visited."""
    import ctypes as C
    tot, vis, pr = C.c_uint64(0), C.c_uint64(0), C.c_int(0)
    check(lib.annk_bf_last_scan(C.byref(tot), C.byref(vis), C.byref(pr)))
    return {"tiles_total": tot.value, "tiles_visited": vis.value, "pruned": bool(pr.value)}


def accuracy_vs_k(graph, vs, k_list, workers: int = 1) -> list:
    """eval.cpp:129-155: [(k', fraction of graph edges inside the exact k'-NN)],
    exact truth and membership counted on the device."""
    g = graph.ids if isinstance(graph, KnnGraph) else np.asarray(graph)
    g = np.ascontiguousarray(g, np.uint32)
    v = _as_vs(vs)
    kl = np.ascontiguousarray(np.asarray(k_list, np.uint32).ravel())
    out = np.empty(max(kl.size, 1), np.float64)
    if g.ndim != 2:
        raise InvalidArgument("accuracy_vs_k: graph must be n x k")
    check(lib.annk_accuracy_vs_k(v.handle, g, g.shape[0], g.shape[1], kl, kl.size, out))
    return [(int(k), float(a)) for k, a in zip(kl, out)]


# ------------------------------------------------------------------ forest

@dataclass
class KdTree:
    """kd_forest.hpp:18-42 (node fields as parallel arrays)."""
    split_dim: np.ndarray
    split_val: np.ndarray
    left: np.ndarray
    right: np.ndarray
    depth: np.ndarray
    even_split: np.ndarray
    point_index: np.ndarray
    root: int
    leaf_count: int
    max_depth: int = 0

    @property
    def n_nodes(self):
        return len(self.split_dim)

    def is_leaf(self, node):
        return self.split_dim[node] == LEAF_MARKER

    def leaf_points(self, node):
        return self.point_index[self.left[node]:self.right[node]]


class KdForest:
    """Device-resident forest (kd_forest.hpp:47-53)."""

    def __init__(self, handle, n, dim, leaf_cap, seed, n_trees):
        self._h = handle
        self.n, self.dim, self.leaf_cap, self.seed, self.n_trees = n, dim, leaf_cap, seed, n_trees
        self._trees = None

    @property
    def handle(self):
        return self._h

    def tree_info(self, t):
        info = np.empty(4, np.uint32)
        check(lib.annk_forest_tree_info(self._h, t, info))
        return dict(num_nodes=int(info[0]), root=int(info[1]), leaf_count=int(info[2]), max_depth=int(info[3]))

    def tree(self, t) -> KdTree:
        inf = self.tree_info(t)
        m = inf["num_nodes"]
        sd = np.empty(m, np.uint32); sv = np.empty(m, np.float32); le = np.empty(m, np.uint32)
        ri = np.empty(m, np.uint32); de = np.empty(m, np.uint32); ev = np.empty(m, np.uint8)
        pi = np.empty(self.n, np.uint32)
        check(lib.annk_forest_export(self._h, t, sd, sv, le, ri, de, ev, pi))
        return KdTree(sd, sv, le, ri, de, ev, pi, inf["root"], inf["leaf_count"], inf["max_depth"])

    @property
    def trees(self):
        if self._trees is None:
            self._trees = [self.tree(t) for t in range(self.n_trees)]
        return self._trees

    @staticmethod
    def pack_trees(trees: Sequence, out=None) -> dict:
        """Concatenated host arrays of `trees` in annk_forest_import's layout;
        `out` (same keys) may supply preallocated (e.g. pinned) buffers."""
        ev_attr = "even_split" if hasattr(trees[0], "even_split") else "even"
        fields = {"split_dim": ("split_dim", np.uint32), "split_val": ("split_val", np.float32),
                  "left": ("left", np.uint32), "right": ("right", np.uint32), "depth": ("depth", np.uint32),
                  "even": (ev_attr, np.uint8), "point_index": ("point_index", np.uint32)}
        packed = {"node_counts": np.array([len(t.split_dim) for t in trees], np.uint32),
                  "roots": np.array([t.root for t in trees], np.uint32)}
        for key, (attr, dt) in fields.items():
            cat = np.concatenate([np.asarray(getattr(t, attr)) for t in trees]).astype(dt)
            if out is not None:
                out[key][...] = cat
                cat = out[key]
            packed[key] = np.ascontiguousarray(cat)
        return packed

    @classmethod
    def import_packed(cls, n, dim, leaf_cap, seed, packed: dict) -> "KdForest":
        """Device forest from pack_trees() arrays (kd_forest.cpp:332-372 load, then upload)."""
        h = C.c_void_p()
        check(lib.annk_forest_import(
            n, dim, leaf_cap, seed, len(packed["roots"]), packed["node_counts"], packed["roots"],
            packed["split_dim"], packed["split_val"], packed["left"], packed["right"], packed["depth"],
            packed["even"], packed["point_index"], C.byref(h)))
        return cls(h, n, dim, leaf_cap, seed, len(packed["roots"]))

    @classmethod
    def from_trees(cls, n, dim, leaf_cap, seed, trees: Sequence) -> "KdForest":
        """Device forest from host trees (e.g. exported by the CPU reference)."""
        return cls.import_packed(n, dim, leaf_cap, seed, cls.pack_trees(trees))

    def search_leaves(self, t: int, queries: np.ndarray, n_leaves: int):
        """kd_forest.cpp:276-305 for a batch; returns a list of leaf-id arrays."""
        q = np.ascontiguousarray(np.atleast_2d(queries), np.float32)
        nq, dim = q.shape
        out = np.empty((nq, max(n_leaves, 1)), np.uint32)
        cnt = np.empty(nq, np.uint32)
        check(lib.annk_search_leaves(self._h, t, q, nq, dim, n_leaves, out, cnt))
        return [out[i, : cnt[i]].copy() for i in range(nq)]

    def descend_from(self, t: int, queries: np.ndarray, start) -> np.ndarray:
        """kd_forest.cpp:266-274 batched."""
        q = np.ascontiguousarray(np.atleast_2d(queries), np.float32)
        nq, dim = q.shape
        st = np.ascontiguousarray(np.broadcast_to(np.asarray(start, np.uint32), (nq,)), np.uint32)
        out = np.empty(nq, np.uint32)
        check(lib.annk_descend_from(self._h, t, q, nq, dim, st, out))
        return out

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib.annk_forest_destroy(h)
            self._h = None


def build_forest(vs, n_trees: int, leaf_cap: int, seed: int, workers: int = 1) -> KdForest:
    """kd_forest.cpp:245-264 — bit-identical trees to the reference for the same seed."""
    v = _as_vs(vs)
    h = C.c_void_p()
    check(lib.annk_forest_build(v.handle, n_trees, leaf_cap, seed, C.byref(h)))
    return KdForest(h, v.n, v.dim, leaf_cap, seed, n_trees)


def search_leaves(forest: KdForest, t: int, q, n_leaves: int) -> np.ndarray:
    return forest.search_leaves(t, np.asarray(q, np.float32)[None, :], n_leaves)[0]


def descend_from(forest: KdForest, t: int, q, node: int) -> int:
    return int(forest.descend_from(t, np.asarray(q, np.float32)[None, :], node)[0])


# ------------------------------------------------------------ refine state

class RefineState:
    """Device-resident RefineState (graph_build.hpp:17-30).  Host views of the
    pools and adjacency lists are materialised on demand."""

    def __init__(self, handle):
        self._h = handle

    @property
    def handle(self):
        return self._h

    def meta(self):
        m = np.empty(8, np.uint64)
        check(lib.annk_state_meta(self._h, m))
        return dict(n=int(m[0]), k=int(m[1]), pool_cap=int(m[2]), sample_cap=int(m[3]), seed=int(m[4]),
                    iteration=int(m[5]), dist_comps=int(m[6]), last_changes=int(m[7]))

    def __getattr__(self, name):
        if name in ("n", "k", "pool_cap", "sample_cap", "seed", "iteration", "dist_comps", "last_changes"):
            return self.meta()[name]
        if name in ("g_new", "g_old", "g_rnew", "g_rold"):
            return self.lists(("g_new", "g_old", "g_rnew", "g_rold").index(name))
        raise AttributeError(name)

    def pools(self):
        """(sizes, ids, dists, flags) with rows of pool_cap slots."""
        m = self.meta()
        n, P = m["n"], m["pool_cap"]
        sizes = np.empty(n, np.uint32)
        ids = np.empty((n, P), np.uint32)
        dists = np.empty((n, P), np.float32)
        flags = np.empty((n, P), np.uint8)
        check(lib.annk_state_export(self._h, sizes, ids, dists, flags))
        return sizes, ids, dists, flags

    def lists(self, which: int):
        n = self.meta()["n"]
        off = np.empty(n + 1, np.uint32)
        check(lib.annk_state_lists(self._h, which, off, None))
        data = np.empty(max(int(off[-1]), 1), np.uint32)
        check(lib.annk_state_lists(self._h, which, off, data.ctypes.data_as(C.c_void_p)))
        return [data[off[i]:off[i + 1]].copy() for i in range(n)]

    @classmethod
    def from_pools(cls, n, k, pool_cap, sample_cap, seed, sizes, ids, dists, flags, iteration=0, dist_comps=0):
        h = C.c_void_p()
        check(lib.annk_state_import(n, k, pool_cap, sample_cap, seed, iteration, dist_comps,
                                    np.ascontiguousarray(sizes, np.uint32), np.ascontiguousarray(ids, np.uint32),
                                    np.ascontiguousarray(dists, np.float32), np.ascontiguousarray(flags, np.uint8),
                                    C.byref(h)))
        return cls(h)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib.annk_state_destroy(h)
            self._h = None


def init_graph(vs, forest: KdForest, k: int, conquer_depth: int, pool_cap: int, sample_cap: int, seed: int,
               workers: int = 1) -> RefineState:
    """graph_build.cpp:230-292."""
    v = _as_vs(vs)
    h = C.c_void_p()
    check(lib.annk_init_graph(v.handle, forest.handle, k, conquer_depth, pool_cap, sample_cap, seed, C.byref(h)))
    return RefineState(h)


def init_random(vs, k: int, pool_cap: int, sample_cap: int, seed: int, workers: int = 1) -> RefineState:
    """graph_build.cpp:294-326 (random-descent baseline start)."""
    v = _as_vs(vs)
    h = C.c_void_p()
    check(lib.annk_init_random(v.handle, k, pool_cap, sample_cap, seed, C.byref(h)))
    return RefineState(h)


class detail:
    """graph_build.hpp:117-133 detail:: entry points."""

    @staticmethod
    def nn_descent_iteration(state: RefineState, vs, workers: int = 1) -> int:
        ch = C.c_uint64(0)
        v = _as_vs(vs)  # keep the handle alive across the call
        check(lib.annk_nn_descent_iteration(state.handle, v.handle, C.byref(ch)))
        return int(ch.value)

    @staticmethod
    def nn_descent_iteration_finalize(state: RefineState, vs, k: int, out_ids: Optional[np.ndarray] = None,
                                      out_dists: Optional[np.ndarray] = None):
        """The last round of a build and finalize as one call
        (graph_build.cpp:105-162 then :346-373): the same changes, pools and
        graph as nn_descent_iteration + finalize, with the finalized rows
        copied out chunk by chunk while the remaining targets are replayed.
        Returns (changes, dist_comps after the round, KnnGraph)."""
        n = state.meta()["n"]
        ids = np.empty((n, k), np.uint32) if out_ids is None else out_ids
        d = np.empty((n, k), np.float32) if out_dists is None else out_dists
        if ids.shape != (n, k) or d.shape != (n, k) or ids.dtype != np.uint32 or d.dtype != np.float32:
            raise InvalidArgument("finalize: output buffers must be n x k uint32 / float32")
        ch, comps = C.c_uint64(0), C.c_uint64(0)
        v = _as_vs(vs)
        check(lib.annk_nn_descent_iteration_finalize(state.handle, v.handle, k, ids, d, C.byref(ch), C.byref(comps)))
        return int(ch.value), int(comps.value), KnnGraph(ids, d)

    @staticmethod
    def nn_expansion_iteration(state: RefineState, vs, workers: int = 1) -> int:
        """graph_build.cpp:164-207 (the NN-expansion baseline) on the device."""
        ch = C.c_uint64(0)
        v = _as_vs(vs)
        check(lib.annk_nn_expansion_iteration(state.handle, v.handle, C.byref(ch)))
        return int(ch.value)

    @staticmethod
    def rebuild_sample_lists(state: RefineState) -> None:
        check(lib.annk_rebuild_sample_lists(state.handle))

    @staticmethod
    def union_reverse_lists(state: RefineState) -> None:
        check(lib.annk_union_reverse_lists(state.handle))

    @staticmethod
    def pool_topk_accuracy(state: RefineState, gt: np.ndarray, rows: Optional[np.ndarray] = None) -> float:
        gt = np.ascontiguousarray(gt, np.uint32)
        acc = C.c_double(0)
        r = None if rows is None else np.ascontiguousarray(rows, np.uint32)
        check(lib.annk_pool_topk_accuracy(state.handle, gt, gt.shape[0], gt.shape[1], ptr(r), C.byref(acc)))
        return float(acc.value)


def refine_nn_descent(state: RefineState, vs, max_iters: int, workers: int = 1,
                      min_change_rate: float = 0.001) -> int:
    """graph_build.cpp:328-335; returns the number of iterations run."""
    it = C.c_uint32(0)
    v = _as_vs(vs)
    check(lib.annk_refine_nn_descent(state.handle, v.handle, max_iters, min_change_rate, C.byref(it)))
    return int(it.value)


def finalize(state: RefineState, vs, k: int, out_ids: Optional[np.ndarray] = None,
             out_dists: Optional[np.ndarray] = None) -> KnnGraph:
    """graph_build.cpp:346-373.  out_ids/out_dists (n x k, C-contiguous) may be
    caller buffers, e.g. pinned host memory for fast device-to-host copies."""
    n = state.meta()["n"]
    ids = np.empty((n, k), np.uint32) if out_ids is None else out_ids
    d = np.empty((n, k), np.float32) if out_dists is None else out_dists
    if ids.shape != (n, k) or d.shape != (n, k) or ids.dtype != np.uint32 or d.dtype != np.float32:
        raise InvalidArgument("finalize: output buffers must be n x k uint32 / float32")
    v = _as_vs(vs)
    check(lib.annk_finalize(state.handle, v.handle, k, ids, d))
    return KnnGraph(ids, d)


# --------------------------------------------------------------- build_graph

STRATEGIES = ("efanna", "random-descent", "nn-expansion", "brute-force", "init-only")


@dataclass
class BuildParams:
    """graph_build.hpp:76-86 (defaults identical)."""
    k: int = 10
    conquer_depth: int = 4
    pool_cap: int = 30
    sample_cap: int = 20
    max_iters: int = 8
    strategy: str = "efanna"
    seed: int = 1
    workers: int = 1
    min_change_rate: float = 0.001


@dataclass
class IterationLog:
    iteration: int = 0
    seconds: float = 0.0
    dist_comps: int = 0
    changes: int = 0
    accuracy: float = -1.0


@dataclass
class BuildStats:
    init_seconds: float = 0.0
    refine_seconds: float = 0.0
    dist_comps: int = 0
    early_stopped: bool = False
    iterations: list = field(default_factory=list)

    def total_seconds(self):
        return self.init_seconds + self.refine_seconds


@dataclass
class BuildResult:
    graph: KnnGraph
    stats: BuildStats
    state: Optional[RefineState] = None


def graph_accuracy(graph, gt: np.ndarray) -> float:
    """eval.cpp:106-127: mean per-row |row ∩ truth| / k (order free)."""
    g = graph.ids if isinstance(graph, KnnGraph) else np.asarray(graph)
    gt = np.asarray(gt)
    if g.shape != gt.shape:
        raise InvalidArgument("graph_accuracy: graph and truth shapes differ")
    if g.shape[0] == 0:
        raise InvalidArgument("graph_accuracy: empty graph")
    s = 0.0
    for i in range(g.shape[0]):
        s += len(np.intersect1d(g[i], gt[i])) / gt.shape[1]
    return s / g.shape[0]


def recall(result_ids, gt_row) -> float:
    """eval.cpp:82-104."""
    a, b = np.asarray(result_ids), np.asarray(gt_row)
    if a.shape != b.shape:
        raise InvalidArgument("recall: result and truth sizes differ")
    if b.size == 0:
        raise InvalidArgument("recall: empty truth row")
    return len(np.intersect1d(a, b)) / b.size


def build_graph(vs, forest: Optional[KdForest], params: BuildParams, gt: Optional[np.ndarray] = None,
                gt_rows: Optional[np.ndarray] = None, keep_state: bool = False) -> BuildResult:
    """graph_build.cpp:395-461 for the device strategies (efanna, init-only,
    brute-force).  Accuracy (when gt is given) is not charged to the build time,
    as in the reference.  gt_rows lets gt cover a seeded sample of points."""
    v = _as_vs(vs)
    st = BuildStats()
    if params.strategy == "brute-force":
        t0 = time.perf_counter()
        comps = []
        g = brute_force_graph(v, params.k, dist_comps=comps)
        st.init_seconds = time.perf_counter() - t0
        st.dist_comps = comps[0]
        acc = graph_accuracy(g, gt) if gt is not None else -1.0
        st.iterations.append(IterationLog(0, st.init_seconds, comps[0], 0, acc))
        return BuildResult(g, st)
    if params.strategy not in ("efanna", "init-only", "random-descent", "nn-expansion"):
        raise InvalidArgument(f"build_graph: unknown strategy {params.strategy}")
    tree_init = params.strategy in ("efanna", "init-only")  # graph_build.cpp:415-416
    if tree_init and forest is None:
        raise InvalidArgument("build_graph: strategy needs a forest")
    lib.annk_synchronize()
    t0 = time.perf_counter()
    if tree_init:
        state = init_graph(v, forest, params.k, params.conquer_depth, params.pool_cap, params.sample_cap,
                           params.seed)
    else:
        state = init_random(v, params.k, params.pool_cap, params.sample_cap, params.seed)
    st.init_seconds = time.perf_counter() - t0

    def log_row(changes):
        m = state.meta()
        acc = detail.pool_topk_accuracy(state, gt, gt_rows) if gt is not None else -1.0
        st.iterations.append(IterationLog(m["iteration"], st.init_seconds + st.refine_seconds,
                                          m["dist_comps"], changes, acc))

    log_row(0)
    iters = 0 if params.strategy == "init-only" else params.max_iters
    threshold = params.min_change_rate * v.n * params.pool_cap
    g = None
    for it in range(iters):
        t1 = time.perf_counter()
        if it == iters - 1 and gt is None and params.strategy != "nn-expansion":
            # the iteration cap makes this the last round whatever `changes` says:
            # replay and finalize overlap the device-to-host copy of the rows
            ch, comps, g = detail.nn_descent_iteration_finalize(state, v, params.k)
            st.refine_seconds += time.perf_counter() - t1
            st.iterations.append(IterationLog(state.meta()["iteration"], st.init_seconds + st.refine_seconds,
                                              comps, ch, -1.0))
            st.early_stopped = ch < threshold
            break
        ch = (detail.nn_expansion_iteration(state, v) if params.strategy == "nn-expansion"
              else detail.nn_descent_iteration(state, v))
        st.refine_seconds += time.perf_counter() - t1
        log_row(ch)
        if ch < threshold:
            st.early_stopped = True
            break
    if g is None:
        g = finalize(state, v, params.k)
    st.dist_comps = state.meta()["dist_comps"]
    return BuildResult(g, st, state if keep_state else None)


# ------------------------------------------------------------------ search

@dataclass
class SearchParams:
    """search.hpp:13-21 (defaults identical)."""
    k_return: int = 10
    pool_size: int = 100
    expansion: int = 100
    iters: int = 4
    n_trees_used: int = 0
    random_seed_count: int = 0
    seed: int = 1


@dataclass
class SearchStats:
    dist_comps: int = 0
    leaves_visited: int = 0
    graph_hops: int = 0
    seed_points: int = 0


@dataclass
class SearchResult:
    ids: np.ndarray
    dists: np.ndarray
    stats: SearchStats


@dataclass
class BatchResult:
    ids: np.ndarray      # nq x k_return
    dists: np.ndarray    # nq x k_return
    stats: np.ndarray    # nq x 4: dist_comps, leaves_visited, graph_hops, seed_points


class GraphSearcher:
    """search.cpp:23-154.  Keeps references to base / forest like the
    reference (caller keeps them alive) and uploads the graph once."""

    def __init__(self, base, forest: Optional[KdForest], graph):
        self.base = _as_vs(base)
        self.forest = forest
        ids = graph.ids if isinstance(graph, KnnGraph) else np.asarray(graph)
        ids = np.ascontiguousarray(ids, np.uint32)
        if ids.ndim != 2:
            raise InvalidArgument("searcher: graph must be n x k")
        h = C.c_void_p()
        check(lib.annk_searcher_create(self.base.handle, forest.handle if forest else None,
                                       ids if ids.size else np.zeros(1, np.uint32), ids.shape[0], ids.shape[1],
                                       C.byref(h)))
        self._h = h

    @staticmethod
    def _params(p: SearchParams, random_init: bool, seed_base: int):
        return SearchParamsC(p.k_return, p.pool_size, p.expansion, p.iters, p.n_trees_used,
                             p.random_seed_count, seed_base, int(random_init))

    def search_batch(self, queries, params: SearchParams, random_init: bool = False,
                     out: Optional[tuple] = None) -> BatchResult:
        """All queries at once; per-query seed = substream(params.seed, qi) as in
        recall_curve (search.cpp:208).  `out` = (ids, dists, stats) caller
        buffers (nq x k_return uint32, nq x k_return float32, nq x 4 uint64),
        e.g. pinned host memory for fast device-to-host copies."""
        cp = self._params(params, random_init, params.seed)
        q = None
        if isinstance(queries, VectorSet):
            nq = queries.n
        else:
            q = np.ascontiguousarray(np.atleast_2d(queries), np.float32)
            nq = q.shape[0]
        kr = params.k_return
        if out is None:
            ids = np.empty((nq, kr), np.uint32)
            d = np.empty((nq, kr), np.float32)
            st = np.empty((nq, 4), np.uint64)
        else:
            ids, d, st = out
            if (ids.shape != (nq, kr) or d.shape != (nq, kr) or st.shape != (nq, 4) or ids.dtype != np.uint32
                    or d.dtype != np.float32 or st.dtype != np.uint64 or not all(
                        a.flags.c_contiguous for a in (ids, d, st))):
                raise InvalidArgument("search: output buffers must be nq x k_return uint32 / float32, nq x 4 uint64")
        if q is None:
            check(lib.annk_search_dataset(self._h, queries.handle, C.byref(cp), ids, d, ptr(st)))
        else:
            check(lib.annk_search(self._h, q, nq, q.shape[1], C.byref(cp), ids, d, ptr(st)))
        return BatchResult(ids, d, st)

    def _one(self, q, params, random_init):
        q = np.asarray(q, np.float32)
        if q.ndim != 1 or q.shape[0] != self.base.dim:
            raise InvalidArgument("search: query length mismatch")
        # single query: SearchParams.seed is used as given (no per-query substream)
        cp = self._params(params, random_init, params.seed)
        cp.seed = params.seed
        ids = np.empty((1, params.k_return), np.uint32)
        d = np.empty((1, params.k_return), np.float32)
        st = np.empty((1, 4), np.uint64)
        check(lib.annk_search(self._h, np.ascontiguousarray(q[None, :]), 1, q.shape[0], C.byref(cp), ids, d,
                              ptr(st)))
        valid = ids[0] != INVALID_ID
        return SearchResult(ids[0][valid], d[0][valid], SearchStats(*[int(x) for x in st[0]]))

    def search(self, q, params: SearchParams) -> SearchResult:
        return self._one(q, params, False)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib.annk_searcher_destroy(h)
            self._h = None


@dataclass
class SweepPoint:
    expansion: int
    pool_size: int


@dataclass
class SweepRow:
    expansion: int = 0
    pool_size: int = 0
    mean_time_us: float = 0.0
    avg_recall: float = 0.0
    avg_dist_comps: float = 0.0
    avg_seed_points: float = 0.0


def recall_curve(base, forest, graph, queries, gt: np.ndarray, sweep: Sequence[SweepPoint],
                 params: SearchParams, random_init: bool = False, workers: int = 1) -> list:
    """search.cpp:182-236.  mean_time_us is the batch wall time / nq."""
    q = _as_vs(queries)
    if q.n == 0:
        raise InvalidArgument("recall_curve: empty query set")
    b = _as_vs(base)
    if q.dim != b.dim:
        raise InvalidArgument("recall_curve: query dim mismatch")
    gt = np.asarray(gt)
    if gt.shape[0] != q.n:
        raise InvalidArgument("recall_curve: ground truth shape")
    if gt.shape[1] < params.k_return:
        raise InvalidArgument("recall_curve: ground truth narrower than k_return")
    s = GraphSearcher(b, forest, graph)
    table = []
    for pt in sweep:
        p = SearchParams(**{**params.__dict__, "expansion": pt.expansion, "pool_size": pt.pool_size})
        t0 = time.perf_counter()
        r = s.search_batch(q, p, random_init)
        dt = time.perf_counter() - t0
        rec = 0.0
        for qi in range(q.n):
            rec += recall(r.ids[qi], gt[qi, : p.k_return])
        table.append(SweepRow(pt.expansion, pt.pool_size, dt * 1e6 / q.n, rec / q.n,
                              float(r.stats[:, 0].astype(np.float64).mean()),
                              float(r.stats[:, 3].astype(np.float64).mean())))
    return table


def state_stats(state: RefineState) -> dict:
    """Device counters of the last NN-descent round (join rows, offers, spills)."""
    out = np.zeros(4, np.uint64)
    check(lib.annk_state_stats(state.handle, out))
    return dict(join_rows=int(out[0]), offers=int(out[1]), spilled=int(out[2]), offer_slots=int(out[3]))
