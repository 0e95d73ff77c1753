"""Python view of the CPU checkers — TEST INFRASTRUCTURE ONLY.

Wraps the C interface in ``oracle/oracle_abi.h``, which two libraries implement:

* ``oracle/liboracle.so``         — our C restatement of the reference (``annkit_oracle.c``)
* ``oracle/_ref/libannkit_ref.so`` — the unmodified reference library plus a thin shim

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg
import this module.  The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
RESTATEMENT_PATH = os.path.join(HERE, "liboracle.so")
REFERENCE_PATH = os.path.join(HERE, "_ref", "libannkit_ref.so")

_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C")
_f32p = np.ctypeslib.ndpointer(np.float32, flags="C")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C")
_vp = C.c_void_p
_u32 = C.c_uint32
_u64 = C.c_uint64


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def _ptr_or_null(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


@dataclass
class Tree:
    split_dim: np.ndarray
    split_val: np.ndarray
    left: np.ndarray
    right: np.ndarray
    depth: np.ndarray
    even: np.ndarray
    point_index: np.ndarray
    root: int
    leaf_count: int

    @property
    def n_nodes(self) -> int:
        return len(self.split_dim)


class OracleLib:
    """One loaded checker (restatement or reference)."""

    def __init__(self, path: str):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.path = path
        L = C.CDLL(path)
        self.L = L
        L.ora_last_error.restype = C.c_char_p
        L.ora_impl_name.restype = C.c_char_p
        L.ora_vs_create.restype = _vp
        L.ora_vs_create.argtypes = [_f32p, _u32, _u32]
        L.ora_vs_free.argtypes = [_vp]
        L.ora_gen_synthetic.argtypes = [_u32, _u32, _u64, _f32p]
        if hasattr(L, "ora_gen_mixture"):  # restatement only (not a reference function)
            L.ora_gen_mixture.argtypes = [_u32, _u32, _u32, C.c_float, C.c_float, C.c_float, C.c_float, C.c_float,
                                          C.c_int, _u64, _u32, _u32, _f32p]
        L.ora_l2_sq.restype = C.c_float
        L.ora_l2_sq.argtypes = [_f32p, _f32p, _u32]
        L.ora_mix64.restype = _u64
        L.ora_mix64.argtypes = [_u64]
        L.ora_substream.restype = _u64
        L.ora_substream.argtypes = [_u64, _u64]
        L.ora_mt19937_64.argtypes = [_u64, _u32, _u64p]
        L.ora_brute_force.argtypes = [_vp, _vp, _u32, _u32, _u32p, _vp, C.POINTER(_u64)]
        L.ora_forest_build.restype = _vp
        L.ora_forest_build.argtypes = [_vp, _u32, _u32, _u64, _u32, C.POINTER(C.c_int)]
        L.ora_forest_free.argtypes = [_vp]
        L.ora_forest_num_trees.restype = _u32
        L.ora_forest_num_trees.argtypes = [_vp]
        L.ora_forest_num_nodes.restype = _u32
        L.ora_forest_num_nodes.argtypes = [_vp, _u32]
        L.ora_forest_export.argtypes = [_vp, _u32, _u32p, _f32p, _u32p, _u32p, _u32p, _u8p, _u32p, _u32p]
        L.ora_forest_import.restype = _vp
        L.ora_forest_import.argtypes = [_u32, _u32, _u32, _u64, _u32, _u32p, _u32p, _u32p, _f32p,
                                        _u32p, _u32p, _u32p, _u8p, _u32p]
        L.ora_search_leaves.argtypes = [_vp, _u32, _f32p, _u32, _u32, _u32p, C.POINTER(_u32)]
        L.ora_descend_from.argtypes = [_vp, _u32, _f32p, _u32, _u32, C.POINTER(_u32)]
        L.ora_init_graph.restype = _vp
        L.ora_init_graph.argtypes = [_vp, _vp, _u32, _u32, _u32, _u32, _u64, _u32, C.POINTER(C.c_int)]
        L.ora_init_random.restype = _vp
        L.ora_init_random.argtypes = [_vp, _u32, _u32, _u32, _u64, _u32, C.POINTER(C.c_int)]
        L.ora_state_import.restype = _vp
        L.ora_state_import.argtypes = [_u32, _u32, _u32, _u32, _u64, _u32, _u64, _u32p, _u32p, _f32p, _u8p]
        L.ora_state_free.argtypes = [_vp]
        L.ora_state_export.argtypes = [_vp, _u32p, _u32p, _f32p, _u8p, _u64p]
        L.ora_state_lists.argtypes = [_vp, C.c_int, _u32p, _vp]
        L.ora_nn_descent_iteration.restype = _u64
        L.ora_nn_descent_iteration.argtypes = [_vp, _vp, _u32]
        L.ora_nn_expansion_iteration.restype = _u64
        L.ora_nn_expansion_iteration.argtypes = [_vp, _vp, _u32]
        L.ora_rebuild_sample_lists.argtypes = [_vp]
        if hasattr(L, "ora_ref_save_forest"):  # reference only: its own file writers/readers
            L.ora_ref_save_forest.argtypes = [_vp, C.c_char_p]
            L.ora_ref_load_forest.restype = _vp
            L.ora_ref_load_forest.argtypes = [C.c_char_p, C.POINTER(C.c_int)]
            L.ora_ref_save_fvecs.argtypes = [_vp, C.c_char_p]
            L.ora_ref_save_ivecs.argtypes = [_u32p, _u32, _u32, C.c_char_p]
            L.ora_ref_accuracy_vs_k.argtypes = [_vp, _u32p, _u32, _u32, _u32p, _u32, _f64p]
        if hasattr(L, "ora_shard_sample"):  # restatement only: shard-mode protocol
            L.ora_shard_sample.argtypes = [_vp, _u32, _u32, _u32p, _u32p, _u32p, _u32p, _u64p]
            L.ora_shard_union.argtypes = [_vp, _u32p, _u32p, _u32p, _u32p]
            L.ora_shard_join.restype = _u64
            L.ora_shard_join.argtypes = [_vp, _vp, _u32, _u32, _u64p, C.POINTER(_u64)]
            L.ora_shard_offers_get.argtypes = [_u32p, _u64p, _u32p]
            L.ora_shard_replay.restype = _u64
            L.ora_shard_replay.argtypes = [_vp, _u32p, _u64p, _u32p, C.c_size_t]
            L.ora_shard_finish.argtypes = [_vp, _u64]
        L.ora_union_reverse_lists.argtypes = [_vp]
        L.ora_refine_nn_descent.argtypes = [_vp, _vp, _u32, _u32, C.c_double]
        L.ora_finalize.argtypes = [_vp, _vp, _u32, _u32p, _f32p]
        L.ora_pool_topk_accuracy.restype = C.c_double
        L.ora_pool_topk_accuracy.argtypes = [_vp, _u32p, _u32, _u32]
        L.ora_build_graph.argtypes = [_vp, _vp, _u32, _u32, _u32, _u32, _u32, C.c_int, _u64, _u32,
                                      C.c_double, _vp, _u32, _u32p, _vp, _f64p, C.POINTER(_u32), _f64p]
        L.ora_search.argtypes = [_vp, _vp, _u32p, _vp, _u32, _u32, _vp, _u32, _u32, _u32, _u32, _u32,
                                 _u32, _u64, C.c_int, _u32, _u32p, _f32p, _u64p, _vp]
        self.name = L.ora_impl_name().decode()

    # ------------------------------------------------------------- helpers
    def _check(self, code: int):
        if code != 0:
            raise OracleError(code, self.L.ora_last_error().decode())

    def gen_synthetic(self, n: int, dim: int, seed: int) -> np.ndarray:
        out = np.empty((n, dim), np.float32)
        self.L.ora_gen_synthetic(n, dim, seed, out)
        return out

    def gen_mixture(self, n, dim, n_centers, center_lo, center_hi, sd, clip_lo, clip_hi, round_to_int, seed,
                    stream_id, workers=None) -> np.ndarray:
        """The BASELINE configs' seeded Gaussian mixture, byte-identical to the
        product's annk_gen_mixture (tests/test_oracle_pin.py pins it)."""
        out = np.empty((n, dim), np.float32)
        w = workers or max(1, min(os.cpu_count() or 1, n // 4096))
        self.L.ora_gen_mixture(n, dim, n_centers, center_lo, center_hi, sd, clip_lo, clip_hi, int(bool(round_to_int)),
                               seed, stream_id, w, out)
        return out

    def mt19937_64(self, seed: int, count: int) -> np.ndarray:
        out = np.empty(count, np.uint64)
        self.L.ora_mt19937_64(seed, count, out)
        return out

    def mix64(self, x: int) -> int:
        return int(self.L.ora_mix64(x))

    def substream(self, seed: int, i: int) -> int:
        return int(self.L.ora_substream(seed, i))

    def l2_sq(self, a: np.ndarray, b: np.ndarray) -> float:
        a = np.ascontiguousarray(a, np.float32)
        b = np.ascontiguousarray(b, np.float32)
        return float(self.L.ora_l2_sq(a, b, len(a)))

    def vs(self, x: np.ndarray) -> "VS":
        return VS(self, x)

    def brute_force(self, base: "VS", queries: "VS | None", k: int, workers: int = 1, with_dists=False):
        nq = queries.n if queries is not None else base.n
        ids = np.empty((nq, k), np.uint32)
        dists = np.empty((nq, k), np.float32) if with_dists else None
        comps = _u64(0)
        self._check(self.L.ora_brute_force(base.h, queries.h if queries else None, k, workers, ids,
                                           _ptr_or_null(dists), C.byref(comps)))
        return (ids, dists, int(comps.value)) if with_dists else ids

    def build_forest(self, vs: "VS", n_trees: int, leaf_cap: int, seed: int, workers: int = 1) -> "Forest":
        st = C.c_int(0)
        h = self.L.ora_forest_build(vs.h, n_trees, leaf_cap, seed, workers, C.byref(st))
        self._check(st.value)
        return Forest(self, h, vs.n, vs.dim, leaf_cap, seed)

    def import_forest(self, n, dim, leaf_cap, seed, trees: list[Tree]) -> "Forest":
        cat = lambda attr, dt: np.ascontiguousarray(np.concatenate([getattr(t, attr) for t in trees]).astype(dt))
        h = self.L.ora_forest_import(
            n, dim, leaf_cap, seed, len(trees),
            np.array([t.n_nodes for t in trees], np.uint32), np.array([t.root for t in trees], np.uint32),
            cat("split_dim", np.uint32), cat("split_val", np.float32), cat("left", np.uint32),
            cat("right", np.uint32), cat("depth", np.uint32), cat("even", np.uint8),
            cat("point_index", np.uint32))
        return Forest(self, h, n, dim, leaf_cap, seed)

    # reference-only file writers/readers (byte-compatibility checks)
    def ref_save_forest(self, forest: "Forest", path: str):
        self._check(self.L.ora_ref_save_forest(forest.h, path.encode()))

    def ref_load_forest(self, path: str, n, dim, leaf_cap, seed) -> "Forest":
        st = C.c_int(0)
        h = self.L.ora_ref_load_forest(path.encode(), C.byref(st))
        self._check(st.value)
        return Forest(self, h, n, dim, leaf_cap, seed)

    def ref_save_fvecs(self, vs: "VS", path: str):
        self._check(self.L.ora_ref_save_fvecs(vs.h, path.encode()))

    def ref_accuracy_vs_k(self, vs: "VS", ids: np.ndarray, k_list) -> list:
        ids = np.ascontiguousarray(ids, np.uint32)
        kl = np.ascontiguousarray(k_list, np.uint32)
        out = np.empty(kl.size, np.float64)
        self._check(self.L.ora_ref_accuracy_vs_k(vs.h, ids, ids.shape[0], ids.shape[1], kl, kl.size, out))
        return out.tolist()

    def ref_save_ivecs(self, ids: np.ndarray, path: str):
        ids = np.ascontiguousarray(ids, np.uint32)
        self._check(self.L.ora_ref_save_ivecs(ids, ids.shape[0], ids.shape[1], path.encode()))

    def init_graph(self, vs, forest, k, conquer_depth, pool_cap, sample_cap, seed, workers=1) -> "State":
        st = C.c_int(0)
        h = self.L.ora_init_graph(vs.h, forest.h, k, conquer_depth, pool_cap, sample_cap, seed, workers,
                                  C.byref(st))
        self._check(st.value)
        return State(self, h, vs.n, pool_cap)

    def init_random(self, vs, k, pool_cap, sample_cap, seed, workers=1) -> "State":
        st = C.c_int(0)
        h = self.L.ora_init_random(vs.h, k, pool_cap, sample_cap, seed, workers, C.byref(st))
        self._check(st.value)
        return State(self, h, vs.n, pool_cap)

    def import_state(self, n, k, pool_cap, sample_cap, seed, iteration, dist_comps, sizes, ids, dists, flags):
        h = self.L.ora_state_import(n, k, pool_cap, sample_cap, seed, iteration, dist_comps,
                                    np.ascontiguousarray(sizes, np.uint32), np.ascontiguousarray(ids, np.uint32),
                                    np.ascontiguousarray(dists, np.float32), np.ascontiguousarray(flags, np.uint8))
        return State(self, h, n, pool_cap)

    def build_graph(self, vs, forest, k=10, conquer_depth=4, pool_cap=30, sample_cap=20, max_iters=8,
                    strategy=0, seed=1, workers=1, min_change_rate=0.001, gt=None):
        ids = np.empty((vs.n, k), np.uint32)
        dists = np.empty((vs.n, k), np.float32)
        log = np.zeros((max_iters + 1, 5), np.float64)
        nlog = _u32(0)
        summ = np.zeros(4, np.float64)
        gtc = None if gt is None else np.ascontiguousarray(gt, np.uint32)
        self._check(self.L.ora_build_graph(vs.h, forest.h if forest else None, k, conquer_depth, pool_cap,
                                           sample_cap, max_iters, strategy, seed, workers, min_change_rate,
                                           _ptr_or_null(gtc), 0 if gt is None else gt.shape[1], ids,
                                           dists.ctypes.data_as(C.c_void_p), log, C.byref(nlog), summ))
        return ids, dists, log[: nlog.value], summ

    def search(self, base, forest, graph_ids, queries, k_return=10, pool_size=100, expansion=100, iters=4,
               n_trees_used=0, random_seed_count=0, seed=1, random_init=False, workers=1, with_time=False):
        nq = queries.n
        gids = np.ascontiguousarray(graph_ids, np.uint32)
        ids = np.empty((nq, k_return), np.uint32)
        dists = np.empty((nq, k_return), np.float32)
        stats = np.empty((nq, 4), np.uint64)
        tus = np.empty(nq, np.float64) if with_time else None
        self._check(self.L.ora_search(base.h, forest.h if forest else None, gids, None, gids.shape[0],
                                      gids.shape[1], queries.h, k_return, pool_size, expansion, iters,
                                      n_trees_used, random_seed_count, seed, int(random_init), workers, ids,
                                      dists, stats, _ptr_or_null(tus)))
        return (ids, dists, stats, tus) if with_time else (ids, dists, stats)


class VS:
    def __init__(self, lib: OracleLib, x: np.ndarray):
        x = np.ascontiguousarray(x, np.float32)
        if x.ndim != 2:
            raise ValueError("expected n x dim")
        self.lib, self.x = lib, x
        self.n, self.dim = x.shape
        self.h = lib.L.ora_vs_create(x if x.size else np.zeros(1, np.float32), self.n, self.dim)

    def __del__(self):
        try:
            self.lib.L.ora_vs_free(self.h)
        except Exception:
            pass


class Forest:
    def __init__(self, lib, h, n, dim, leaf_cap, seed):
        self.lib, self.h, self.n, self.dim, self.leaf_cap, self.seed = lib, h, n, dim, leaf_cap, seed

    def __del__(self):
        try:
            self.lib.L.ora_forest_free(self.h)
        except Exception:
            pass

    @property
    def n_trees(self):
        return int(self.lib.L.ora_forest_num_trees(self.h))

    def tree(self, t: int) -> Tree:
        L = self.lib.L
        m = int(L.ora_forest_num_nodes(self.h, t))
        sd = np.empty(m, np.uint32); sv = np.empty(m, np.float32); le = np.empty(m, np.uint32)
        ri = np.empty(m, np.uint32); de = np.empty(m, np.uint32); ev = np.empty(m, np.uint8)
        pi = np.empty(self.n, np.uint32); rl = np.empty(2, np.uint32)
        L.ora_forest_export(self.h, t, sd, sv, le, ri, de, ev, pi, rl)
        return Tree(sd, sv, le, ri, de, ev, pi, int(rl[0]), int(rl[1]))

    def trees(self):
        return [self.tree(t) for t in range(self.n_trees)]

    def search_leaves(self, t, q, n_leaves):
        q = np.ascontiguousarray(q, np.float32)
        out = np.empty(max(n_leaves, 1), np.uint32)
        cnt = _u32(0)
        self.lib._check(self.lib.L.ora_search_leaves(self.h, t, q, len(q), n_leaves, out, C.byref(cnt)))
        return out[: cnt.value].copy()

    def descend_from(self, t, q, node):
        q = np.ascontiguousarray(q, np.float32)
        out = _u32(0)
        self.lib._check(self.lib.L.ora_descend_from(self.h, t, q, len(q), node, C.byref(out)))
        return int(out.value)


class State:
    def __init__(self, lib, h, n, pool_cap):
        self.lib, self.h, self.n, self.pool_cap = lib, h, n, pool_cap

    def __del__(self):
        try:
            self.lib.L.ora_state_free(self.h)
        except Exception:
            pass

    def export(self):
        n, P = self.n, self.pool_cap
        sizes = np.empty(n, np.uint32)
        ids = np.zeros((n, P), np.uint32)
        dists = np.zeros((n, P), np.float32)
        flags = np.zeros((n, P), np.uint8)
        meta = np.empty(3, np.uint64)
        self.lib.L.ora_state_export(self.h, sizes, ids, dists, flags, meta)
        return dict(sizes=sizes, ids=ids, dists=dists, flags=flags, iteration=int(meta[0]),
                    dist_comps=int(meta[1]), last_changes=int(meta[2]))

    def lists(self, which: int):
        off = np.empty(self.n + 1, np.uint32)
        self.lib.L.ora_state_lists(self.h, which, off, None)
        data = np.empty(max(int(off[-1]), 1), np.uint32)
        self.lib.L.ora_state_lists(self.h, which, off, data.ctypes.data_as(C.c_void_p))
        return [data[off[i]:off[i + 1]].copy() for i in range(self.n)]

    def nn_descent_iteration(self, vs, workers=1) -> int:
        return int(self.lib.L.ora_nn_descent_iteration(self.h, vs.h, workers))

    def nn_expansion_iteration(self, vs, workers=1) -> int:
        return int(self.lib.L.ora_nn_expansion_iteration(self.h, vs.h, workers))

    def rebuild_sample_lists(self):
        self.lib.L.ora_rebuild_sample_lists(self.h)

    # shard-mode protocol (see annkit_oracle.c); row buffers are full-n arrays
    def shard_sample(self, lo, hi, fnew, cnew, fold, cold, thr):
        self.lib.L.ora_shard_sample(self.h, lo, hi, fnew, cnew, fold, cold, thr)

    def shard_union(self, fnew, cnew, fold, cold):
        self.lib.L.ora_shard_union(self.h, fnew, cnew, fold, cold)

    def shard_join(self, vs, lo, hi, thr):
        m = C.c_uint64(0)
        comps = int(self.lib.L.ora_shard_join(self.h, vs.h, lo, hi, thr, C.byref(m)))
        tgt = np.empty(max(m.value, 1), np.uint32)
        key = np.empty(max(m.value, 1), np.uint64)
        src = np.empty(max(m.value, 1), np.uint32)
        self.lib.L.ora_shard_offers_get(tgt, key, src)
        return comps, tgt[:m.value], key[:m.value], src[:m.value]

    def shard_replay(self, tgt, key, src):
        """Offers replayed into their pools in the reference's order (source
        point ascending, a source's offers as given); returns accepted inserts."""
        tgt = np.ascontiguousarray(tgt, np.uint32)
        key = np.ascontiguousarray(key, np.uint64)
        src = np.ascontiguousarray(src, np.uint32)
        return int(self.lib.L.ora_shard_replay(self.h, tgt, key, src, tgt.size))

    def shard_finish(self, changes):
        self.lib.L.ora_shard_finish(self.h, int(changes))

    def union_reverse_lists(self):
        self.lib.L.ora_union_reverse_lists(self.h)

    def refine(self, vs, max_iters, workers=1, min_change_rate=0.001):
        self.lib._check(self.lib.L.ora_refine_nn_descent(self.h, vs.h, max_iters, workers, min_change_rate))

    def finalize(self, vs, k):
        ids = np.empty((self.n, k), np.uint32)
        d = np.empty((self.n, k), np.float32)
        self.lib._check(self.lib.L.ora_finalize(self.h, vs.h, k, ids, d))
        return ids, d

    def pool_topk_accuracy(self, gt: np.ndarray) -> float:
        gt = np.ascontiguousarray(gt, np.uint32)
        return float(self.lib.L.ora_pool_topk_accuracy(self.h, gt, gt.shape[0], gt.shape[1]))


_cache: dict[str, OracleLib] = {}


def load(which: str = "oracle") -> OracleLib:
    """which: 'oracle' (C restatement) or 'reference' (oracle/_ref)."""
    path = RESTATEMENT_PATH if which == "oracle" else REFERENCE_PATH
    if path not in _cache:
        _cache[path] = OracleLib(path)
    return _cache[path]


def reference_available() -> bool:
    return os.path.exists(REFERENCE_PATH)
