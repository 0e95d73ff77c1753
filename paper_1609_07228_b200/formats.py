"""The reference's on-disk formats, read and written from device handles
(SURVEY §8(f) row 1): indices built on the GPU can be loaded by the CPU
reference and vice versa.

* fvecs / ivecs (dataset.cpp:96-200): per record an int32 dimension, then that
  many little-endian float32 / int32 values; no header.  Loading rejects
  non-positive or inconsistent dimensions, non-finite floats and negative ids
  with the reference's error classes.
* AKF1 forests (kd_forest.cpp:307-372): magic "AKF1", u32 version 1, u32 n,
  dim, n_trees, leaf_cap, u64 seed; per tree u32 node_count, u32 root, then
  node_count packed 21-byte nodes (u32 split_dim, f32 split_val, u32 left,
  u32 right, u32 depth, u8 even_split) and n u32 point_index entries.
  Loading runs the reference's validate_tree checks (kd_forest.cpp:175-243),
  vectorised.
* graphs (knn_graph.cpp:5-37): ids as ivecs, dists (optional) as fvecs.

Host byte layout only; the arrays move to / from the device through the
C-ABI (annk_forest_export / annk_forest_import, annk_dataset_create).
"""
from __future__ import annotations

import os
from typing import Optional

import numpy as np

from . import api

MAGIC = b"AKF1"
VERSION = 1
_NODE = np.dtype([("split_dim", "<u4"), ("split_val", "<f4"), ("left", "<u4"), ("right", "<u4"),
                  ("depth", "<u4"), ("even", "u1")])  # packed: 21 bytes, as written by the reference
assert _NODE.itemsize == 21


class FormatError(RuntimeError):
    """dataset.hpp:15-19 format_error: malformed file structure."""


class DataError(RuntimeError):
    """dataset.hpp:21-24 data_error: well-formed file, invalid values."""


# ------------------------------------------------------------ fvecs/ivecs

def _read_records(path: str, kind: str):
    try:
        size = os.path.getsize(path)
        raw = np.fromfile(path, dtype="<i4", count=size // 4)
    except OSError as e:
        raise FormatError(f"cannot open file for reading: {path}") from e
    words = raw.size
    if words == 0:
        if size % 4:
            raise FormatError(f"truncated record 0 at byte 0 in {path}")
        return np.zeros((0, 0), "<i4")
    d = int(raw[0])
    if d < 1:
        raise FormatError(f"record 0 at byte 0 declares dimension {d} in {path}")
    if words % (d + 1) or size % 4:
        # walk to the first inconsistent / cut record for the message: a record
        # cut short names the byte where its first missing value starts
        rec, off = 0, 0
        while True:
            if off == words:
                raise FormatError(f"truncated record {rec} at byte {4 * off} in {path}")
            dd = int(raw[off])
            if dd < 1:
                raise FormatError(f"record {rec} at byte {off * 4} declares dimension {dd} in {path}")
            if dd != d:
                raise FormatError(f"record {rec} has dimension {dd}, expected {d} in {path}")
            if off + 1 + dd > words:
                raise FormatError(f"truncated record {rec} at byte {4 * words} in {path}")
            off += dd + 1
            rec += 1
    rows = raw.reshape(-1, d + 1)
    bad = np.nonzero(rows[:, 0] != d)[0]
    if bad.size:
        r = int(bad[0])
        dd = int(rows[r, 0])
        if dd < 1:
            raise FormatError(f"record {r} at byte {r * (d + 1) * 4} declares dimension {dd} in {path}")
        raise FormatError(f"record {r} has dimension {dd}, expected {d} in {path}")
    return rows[:, 1:]


def validate_truth(ids: np.ndarray, base_n: int) -> None:
    """GroundTruth::validate_against (dataset.cpp:78-95 contract): every id
    inside the base set and no id twice in a row, else DataError."""
    if ids.size == 0:
        return
    over = np.argwhere(ids >= base_n)
    if over.size:
        r, c = map(int, over[0])
        raise DataError(f"row {r} holds id {int(ids[r, c])} outside base set of size {base_n}")
    srt = np.sort(ids, axis=1)
    dup = np.argwhere(srt[:, 1:] == srt[:, :-1])
    if dup.size:
        r, c = map(int, dup[0])
        raise DataError(f"row {r} holds duplicate id {int(srt[r, c])}")


def load_fvecs(path: str) -> np.ndarray:
    """dataset.cpp:96-133 load_fvecs -> n x dim float32."""
    body = _read_records(path, "fvecs")
    x = np.ascontiguousarray(body).view("<f4").astype(np.float32)
    if x.size and not np.isfinite(x).all():
        r, c = map(int, np.argwhere(~np.isfinite(x))[0])
        raise DataError(f"non-finite value in record {r} component {c} in {path}")
    return x


def save_fvecs(x: np.ndarray, path: str) -> None:
    """dataset.cpp:135-147 save_fvecs."""
    x = np.ascontiguousarray(x, np.float32)
    n, dim = x.shape
    out = np.empty((n, dim + 1), "<u4")
    out[:, 0] = dim
    out[:, 1:] = x.view("<u4")
    out.tofile(path)


def load_ivecs(path: str) -> np.ndarray:
    """dataset.cpp:149-184 load_ivecs -> n x k uint32."""
    body = _read_records(path, "ivecs")
    if body.size and (body < 0).any():
        r, c = map(int, np.argwhere(body < 0)[0])
        raise DataError(f"negative id in record {r} component {c} in {path}")
    return np.ascontiguousarray(body).astype(np.uint32)


def save_ivecs(ids: np.ndarray, path: str) -> None:
    """dataset.cpp:186-200 save_ivecs (ids must fit an int32 payload)."""
    ids = np.ascontiguousarray(ids, np.uint32)
    if ids.size and int(ids.max()) > 0x7FFFFFFF:
        raise DataError(f"id {int(ids.max())} does not fit an int32 payload")
    n, k = ids.shape
    out = np.empty((n, k + 1), "<u4")
    out[:, 0] = k
    out[:, 1:] = ids
    out.tofile(path)


def load_dataset(path: str) -> api.VectorSet:
    """fvecs file -> device VectorSet."""
    return api.VectorSet(load_fvecs(path))


# ------------------------------------------------------------------ graph

def save_graph(g: api.KnnGraph, ids_path: str, dists_path: Optional[str] = None) -> None:
    """knn_graph.cpp:5-19."""
    save_ivecs(g.ids, ids_path)
    if dists_path is not None:
        if g.dists is None:
            raise api.InvalidArgument("save_graph: graph has no distances")
        save_fvecs(g.dists, dists_path)


def load_graph(ids_path: str, dists_path: Optional[str] = None) -> api.KnnGraph:
    """knn_graph.cpp:21-37."""
    ids = load_ivecs(ids_path)
    d = None
    if dists_path is not None:
        d = load_fvecs(dists_path)
        if d.shape != ids.shape:
            raise FormatError(f"distance file {dists_path} has shape {d.shape[0]}x{d.shape[1]}, "
                              f"graph is {ids.shape[0]}x{ids.shape[1]}")
    return api.KnnGraph(ids, d)


# ----------------------------------------------------------------- forest

def save_forest(forest, path: str) -> None:
    """kd_forest.cpp:307-330 save_forest, from a device forest (or any forest
    exposing n, dim, n_trees, leaf_cap, seed and tree(t) arrays)."""
    with open(path, "wb") as fh:
        fh.write(MAGIC)
        np.array([VERSION, forest.n, forest.dim, forest.n_trees, forest.leaf_cap], "<u4").tofile(fh)
        np.array([forest.seed], "<u8").tofile(fh)
        for t in range(forest.n_trees):
            tr = forest.tree(t)
            even = tr.even_split if hasattr(tr, "even_split") else tr.even
            np.array([len(tr.split_dim), tr.root], "<u4").tofile(fh)
            rec = np.empty(len(tr.split_dim), _NODE)
            rec["split_dim"], rec["split_val"], rec["left"] = tr.split_dim, tr.split_val, tr.left
            rec["right"], rec["depth"], rec["even"] = tr.right, tr.depth, even
            rec.tofile(fh)
            np.asarray(tr.point_index).astype("<u4").tofile(fh)


def validate_tree(tr: api.KdTree, n: int, dim: int, leaf_cap: int) -> None:
    """kd_forest.cpp:175-243 validate_tree (same conditions, same error class)."""
    m = tr.n_nodes
    if m == 0 or tr.root >= m:
        raise FormatError("forest file: bad tree root")
    pi = np.asarray(tr.point_index)
    if pi.size != n:
        raise FormatError("forest file: point_index size mismatch")
    if (pi >= n).any():
        raise FormatError("forest file: point id out of range")
    if (np.bincount(pi, minlength=n) != 1).any():
        raise FormatError("forest file: point_index is not a permutation")
    depth = np.asarray(tr.depth, np.int64)
    if depth[tr.root] != 0:
        raise FormatError("forest file: root depth not 0")
    max_depth = 16
    mm = n
    while mm > 1:
        max_depth += 4
        mm //= 2
    sd = np.asarray(tr.split_dim)
    left, right = np.asarray(tr.left, np.int64), np.asarray(tr.right, np.int64)
    leaf = sd == api.LEAF_MARKER
    inner = ~leaf
    # topology: every node but the root is some internal node's child exactly once
    kids = np.concatenate([left[inner], right[inner]])
    if kids.size and ((kids >= m).any()):
        raise FormatError("forest file: child id out of range")
    refs = np.bincount(kids, minlength=m) if kids.size else np.zeros(m, np.int64)
    expect = np.ones(m, np.int64)
    expect[tr.root] = 0
    if (refs > expect).any():
        raise FormatError("forest file: malformed tree topology")
    if (refs < expect).any():
        raise FormatError("forest file: unreachable nodes present")
    if (depth > max_depth).any():
        raise FormatError("forest file: implausible tree depth")
    if ((sd[inner] >= dim)).any():
        raise FormatError("forest file: split dimension out of range")
    if inner.any() and ((depth[left[inner]] != depth[inner] + 1).any() or
                        (depth[right[inner]] != depth[inner] + 1).any()):
        raise FormatError("forest file: child depth mismatch")
    lo, hi = left[leaf], right[leaf]
    if ((lo >= hi) | (hi > n) | (hi - lo > leaf_cap)).any():
        raise FormatError("forest file: leaf range violates 1..leaf_cap")
    # ranges bottom-up: an internal node's left range must end where its right begins
    rlo = np.where(leaf, left, -1)
    rhi = np.where(leaf, right, -1)
    idx = np.nonzero(inner)[0]
    for dlev in sorted(set(depth[idx].tolist()), reverse=True):
        ids = idx[depth[idx] == dlev]
        l, r = left[ids], right[ids]
        if (rhi[l] != rlo[r]).any():
            raise FormatError("forest file: left subtree does not precede right subtree")
        rlo[ids], rhi[ids] = rlo[l], rhi[r]
    if rlo[tr.root] != 0 or rhi[tr.root] != n:
        raise FormatError("forest file: leaf ranges do not cover all points")


def parse_forest(path: str):
    """kd_forest.cpp:332-372 load_forest, host side: (n, dim, leaf_cap, seed, [KdTree])."""
    try:
        blob = np.fromfile(path, np.uint8)
    except OSError as e:
        raise FormatError(f"cannot open file for reading: {path}") from e
    off = 0

    def take(nbytes):
        nonlocal off
        if off + nbytes > blob.size:
            raise FormatError(f"unexpected end of file in {path}")
        b = blob[off:off + nbytes]
        off += nbytes
        return b

    if take(4).tobytes() != MAGIC:
        raise FormatError(f"not a forest file: {path}")
    ver, n, dim, n_trees, leaf_cap = take(20).view("<u4").tolist()
    if ver != VERSION:
        raise FormatError(f"unsupported forest version in {path}")
    seed = int(take(8).view("<u8")[0])
    if n < 1 or dim < 1 or n_trees < 1 or leaf_cap < 1:
        raise FormatError(f"forest file: degenerate header in {path}")
    trees = []
    for _ in range(n_trees):
        count, root = take(8).view("<u4").tolist()
        if count == 0 or count > 2 * n:
            raise FormatError(f"forest file: implausible node count in {path}")
        rec = take(count * _NODE.itemsize).view(_NODE)
        pi = take(4 * n).view("<u4").astype(np.uint32)
        tr = api.KdTree(rec["split_dim"].astype(np.uint32), rec["split_val"].astype(np.float32),
                        rec["left"].astype(np.uint32), rec["right"].astype(np.uint32),
                        rec["depth"].astype(np.uint32), (rec["even"] != 0).astype(np.uint8), pi, int(root),
                        int((rec["split_dim"] == api.LEAF_MARKER).sum()))
        validate_tree(tr, n, dim, leaf_cap)
        trees.append(tr)
    if off != blob.size:
        raise FormatError(f"forest file: trailing bytes in {path}")
    return n, dim, leaf_cap, seed, trees


def load_forest(path: str) -> api.KdForest:
    """kd_forest.cpp:332-372 load_forest -> device forest."""
    n, dim, leaf_cap, seed, trees = parse_forest(path)
    return api.KdForest.from_trees(n, dim, leaf_cap, seed, trees)
