"""CPU engine for the sharded-build protocol (paper_1609_07228_b200/sharded.py),
over the C oracle's shard primitives — TEST INFRASTRUCTURE: lets the gloo /
thread tests drive the exact driver code the GPUs run, without a GPU."""
from __future__ import annotations

import numpy as np
import torch

from paper_1609_07228_b200._lib import (ANNK_ROWS_CNEW, ANNK_ROWS_COLD, ANNK_ROWS_FNEW, ANNK_ROWS_FOLD,
                                        ANNK_ROWS_THR)


class OracleShard:
    """Same interface as sharded.DeviceShard; `state` is a full oracle
    RefineState of which only the rows [lo, hi) are maintained."""

    def __init__(self, lib, vs, state, n, P, S, lo, hi):
        self.lib, self.vs, self.st = lib, vs, state
        self.n, self.P, self.S, self.lo, self.hi = n, P, S, lo, hi
        self.rows = {
            ANNK_ROWS_FNEW: np.zeros((n, S), np.uint32),
            ANNK_ROWS_CNEW: np.zeros((n, 1), np.uint32),
            ANNK_ROWS_FOLD: np.zeros((n, P), np.uint32),
            ANNK_ROWS_COLD: np.zeros((n, 1), np.uint32),
            ANNK_ROWS_THR: np.zeros((n, 1), np.uint64),
        }
        self.comps = 0
        self.local_tgt = self.local_key = None
        self.recv = []

    def sample(self):
        r = self.rows
        self.st.shard_sample(self.lo, self.hi, r[ANNK_ROWS_FNEW], r[ANNK_ROWS_CNEW], r[ANNK_ROWS_FOLD],
                             r[ANNK_ROWS_COLD], r[ANNK_ROWS_THR])

    def get_rows(self, kind):
        a = self.rows[kind][self.lo:self.hi]
        dt = np.int64 if kind == ANNK_ROWS_THR else np.int32
        return torch.from_numpy(np.ascontiguousarray(a).view(dt).copy())

    def put_rows(self, kind, lo, hi, t):
        dst = self.rows[kind]
        dst[lo:hi] = t.numpy().view(dst.dtype).reshape(hi - lo, dst.shape[1])

    def union(self):
        r = self.rows
        self.st.shard_union(r[ANNK_ROWS_FNEW], r[ANNK_ROWS_CNEW], r[ANNK_ROWS_FOLD], r[ANNK_ROWS_COLD])

    def join(self) -> int:
        c, tgt, key = self.st.shard_join(self.vs, self.lo, self.hi, self.rows[ANNK_ROWS_THR].reshape(-1))
        self.comps += c
        self.local_tgt, self.local_key = tgt, key
        self.recv = []
        return c

    def pack(self, lo, hi):
        sel = (self.local_tgt >= lo) & (self.local_tgt < hi)
        tgt, key = self.local_tgt[sel], self.local_key[sel]
        order = np.argsort(tgt, kind="stable")
        counts = np.bincount(tgt - lo, minlength=hi - lo).astype(np.uint32)
        return (torch.from_numpy(counts.view(np.int32).copy()),
                torch.from_numpy(key[order].view(np.int64).copy()))

    def add(self, counts, keys):
        c = counts.numpy().view(np.uint32).astype(np.int64)
        tgt = np.repeat(np.arange(self.lo, self.hi, dtype=np.uint32), c)
        self.recv.append((tgt, keys.numpy().view(np.uint64)))

    def merge(self) -> int:
        sel = (self.local_tgt >= self.lo) & (self.local_tgt < self.hi)
        tgts = [self.local_tgt[sel]] + [t for t, _ in self.recv]
        keys = [self.local_key[sel]] + [k for _, k in self.recv]
        return self.st.shard_merge(self.lo, self.hi, np.concatenate(tgts), np.concatenate(keys))

    def dist_comps(self) -> int:
        return self.comps

    def pools(self):
        p = self.st.export()
        return tuple(p[k][self.lo:self.hi] for k in ("sizes", "ids", "dists", "flags"))
