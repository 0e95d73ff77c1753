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
        self.local = None
        self.recv = []
        self.piece_changes = 0
        self.join_pieces = 1
        self.limit = 1 << 62  # offers one join may hold (tests lower it to force pieces)

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

    def join_range(self, ilo, ihi):
        """Join of the owned sources in [ilo, ihi): (comps, offers, ok)."""
        lo, hi = max(self.lo, ilo), min(self.hi, ihi)
        if hi <= lo:
            c, tgt, key, src = 0, np.empty(0, np.uint32), np.empty(0, np.uint64), np.empty(0, np.uint32)
        else:
            c, tgt, key, src = self.st.shard_join(self.vs, lo, hi, self.rows[ANNK_ROWS_THR].reshape(-1))
        if tgt.size >= self.limit:  # refused, as the device join refuses an oversized launch
            return 0, int(tgt.size), False
        self.comps += c
        self.local = (tgt, key, src)
        self.recv = []
        return c, int(tgt.size), True

    def join(self) -> int:
        c, _, ok = self.join_range(0, self.n)
        assert ok
        return c

    def pack(self, lo, hi):
        tgt, key, src = self.local
        sel = (tgt >= lo) & (tgt < hi)
        tgt, key, src = tgt[sel], key[sel], src[sel]
        order = np.argsort(tgt, kind="stable")
        counts = np.bincount(tgt - lo, minlength=hi - lo).astype(np.uint32)
        return (torch.from_numpy(counts.view(np.int32).copy()),
                torch.from_numpy(key[order].view(np.int64).copy()),
                torch.from_numpy(src[order].view(np.int32).copy()))

    def add(self, counts, keys, srcs):
        c = counts.numpy().view(np.uint32).astype(np.int64)
        tgt = np.repeat(np.arange(self.lo, self.hi, dtype=np.uint32), c)
        self.recv.append((tgt, keys.numpy().view(np.uint64), srcs.numpy().view(np.uint32)))

    def _replay(self) -> int:
        tgt, key, src = self.local
        sel = (tgt >= self.lo) & (tgt < self.hi)
        parts = [(tgt[sel], key[sel], src[sel])] + self.recv
        return self.st.shard_replay(*(np.concatenate([p[j] for p in parts]) for j in range(3)))

    def merge(self) -> int:
        ch = self._replay()
        self.st.shard_finish(ch)
        return ch

    def merge_piece(self) -> int:
        ch = self._replay()
        self.piece_changes += ch
        return ch

    def finish_round(self) -> int:
        ch, self.piece_changes = self.piece_changes, 0
        self.st.shard_finish(ch)
        return ch

    def dist_comps(self) -> int:
        return self.comps

    def pools(self):
        p = self.st.export()
        return tuple(p[k][self.lo:self.hi] for k in ("sizes", "ids", "dists", "flags"))
