"""Multi-GPU graph build: one process per GPU, pools sharded by point.

Rank r owns the points ``shard_ranges(n, G)[r]``.  Every rank holds the whole
dataset and the whole forest (the forest build is one CTA per tree and
latency-bound per tree, so splitting trees across GPUs would not shorten it).
One NN-descent round (graph_build.cpp:59-162) runs as:

1. ``sample``   forward lists + start-of-round tails of the owned points
2. all-gather   those rows (``annk_state_rows``: FNEW, CNEW, FOLD, COLD, THR)
3. ``union``    reverse lists from all forward rows, ``sample_down``, union
                (same RNG streams on every rank, so every rank agrees)
4. ``join``     local join of the owned points; offers may target any point
                and carry their source point
5. all-to-all   offers routed to the rank owning their target
6. ``merge``    the owned pools replay their offers in the reference's order
                (source point ascending, then the source's pair order)
7. all-reduce   dist_comps and changes

Because the join only reads the snapshot lists and the merge replays the
reference's insert order, pools, flags and ``changes`` equal the single-GPU
build and the reference's single-worker build exactly.  A round too large for
one join launch is joined in global source ranges, ascending, each exchanged
and replayed before the next.

The protocol is written once against two small interfaces:

* an *engine* (``DeviceShard`` here; the CPU oracle engine used by the gloo
  tests lives in ``tests/``), and
* a *comm* (``TorchComm`` over ``torch.distributed`` — NCCL on GPUs, gloo on
  CPU — or ``ThreadComm`` for several virtual ranks in one process).
"""
from __future__ import annotations

import math
import os
import threading
from dataclasses import dataclass
from typing import Callable, List, Optional, Sequence

import numpy as np

from . import api
from ._lib import (ANNK_ROWS_CNEW, ANNK_ROWS_COLD, ANNK_ROWS_FNEW, ANNK_ROWS_FOLD, ANNK_ROWS_THR, C, check,
                   lib)

ROW_KINDS = (ANNK_ROWS_FNEW, ANNK_ROWS_CNEW, ANNK_ROWS_FOLD, ANNK_ROWS_COLD, ANNK_ROWS_THR)


def shard_ranges(n: int, size: int) -> List[tuple]:
    """Contiguous point ranges, sizes differing by at most one."""
    if size < 1:
        raise api.InvalidArgument("shard_ranges: size must be >= 1")
    base, rem = divmod(n, size)
    out, lo = [], 0
    for r in range(size):
        hi = lo + base + (1 if r < rem else 0)
        out.append((lo, hi))
        lo = hi
    return out


def row_width(kind: int, P: int, S: int) -> int:
    return {ANNK_ROWS_FNEW: S, ANNK_ROWS_CNEW: 1, ANNK_ROWS_FOLD: P, ANNK_ROWS_COLD: 1, ANNK_ROWS_THR: 1}[kind]


def row_dtype(kind: int):
    import torch
    return torch.int64 if kind == ANNK_ROWS_THR else torch.int32


# ------------------------------------------------------------------ comms

class TorchComm:
    """Collectives over the default torch.distributed group (NCCL or gloo)."""

    def __init__(self, device: str = "cpu"):
        import torch.distributed as dist
        self.dist = dist
        self.rank = dist.get_rank()
        self.size = dist.get_world_size()
        self.device = device

    def _sync(self):
        if self.device != "cpu":
            import torch
            torch.cuda.synchronize()

    def allgather(self, x):
        """Tensors of possibly different first dimension -> list per rank."""
        import torch
        n = torch.tensor([x.shape[0]], dtype=torch.int64, device=self.device)
        ns = [torch.zeros_like(n) for _ in range(self.size)]
        self.dist.all_gather(ns, n)
        sizes = [int(v.item()) for v in ns]
        m = max(sizes)
        pad = torch.zeros((m,) + tuple(x.shape[1:]), dtype=x.dtype, device=self.device)
        pad[:x.shape[0]] = x
        outs = [torch.empty_like(pad) for _ in range(self.size)]
        self.dist.all_gather(outs, pad)
        self._sync()
        return [o[:s] for o, s in zip(outs, sizes)]

    def alltoall(self, sends: Sequence):
        """sends[r]: 1-D tensor for rank r (or None for self) -> list of received tensors."""
        import torch
        dt = next(s.dtype for s in sends if s is not None) if any(s is not None for s in sends) else torch.int64
        lens = torch.tensor([0 if s is None else s.numel() for s in sends], dtype=torch.int64, device=self.device)
        all_lens = [torch.zeros_like(lens) for _ in range(self.size)]
        self.dist.all_gather(all_lens, lens)
        recv_len = [int(all_lens[r][self.rank].item()) for r in range(self.size)]
        recvs = [None] * self.size
        ops = []
        for r in range(self.size):
            if r == self.rank:
                continue
            if sends[r] is not None and sends[r].numel():
                ops.append(self.dist.P2POp(self.dist.isend, sends[r].contiguous(), r))
            if recv_len[r]:
                recvs[r] = torch.empty(recv_len[r], dtype=dt, device=self.device)
                ops.append(self.dist.P2POp(self.dist.irecv, recvs[r], r))
            else:
                recvs[r] = torch.empty(0, dtype=dt, device=self.device)
        if ops:
            for w in self.dist.batch_isend_irecv(ops):
                w.wait()
        self._sync()
        return recvs

    def allreduce_sum(self, v: int) -> int:
        import torch
        t = torch.tensor([int(v)], dtype=torch.int64, device=self.device)
        self.dist.all_reduce(t)
        return int(t.item())

    def allreduce_sumf(self, v: float) -> float:
        import torch
        t = torch.tensor([float(v)], dtype=torch.float64, device=self.device)
        self.dist.all_reduce(t)
        return float(t.item())

    def barrier(self):
        self.dist.barrier()


class ThreadGroup:
    def __init__(self, size: int):
        self.size = size
        self.barrier = threading.Barrier(size)
        self.slots = [None] * size


class ThreadComm:
    """Several virtual ranks in one process (one thread each)."""

    def __init__(self, group: ThreadGroup, rank: int):
        self.g, self.rank, self.size, self.device = group, rank, group.size, "cpu"

    def _exchange(self, v):
        self.g.slots[self.rank] = v
        self.g.barrier.wait()
        out = list(self.g.slots)
        self.g.barrier.wait()
        return out

    def allgather(self, x):
        return [t.clone() for t in self._exchange(x)]

    def alltoall(self, sends):
        allsends = self._exchange(list(sends))
        return [None if r == self.rank else allsends[r][self.rank] for r in range(self.size)]

    def allreduce_sum(self, v: int) -> int:
        return int(sum(self._exchange(int(v))))

    def allreduce_sumf(self, v: float) -> float:
        return float(sum(self._exchange(float(v))))

    def barrier(self):
        self._exchange(None)


def run_threads(size: int, fn: Callable[[ThreadComm], object]) -> list:
    """Runs fn(comm) for `size` virtual ranks; returns their results in rank order."""
    g = ThreadGroup(size)
    res, err = [None] * size, [None] * size

    def body(r):
        try:
            res[r] = fn(ThreadComm(g, r))
        except BaseException as e:  # noqa: BLE001 - re-raised below
            err[r] = e
            g.barrier.abort()

    ts = [threading.Thread(target=body, args=(r,)) for r in range(size)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for e in err:
        if e is not None and not isinstance(e, threading.BrokenBarrierError):
            raise e
    for e in err:
        if e is not None:
            raise e
    return res


# ----------------------------------------------------------------- engine

_LIB_LOCK = threading.RLock()  # the library runs one stream: virtual ranks take turns


class DeviceShard:
    """Engine over the device library: one RefineState owning [lo, hi)."""

    def __init__(self, vs, forest, k, conquer_depth, pool_cap, sample_cap, seed, lo, hi,
                 buffer_device: str = "cpu"):
        self.vs = api._as_vs(vs)
        self.n, self.lo, self.hi = self.vs.n, lo, hi
        self.P, self.S, self.k = pool_cap, sample_cap, k
        self.buffer_device = buffer_device
        h = C.c_void_p()
        with _LIB_LOCK:
            check(lib.annk_init_graph_shard(self.vs.handle, forest.handle, k, conquer_depth, pool_cap, sample_cap,
                                            seed, lo, hi, C.byref(h)))
        self.state = api.RefineState(h)
        self.join_pieces = 1
        self.limit = int(os.environ.get("ANNK_JOIN_MAX_OFFERS", str(1 << 32)))

    def _tensor(self, shape, dtype):
        import torch
        return torch.empty(shape, dtype=dtype, device=self.buffer_device)

    def sample(self):
        with _LIB_LOCK:
            check(lib.annk_shard_sample(self.state.handle))

    def get_rows(self, kind):
        t = self._tensor((self.hi - self.lo, row_width(kind, self.P, self.S)), row_dtype(kind))
        with _LIB_LOCK:
            check(lib.annk_state_rows(self.state.handle, kind, 0, self.lo, self.hi, C.c_void_p(t.data_ptr())))
        return t

    def put_rows(self, kind, lo, hi, t):
        t = t.contiguous()
        with _LIB_LOCK:
            check(lib.annk_state_rows(self.state.handle, kind, 1, lo, hi, C.c_void_p(t.data_ptr())))

    def union(self):
        with _LIB_LOCK:
            check(lib.annk_shard_union(self.state.handle))

    def join_range(self, ilo, ihi):
        """Join of the owned sources in [ilo, ihi): (comps, offers, ok); ok is
        False when the range's offers exceed one join launch."""
        c, o, ok = C.c_uint64(0), C.c_uint64(0), C.c_uint32(0)
        with _LIB_LOCK:
            check(lib.annk_shard_join_range(self.state.handle, self.vs.handle, ilo, ihi, C.byref(c), C.byref(o),
                                            C.byref(ok)))
        return c.value, o.value, bool(ok.value)

    def join(self) -> int:
        c = C.c_uint64(0)
        with _LIB_LOCK:
            check(lib.annk_shard_join(self.state.handle, self.vs.handle, C.byref(c)))
        return c.value

    def pack(self, lo, hi):
        import torch
        tot = C.c_uint64(0)
        with _LIB_LOCK:
            check(lib.annk_shard_offers_count(self.state.handle, lo, hi, C.byref(tot)))
            counts = self._tensor(hi - lo, torch.int32)
            keys = self._tensor(tot.value, torch.int64)
            srcs = self._tensor(tot.value, torch.int32)
            check(lib.annk_shard_offers_pack(self.state.handle, lo, hi, C.c_void_p(counts.data_ptr()),
                                             C.c_void_p(keys.data_ptr()), C.c_void_p(srcs.data_ptr())))
        return counts, keys, srcs

    def add(self, counts, keys, srcs):
        counts, keys, srcs = counts.contiguous(), keys.contiguous(), srcs.contiguous()
        with _LIB_LOCK:
            check(lib.annk_shard_offers_add(self.state.handle, self.lo, self.hi, C.c_void_p(counts.data_ptr()),
                                            C.c_void_p(keys.data_ptr()) if keys.numel() else None,
                                            C.c_void_p(srcs.data_ptr()) if srcs.numel() else None))

    def merge(self) -> int:
        c = C.c_uint64(0)
        with _LIB_LOCK:
            check(lib.annk_shard_merge(self.state.handle, C.byref(c)))
        return c.value

    def merge_piece(self) -> int:
        c = C.c_uint64(0)
        with _LIB_LOCK:
            check(lib.annk_shard_merge_piece(self.state.handle, C.byref(c)))
        return c.value

    def finish_round(self) -> int:
        c = C.c_uint64(0)
        with _LIB_LOCK:
            check(lib.annk_shard_finish_round(self.state.handle, C.byref(c)))
        return c.value

    def dist_comps(self) -> int:
        return self.state.meta()["dist_comps"]

    def finalize(self, k=None) -> api.KnnGraph:
        """Rows [lo, hi) of the final graph."""
        k = self.k if k is None else k
        m = self.hi - self.lo
        ids = np.empty((m, k), np.uint32)
        d = np.empty((m, k), np.float32)
        with _LIB_LOCK:
            check(lib.annk_finalize(self.state.handle, self.vs.handle, k, ids, d))
        return api.KnnGraph(ids, d)

    def pools(self):
        """(sizes, ids, dists, flags) of the owned rows."""
        with _LIB_LOCK:
            p = self.state.pools()
        return tuple(v[self.lo:self.hi] for v in p)

    def accuracy_sum(self, gt_rows: np.ndarray, rows: np.ndarray) -> tuple:
        """graph_build.cpp:209-226 over the owned sample rows: (sum of per-row
        scores, row count); the driver all-reduces both."""
        sel = (rows >= self.lo) & (rows < self.hi)
        m = int(sel.sum())
        if m == 0:
            return 0.0, 0
        with _LIB_LOCK:
            acc = api.detail.pool_topk_accuracy(self.state, gt_rows[sel], rows[sel])
        return acc * m, m


def sharded_accuracy(e, comm, gt_rows, rows) -> float:
    s, m = e.accuracy_sum(gt_rows, rows)
    return comm.allreduce_sumf(s) / max(comm.allreduce_sum(m), 1)


def allgather_graph(g: api.KnnGraph, comm) -> api.KnnGraph:
    """Full graph on every rank from the ranks' finalized rows."""
    import torch
    ids = torch.from_numpy(g.ids.view(np.int32)).to(comm.device)
    d = torch.from_numpy(g.dists).to(comm.device)
    all_ids = comm.allgather(ids)
    all_d = comm.allgather(d)
    return api.KnnGraph(np.ascontiguousarray(torch.cat(all_ids).cpu().numpy().view(np.uint32)),
                        np.ascontiguousarray(torch.cat(all_d).cpu().numpy()))


# --------------------------------------------------------------- protocol

def _exchange(e, comm, ranges, me):
    """all-to-all of the offers by target owner (keys and their source points)."""
    packs = [None if r == me else e.pack(*ranges[r]) for r in range(comm.size)]
    counts = comm.alltoall([None if p is None else p[0] for p in packs])
    keys = comm.alltoall([None if p is None else p[1] for p in packs])
    srcs = comm.alltoall([None if p is None else p[2] for p in packs])
    for r in range(comm.size):
        if r != me:
            e.add(counts[r], keys[r], srcs[r])


def nn_descent_round(e, comm) -> tuple:
    """One sharded NN-descent round; returns (global changes, global new comps)."""
    ranges = shard_ranges(e.n, comm.size)
    me = comm.rank
    e.sample()
    for kind in ROW_KINDS:
        parts = comm.allgather(e.get_rows(kind))
        for r, part in enumerate(parts):
            if r != me:
                e.put_rows(kind, ranges[r][0], ranges[r][1], part)
    e.union()
    pieces = e.join_pieces
    if pieces <= 1:
        comps, offers, ok = e.join_range(0, e.n)
        if comm.allreduce_sum(0 if ok else 1) == 0:
            _exchange(e, comm, ranges, me)
            changes = e.merge()
            return comm.allreduce_sum(changes), comm.allreduce_sum(comps)
        # some rank's offers do not fit one launch: the round runs in global source ranges
        pieces = max(2, math.ceil(2 * comm.allreduce_sum(offers) / (comm.size * e.limit)) + 1)
    # pieces in ascending source order, each replayed before the next: the
    # reference's order (graph_build.cpp:129 walks the points ascending)
    comps_total, max_piece, pos = 0, 0, 0
    while pos < e.n:
        end = min(e.n, pos + max(1, -(-e.n // pieces)))
        comps, offers, ok = e.join_range(pos, end)
        if comm.allreduce_sum(0 if ok else 1):
            pieces *= 2
            continue
        _exchange(e, comm, ranges, me)
        e.merge_piece()
        comps_total += comps
        max_piece = max(max_piece, offers)
        pos = end
    changes = e.finish_round()
    e.join_pieces = 1 if 2 * max_piece * pieces < e.limit else pieces
    return comm.allreduce_sum(changes), comm.allreduce_sum(comps_total)


@dataclass
class ShardedLog:
    iteration: int
    changes: int
    dist_comps: int  # cumulative, all ranks


def refine_sharded(e, comm, max_iters: int, min_change_rate: float = 0.001,
                   init_comps: Optional[int] = None,
                   on_iteration: Optional[Callable[[int], bool]] = None) -> List[ShardedLog]:
    """graph_build.cpp:328-335 over shards.  on_iteration(it) -> True stops early."""
    total = comm.allreduce_sum(e.dist_comps() if init_comps is None else init_comps)
    thr = min_change_rate * e.n * e.P
    logs = []
    for it in range(max_iters):
        ch, comps = nn_descent_round(e, comm)
        total += comps
        logs.append(ShardedLog(it + 1, ch, total))
        if on_iteration is not None and on_iteration(it + 1):
            break
        if ch < thr:
            break
    return logs
