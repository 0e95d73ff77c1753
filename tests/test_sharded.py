"""Sharded (multi-GPU) build protocol, SURVEY §8(e).

CPU: the driver in paper_1609_07228_b200/sharded.py runs over the C oracle's
shard primitives, as virtual ranks (threads) and as a world_size-2 gloo job;
the owned pools, concatenated in rank order, must equal the single-process
oracle's pools bit for bit, and the all-reduced dist_comps and `changes` its
counts (the reference's sequential accepted-insert count).
GPU: the same driver over device shards (virtual ranks on one GPU, and two
processes sharing one GPU over gloo).
"""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch

from paper_1609_07228_b200 import sharded as SH
from tests.helpers import ora
from tests.shard_engines import OracleShard

N, DIM, TREES, LEAF, K, DEP, P, S, SEED, ITERS = 1500, 12, 3, 8, 10, 2, 20, 8, 5, 3


def _data(o):
    return o.gen_synthetic(N, DIM, SEED)


def _single(o, x):
    vs = o.vs(x)
    f = o.build_forest(vs, TREES, LEAF, SEED)
    st = o.init_graph(vs, f, K, DEP, P, S, SEED)
    comps = [st.export()["dist_comps"]]
    changes = []
    for _ in range(ITERS):
        changes.append(st.nn_descent_iteration(vs))
        comps.append(st.export()["dist_comps"])
    return st.export(), [b - a for a, b in zip(comps, comps[1:])] + changes


def _oracle_rank(o, x, comm, limit=None):
    vs = o.vs(x)
    f = o.build_forest(vs, TREES, LEAF, SEED)
    st = o.init_graph(vs, f, K, DEP, P, S, SEED)
    lo, hi = SH.shard_ranges(N, comm.size)[comm.rank]
    e = OracleShard(o, vs, st, N, P, S, lo, hi)
    if limit:
        e.limit = limit
    comps, changes = [], []
    for _ in range(ITERS):
        ch, c = SH.nn_descent_round(e, comm)
        comps.append(c)
        changes.append(ch)
    return e.pools(), comps + changes


def _check(parts, ref, ref_comps):
    sizes = np.concatenate([p[0][0] for p in parts])
    ids = np.concatenate([p[0][1] for p in parts])
    dists = np.concatenate([p[0][2] for p in parts])
    flags = np.concatenate([p[0][3] for p in parts])
    np.testing.assert_array_equal(sizes, ref["sizes"])
    for i in range(N):
        m = int(sizes[i])
        np.testing.assert_array_equal(ids[i, :m], ref["ids"][i, :m], err_msg=f"ids row {i}")
        np.testing.assert_array_equal(dists[i, :m].view(np.uint32), ref["dists"][i, :m].view(np.uint32))
        np.testing.assert_array_equal(flags[i, :m] & 1, ref["flags"][i, :m] & 1, err_msg=f"flags row {i}")
    for p in parts:
        assert p[1] == ref_comps


def test_shard_ranges_cover_and_balance():
    for n, g in [(10, 3), (7, 7), (1000, 8), (5, 1)]:
        r = SH.shard_ranges(n, g)
        assert r[0][0] == 0 and r[-1][1] == n
        assert all(a[1] == b[0] for a, b in zip(r, r[1:]))
        sz = [hi - lo for lo, hi in r]
        assert max(sz) - min(sz) <= 1


@pytest.mark.parametrize("size", [2, 3])
def test_thread_ranks_match_single_process(size):
    o = ora()
    x = _data(o)
    ref, ref_comps = _single(o, x)
    parts = SH.run_threads(size, lambda comm: _oracle_rank(o, x, comm))
    _check(parts, ref, ref_comps)


def test_thread_ranks_piecewise_rounds_match_single_process():
    # a join limit below a rank's offer volume: every round runs in global
    # source ranges, exchanged and replayed one after another
    o = ora()
    x = _data(o)
    ref, ref_comps = _single(o, x)
    parts = SH.run_threads(2, lambda comm: _oracle_rank(o, x, comm, limit=3000))
    _check(parts, ref, ref_comps)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gloo_worker(rank, world, port, outdir):
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        o = ora()
        pools, comps = _oracle_rank(o, _data(o), SH.TorchComm("cpu"))
        np.savez(os.path.join(outdir, f"rank{rank}.npz"), sizes=pools[0], ids=pools[1], dists=pools[2],
                 flags=pools[3], comps=np.array(comps, np.int64))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_matches_single_process():
    o = ora()
    ref, ref_comps = _single(o, _data(o))
    with tempfile.TemporaryDirectory() as d:
        torch.multiprocessing.spawn(_gloo_worker, args=(2, _free_port(), d), nprocs=2, join=True)
        parts = []
        for r in range(2):
            z = np.load(os.path.join(d, f"rank{r}.npz"))
            parts.append(((z["sizes"], z["ids"], z["dists"], z["flags"]), [int(c) for c in z["comps"]]))
    _check(parts, ref, ref_comps)


@pytest.mark.gpu
@pytest.mark.parametrize("size", [2, 3])
def test_device_shards_match_oracle(size):
    import paper_1609_07228_b200 as A
    o = ora()
    x = _data(o)
    ref, ref_comps = _single(o, x)
    vs = A.VectorSet(x)
    f = A.build_forest(vs, TREES, LEAF, SEED)

    def rank(comm):
        lo, hi = SH.shard_ranges(N, comm.size)[comm.rank]
        e = SH.DeviceShard(vs, f, K, DEP, P, S, SEED, lo, hi)
        comps, changes = [], []
        for _ in range(ITERS):
            ch, c = SH.nn_descent_round(e, comm)
            comps.append(c)
            changes.append(ch)
        return e.pools(), comps + changes, e.finalize()

    parts = SH.run_threads(size, rank)
    _check([(p[0], p[1]) for p in parts], ref, ref_comps)
    # finalize rows of the shards == single-state finalize
    st = A.init_graph(vs, f, K, DEP, P, S, SEED)
    for _ in range(ITERS):
        A.detail.nn_descent_iteration(st, vs)
    g = A.finalize(st, vs, K)
    np.testing.assert_array_equal(np.concatenate([p[2].ids for p in parts]), g.ids)
    np.testing.assert_array_equal(np.concatenate([p[2].dists for p in parts]).view(np.uint32),
                                  g.dists.view(np.uint32))


@pytest.mark.gpu
def test_device_shard_integer_mixture_u8_path():
    import paper_1609_07228_b200 as A
    from tests.helpers import mixture
    o = ora()
    x = mixture(4000, 128, 20, 9)
    vs_o = o.vs(x)
    fo = o.build_forest(vs_o, 4, 8, 3)
    so = o.init_graph(vs_o, fo, 10, 4, 30, 10, 3)
    for _ in range(2):
        so.nn_descent_iteration(vs_o)
    ref = so.export()
    vs = A.VectorSet(x)
    f = A.build_forest(vs, 4, 8, 3)

    def rank(comm):
        lo, hi = SH.shard_ranges(4000, comm.size)[comm.rank]
        e = SH.DeviceShard(vs, f, 10, 4, 30, 10, 3, lo, hi)
        for _ in range(2):
            SH.nn_descent_round(e, comm)
        return e.pools()

    parts = SH.run_threads(2, rank)
    sizes = np.concatenate([p[0] for p in parts])
    ids = np.concatenate([p[1] for p in parts])
    np.testing.assert_array_equal(sizes, ref["sizes"])
    for i in range(4000):
        m = int(sizes[i])
        np.testing.assert_array_equal(ids[i, :m], ref["ids"][i, :m])


def _nccl_worker(rank, world, port, outdir):
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        import paper_1609_07228_b200 as A
        o = ora()
        x = _data(o)
        vs = A.VectorSet(x)
        f = A.build_forest(vs, TREES, LEAF, SEED)
        lo, hi = SH.shard_ranges(N, world)[rank]
        e = SH.DeviceShard(vs, f, K, DEP, P, S, SEED, lo, hi, buffer_device="cuda")
        comm = SH.TorchComm("cuda")
        rounds = [SH.nn_descent_round(e, comm) for _ in range(ITERS)]
        comps = [r[1] for r in rounds] + [r[0] for r in rounds]
        pools = e.pools()
        np.savez(os.path.join(outdir, f"rank{rank}.npz"), sizes=pools[0], ids=pools[1], dists=pools[2],
                 flags=pools[3], comps=np.array(comps, np.int64))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_nccl_single_rank_device_buffers():
    # the multi-GPU bench path (NCCL collectives on CUDA tensors) with one rank
    o = ora()
    ref, ref_comps = _single(o, _data(o))
    with tempfile.TemporaryDirectory() as d:
        torch.multiprocessing.spawn(_nccl_worker, args=(1, _free_port(), d), nprocs=1, join=True)
        z = np.load(os.path.join(d, "rank0.npz"))
        parts = [((z["sizes"], z["ids"], z["dists"], z["flags"]), [int(c) for c in z["comps"]])]
    _check(parts, ref, ref_comps)


def _gloo_device_worker(rank, world, port, outdir, limit):
    import torch.distributed as dist
    if limit:
        os.environ["ANNK_JOIN_MAX_OFFERS"] = str(limit)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        import paper_1609_07228_b200 as A
        o = ora()
        x = _data(o)
        vs = A.VectorSet(x)
        f = A.build_forest(vs, TREES, LEAF, SEED)
        lo, hi = SH.shard_ranges(N, world)[rank]
        e = SH.DeviceShard(vs, f, K, DEP, P, S, SEED, lo, hi)
        comm = SH.TorchComm("cpu")
        rounds = [SH.nn_descent_round(e, comm) for _ in range(ITERS)]
        pools = e.pools()
        np.savez(os.path.join(outdir, f"rank{rank}.npz"), sizes=pools[0], ids=pools[1], dists=pools[2],
                 flags=pools[3], comps=np.array([r[1] for r in rounds] + [r[0] for r in rounds], np.int64))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("limit", [0, 3000])
def test_gloo_world2_device_shards_two_processes(limit):
    # two processes (one DeviceShard each) on one GPU over gloo; limit > 0
    # forces every round through the piecewise path
    o = ora()
    ref, ref_comps = _single(o, _data(o))
    with tempfile.TemporaryDirectory() as d:
        torch.multiprocessing.spawn(_gloo_device_worker, args=(2, _free_port(), d, limit), nprocs=2, join=True)
        parts = []
        for r in range(2):
            z = np.load(os.path.join(d, f"rank{r}.npz"))
            parts.append(((z["sizes"], z["ids"], z["dists"], z["flags"]), [int(c) for c in z["comps"]]))
    _check(parts, ref, ref_comps)
