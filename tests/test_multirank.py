"""CPU, world_size 2 over gloo: the N>1 host logic (replica timing reduction as
bench.py uses it, and the deterministic contiguous partitioner)."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1506_05957_b200.parallel import partition_contiguous, reduce_timing


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ms, n = reduce_timing(10.0 + 5.0 * rank, 4 + rank)
        w = np.random.default_rng(0).uniform(0.5, 2.0, 101)
        b = partition_contiguous(w, world)
        out.put((rank, ms, n, b.tolist()))
    finally:
        dist.destroy_process_group()


def test_two_rank_reduction_and_partition():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    assert all(r[1] == 15.0 for r in res)          # max over ranks
    assert all(r[2] == 9.0 for r in res)           # sum over ranks
    assert res[0][3] == res[1][3]                  # identical split on every rank


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_partition_covers_in_order(world):
    w = np.random.default_rng(world).uniform(0.1, 3.0, 257)
    b = partition_contiguous(w, world)
    assert b[0] == 0 and b[-1] == len(w)
    assert np.all(np.diff(b) >= 0)
    loads = [w[b[r]:b[r + 1]].sum() for r in range(world)]
    assert max(loads) <= w.sum() / world + w.max() + 1e-12


def test_single_process_reduction_is_identity():
    assert reduce_timing(3.0, 2) == (3.0, 2.0)


def _bytes_worker(rank, world, port, out):
    import torch.distributed as dist

    from paper_1506_05957_b200.parallel import broadcast_bytes

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        got = broadcast_bytes(bytes(range(128)) if rank == 0 else None)
        out.put((rank, got))
    finally:
        dist.destroy_process_group()


def test_two_rank_nccl_id_broadcast():
    """The shard setup shares rank 0's 128-byte NCCL id with every rank."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bytes_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(r[1] == bytes(range(128)) for r in res)


def _gloo_collectives_worker(rank, world, port, out):
    import torch.distributed as dist

    from paper_1506_05957_b200.parallel import gloo_collectives

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ag, ar = gloo_collectives(world)
        send = np.arange(5, dtype=np.float64) + 10.0 * rank
        out.put((rank, ag(send.copy()).tolist(), ar(send.copy()).tolist()))
    finally:
        dist.destroy_process_group()


def test_host_transport_collectives_over_gloo():
    """The (allgather, allreduce) pair the host transport of a sharded operator calls
    (parallel.gloo_collectives -> fmmbem_op_shard_host): rank-ordered gather, in-place sum."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_collectives_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want_g = list(np.arange(5.0)) + list(np.arange(5.0) + 10.0)
    want_r = list(2 * np.arange(5.0) + 10.0)
    for _, g, r in res:
        assert g == want_g and r == want_r
