"""Multi-GPU host logic: one process per GPU (torch.distributed for the plumbing).

The partitioned solve (csrc/shard.cu + csrc/gmres.cu): the target leaves and
the source leaves are split into contiguous, work-balanced ranges (``partition_contiguous``);
each rank does the P2M of its source leaves, all-gathers the leaf multipoles, and runs M2L /
P2P / the epilogue for its own target leaves.  GMRES keeps only each rank's rows of the
Krylov vectors: v_k is all-gathered before every apply and the Gram-Schmidt dot products are
all-reduced (CGS2).  The collectives go over NCCL (``shard_operator(..., transport="nccl")``,
one GPU per rank, captured in the per-order CUDA graphs) or over a host transport
(``transport="gloo"``: torch.distributed on CPU tensors behind the C callbacks; used to run
two ranks on one GPU in the tests).  Multi-GPU timings: unmeasured on hardware (no multi-GPU
node in this build's runs).
"""

from __future__ import annotations

import numpy as np


def partition_contiguous(weights, world: int) -> np.ndarray:
    """Split items 0..n-1 (kept in order) into `world` contiguous ranges of ~equal weight.

    Returns boundaries b (world+1,) with rank r owning [b[r], b[r+1]).  Every
    rank computes the same split from the same weights (deterministic).
    """
    w = np.asarray(weights, dtype=np.float64)
    if world < 1:
        raise ValueError("world must be >= 1")
    n = len(w)
    c = np.concatenate([[0.0], np.cumsum(w)])
    total = c[-1]
    b = np.zeros(world + 1, dtype=np.int64)
    b[world] = n
    for r in range(1, world):
        target = total * r / world
        k = int(np.searchsorted(c, target, side="left"))
        k = min(max(k, b[r - 1]), n)
        # pick the closer of k-1 / k
        if k > b[r - 1] and abs(c[k - 1] - target) <= abs(c[k] - target):
            k -= 1
        b[r] = k
    return b


def leaf_bounds(op, world: int):
    """(target, source) leaf bounds for `world` ranks from the operator's work weights."""
    return (partition_contiguous(op.leaf_work("tgt"), world),
            partition_contiguous(op.leaf_work("src"), world))


def nccl_unique_id() -> bytes:
    import ctypes

    from . import _native as N

    buf = ctypes.create_string_buffer(128)
    N.check(N.load().fmmbem_nccl_unique_id(buf))
    return buf.raw


def broadcast_bytes(data: bytes | None, src: int = 0) -> bytes:
    """Share a small byte string from rank `src` (torch.distributed object broadcast)."""
    import torch.distributed as dist

    obj = [data]
    dist.broadcast_object_list(obj, src=src)
    return obj[0]


def gloo_collectives(world: int):
    """(allgather, allreduce) on host float64 arrays over the current torch.distributed group."""
    import torch
    import torch.distributed as dist

    def allgather(send):
        t = torch.from_numpy(send)
        out = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(out, t)
        return torch.cat(out).numpy()

    def allreduce(buf):
        t = torch.from_numpy(buf)
        dist.all_reduce(t)
        return t.numpy()

    return allgather, allreduce


def shard_operator(op, rank: int, world: int, transport: str = "nccl"):
    """Partition op's work over the torch.distributed world.

    Every rank computes the same bounds.  transport "nccl": one GPU per rank, rank 0 creates
    the NCCL id and shares it; "gloo": the collectives run on host buffers through
    torch.distributed (any backend), e.g. several ranks sharing one GPU.
    """
    tb, sb = leaf_bounds(op, world)
    if transport == "nccl":
        uid = broadcast_bytes(nccl_unique_id() if rank == 0 else None)
        op.shard(rank, world, tb, sb, uid)
    elif transport == "gloo":
        op.shard_host(rank, world, tb, sb, *gloo_collectives(world))
    else:
        raise ValueError(f"unknown transport {transport!r}")
    return tb, sb


def reduce_timing(local_ms: float, local_count: float, device=None):
    """(max over ranks of the device time, sum over ranks of the work units).

    Uses torch.distributed when it is initialised (nccl on GPUs, gloo in the
    CPU tests); identity for a single process.
    """
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        return float(local_ms), float(local_count)
    dev = device if device is not None else "cpu"
    t = torch.tensor([float(local_ms)], dtype=torch.float64, device=dev)
    n = torch.tensor([float(local_count)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.all_reduce(n, op=dist.ReduceOp.SUM)
    return float(t.item()), float(n.item())
