"""Two ranks of the partitioned solve as two processes sharing the one GPU.

The collectives go through the host transport (torch.distributed / gloo behind the C
callbacks): every rank's kernels run on its own, the processes meet only on the host inside
each all-gather / all-reduce, so no kernel waits on another process's kernel.  This runs the
real pack -> exchange -> unpack path of the leaf multipoles, the y slices and the partitioned
Krylov vectors (all-gather of v_k, all-reduced CGS2 dot products), which a single process
cannot.  Bars: the sharded mat-vec equals the unpartitioned one to roundoff (its upward pass
is P2M + M2M instead of the direct basis pass: <= 1e-13); the partitioned GMRES (CGS2 on row
slices) takes the same orders and iterations and its solution agrees to <= 1e-10.
"""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rank_main(rank, world, port, name, out):
    import sys

    import torch
    import torch.distributed as dist

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1506_05957_b200.configs import CONFIGS
        from paper_1506_05957_b200.operator import GpuBemOperator
        from paper_1506_05957_b200.parallel import shard_operator
        from paper_1506_05957_b200.solver import solve

        torch.cuda.set_device(0)
        cfg = CONFIGS[name]
        op = GpuBemOperator(cfg.mesh(), cfg.formulation, theta=cfg.theta, n_crit=cfg.n_crit, mu=cfg.mu)
        x = np.random.default_rng(1).uniform(-1.0, 1.0, op.shape[0])
        b = op.assemble_rhs(cfg.boundary_data(op.centroids, op.normals))
        y_ref = op.apply(x, cfg.p_initial)
        ref = solve(op, b, eta=cfg.tol, p_initial=cfg.p_initial, p_min=cfg.p_min)
        tb, sb = shard_operator(op, rank, world, transport="gloo")
        y = op.apply(x, cfg.p_initial)
        res = solve(op, b, eta=cfg.tol, p_initial=cfg.p_initial, p_min=cfg.p_min)
        op.unshard()
        out.put((rank, np.linalg.norm(y - y_ref) / np.linalg.norm(y_ref), res.orders, ref.orders,
                 float(np.linalg.norm(res.x - ref.x) / np.linalg.norm(ref.x)), res.x,
                 [int(v) for v in tb]))
    except Exception as exc:  # surfaced by the parent
        out.put((rank, repr(exc)))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["cfg1", "stokes_ico3"])
def test_two_ranks_over_the_host_transport(name):
    import torch.multiprocessing as mp

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, name, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
    res.sort(key=lambda r: r[0])
    for r in res:
        assert len(r) > 2, r[1]
    for rank, apply_err, orders, ref_orders, x_err, _, tb in res:
        assert tb[0] == 0 < tb[1] < tb[2]          # both ranks own target leaves
        assert apply_err <= 1e-13, (rank, apply_err)
        assert orders == ref_orders, (rank, orders, ref_orders)
        assert x_err <= 1e-10, (rank, x_err)
    assert np.array_equal(res[0][5], res[1][5])   # every rank returns the same whole solution
    for p in procs:
        assert p.exitcode == 0
