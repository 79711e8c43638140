"""GPU: the row-partitioned solve (paper_1907_04417_b200.distributed) with the
device kernels.  World size 1 in-process (bit-identical to the single-GPU
operator), and world size 2 as two processes on the one GPU with gloo staging
(ranks wait on each other only on the host, never inside a kernel)."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from _fixtures import golden, hierarchy
from oracle.oracle import OracleOperator, oracle_pcg

pytestmark = pytest.mark.gpu


def test_distributed_world1_bit_identical():
    import paper_1907_04417_b200 as mv
    from paper_1907_04417_b200.distributed import DistributedSolver

    from paper_1907_04417_b200.distributed import DeviceBackend

    d = golden("c1")
    mats, pros = hierarchy(d, "mv")
    exact = mv.GpuConfig(exact_gs=True)  # same schedules' bits whatever kernel each level gets
    s = DistributedSolver(mats, pros, backend=DeviceBackend(exact))
    op = s.op
    z = op.be.vec(op.n_own)
    op.apply(op.be.from_host(d["b"]), z)
    ref = mv.GpuMultigridOperator(mats, pros, config=exact).apply(d["b"])
    assert np.array_equal(z.cpu().numpy(), ref)
    x, rep = s.solve(d["b"])
    _, hist, nit, _ = oracle_pcg(OracleOperator(mats, pros), d["b"])
    assert rep.iterations == nit
    assert np.max(np.abs(rep.residual_history - hist) / hist) <= 1e-10


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    import torch

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1907_04417_b200.distributed import DistributedSolver

        d = golden("c1")
        mats, pros = hierarchy(d, "mv")
        s = DistributedSolver(mats, pros)
        op = s.op
        z = op.be.vec(op.n_own)
        op.apply(op.be.from_host(s.own_rows(d["b"])), z)
        x, rep = s.solve(d["b"])
        out[rank] = (z.cpu().numpy(), x, rep.iterations, rep.residual_history)
    finally:
        dist.destroy_process_group()


def test_distributed_two_ranks_one_gpu():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    d = golden("c1")
    mats, pros = hierarchy(d, "mv")
    ref = OracleOperator(mats, pros)
    z_ref = ref.apply(d["b"])
    z = np.concatenate([out[r][0] for r in range(world)])
    assert np.max(np.abs(z - z_ref)) / np.max(np.abs(z_ref)) <= 1e-10
    _, hist, nit, _ = oracle_pcg(ref, d["b"])
    assert abs(out[0][2] - nit) <= 1 and out[0][2] == out[1][2]
    h = out[0][3]
    m = min(len(h), len(hist))
    assert np.max(np.abs(h[:m] - hist[:m]) / hist[:m]) <= 1e-10
