"""Row-partitioned solve (paper_1907_04417_b200.distributed) on
the CPU: partition and halo plans, and the whole relay / halo / gather
algorithm under gloo with world sizes 1-3, with the oracle as arithmetic
(tests/_dist_backend.py), against the single-process oracle solve."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from _fixtures import golden, hierarchy, laplacian_2d
from oracle.oracle import OracleOperator, oracle_pcg
from paper_1907_04417_b200.distributed import (DistributedSolver, DistributedVCycle, RowPartition, make_halo,
                                               plan_rank)


def test_partition_balanced():
    A = laplacian_2d(10)
    for nr in (1, 2, 3, 7, 100):
        p = RowPartition.balanced(A, nr)
        assert p.offsets[0] == 0 and p.offsets[-1] == 100 and np.all(np.diff(p.offsets) >= 1)
        nnz = np.diff(A.indptr[p.offsets])
        assert nnz.max() - nnz.min() <= 2 * 5 + 5  # within a couple of rows of balanced
    with pytest.raises(ValueError):
        RowPartition.balanced(A, 101)


def test_halo_plans_are_consistent():
    A = laplacian_2d(12)
    part = RowPartition.balanced(A, 4)
    need = [np.unique(A.indices[A.indptr[part.offsets[q]]:A.indptr[part.offsets[q + 1]]]) for q in range(4)]
    halos = [make_halo(part, r, need) for r in range(4)]
    for r, h in enumerate(halos):
        for q, sl in h.recv.items():
            # what q sends to r is exactly the ghosts r receives from q, in order
            assert np.array_equal(halos[q].send[r] + halos[q].lo, h.ghosts[sl])
        assert set(h.recv) == {q for q in range(4) if r in halos[q].send}
        lo_g = h.ghosts[:h.n_lower]
        assert np.all(lo_g < h.lo) and np.all(h.ghosts[h.n_lower:] >= h.hi)


def test_plan_local_blocks_reassemble():
    d = golden("c1")
    mats, pros = hierarchy(d, "mv")
    A, P = mats[0], pros[0]
    part = RowPartition.balanced(A, 3)
    x = np.random.default_rng(0).standard_normal(A.shape[0])
    t = np.random.default_rng(1).standard_normal(A.shape[0])
    R = P.T.tocsr()
    rc = np.zeros(P.shape[1])
    for r in range(3):
        pl = plan_rank(A, P, part, r)
        h = pl.xhalo
        xe = np.concatenate([x[h.ghosts[:h.n_lower]], x[h.lo:h.hi], x[h.ghosts[h.n_lower:]]])
        assert np.array_equal(pl.A_ext @ xe, (A @ x)[h.lo:h.hi])       # CSR order kept: bit-exact
        th = pl.thalo
        te = np.concatenate([t[th.ghosts[:th.n_lower]], t[th.lo:th.hi], t[th.ghosts[th.n_lower:]]])
        rc[pl.coarse_own] = pl.R_ext @ te
    assert np.array_equal(rc, R @ t)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out, direct=None):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from _dist_backend import OracleBackend
        from paper_1907_04417_b200.distributed import Comm

        d = golden("c1")
        mats, pros = hierarchy(d, "mv")
        s = DistributedSolver(mats, pros, comm=Comm(direct=direct), backend=OracleBackend())
        op = s.op
        z = op.be.vec(op.n_own)
        op.apply(op.be.from_host(s.own_rows(d["b"])), z)
        x, rep = s.solve(d["b"])
        out[rank] = (z.numpy().copy(), x, rep.iterations, rep.residual_history)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,direct", [(1, None), (2, None), (3, None), (2, True), (3, True)])
def test_distributed_pcg_gloo(world, direct):
    """direct=True hands the tensors to the backend unstaged -- the NCCL code
    path (views of the extended vectors as receive buffers), run by gloo."""
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out, direct), nprocs=world, join=True)
    d = golden("c1")
    mats, pros = hierarchy(d, "mv")
    ref = OracleOperator(mats, pros)
    z_ref = ref.apply(d["b"])
    z = np.concatenate([out[r][0] for r in range(world)])
    err = np.max(np.abs(z - z_ref)) / np.max(np.abs(z_ref))
    if world == 1:
        assert err == 0.0           # no ghosts: the single-GPU recipe, bit for bit
    assert err <= 1e-10
    _, hist, nit, _ = oracle_pcg(ref, d["b"])
    x = np.concatenate([out[r][1] for r in range(world)])
    for r in range(world):
        assert abs(out[r][2] - nit) <= 1
    h = out[0][3]
    m = min(len(h), len(hist))
    assert np.max(np.abs(h[:m] - hist[:m]) / hist[:m]) <= 1e-10
    assert np.linalg.norm(d["b"] - mats[0] @ x) <= 1e-6 * np.linalg.norm(d["b"]) * 1.0001


def _worker_pipelined(rank, world, port, out, tag):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    be = None
    try:
        from _dist_backend import PipelinedOracleBackend
        from paper_1907_04417_b200.distributed import Comm

        d = golden("c1")
        mats, pros = hierarchy(d, "mv")
        be = PipelinedOracleBackend(tag)
        s = DistributedSolver(mats, pros, comm=Comm(), backend=be)
        op = s.op
        assert op.pipelined
        z = op.be.vec(op.n_own)
        op.apply(op.be.from_host(s.own_rows(d["b"])), z)
        x, rep = s.solve(d["b"])
        out[rank] = (z.numpy().copy(), x, rep.iterations, rep.residual_history)
        dist.barrier()
    finally:
        if be is not None:
            be.close()
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_distributed_pipelined_sweeps_gloo(world):
    """The pipelined fine-level sweeps (every rank sweeps at once, polling its
    ghosts, which their owners -- other processes -- store into its shared
    extended x as they finish them): the same dependency order and the same
    CSR summation order as the serial loop, so one V-cycle is bit-identical to
    the single-process oracle's (the relay folds the upper ghosts out of
    order: 1e-10).  PCG as the single-process solve (dots: tolerance)."""
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_worker_pipelined, args=(world, port, out, f"t{port}"), nprocs=world, join=True)
    d = golden("c1")
    mats, pros = hierarchy(d, "mv")
    ref = OracleOperator(mats, pros)
    z = np.concatenate([out[r][0] for r in range(world)])
    assert np.array_equal(z, ref.apply(d["b"]))
    _, hist, nit, _ = oracle_pcg(ref, d["b"])
    for r in range(world):
        assert out[r][2] == nit
    h = out[0][3]
    assert np.max(np.abs(h - hist[:len(h)]) / hist[:len(h)]) <= 1e-10
    x = np.concatenate([out[r][1] for r in range(world)])
    assert np.linalg.norm(d["b"] - mats[0] @ x) <= 1e-6 * np.linalg.norm(d["b"]) * 1.0001


def test_cycle_needs_two_levels():
    from _dist_backend import OracleBackend

    with pytest.raises(ValueError):
        DistributedVCycle([laplacian_2d(4)], [], backend=OracleBackend())
