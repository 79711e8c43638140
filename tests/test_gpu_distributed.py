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
from oracle.oracle import OracleOperator, oracle_gs, oracle_pcg

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

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
        s = DistributedSolver(mats, pros)  # gloo on one GPU: the relay (no kernel waits on a peer)
        op = s.op
        assert not op.pipelined
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


def test_pipelined_ext_sweeps_bit_exact_sequential():
    """The pipelined fine-level sweep kernel (mvamg_gs_row_sweep_ext_f64) of a
    2- and 3-rank row partition, run rank after rank on one GPU (forward in
    rank order, backward in reverse -- no kernel waits on another concurrently
    running one): each rank's rows over its extended layout, ghost inputs read
    from the slots its peers' kernels stored into, CSR summation order kept --
    bit-identical to the serial sweep of the whole matrix."""
    import torch

    from paper_1907_04417_b200.device import GpuConfig
    from paper_1907_04417_b200.distributed import DeviceBackend, RowPartition, plan_rank

    d = golden("c1")
    mats, pros = hierarchy(d, "mv")
    A, P = mats[0], pros[0]
    n = A.shape[0]
    rng = np.random.default_rng(7)
    b, x0 = rng.standard_normal(n), rng.standard_normal(n)
    be = DeviceBackend(GpuConfig(exact_gs=True))
    for nr in (2, 3):
        part = RowPartition.balanced(A, nr)
        plans = [plan_rank(A, P, part, r) for r in range(nr)]
        xps = [torch.empty(p.xhalo.n_own + p.xhalo.n_ghost, dtype=torch.float64, device="cuda") for p in plans]
        peers = torch.tensor([t.data_ptr() for t in xps], dtype=torch.int64, device="cuda")
        for mode, direction in ((0, "forward"), (2, "backward")):
            want = np.zeros(n) if mode == 0 else x0.copy()
            oracle_gs(A, b, want, direction)
            for t in xps:
                be.fill_sentinel(t)
            order = range(nr) if mode == 0 else range(nr - 1, -1, -1)
            got = np.empty(n)
            for r in order:
                pl, h = plans[r], plans[r].xhalo
                mirror = pl.mirror_fwd if mode == 0 else pl.mirror_bwd
                pp = be.pipe_plan(pl.M_ext, (h.n_lower, h.n_lower + h.n_own), mode, mirror)
                xo = None
                if mode == 2:
                    ext = np.concatenate([x0[h.ghosts[:h.n_lower]], x0[h.lo:h.hi], x0[h.ghosts[h.n_lower:]]])
                    xo = torch.from_numpy(ext).cuda()
                be.pipe_sweep(pp, torch.from_numpy(b[h.lo:h.hi].copy()).cuda(), xo, xps[r], peers)
                got[h.lo:h.hi] = xps[r][h.n_lower:h.n_lower + h.n_own].cpu().numpy()
            assert np.array_equal(got, want), (nr, direction)


def test_ipc_handle_opened_by_another_process():
    """mvamg_ipc_handle / mvamg_ipc_open: a child process opens this process's
    buffer and stores into it (what a peer rank's pipelined sweep does)."""
    import ctypes
    import subprocess
    import sys

    import torch

    from paper_1907_04417_b200 import _lib

    L = _lib.load()
    buf = torch.zeros(16, dtype=torch.float64, device="cuda")
    h = ctypes.create_string_buffer(64)
    _lib.check(L.mvamg_ipc_handle(ctypes.c_void_p(buf.data_ptr()), h), "ipc_handle")
    torch.cuda.synchronize()
    code = (
        "import ctypes, sys, torch\n"
        "sys.path.insert(0, %r)\n"
        "from paper_1907_04417_b200 import _lib\n"
        "L = _lib.load()\n"
        "p = ctypes.c_void_p()\n"
        "_lib.check(L.mvamg_ipc_open(ctypes.create_string_buffer(bytes.fromhex(%r), 64), ctypes.byref(p)), 'open')\n"
        "src = torch.arange(16, dtype=torch.float64, device='cuda')\n"
        "idx = torch.arange(16, dtype=torch.int32, device='cuda')\n"
        "_lib.check(L.mvamg_gather_f64(16, ctypes.c_void_p(idx.data_ptr()), ctypes.c_void_p(src.data_ptr()), p, None), 'gather')\n"
        "torch.cuda.synchronize()\n"
        "_lib.check(L.mvamg_ipc_close(p), 'close')\n" % (ROOT, h.raw.hex()))
    subprocess.run([sys.executable, "-c", code], check=True, timeout=300)
    assert np.array_equal(buf.cpu().numpy(), np.arange(16.0))
