"""Process-group plumbing of bench.py's N > 1 path on CPU: world-size-2 gloo
process groups run the barrier and the max-over-ranks device time around CPU
oracle solves (the row-partitioned solve itself: tests/test_distributed.py)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from _fixtures import laplacian_2d


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WORLD_SIZE=str(ws), RANK=str(rank),
                      LOCAL_RANK=str(rank))
    from paper_1907_04417_b200 import replicas

    dist = replicas.init("gloo")
    try:
        from oracle.oracle import OracleOperator, oracle_pcg

        A = laplacian_2d(24)
        rng = np.random.default_rng(rank)  # each replica solves its own rhs
        b = rng.uniform(-1, 1, A.shape[0])
        op = OracleOperator([A], [])
        dist.barrier()
        x, hist, nit, conv = oracle_pcg(op, b, precond="none", rtol=1e-8)
        t_local = 0.25 * (rank + 1)  # stand-in device time per rank
        t_max = replicas.max_over_ranks(t_local, dist)
        res = float(np.linalg.norm(b - A @ x) / np.linalg.norm(b))
        q.put((rank, t_max, res, conv, replicas.parallelism(ws)))
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_replicas_world2_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=100) for _ in procs)
    for p in procs:
        p.join(timeout=30)
        assert p.exitcode == 0
    for rank, t_max, res, conv, par in out:
        assert t_max == 0.5  # max over ranks, identical on both
        assert conv and res <= 1e-8
        assert par.startswith("row-partitioned fine level over 2 GPUs")


def test_single_process_identity():
    from paper_1907_04417_b200 import replicas

    assert replicas.max_over_ranks(1.5, None) == 1.5
    assert replicas.parallelism(1) == "single GPU"
