"""CPU: the chain-scan GS planner (paper_1907_04417_b200/gs_scan.py).  A
sequential executor of the plan's records (test-only) must reproduce the
reference sweep (oracle, _kernels.py:15-38) within rounding, and every wait
must cover the segment's sources."""

import numpy as np
import pytest
import scipy.sparse as sp

from _fixtures import golden, hierarchy, laplacian_1d, laplacian_2d, laplacian_3d
from oracle.oracle import oracle_gs
from paper_1907_04417_b200 import problems
from paper_1907_04417_b200.gs_scan import MAX_DEPS, plan_scan


def run_plan(p, A, b, x_old):
    """Execute a ScanPlan row by row in sweep order (what the kernel computes),
    checking that every source is covered by a wait of its segment."""
    A = sp.csr_matrix(A)
    n = A.shape[0]
    fwd = p.mode < 2
    old = p.mode % 2 == 1
    nv = p.nv
    recv = p.recv.reshape(-1, nv, 32, 2)
    addr = p.addr.reshape(-1, 32, 4)
    info = p.seginfo
    o0 = np.zeros(recv.shape[0] * 32)
    for i in range(n):
        s = b[i]
        if old:
            for k in range(A.indptr[i], A.indptr[i + 1]):
                j = A.indices[k]
                if (j > i) if fwd else (j < i):
                    s -= A.data[k] * x_old[j]
        o0[p.rec[i]] = s * p.rdiag[i]
    xs = np.zeros(n)  # sweep order
    for L in range(p.nchains):
        cs, ln = p.chain_start[L], p.chain_len[L]
        carry = 0.0
        for q in range(ln):
            r = (p.seg_ptr[L] + q // 32) * 32 + q % 32
            g, lane = r // 32, r % 32
            waits = [int(x) for x in (info["wait0"][g], info["wait1"][g]) if x]
            o = o0[r]
            flat = recv[g, :, lane, :].ravel()
            for k in range(p.K):
                a = int(addr[g, lane, k])
                d, pos = a >> 20, a & 0xFFFFF
                if d == 0:
                    assert flat[k + 1] == 0.0
                    continue
                assert any((x >> 20) == d and (x & 0xFFFFF) >= pos // 32 + 1 for x in waits), (L, q)
                o -= flat[k + 1] * xs[p.chain_start[L - d] + pos]
            if lane == 31 and info["defer"][g]:
                dv, dpos = int(info["defer"][g]), int(info["defpos"][g])
                d = dv >> 20
                assert (dv & 0xFFFFF) >= dpos // 32 + 1
                o -= info["defcoef"][g] * xs[p.chain_start[L - d] + dpos]
            x = o + flat[0] * carry
            xs[cs + q] = x
            carry = x
    return xs if fwd else xs[::-1]


def cases():
    yield "lap1d", laplacian_1d(50)
    yield "lap2d", laplacian_2d(20)
    yield "lap3d", laplacian_3d(6)
    yield "q1aniso", problems.anisotropic_q1(24)
    yield "jump3d", problems.jump_3d(8, 4, 1)
    yield "c1_fine", hierarchy(golden("c1"), "mv")[0][0]


@pytest.mark.parametrize("name,A", list(cases()), ids=[c[0] for c in cases()])
@pytest.mark.parametrize("mode", [0, 1, 2, 3])
def test_plan_executes_the_reference_sweep(name, A, mode):
    p = plan_scan(A, mode)
    assert p is not None
    n = A.shape[0]
    rng = np.random.default_rng(mode)
    b = rng.standard_normal(n)
    x0 = rng.standard_normal(n)
    want = np.zeros(n) if mode % 2 == 0 else x0.copy()
    oracle_gs(A, b, want, "forward" if mode < 2 else "backward")
    got = run_plan(p, A, b, x0)
    assert np.max(np.abs(got - want)) <= 1e-12 * np.max(np.abs(want))


def test_plan_shapes():
    p = plan_scan(problems.anisotropic_q1(64), 0)
    assert p.nchains == 64 and p.W == 1 and p.K == 3
    assert p.depth <= 64 + 2 + 2   # wavefront: one segment step per line (deferral) + the last line
    p3 = plan_scan(laplacian_3d(8), 0)
    assert p3.W == 8 and p3.K == 2


def test_plan_rejects_unchained():
    # interleaved dofs: row i rarely couples to i - 1
    A = laplacian_2d(12)
    n = A.shape[0]
    perm = np.concatenate([np.arange(0, n, 2), np.arange(1, n, 2)])
    B = sp.csr_matrix(A[perm][:, perm])
    p = plan_scan(B, 0)
    assert p is None or p.nchains > n // 4
