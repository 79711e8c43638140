"""Host-side schedule builders of the GS kernels (CPU, no GPU needed): the
streamed level-set plan (mvamg_gs_stream_plan), the blocked chain order and
the modular window of the lean wavefront (chain_block_order, mvamg_gs_schedule
with wpos), and row schedules over a row range (mvamg_gs_rows, the pipelined
row partition).  Each plan is decoded here and checked against the sweep's
dependency DAG (_kernels.py:15-38): every row exactly once, every input of a
row in an earlier batch / round, nothing the kernel could read before it is
final."""

import ctypes

import numpy as np
import pytest
import scipy.sparse as sp

from _fixtures import laplacian_1d, laplacian_2d, laplacian_3d, random_spd_csr

from paper_1907_04417_b200 import _lib, problems
from paper_1907_04417_b200.device import GpuConfig, _gs_ring, chain_block_order, gs_analyse, gs_schedule

vp = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731


def _stream_plan(A, mode, slot, ncta):
    A = sp.csr_matrix(A)
    L = _lib.load()
    ip = np.ascontiguousarray(A.indptr, dtype=np.int32)
    ix = np.ascontiguousarray(A.indices, dtype=np.int32)
    v = np.ascontiguousarray(A.data, dtype=np.float64)
    nb, ns, nl = ctypes.c_longlong(), ctypes.c_int(), ctypes.c_int()
    _lib.check(L.mvamg_gs_stream_plan(A.shape[0], vp(ip), vp(ix), vp(v), mode, slot, ncta, ctypes.byref(nb),
                                      ctypes.byref(ns), ctypes.byref(nl), None, None), "plan")
    blob = np.zeros(max(16, nb.value), dtype=np.uint8)
    off = np.zeros(ns.value * ncta + 1, dtype=np.int64)
    _lib.check(L.mvamg_gs_stream_plan(A.shape[0], vp(ip), vp(ix), vp(v), mode, slot, ncta, ctypes.byref(nb),
                                      ctypes.byref(ns), ctypes.byref(nl), vp(blob), vp(off)), "plan")
    return blob, off, ns.value


def _decode(blob, off, nstages, ncta, n):
    """[(stage, batch, cta, row, [columns])] in execution order."""
    R = -(-n // ncta) if ncta > 1 else n
    out = []
    for s in range(nstages):
        for c in range(ncta):
            st = blob[off[s * ncta + c]:off[s * ncta + c + 1]]
            hdr = st[:16].view(np.uint32)
            nb, nr, ne = int(hdr[0]), int(hdr[1]), int(hdr[2])
            assert off[s * ncta + c + 1] - off[s * ncta + c] <= 1 << 20
            bt = st[16:16 + 8 * nb].view(np.uint32).reshape(nb, 2)
            rows_off = (16 + 8 * nb + 15) & ~15
            coef_off = rows_off + 32 * nr
            src_off = (coef_off + 8 * ne + 15) & ~15
            rows = st[rows_off:rows_off + 32 * nr].view(np.uint32).reshape(nr, 8)
            src = st[src_off:src_off + 4 * ne].view(np.uint32)
            for b in range(nb):
                for r in range(int(bt[b, 0]), int(bt[b, 0] + bt[b, 1])):
                    loc, cnt, ebeg = int(rows[r, 0]), int(rows[r, 1]), int(rows[r, 2])
                    cols = src[ebeg:ebeg + cnt]
                    if ncta > 1:
                        cols = (cols >> 24) * R + (cols & 0xFFFFFF)
                        loc += c * R
                    out.append((s, b, c, loc, [int(j) for j in cols]))
    return out


@pytest.mark.parametrize("mode", [0, 1, 2, 3])
@pytest.mark.parametrize("slot,ncta", [(65536, 1), (2048, 1), (4096, 4)])
def test_stream_plan_respects_the_dag(mode, slot, ncta):
    if ncta > 1 and mode & 1:
        pytest.skip("cluster plans are zero-guess only")
    fwd, old = mode < 2, bool(mode & 1)
    for A in (laplacian_2d(20).tocsr(), random_spd_csr(300, density=0.03, seed=2), problems.jump_3d(8, 4, 1)):
        n = A.shape[0]
        blob, off, ns = _stream_plan(A, mode, slot, ncta)
        ents = _decode(blob, off, ns, ncta, n)
        assert sorted(e[3] for e in ents) == list(range(n))            # every row once
        when = {e[3]: (e[0], e[1]) for e in ents}
        for s, b, c, i, cols in ents:
            row = A.indices[A.indptr[i]:A.indptr[i + 1]]
            keep = [j for j in row if j != i and (old or (j < i if fwd else j > i))]
            assert cols == keep                                         # the row's entries, CSR order
            for j in row:
                if j == i:
                    continue
                if (j < i) == fwd:                                      # an input: final before i
                    assert when[j] < (s, b), (i, j)
                elif old:                                               # an old value: read before overwritten
                    assert when[j] > (s, b), (i, j)


def test_chain_block_order_and_schedule():
    A = laplacian_3d(32).tocsr()
    p = gs_analyse(A)
    assert p.chain_order is not None
    assert np.array_equal(np.sort(p.chain_order), np.arange(p.nchains))
    C, R, D, slot, S = _gs_ring(A, GpuConfig())
    for m in (0, 2):
        gs_schedule(A, p, m, R=R, uniform_S=S)       # verifies: inputs only from earlier warps
    assert chain_block_order(laplacian_2d(64).tocsr(), np.arange(0, 64 * 64 + 1, 64, dtype=np.int32), 64) is None


def test_modular_window_is_verified():
    cfg = GpuConfig(lean_wpos=2, max_threads=32)
    A = laplacian_2d(64).tocsr()
    p = gs_analyse(A, cfg)
    assert p.wpos == 2 and p.threads == 32
    C, R, D, slot, S = _gs_ring(A, cfg)
    gs_schedule(A, p, 0, R=R, uniform_S=S)            # 5-point: position lag 0, two slots suffice
    Q = problems.anisotropic_q1(64)                   # 9-point reads (x+1, y-1): needs more
    pq = gs_analyse(Q, cfg)
    Cq, Rq, Dq, sq, Sq = _gs_ring(Q, cfg)
    with pytest.raises(ValueError, match="too short"):
        gs_schedule(Q, pq, 0, R=Rq, uniform_S=Sq)


def test_row_schedule_over_a_row_range():
    A = laplacian_1d(50).tocsr()
    L = _lib.load()
    ip, ix = np.ascontiguousarray(A.indptr, dtype=np.int32), np.ascontiguousarray(A.indices, dtype=np.int32)
    v = np.ascontiguousarray(A.data)
    ns, nl = ctypes.c_longlong(), ctypes.c_int()
    lo, hi = 10, 30
    _lib.check(L.mvamg_gs_rows(50, vp(ip), vp(ix), vp(v), 0, 0, ctypes.byref(ns), ctypes.byref(nl), None, None,
                               None, None, None, None, None, None, None, lo, hi), "gs_rows")
    n = hi - lo
    rowid, cnt, crit = (np.empty(n, dtype=np.int32) for _ in range(3))
    dg, rdg = np.empty(n), np.empty(n)
    perm = np.full(50, -1, dtype=np.int32)
    wofs = np.empty(-(-n // 32) + 1, dtype=np.int32)
    coef = np.empty(max(32, 32 * ns.value))
    src = np.empty(max(32, 32 * ns.value), dtype=np.int32)
    _lib.check(L.mvamg_gs_rows(50, vp(ip), vp(ix), vp(v), 0, 0, ctypes.byref(ns), ctypes.byref(nl), vp(rowid),
                               vp(cnt), vp(crit), vp(dg), vp(rdg), vp(perm), vp(wofs), vp(coef), vp(src), lo, hi),
               "gs_rows")
    assert sorted(rowid.tolist()) == list(range(lo, hi))           # only the own rows are positions
    assert np.all(perm[:lo] == -1) and np.all(perm[hi:] == -1)     # ghosts are never written
    assert list(rowid) == list(range(lo, hi))                      # a chain: topological = natural order
    assert src[0] == lo - 1                                        # the first row reads its lower ghost
