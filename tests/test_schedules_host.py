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


# ---- cluster dataflow plan (mvamg_gs_cluster_plan, gs_cluster.cuh) -------------------------------
def _cluster_plan(A, mode, ncta, wpc, page=2048, grid=0):
    A = sp.csr_matrix(A)
    n = A.shape[0]
    L = _lib.load()
    ip = np.ascontiguousarray(A.indptr, dtype=np.int32)
    ix = np.ascontiguousarray(A.indices, dtype=np.int32)
    v = np.ascontiguousarray(A.data, dtype=np.float64)
    npg, nl, sl, hits = ctypes.c_longlong(), ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    head = (n, vp(ip), vp(ix), vp(v), mode, grid, ncta, wpc, page, ctypes.byref(npg), ctypes.byref(nl),
            ctypes.byref(sl), ctypes.byref(hits))
    _lib.check(L.mvamg_gs_cluster_plan(*head, None, None, None, None, None), "plan")
    G = ncta * wpc
    wptr, wpage = np.empty(G + 1, dtype=np.int32), np.empty(G + 1, dtype=np.int32)
    rowid, perm = np.empty(max(1, n), dtype=np.int32), np.empty(max(1, n), dtype=np.int32)
    blob = np.zeros(max(1, npg.value) * page, dtype=np.uint8)
    _lib.check(L.mvamg_gs_cluster_plan(*head, vp(wptr), vp(wpage), vp(rowid), vp(perm), vp(blob)), "plan")
    return dict(wptr=wptr, wpage=wpage, rowid=rowid, perm=perm, blob=blob, nlev=nl.value, slots=sl.value,
                local=hits.value, page=page, npages=npg.value, grid=grid)


def _cluster_streams(pl, G):
    """Per worker, its rows in order: (cnt, early, row, slot, diag, coef[], src[]) decoded as the kernel reads them."""
    page, blob = pl["page"], pl["blob"]
    out = []
    for g in range(G):
        rows = []
        for pg in range(pl["wpage"][g], pl["wpage"][g + 1]):
            base = pg * page
            nrows = int(blob[base:base + 4].view(np.int32)[0])
            off = base + 16
            for _ in range(nrows):
                assert off % 16 == 0
                cnt, ne, row, slot = (int(t) for t in blob[off:off + 16].view(np.int32))
                dg, rdg = blob[off + 16:off + 32].view(np.float64)
                assert rdg == 1.0 / dg
                cf = blob[off + 32:off + 32 + 8 * cnt].view(np.float64)
                sc = blob[off + 32 + 8 * cnt:off + 32 + 12 * cnt].view(np.uint32)
                assert 0 <= ne <= cnt and cnt - ne <= 4
                rows.append((cnt, ne, row, slot, float(dg), cf, sc))
                off += (32 + 12 * cnt + 15) & ~15
            assert off <= base + page                              # no record straddles a page
        assert len(rows) == pl["wptr"][g + 1] - pl["wptr"][g]
        for t, rw in enumerate(rows):
            assert pl["rowid"][pl["wptr"][g] + t] == rw[2] and pl["perm"][rw[2]] == pl["wptr"][g] + t
        out.append(rows)
    return out


def _cluster_emulate(A, pl, ncta, wpc, mode, b, x_old):
    """Run the plan as the kernel does -- every worker takes its rows in order, a
    row only when all its polled inputs are published -- and return x."""
    n = A.shape[0]
    G = ncta * wpc
    streams = _cluster_streams(pl, G)
    xs = np.full((ncta, pl["slots"]), np.nan)
    xg = np.full(n, np.nan)                                          # x_new in global memory (grid form)
    grid = pl["grid"]
    cur = [0] * G
    x = np.zeros(n)
    left = n
    while left:
        progressed = False
        for g in range(G):
            if cur[g] >= len(streams[g]):
                continue
            cnt, ne, row, slot, dg, cf, sc = streams[g][cur[g]]
            vals = np.empty(cnt)
            for u in range(cnt):
                s = int(sc[u])
                if s >> 31:
                    vals[u] = x_old[s & 0x7fffffff]
                elif not grid:
                    vals[u] = xs[(s >> 24) & 15, s & 0xffffff]
                elif s >> 30:                                        # a late input this CTA owns: its shared slot
                    assert u >= ne
                    vals[u] = xs[g % ncta, s & 0xffffff]
                else:
                    vals[u] = xg[s]
            if np.isnan(vals).any():
                continue
            xi = (b[row] - np.dot(cf, vals)) / dg
            if slot >= 0:                                           # grid form: only rows polled in this CTA
                assert np.isnan(xs[g % ncta, slot])                 # every slot is written once
                xs[g % ncta, slot] = xi
            else:
                assert grid
            xg[row] = xi
            x[row] = xi
            cur[g] += 1
            left -= 1
            progressed = True
        assert progressed, "the plan deadlocks"
    return x


@pytest.mark.parametrize("ncta,wpc,grid", [(1, 1, 0), (2, 3, 0), (4, 8, 0), (16, 32, 0), (1, 2, 1), (37, 5, 1),
                                           (148, 8, 1)])
def test_cluster_plan_is_the_serial_sweep(ncta, wpc, grid):
    rng = np.random.default_rng(5)
    cases = [laplacian_1d(70), laplacian_2d(13), random_spd_csr(300, density=0.05, seed=1),
             random_spd_csr(90, density=0.9, seed=2), sp.diags(np.linspace(1, 2, 9)).tocsr(),
             sp.csr_matrix(np.array([[2.0]]))]
    for A in cases:
        A = sp.csr_matrix(A)
        n = A.shape[0]
        d = A.diagonal()
        b, x0 = rng.standard_normal(n), rng.standard_normal(n)
        for mode in range(4):
            pl = _cluster_plan(A, mode, ncta, wpc, grid=grid)
            x_old = np.zeros(n) if mode % 2 == 0 else x0
            got = _cluster_emulate(A, pl, ncta, wpc, mode, b, x_old)
            want = x_old.copy()                                     # the serial loop, _kernels.py:15-38
            for i in (range(n) if mode < 2 else range(n - 1, -1, -1)):
                s = b[i]
                for k in range(A.indptr[i], A.indptr[i + 1]):
                    j = A.indices[k]
                    if j != i:
                        s -= A.data[k] * want[j]
                want[i] = s / d[i]
            assert np.max(np.abs(got - want)) <= 1e-13 * max(1.0, np.max(np.abs(want))), (n, mode)
            assert sorted(pl["rowid"][:n].tolist()) == list(range(n))
            counts = np.diff(pl["wptr"])
            assert counts.sum() == n


def test_cluster_plan_balance_and_locality():
    """Rows follow their latest input's CTA where the level's share allows, and no CTA ends up with much more
    than its share of the rows (its x slice must fit shared memory)."""
    A = random_spd_csr(4000, density=0.01, seed=3)
    pl = _cluster_plan(A, 0, 16, 8)
    assert pl["local"] >= 0.5 * 4000
    assert pl["slots"] <= 1.25 * 4000 / 16 + 8
    per_worker = np.diff(pl["wptr"])
    assert per_worker.max() <= 1.25 * 4000 / 128 + 2


def test_cluster_plan_long_rows_need_larger_pages():
    n = 400
    D = sp.csr_matrix(np.ones((n, n)) * 0.01 + np.eye(n) * n)
    L = _lib.load()
    ip, ix = np.ascontiguousarray(D.indptr, dtype=np.int32), np.ascontiguousarray(D.indices, dtype=np.int32)
    v = np.ascontiguousarray(D.data)
    npg, nl, sl, hits = ctypes.c_longlong(), ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    rc = L.mvamg_gs_cluster_plan(n, vp(ip), vp(ix), vp(v), 0, 0, 2, 2, 2048, ctypes.byref(npg), ctypes.byref(nl),
                                 ctypes.byref(sl), ctypes.byref(hits), None, None, None, None, None)
    assert rc == _lib.E_ARG                                        # 399 entries: 4,832 bytes > one 2 KiB page
    pl = _cluster_plan(D, 0, 2, 2, page=8192)
    rng = np.random.default_rng(0)
    b = rng.standard_normal(n)
    got = _cluster_emulate(D, pl, 2, 2, 0, b, np.zeros(n))
    want = np.linalg.solve(np.tril(D.toarray()), b)
    assert np.max(np.abs(got - want)) <= 1e-13 * np.max(np.abs(want))
