"""CPU-only setup (oracle/host_setup.py, bench.py's reference arm) and the
hierarchy cache (paper_1907_04417_b200/hcache.py).

The reference arm must build its hierarchy on host cores only; these tests pin
that setup to the reference's own C1 fit (golden fixture made by the unmodified
reference) and its natives (greedy acceptance, batched Jacobi SVD) to the
product's host restatements, bit for bit."""

import os
import subprocess
import sys

import numpy as np
import pytest
import scipy.sparse as sp

from _fixtures import golden, hierarchy, laplacian_2d
from oracle.host_setup import fit_host, host_matching, host_svd
from oracle.oracle import OracleOperator, oracle_pcg

from paper_1907_04417_b200 import hcache, problems

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def rel(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


@pytest.fixture(scope="module")
def c1_fit():
    return fit_host(problems.poisson_2d(128))


def test_c1_host_fit_matches_reference(c1_fit):
    """Same aggregates / kept counts (patterns), values to rounding, same PCG
    iterations and history as the reference's own C1 fit and solve."""
    mats, pros, info = c1_fit
    d = golden("c1")
    rm, rp = hierarchy(d, "mv")
    assert [M.shape[0] for M in mats] == [M.shape[0] for M in rm]
    assert info["bootstrap_stages"] == int(d["n_comp"])
    for k in range(len(pros)):
        assert np.array_equal(pros[k].indptr, rp[k].indptr) and np.array_equal(pros[k].indices, rp[k].indices)
        assert rel(pros[k].data, rp[k].data) <= 1e-10
    for k in range(1, len(mats)):
        assert np.array_equal(mats[k].indices, rm[k].indices)
        assert rel(mats[k].data, rm[k].data) <= 1e-10
    _, hist, nit, conv = oracle_pcg(OracleOperator(mats, pros), d["b"])
    assert conv and nit == int(d["pcg_nit"])
    assert rel(hist, d["pcg_hist"]) <= 1e-10


def test_host_matching_equals_product_greedy():
    from paper_1907_04417_b200.setup import edge_weights, greedy_matching

    A = problems.anisotropic_q1(24)
    w = np.random.default_rng(3).uniform(0.5, 1.5, A.shape[0])
    p1, u1 = host_matching(A, w)
    i, j, c = edge_weights(A, w)
    p2, u2 = greedy_matching(i, j, c, A.shape[0])
    assert np.array_equal(p1, p2) and np.array_equal(u1, u2)


def test_host_svd_equals_product_restatement():
    import ctypes

    from paper_1907_04417_b200 import _lib

    rng = np.random.default_rng(7)
    sizes = rng.integers(1, 65, 200)
    rp = np.zeros(201, dtype=np.int32)
    rp[1:] = np.cumsum(sizes)
    nv = 5
    local = rng.standard_normal((rp[-1], nv))
    local[rp[3]:rp[4]] = 0.0                                   # zero block
    local[rp[5]:rp[6], 1] = local[rp[5]:rp[6], 0]              # duplicate column
    local[rp[7]:rp[8]] *= 1e-150
    code, U, sig, failed = host_svd(rp, local, nv)
    assert code == 0 and failed == -1
    Uh, sh = np.empty_like(local), np.empty((200, nv))
    f = ctypes.c_int(-1)
    vp = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    assert _lib.load().mvamg_jacobi_svd_batch(200, vp(rp), nv, vp(local), 60, 1e-14, vp(Uh), vp(sh),
                                              ctypes.byref(f)) == 0
    assert np.array_equal(U.view(np.int64), Uh.view(np.int64))
    assert np.array_equal(sig.view(np.int64), sh.view(np.int64))


def test_host_setup_never_maps_the_gpu_library():
    code = ("import sys; sys.path.insert(0, %r); sys.path.insert(0, %r)\n"
            "from oracle.host_setup import fit_host\n"
            "from paper_1907_04417_b200 import problems\n"
            "fit_host(problems.poisson_2d(32))\n"
            "maps = open('/proc/self/maps').read()\n"
            "assert 'libmvamg_b200' not in maps, 'GPU library mapped'\n"
            "assert 'libmvamg_oracle' in maps\n" % (ROOT, os.path.join(ROOT, "tests")))
    subprocess.run([sys.executable, "-c", code], check=True)


def test_hcache_roundtrip(tmp_path, monkeypatch, c1_fit):
    monkeypatch.setenv("MVAMG_HCACHE", str(tmp_path))
    mats, pros, info = c1_fit
    A, b = mats[0], np.ones(mats[0].shape[0])
    k = hcache.key("c1", A, b, {"p": 1})
    assert k != hcache.key("c1", A, b + 1.0, {"p": 1}) and k != hcache.key("c1", A, b, {"p": 2})
    assert hcache.load(k) is None
    hcache.save(k, mats, pros, info["components"], {"setup": "test"})
    m2, p2, c2, meta = hcache.load(k)
    assert meta["setup"] == "test" and len(c2) == len(info["components"])
    for X, Y in zip(mats + pros, m2 + p2):
        assert (X != Y).nnz == 0 and X.shape == Y.shape
    for (cm, cp), (dm, dp) in zip(info["components"], c2):
        assert len(cm) == len(dm) and all((X != Y).nnz == 0 for X, Y in zip(cm + cp, dm + dp))


def test_kcycle_byte_model_visits():
    """K-cycle byte model: a 4-level hierarchy visits levels
    1, 2 twice / four times and the coarsest as often as level 2."""
    from paper_1907_04417_b200.roofline import abytes, cycle_bytes, kcycle_bytes

    A = sp.csr_matrix(laplacian_2d(8))
    mats = [A, sp.identity(16, format="csr"), sp.identity(8, format="csr"), sp.identity(4, format="csr")]
    pros = [sp.csr_matrix(np.ones((64, 16))), sp.csr_matrix(np.ones((16, 8))), sp.csr_matrix(np.ones((8, 4)))]
    v = [1, 2, 4, 4]
    exp = 0
    for k in range(3):
        nk, nk1, P = mats[k].shape[0], mats[k + 1].shape[0], pros[k]
        exp += v[k] * (2 * abytes(mats[k]) + 12 * P.nnz + 4 * (nk + 1) + 12 * P.nnz + 4 * (nk1 + 1) + 64 * nk + 16 * nk1)
        if k + 1 < 3:
            exp += 2 * v[k] * (abytes(mats[k + 1]) + 80 * nk1)
    exp += v[3] * (8 * 16 + 16 * 4)
    assert kcycle_bytes(mats, pros, 2) == exp
    assert kcycle_bytes(mats, pros, 1) < exp and cycle_bytes(mats, pros) < exp
