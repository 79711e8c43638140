"""The CPU oracle (oracle/) pinned against the reference's own outputs.

Golden fixtures come from the unmodified reference (tests/golden/make_golden.py).
Bit-exact for SpMV and GS (verified); tolerance for
anything that passes through np.dot / LAPACK (OpenBLAS is not sequential).
"""

import numpy as np
import pytest

from _fixtures import golden, hierarchy, laplacian_1d
from oracle.oracle import OracleOperator, oracle_composite, oracle_gs, oracle_pcg, oracle_spmv

REL = 1e-12


def rel(a, b):
    return np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300)


@pytest.fixture(scope="module")
def c1():
    d = golden("c1")
    mats, pros = hierarchy(d, "mv")
    return d, mats, pros, OracleOperator(mats, pros)


@pytest.fixture(scope="module")
def comps(c1):
    d, mats, _, _ = c1
    out = []
    for c in range(int(d["n_comp"])):
        m, p = hierarchy(d, f"c{c}", fine=mats[0])
        out.append(OracleOperator(m, p, cycle="K", inner_fcg_iters=2))
    return out


def test_gs_hand_recurrence():
    # pkg/tests/test_cycles.py:30-38
    A = laplacian_1d(3)
    x = np.ones(3)
    oracle_gs(A, np.zeros(3), x, "forward")
    assert np.allclose(x, [0.5, 0.75, 0.375], atol=1e-15)
    x = np.ones(3)
    oracle_gs(A, np.zeros(3), x, "backward")
    assert np.allclose(x, [0.375, 0.75, 0.5], atol=1e-15)


def test_spmv_hand_values():
    # pkg/tests/test_sparse.py:16-18
    assert np.array_equal(oracle_spmv(laplacian_1d(3), np.ones(3)), [1.0, 0.0, 1.0])


def test_spmv_gs_bit_exact(c1):
    d, mats, _, _ = c1
    assert np.array_equal(oracle_spmv(mats[0], d["r1"]), d["spmv_A0_r1"])
    x = np.zeros(mats[0].shape[0])
    oracle_gs(mats[0], d["b"], x, "forward")
    assert np.array_equal(x, d["gsf_A0_b"])
    x = d["x2"].copy()
    oracle_gs(mats[0], d["b"], x, "backward")
    assert np.array_equal(x, d["gsb_A0_b_x2"])


def test_transfer_bit_exact(c1):
    d, mats, pros, _ = c1
    for k, P in enumerate(pros):
        assert np.array_equal(oracle_spmv(P.T.tocsr(), d[f"restrict_in{k}"]), d[f"restrict_out{k}"])
        assert np.array_equal(oracle_spmv(P, d[f"prolong_in{k}"]), d[f"prolong_out{k}"])


def test_vcycle_apply(c1):
    d, _, _, op = c1
    assert rel(op.apply(d["b"]), d["apply_b"]) <= REL
    assert rel(op.apply(d["r1"]), d["apply_r1"]) <= REL
    assert rel(op.error_propagation(d["x2"]), d["errprop_x2"]) <= REL


def test_pcg_history(c1):
    d, _, _, op = c1
    x, hist, nit, conv = oracle_pcg(op, d["b"])
    assert conv and nit == int(d["pcg_nit"])
    assert np.max(np.abs(hist - d["pcg_hist"]) / d["pcg_hist"]) <= 1e-10
    assert rel(x, d["pcg_x"]) <= 1e-10


def test_kcycle_and_composite(c1, comps):
    d = c1[0]
    assert rel(comps[0].apply(d["r3"]), d["kapply_c0_r3"]) <= REL
    assert rel(comps[-1].apply(d["r3"]), d["kapply_c3_r3"]) <= REL
    assert rel(comps[1].error_propagation(d["r3"]), d["kerr_c1_r3"]) <= REL
    assert rel(oracle_composite(comps, d["x4"]), d["comp_x4"]) <= 1e-11


def test_composite_pcg(c1, comps):
    d = c1[0]
    x, hist, nit, conv = oracle_pcg(comps[0], d["b"], "composite", comps)
    assert nit == int(d["h2pcg_nit"])
    assert np.max(np.abs(hist - d["h2pcg_hist"]) / d["h2pcg_hist"]) <= 1e-10


def test_small_cases():
    d = golden("small")
    m, p = hierarchy(d, "lap16")
    assert rel(OracleOperator(m, p).apply(d["lap16_r"]), d["lap16_v"]) <= REL
    assert rel(OracleOperator(m, p, cycle="K", inner_fcg_iters=2).apply(d["lap16_r"]), d["lap16_k2"]) <= REL
    assert rel(OracleOperator(m, p, cycle="K", inner_fcg_iters=1).apply(d["lap16_r"]), d["lap16_k1"]) <= REL
    m, p = hierarchy(d, "ani2")
    op = OracleOperator(m, p)
    assert rel(op.apply(d["ani2_r"]), d["ani2_v"]) <= REL
    assert rel(op.error_propagation(d["ani2_r"]), d["ani2_e"]) <= REL
    _, hist, nit, _ = oracle_pcg(op, np.ones(m[0].shape[0]), rtol=1e-8)
    assert nit == len(d["ani2_pcg_hist"]) - 1
