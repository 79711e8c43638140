"""GPU: the device Galerkin product (csrc/galerkin.cuh, mvamg_galerkin_f64)
bit for bit against the reference's coarse matrices, the CPU oracle and the
reference's scipy call (pkg/src/mvamg/sparse.py:50-66)."""

import numpy as np
import pytest
import scipy.sparse as sp

from _galerkin_cases import aggregation_case, edge_cases, golden_levels, overflow_case
from oracle.oracle import oracle_galerkin
from paper_1907_04417_b200 import problems
from paper_1907_04417_b200.device import galerkin_product_device
from paper_1907_04417_b200.setup import galerkin_product

pytestmark = pytest.mark.gpu


def same_csr(A, B):
    return (A.shape == B.shape and np.array_equal(A.indptr, B.indptr) and np.array_equal(A.indices, B.indices)
            and np.array_equal(A.data.view(np.int64), B.data.view(np.int64)))


def test_galerkin_golden_hierarchies():
    checked = 0
    for name, P, A, want in golden_levels():
        G = galerkin_product_device(P, A)
        assert same_csr(G, oracle_galerkin(P, A)), name
        if want is not None:
            assert same_csr(G, want), name
            checked += 1
    assert checked == 12


@pytest.mark.parametrize("case", edge_cases(), ids=lambda c: c[0])
def test_galerkin_edge_cases(case):
    _, P, A = case
    assert same_csr(galerkin_product_device(P, A), oracle_galerkin(P, A))


def test_galerkin_overflow_rows():
    # row 0 has 1500 distinct columns: the global-memory table path
    P, A = overflow_case()
    assert same_csr(galerkin_product_device(P, A), galerkin_product(P, A))


def test_galerkin_dimension_mismatch():
    with pytest.raises(ValueError):
        galerkin_product_device(sp.eye(4, format="csr"), sp.eye(5, format="csr"))


def test_galerkin_setup_levels():
    # multi-vector-shaped block prolongators (2-5 nnz/row) and a pairwise one
    for P, A in (aggregation_case(), aggregation_case(grid=96, agg=8, nsv=5, seed=2)):
        assert same_csr(galerkin_product_device(P, A), galerkin_product(P, A))


def test_galerkin_full_size_c2():
    # C2's fine operator (Q1 anisotropic 1024^2, n = 1,048,576) with an
    # 8x8-aggregate, 5-vector block prolongator: 9.4M + 5.2M nonzeros in
    A = problems.anisotropic_q1(1024)
    g = 1024
    rng = np.random.default_rng(0)
    n = g * g
    ii, jj = np.divmod(np.arange(n), g)
    aid = (ii // 8) * (g // 8) + jj // 8
    nsv = 5
    P = sp.csr_matrix((rng.standard_normal(n * nsv), (np.repeat(np.arange(n), nsv),
                                                      (aid[:, None] * nsv + np.arange(nsv)).ravel())),
                      shape=(n, (g // 8) ** 2 * nsv))
    t = {}
    G = galerkin_product_device(P, A, timing=t)
    assert same_csr(G, galerkin_product(P, A))
    assert t["total_ms"] > 0


def _host_matching(A, w):
    from paper_1907_04417_b200.setup import edge_weights, greedy_matching

    i, j, c = edge_weights(A, w)
    return greedy_matching(i, j, c, A.shape[0])


def test_device_matching_equals_greedy():
    """The GPU locally dominant matching gives the reference greedy's pairs, in
    its acceptance order, and its unmatched set (matching.py:78-122), on the
    golden hierarchies' levels with smooth vectors, random weights, ties
    (constant weights on a uniform grid) and C2's fine operator."""
    from _fixtures import laplacian_2d
    from paper_1907_04417_b200.setup import greedy_matching_device

    rng = np.random.default_rng(5)
    cases = []
    for name, P, A, _ in golden_levels():
        cases.append((name, A, rng.uniform(0.5, 1.5, A.shape[0])))
    cases.append(("lap2d_ties", laplacian_2d(40), np.ones(1600)))
    cases.append(("q1_smooth", problems.anisotropic_q1(64), np.cos(np.arange(64 * 64) / 300.0)))
    cases.append(("c2_fine", problems.anisotropic_q1(1024), rng.standard_normal(1024 * 1024)))
    for name, A, w in cases:
        A = sp.csr_matrix(A)
        p_h, u_h = _host_matching(A, w)
        p_d, u_d = greedy_matching_device(A, w)
        assert np.array_equal(p_h, p_d), name
        assert np.array_equal(u_h, u_d), name


def test_fit_with_device_matching_is_identical():
    """A whole fit with the device matching gives the same hierarchy as with
    the host greedy (elasticity 64^2: four bootstrap stages)."""
    import paper_1907_04417_b200 as mv

    A = problems.elasticity_q1(64)
    e1 = mv.MultiVectorAMG(config=mv.GpuConfig(device_matching=True)).fit(A)
    e0 = mv.MultiVectorAMG(config=mv.GpuConfig(device_matching=False)).fit(A)
    for M0, M1 in zip(e0.hierarchy_.matrices, e1.hierarchy_.matrices):
        assert same_csr(M0, M1)
    assert len(e0.hierarchy_.matrices) == len(e1.hierarchy_.matrices)
