"""CPU: the oracle's Galerkin restatement (oracle/mvamg_oracle.c or_galerkin)
pinned against the reference's own coarse matrices (golden fixtures) and the
reference's call itself (scipy, pkg/src/mvamg/sparse.py:50-66)."""

import numpy as np
import pytest

from _galerkin_cases import aggregation_case, edge_cases, golden_levels, overflow_case
from oracle.oracle import oracle_galerkin
from paper_1907_04417_b200.setup import galerkin_product


def same_csr(A, B):
    return (A.shape == B.shape and np.array_equal(A.indptr, B.indptr) and np.array_equal(A.indices, B.indices)
            and np.array_equal(A.data.view(np.int64), B.data.view(np.int64)))


def test_oracle_galerkin_golden():
    checked = 0
    for name, P, A, want in golden_levels():
        G = oracle_galerkin(P, A)
        assert same_csr(G, galerkin_product(P, A)), name
        if want is not None:
            assert same_csr(G, want), name
            checked += 1
    assert checked == 12


@pytest.mark.parametrize("case", edge_cases(), ids=lambda c: c[0])
def test_oracle_galerkin_edge_cases(case):
    _, P, A = case
    assert same_csr(oracle_galerkin(P, A), galerkin_product(P, A))


def test_oracle_galerkin_drops_exact_zeros():
    cases = dict((c[0], c[1:]) for c in edge_cases())
    G = oracle_galerkin(*cases["cancel_G"])       # [[6, 0], [0, 2]]: the zero is not stored
    assert G.nnz == 2 and G.toarray().tolist() == [[6.0, 0.0], [0.0, 2.0]]
    G = oracle_galerkin(*cases["cancel_AP"])      # A P has an exact-zero column 0
    assert G.toarray().tolist() == [[0.0, 0.0], [0.0, 2.0]] and G.nnz == 1


def test_oracle_galerkin_overflow_and_aggregation():
    for P, A in (overflow_case(), aggregation_case()):
        assert same_csr(oracle_galerkin(P, A), galerkin_product(P, A))
