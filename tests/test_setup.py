"""Host setup restatement against the reference's own hierarchies (golden
fixtures from the unmodified reference, tests/golden/make_golden.py)."""

import numpy as np
import pytest
import scipy.sparse as sp

from _fixtures import golden, hierarchy, laplacian_2d
from paper_1907_04417_b200 import problems
from paper_1907_04417_b200.setup import (CoarseningParams, build_multivector_hierarchy,
                                         build_pairwise_hierarchy, edge_weights, galerkin_product,
                                         greedy_matching)


def same_csr(A, B):
    A, B = sp.csr_matrix(A), sp.csr_matrix(B)
    return (A.shape == B.shape and np.array_equal(A.indptr, B.indptr) and np.array_equal(A.indices, B.indices)
            and np.array_equal(A.data, B.data))


def test_matching_hand_example():
    # weight of a 2x2 block [[2, -1], [-1, 2]] with w = 1 is 1 - 2(-1)/(2+2) = 1.5
    A = sp.csr_matrix(np.array([[2.0, -1.0], [-1.0, 2.0]]))
    i, j, c = edge_weights(A, np.ones(2))
    assert c.tolist() == [1.5]
    pairs, unmatched = greedy_matching(i, j, c, 2)
    assert pairs.tolist() == [[0, 1]] and unmatched.size == 0


@pytest.mark.parametrize("name,mcs", [("lap16", 8), ("ani2", 40)])
def test_pairwise_hierarchy_bit_exact(name, mcs):
    d = golden("small")
    mats, pros = hierarchy(d, name)
    h = build_pairwise_hierarchy(mats[0], np.ones(mats[0].shape[0]), CoarseningParams(min_coarse_size=mcs))
    assert h.nl == len(mats)
    for k in range(1, h.nl):
        assert same_csr(h.matrices[k], mats[k]), k
        assert same_csr(h.prolongators[k - 1], pros[k - 1]), k


def test_c1_component_and_multivector_hierarchy_bit_exact():
    d = golden("c1")
    mv_mats, mv_pros = hierarchy(d, "mv")
    A = mv_mats[0]
    vecs = list(d["smooth_vectors"])
    # component 4 of the bootstrap was built from smooth vector 4 (index 3)
    c_mats, c_pros = hierarchy(d, "c3", fine=A)
    h = build_pairwise_hierarchy(A, vecs[3])
    assert h.nl == len(c_mats)
    for k in range(1, h.nl):
        assert same_csr(h.matrices[k], c_mats[k]), k
        assert same_csr(h.prolongators[k - 1], c_pros[k - 1]), k
    mvh = build_multivector_hierarchy(A, h, vecs[:5])
    assert mvh.sizes() == [M.shape[0] for M in mv_mats]
    for k in range(1, mvh.nl):
        assert same_csr(mvh.prolongator_matrices[k - 1], mv_pros[k - 1]), k
        assert same_csr(mvh.matrices[k], mv_mats[k]), k


def test_galerkin_matches_dense():
    rng = np.random.default_rng(3)
    A = laplacian_2d(6)
    P = sp.csr_matrix(rng.standard_normal((36, 7)) * (rng.random((36, 7)) < 0.3))
    G = galerkin_product(P, A).toarray()
    ref = P.T.toarray() @ A.toarray() @ P.toarray()
    assert np.max(np.abs(G - ref)) <= 1e-13 * np.max(np.abs(ref))
    assert (galerkin_product(P, A) != galerkin_product(P, A).T).nnz == 0


def test_generators_valid():
    for A in (problems.poisson_2d(8), problems.anisotropic_q1(12), problems.jump_3d(8, 4, 1),
              problems.elasticity_q1(6)):
        assert (A != A.T).nnz == 0
        assert np.all(A.diagonal() > 0)
        assert np.linalg.eigvalsh(A.toarray()).min() > 0
    assert (problems.poisson_2d(128) != hierarchy(golden("c1"), "mv")[0][0]).nnz == 0
