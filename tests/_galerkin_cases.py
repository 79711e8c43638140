"""Galerkin-product test operands (shared by the CPU oracle pin and the GPU
parity tests): the reference's own hierarchies, hand edge cases, exact-zero
cancellations and the overflow (long-row) path."""

import numpy as np
import scipy.sparse as sp

from _fixtures import golden, hierarchy, laplacian_1d, laplacian_2d, random_spd_csr

# levels whose stored A_{k+1} the reference formed as galerkin_product(P_k, A_k)
# (pkg/src/mvamg/multivector.py:307, pairwise.py:206; the double-pairwise levels
# of the other components compose two products and are checked op-by-op only)
GOLDEN_DIRECT = [("c1", "mv", [0, 1, 2]), ("c1", "c0", [0, 1, 2, 3, 4]), ("small", "lap16", [0, 1, 2]),
                 ("small", "ani2", [2])]


def golden_levels():
    """(name, P_k, A_k, A_{k+1} or None) over every stored hierarchy level."""
    out = []
    d1 = golden("c1")
    fine = hierarchy(d1, "mv")[0][0]
    direct = {(f, p): ks for f, p, ks in GOLDEN_DIRECT}
    for f, prefs in (("c1", ["mv", "c0", "c1", "c2", "c3"]), ("small", ["lap16", "ani2"])):
        d = golden(f)
        for p in prefs:
            mats, pros = hierarchy(d, p, fine=fine if f == "c1" else None)
            for k in range(len(pros)):
                want = mats[k + 1] if k in direct.get((f, p), []) else None
                out.append((f"{f}/{p}/{k}", pros[k], mats[k], want))
    return out


def cancellation_case(seed=0, n=60, nc=12):
    """Small-integer operands so that A P and P'A P hit exact zeros (dropped)."""
    rng = np.random.default_rng(seed)
    A = sp.random(n, n, density=0.15, random_state=rng, data_rvs=lambda k: rng.integers(-2, 3, k).astype(float))
    A = (A + A.T).tocsr()
    A.setdiag(4.0)
    A.eliminate_zeros()
    P = sp.random(n, nc, density=0.25, random_state=rng, data_rvs=lambda k: rng.choice([-1.0, 1.0, 0.5], k))
    return P.tocsr(), A.tocsr()


def edge_cases():
    out = []
    A = laplacian_1d(7)
    out.append(("empty_P", sp.csr_matrix((7, 3)), A))                       # all-zero prolongator
    Pz = sp.csr_matrix(np.array([[1.0, 0], [1, 0], [0, 0], [0, 1], [0, 1], [0, 0], [0, 0]]))
    out.append(("zero_rows", Pz, A))                                          # rows outside every aggregate
    out.append(("one_coarse", sp.csr_matrix(np.ones((7, 1))), A))
    out.append(("identity", sp.eye(7, format="csr"), A))
    out.append(("1x1", sp.csr_matrix(np.array([[2.0]])), sp.csr_matrix(np.array([[3.0]]))))
    # a coarse column no fine row touches (an empty row of P^T and of G)
    out.append(("empty_col", sp.csr_matrix(np.array([[1.0, 0, 0], [0.5, 0, 1], [0, 0, 1], [0, 0, 2],
                                                     [1, 0, 0], [0, 0, 1], [1, 0, 0]])), A))
    # exact cancellations: G = P'(A P) has exact-zero off-diagonals, and A P an
    # exact-zero column (both dropped by csr_matmat)
    out.append(("cancel_G", sp.csr_matrix(np.array([[1.0, 1.0], [1.0, -1.0]])),
                sp.csr_matrix(np.array([[2.0, 1.0], [1.0, 2.0]]))))
    out.append(("cancel_AP", sp.csr_matrix(np.array([[1.0, 0.0], [1.0, 0.0], [0.0, 1.0]])),
                sp.csr_matrix(np.array([[1.0, -1.0, 0.0], [-1.0, 1.0, 0.0], [0.0, 0.0, 2.0]]))))
    for s in range(3):
        out.append((f"cancel{s}", *cancellation_case(s)))
    out.append(("random_spd", sp.random(80, 9, density=0.3, random_state=5, format="csr"), random_spd_csr(80, 0.1, 3)))
    return out


def overflow_case(n=1500):
    """A star (row 0 couples to everyone) with P = I: row 0 of A P and of P'A P
    has n distinct columns -- past the shared-memory table, onto the global one."""
    r = np.concatenate([np.zeros(n - 1, int), np.arange(1, n)])
    c = np.concatenate([np.arange(1, n), np.zeros(n - 1, int)])
    A = sp.csr_matrix((np.full(2 * (n - 1), -1.0), (r, c)), shape=(n, n)) + sp.diags(np.full(n, float(n)))
    rng = np.random.default_rng(7)
    P = sp.diags(rng.uniform(0.5, 1.5, n)).tocsr()
    return P.tocsr(), A.tocsr()


def aggregation_case(grid=64, agg=4, nsv=3, seed=1):
    """Multi-vector-shaped P on a 2D Laplacian: agg x agg aggregates, nsv random
    columns each (2-5 nnz per row, like the reference's block prolongators)."""
    rng = np.random.default_rng(seed)
    A = laplacian_2d(grid)
    n = grid * grid
    ii, jj = np.divmod(np.arange(n), grid)
    aid = (ii // agg) * (grid // agg) + jj // agg
    rows = np.repeat(np.arange(n), nsv)
    cols = (aid[:, None] * nsv + np.arange(nsv)[None, :]).ravel()
    P = sp.csr_matrix((rng.standard_normal(n * nsv), (rows, cols)), shape=(n, (grid // agg) ** 2 * nsv))
    return P, A
