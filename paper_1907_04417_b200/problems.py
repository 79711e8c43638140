"""Synthetic SPD test problems for the benchmark configurations (BASELINE.json).

The reference ships only P1 anisotropic diffusion on structured triangles
(pkg/src/mvamg/problems.py:41-94); configurations 2-5 name Q1, 3D
jumping-coefficient and plane-strain elasticity problems that it does not
generate.  These generators are written fresh, vectorised with
numpy/scipy, and return canonical float64 CSR matrices with exactly symmetric
stored values and a positive diagonal (the checks of
pkg/src/mvamg/validation.py:10-26).

    C1  poisson_2d(128)                          5-point Laplacian, n = 16,384
    C2  anisotropic_q1(1024, 1e-3, pi/6)         Q1 bilinear 9-point, n = 1,048,576
    C3  jump_3d(128, block=16, seed=1)           7-point FV, 10^k coefficients, n = 2,097,152
    C4  elasticity_q1(512, E=1, nu=0.45)         plane strain, 2 dofs/node, n = 525,312
    C5  jump_3d(320, block=16, seed=1)           n = 32,768,000
Right-hand sides follow the reference's RNG idiom
(np.random.default_rng(seed).uniform(-1, 1, n), pkg/src/mvamg/bootstrap.py:127).
"""

import numpy as np
import scipy.sparse as sp

from .device import as_csr


def _finish(A):
    A = sp.csr_matrix(A)
    A = ((A + A.T) * 0.5).tocsr()  # exact stored-value symmetry
    A.eliminate_zeros()
    return as_csr(A)


def poisson_2d(g):
    """5-point Laplacian on a g x g interior grid (4 on the diagonal, -1 off),
    identical to the reference's P1 stiffness for K = I."""
    T = sp.diags([-np.ones(g - 1), 2.0 * np.ones(g), -np.ones(g - 1)], [-1, 0, 1], format="csr")
    eye = sp.eye(g, format="csr")
    return as_csr((sp.kron(eye, T) + sp.kron(T, eye)).tocsr())


def anisotropy_tensor(eps, theta):
    c, s = np.cos(theta), np.sin(theta)
    return np.array([[eps + c * c, c * s], [c * s, eps + s * s]])


def _q1_element(K):
    """4x4 bilinear element stiffness on a square cell for constant tensor K
    (2x2 Gauss quadrature, exact for Q1); scale invariant in 2D.  Local node
    order (0,0), (1,0), (1,1), (0,1)."""
    g = 1.0 / np.sqrt(3.0)
    pts = [(0.5 - 0.5 * g, 0.5 - 0.5 * g), (0.5 + 0.5 * g, 0.5 - 0.5 * g),
           (0.5 + 0.5 * g, 0.5 + 0.5 * g), (0.5 - 0.5 * g, 0.5 + 0.5 * g)]
    Ke = np.zeros((4, 4))
    for (x, y) in pts:
        # gradients of (1-x)(1-y), x(1-y), xy, (1-x)y
        G = np.array([[-(1 - y), -(1 - x)], [(1 - y), -x], [y, x], [-y, (1 - x)]])
        Ke += 0.25 * G @ K @ G.T
    return 0.5 * (Ke + Ke.T)


def _assemble_cells(g, Ke, dofs_per_node=1):
    """Assemble a cell-constant element matrix on a (g+1) x (g+1) cell grid of
    (g+2)^2 nodes and eliminate the Dirichlet boundary (all four sides).  Dof
    of interior node (i, j): ((j-1) g + (i-1)) * dofs_per_node + c."""
    N = g + 2
    ci, cj = np.meshgrid(np.arange(N - 1), np.arange(N - 1), indexing="ij")
    ci, cj = ci.ravel(), cj.ravel()
    nodes = np.stack([cj * N + ci, cj * N + ci + 1, (cj + 1) * N + ci + 1, (cj + 1) * N + ci])  # 4 x ncell
    m = dofs_per_node
    ldofs = (nodes[:, None, :] * m + np.arange(m)[None, :, None]).reshape(4 * m, -1)  # local order node-major
    rows = np.repeat(ldofs, 4 * m, axis=0).ravel()
    cols = np.tile(ldofs, (4 * m, 1)).ravel()
    vals = np.repeat(Ke.ravel(), ldofs.shape[1])
    A = sp.coo_matrix((vals, (rows, cols)), shape=(N * N * m, N * N * m)).tocsr()
    ii, jj = np.meshgrid(np.arange(1, g + 1), np.arange(1, g + 1), indexing="xy")
    interior_nodes = (jj.ravel() * N + ii.ravel()).astype(np.int64)
    keep = (interior_nodes[:, None] * m + np.arange(m)[None, :]).ravel()
    return A[keep][:, keep]


def anisotropic_q1(g, eps=1e-3, theta=np.pi / 6):
    """C2: Q1 bilinear FEM for -div(K grad u) on g x g interior nodes, K the
    rotated anisotropy tensor of pkg/src/mvamg/problems.py:20-38."""
    return _finish(_assemble_cells(g, _q1_element(anisotropy_tensor(eps, theta))))


def jump_coefficients(g, block=16, seed=1, kmin=-3, kmax=3):
    """Cell coefficients 10^k, k uniform in {kmin..kmax} per block^3 block."""
    nb = -(-g // block)
    rng = np.random.default_rng(seed)
    kb = rng.integers(kmin, kmax + 1, size=(nb, nb, nb))
    idx = np.arange(g) // block
    k = kb[idx[:, None, None], idx[None, :, None], idx[None, None, :]]
    return 10.0 ** k.astype(np.float64)  # indexed [z, y, x]


def jump_3d(g, block=16, seed=1):
    """C3 / C5: 7-point cell-centred finite volumes on a g^3 grid, piecewise
    constant coefficient, harmonic-mean face coefficients, Dirichlet (the
    boundary face uses the cell's own coefficient at half distance).  Natural
    lexicographic ordering x fastest; n = g^3."""
    c = jump_coefficients(g, block, seed)
    n = g ** 3
    lin = np.arange(n).reshape(g, g, g)
    diag = np.zeros((g, g, g))
    rows, cols, vals = [], [], []
    for axis in range(3):
        a = np.moveaxis(c, axis, 0)
        li = np.moveaxis(lin, axis, 0)
        h = 2.0 * a[:-1] * a[1:] / (a[:-1] + a[1:])  # harmonic mean on interior faces
        rows += [li[:-1].ravel(), li[1:].ravel()]
        cols += [li[1:].ravel(), li[:-1].ravel()]
        vals += [-h.ravel(), -h.ravel()]
        d = np.zeros_like(a)
        d[:-1] += h
        d[1:] += h
        d[0] += 2.0 * a[0]   # Dirichlet faces
        d[-1] += 2.0 * a[-1]
        diag += np.moveaxis(d, 0, axis)
    rows.append(lin.ravel())
    cols.append(lin.ravel())
    vals.append(diag.ravel())
    A = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                      shape=(n, n)).tocsr()
    return _finish(A)


def _q1_elasticity_element(E=1.0, nu=0.45):
    """8x8 bilinear plane-strain element stiffness on a unit square (2x2
    Gauss); dof order (u, v) per local node (0,0), (1,0), (1,1), (0,1)."""
    lam = E * nu / ((1 + nu) * (1 - 2 * nu))
    mu = E / (2 * (1 + nu))
    Dm = np.array([[lam + 2 * mu, lam, 0.0], [lam, lam + 2 * mu, 0.0], [0.0, 0.0, mu]])
    g = 1.0 / np.sqrt(3.0)
    pts = [(0.5 - 0.5 * g, 0.5 - 0.5 * g), (0.5 + 0.5 * g, 0.5 - 0.5 * g),
           (0.5 + 0.5 * g, 0.5 + 0.5 * g), (0.5 - 0.5 * g, 0.5 + 0.5 * g)]
    Ke = np.zeros((8, 8))
    for (x, y) in pts:
        G = np.array([[-(1 - y), -(1 - x)], [(1 - y), -x], [y, x], [-y, (1 - x)]])
        B = np.zeros((3, 8))
        B[0, 0::2] = G[:, 0]
        B[1, 1::2] = G[:, 1]
        B[2, 0::2] = G[:, 1]
        B[2, 1::2] = G[:, 0]
        Ke += 0.25 * B.T @ Dm @ B
    return 0.5 * (Ke + Ke.T)


def elasticity_q1(ne=512, E=1.0, nu=0.45):
    """C4: Q1 plane-strain elasticity on ne x ne elements of the unit square,
    clamped on the left edge (x = 0), all other edges free; 2 dofs per node
    interleaved (u, v).  n = 2 ne (ne + 1)."""
    Ke = _q1_elasticity_element(E, nu)
    N = ne + 1  # nodes per side
    ci, cj = np.meshgrid(np.arange(ne), np.arange(ne), indexing="ij")
    ci, cj = ci.ravel(), cj.ravel()
    nodes = np.stack([cj * N + ci, cj * N + ci + 1, (cj + 1) * N + ci + 1, (cj + 1) * N + ci])
    ldofs = (nodes[:, None, :] * 2 + np.arange(2)[None, :, None]).reshape(8, -1)
    rows = np.repeat(ldofs, 8, axis=0).ravel()
    cols = np.tile(ldofs, (8, 1)).ravel()
    vals = np.repeat(Ke.ravel(), ldofs.shape[1])
    A = sp.coo_matrix((vals, (rows, cols)), shape=(2 * N * N, 2 * N * N)).tocsr()
    xi = np.tile(np.arange(N), N)
    keep_nodes = np.flatnonzero(xi > 0)  # clamp x = 0
    keep = (keep_nodes[:, None] * 2 + np.arange(2)[None, :]).ravel()
    return _finish(A[keep][:, keep])


def elasticity_rhs(A, seed=0, noise=0.1):
    """Uniform downward body load plus seeded noise (config 4)."""
    n = A.shape[0]
    b = np.zeros(n)
    b[1::2] = -1.0 / n
    return b + noise / n * np.random.default_rng(seed).uniform(-1.0, 1.0, n)


def rhs_uniform(n, seed=0):
    """Reference RNG idiom: default_rng(seed).uniform(-1, 1, n)."""
    return np.random.default_rng(seed).uniform(-1.0, 1.0, n)


CONFIGS = {
    "c1": dict(build=lambda: poisson_2d(128), desc="C1: 2D Poisson 5-point, 128x128 interior (n=16,384)"),
    "c2": dict(build=lambda: anisotropic_q1(1024, 1e-3, np.pi / 6),
               desc="C2: 2D rotated anisotropic diffusion, Q1 9-point, 1024x1024 (n=1,048,576), eps=1e-3, theta=pi/6"),
    "c3": dict(build=lambda: jump_3d(128, 16, 1),
               desc="C3: 3D 7-point FV, 128^3 (n=2,097,152), 10^k per 16^3 block, harmonic faces"),
    "c4": dict(build=lambda: elasticity_q1(512, 1.0, 0.45),
               desc="C4: 2D Q1 plane-strain elasticity, 512x512 elements (n=525,312), E=1, nu=0.45, clamped left edge"),
    "c5": dict(build=lambda: jump_3d(320, 16, 1),
               desc="C5: 3D 7-point FV, 320^3 (n=32,768,000), jumping coefficients"),
}
