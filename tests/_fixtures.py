"""Shared test inputs: golden fixtures (made by tests/golden/make_golden.py from
the unmodified reference) and small matrix generators restating the reference
test fixtures (pkg/tests/conftest.py:8-29)."""

import os

import numpy as np
import scipy.sparse as sp

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
_cache = {}


def golden(name):
    if name not in _cache:
        _cache[name] = dict(np.load(os.path.join(GOLDEN, name + ".npz")))
    return _cache[name]


def csr(d, key):
    return sp.csr_matrix((d[key + "_data"], d[key + "_indices"], d[key + "_indptr"]),
                         shape=tuple(d[key + "_shape"]))


def hierarchy(d, prefix, fine=None):
    """(matrices, prolongators) stored under prefix (mv / c0.. / lap16 / ani2)."""
    L = int(d[prefix + "_nlev"])
    mats = []
    for k in range(L):
        key = f"{prefix}_A{k}"
        if key + "_data" in d:
            mats.append(csr(d, key))
        else:
            mats.append(fine)
    pros = [csr(d, f"{prefix}_P{k}") for k in range(L - 1)]
    return mats, pros


def c1_fine():
    d = golden("c1")
    return csr(d, "mv_A0")


def laplacian_1d(n):
    return sp.diags([-np.ones(n - 1), 2 * np.ones(n), -np.ones(n - 1)], [-1, 0, 1]).tocsr()


def laplacian_2d(grid):
    T = laplacian_1d(grid)
    eye = sp.eye(grid, format="csr")
    return (sp.kron(eye, T) + sp.kron(T, eye)).tocsr()


def laplacian_3d(g):
    T = laplacian_1d(g)
    I = sp.eye(g, format="csr")
    return (sp.kron(sp.kron(I, I), T) + sp.kron(sp.kron(I, T), I) + sp.kron(sp.kron(T, I), I)).tocsr()


def random_spd_csr(n, density=0.2, seed=0):
    """Symmetric random pattern made diagonally dominant (SPD)."""
    rng = np.random.default_rng(seed)
    R = sp.random(n, n, density=density, random_state=rng, data_rvs=lambda k: rng.uniform(-1, 1, k))
    S = (R + R.T).tocsr()
    S.setdiag(0.0)
    S.eliminate_zeros()
    row_abs = np.asarray(abs(S).sum(axis=1)).ravel()
    return (S + sp.diags(row_abs + 1.0)).tocsr()
