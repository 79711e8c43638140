"""Hierarchy / vector digests shared by the reference golden generator
(tests/golden/make_golden_large.py, runs the unmodified reference) and the
GPU tests that re-fit the same workloads on the box (tests/test_gpu_reference_large.py).
Fixed dtypes (int64 indices, float64 values) so a digest depends only on the
values, not on scipy's index dtype choice."""

import hashlib

import numpy as np
import scipy.sparse as sp


def csr_digest(M):
    """SHA-256 over (shape, indptr, indices, data)."""
    M = sp.csr_matrix(M)
    h = hashlib.sha256()
    h.update(np.asarray(M.shape, dtype=np.int64).tobytes())
    h.update(np.ascontiguousarray(M.indptr, dtype=np.int64).tobytes())
    h.update(np.ascontiguousarray(M.indices, dtype=np.int64).tobytes())
    h.update(np.ascontiguousarray(M.data, dtype=np.float64).tobytes())
    return h.hexdigest()


def vec_digest(x):
    return hashlib.sha256(np.ascontiguousarray(x, dtype=np.float64).tobytes()).hexdigest()


def diagnostics(mats, pros):
    """Per level: size, nnz, diagonal range, Gershgorin bound, and for the
    prolongators max |P'P - I| and the largest column norm (orthonormality of
    the multi-vector blocks, pkg/src/mvamg/multivector.py:181-212)."""
    out = []
    for k, A in enumerate(mats):
        A = sp.csr_matrix(A)
        d = A.diagonal()
        ent = {"level": k, "n": int(A.shape[0]), "nnz": int(A.nnz), "diag_min": float(d.min()),
               "diag_max": float(d.max()),
               "gershgorin_max": float(np.max(np.asarray(abs(A).sum(axis=1)).ravel()))}
        if k < len(pros):
            P = sp.csr_matrix(pros[k])
            G = (P.T @ P).tocsr() - sp.eye(P.shape[1], format="csr")
            ent["ptp_minus_i_max"] = float(abs(G).max()) if G.nnz else 0.0
            ent["p_col_norm_max"] = float(np.sqrt(np.asarray(P.multiply(P).sum(axis=0)).ravel().max()))
        out.append(ent)
    return out


def coarsest_condition(AL, limit=12000):
    AL = sp.csr_matrix(AL)
    if AL.shape[0] > limit:
        return None
    w = np.linalg.eigvalsh(AL.toarray())
    return {"lambda_min": float(w[0]), "lambda_max": float(w[-1]),
            "cond": float(w[-1] / w[0]) if w[0] > 0 else float("inf"),
            "n_nonpositive": int(np.count_nonzero(w <= 0))}


def pattern_digest(M):
    """SHA-256 over (shape, indptr, indices): the sparsity pattern only (for
    P this is the aggregate structure and the kept count per aggregate)."""
    M = sp.csr_matrix(M)
    h = hashlib.sha256()
    h.update(np.asarray(M.shape, dtype=np.int64).tobytes())
    h.update(np.ascontiguousarray(M.indptr, dtype=np.int64).tobytes())
    h.update(np.ascontiguousarray(M.indices, dtype=np.int64).tobytes())
    return h.hexdigest()


def moments(M):
    """Value moments for a tolerance comparison of two matrices with the same
    pattern: sum |a|, sum a^2, and sum a * cos(k) over the stored entries."""
    d = np.asarray(sp.csr_matrix(M).data, dtype=np.float64)
    k = np.arange(d.shape[0], dtype=np.float64)
    return [float(np.sum(np.abs(d))), float(np.sum(d * d)), float(np.sum(d * np.cos(k)))]


def hierarchy_record(mats, pros):
    """Digests of a multi-vector hierarchy: exact values, patterns, moments."""
    return {"levels": [int(sp.csr_matrix(M).shape[0]) for M in mats],
            "nnz_levels": [int(sp.csr_matrix(M).nnz) for M in mats],
            "nnz_P": [int(sp.csr_matrix(P).nnz) for P in pros],
            "A_sha256": [csr_digest(M) for M in mats],
            "P_sha256": [csr_digest(P) for P in pros],
            "A_pattern": [pattern_digest(M) for M in mats],
            "P_pattern": [pattern_digest(P) for P in pros],
            "A_moments": [moments(M) for M in mats],
            "P_moments": [moments(P) for P in pros]}
