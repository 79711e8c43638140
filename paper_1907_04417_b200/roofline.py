"""Algorithmic byte model of the solve path and roofline helpers.

int32 indices, fp64 values; Abytes(M) = 12 nnz(M) + 4 (rows(M) + 1).
  B_cycle = sum_{k<L} [ 2 Abytes(A_k) + (12 nnz(P_k) + 4 (n_k+1)) + (12 nnz(P_k) + 4 (n_{k+1}+1))
                        + 64 n_k + 16 n_{k+1} ] + 8 n_L^2 + 16 n_L
  B_pcg   = B_cycle + Abytes(A_0) + 80 n_0
These count each operand once per use (what an ideal fused implementation must
move); kernels that re-read more show up as traffic above the model in ncu.
"""

import json
import os


def abytes(M):
    return 12 * M.nnz + 4 * (M.shape[0] + 1)


def cycle_bytes(matrices, prolongators):
    L = len(matrices)
    B = 0
    for k in range(L - 1):
        A, P = matrices[k], prolongators[k]
        nk, nk1 = A.shape[0], matrices[k + 1].shape[0]
        B += 2 * abytes(A) + (12 * P.nnz + 4 * (nk + 1)) + (12 * P.nnz + 4 * (nk1 + 1))
        B += 64 * nk + 16 * nk1
    nL = matrices[-1].shape[0]
    return B + 8 * nL * nL + 16 * nL


def pcg_iteration_bytes(matrices, prolongators):
    A0 = matrices[0]
    return cycle_bytes(matrices, prolongators) + abytes(A0) + 80 * A0.shape[0]


def gs_sweep_bytes(A, zero_init):
    """One GS sweep.  From x = 0 (forward pre-smoothing) only the lower
    triangle and the diagonal are read (the upper neighbours are still zero):
    12 nnz(L+D) + 4 (n+1) + b, diag, x_new.  From x_old: all of A + b, diag,
    x_old, x_new."""
    n = A.shape[0]
    if zero_init:
        import scipy.sparse as sp

        nnz_ld = int(sp.tril(A).nnz)
        return 12 * nnz_ld + 4 * (n + 1) + 8 * n * 3
    return abytes(A) + 8 * n * 4


def kcycle_bytes(matrices, prolongators, inner=2):
    """SURVEY.md 8(d) composite model: one K-cycle application.  Level k is
    visited v_k times (v_0 = 1; v_{k+1} = inner * v_k where level k+1 runs an
    inner FCG, i.e. k + 1 < L - 1, else v_k); each visit costs the V-cycle's
    per-level terms, each inner FCG step Abytes(A_{k+1}) + 80 n_{k+1}
    (cycles.py:157-167, krylov.py:75-107)."""
    L = len(matrices)
    v = [1] * L
    for k in range(L - 1):
        v[k + 1] = inner * v[k] if k + 1 < L - 1 else v[k]
    B = 0
    for k in range(L - 1):
        A, P = matrices[k], prolongators[k]
        nk, nk1 = A.shape[0], matrices[k + 1].shape[0]
        per = 2 * abytes(A) + (12 * P.nnz + 4 * (nk + 1)) + (12 * P.nnz + 4 * (nk1 + 1)) + 64 * nk + 16 * nk1
        B += v[k] * per
        if k + 1 < L - 1:
            B += inner * v[k] * (abytes(matrices[k + 1]) + 80 * nk1)
    nL = matrices[-1].shape[0]
    return B + v[L - 1] * (8 * nL * nL + 16 * nL)


def composite_application_bytes(components, inner=2):
    """B_H2 = sum_i 2 (Abytes(A_0) + 16 n_0 + B_Kcycle(i)) per symmetrized
    application (bootstrap.py:98-113; as a preconditioner the residual update
    replaces the error update, same traffic)."""
    B = 0
    for mats, pros in components:
        A0 = mats[0]
        B += 2 * (abytes(A0) + 16 * A0.shape[0] + kcycle_bytes(mats, pros, inner))
    return B


def measured_peak_gbs(repo_root):
    """(hbm GB/s, source) from MEASURED_PEAKS.json, else the recipe's fallback."""
    path = os.path.join(repo_root, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"
