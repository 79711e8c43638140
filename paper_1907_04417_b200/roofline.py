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
    """One GS sweep: A once, b, diag, x_new (+ x_old unless zero-init)."""
    n = A.shape[0]
    return abytes(A) + 8 * n * (3 if zero_init else 4)


def measured_peak_gbs(repo_root):
    """(hbm GB/s, source) from MEASURED_PEAKS.json, else the recipe's fallback."""
    path = os.path.join(repo_root, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"
