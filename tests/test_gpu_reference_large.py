"""Parity at BASELINE configurations C2-C4 pinned to the unmodified reference.

tests/golden/<cfg>_ref.json were made in the build container by running the
reference's own MultiVectorAMG().fit / solve (estimator.py:94-145) on the
repo's generator output (tests/golden/make_golden_large.py; the hierarchies
themselves are far too large to commit, so the records hold digests).  On the
box these tests fit the same matrices with this repo's GPU setup, solve on the
GPU, and require:

  * index work bit-exact: the same level sizes, nnz, and sparsity patterns of
    every A_k and P_k (the aggregates and the kept SVD columns per aggregate);
  * values to rounding: per-level value moments within 1e-9 relative.  The
    values are not bit-identical because the reference's test phase forms its
    dots with OpenBLAS (blocked, FMA, thread-count dependent),
    so its smooth vectors differ from any other implementation's -- and from
    its own run with another OPENBLAS_NUM_THREADS -- in the last bits;
  * the same bootstrap stage count and stage rho within 1e-9;
  * the H1 PCG solve: the reference's iteration count exactly and its residual
    history within 1e-10 relative per iteration (north star).
"""

import json
import os

import numpy as np
import pytest

from _digest import hierarchy_record

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _rel(a, b):
    return max(abs(x - y) / max(abs(y), 1e-300) for x, y in zip(a, b))


@pytest.mark.parametrize("cfg", ["c4", "c3", "c2"])
def test_fit_and_solve_match_reference(cfg):
    from paper_1907_04417_b200 import problems
    from paper_1907_04417_b200.estimator import MultiVectorAMG

    ref = json.load(open(os.path.join(GOLDEN, f"{cfg}_ref.json")))
    A = problems.CONFIGS[cfg]["build"]()
    b = problems.elasticity_rhs(A) if cfg == "c4" else problems.rhs_uniform(A.shape[0], 0)
    est = MultiVectorAMG().fit(A)
    rec = hierarchy_record(list(est.hierarchy_.matrices), list(est.hierarchy_.prolongator_matrices))
    assert rec["levels"] == ref["levels"]
    assert rec["nnz_levels"] == ref["nnz_levels"] and rec["nnz_P"] == ref["nnz_P"]
    assert rec["A_pattern"] == ref["A_pattern"]
    assert rec["P_pattern"] == ref["P_pattern"]
    assert rec["A_sha256"][0] == ref["A_sha256"][0]          # the generator's matrix itself
    for mine, theirs in zip(rec["A_moments"] + rec["P_moments"], ref["A_moments"] + ref["P_moments"]):
        assert _rel(mine, theirs) <= 1e-9
    stages = [float(s.rho) for s in est.composite_.stage_records]
    assert len(stages) == len(ref["stage_rho"])
    assert _rel(stages, ref["stage_rho"]) <= 1e-9
    x, rep = est.solve(b)
    hist, rh = np.asarray(rep.residual_history), np.asarray(ref["residual_history"])
    assert rep.iterations == ref["nit"]
    assert float(np.max(np.abs(hist - rh) / rh)) <= 1e-10
    assert rep.converged and np.linalg.norm(b - A @ x) <= 2e-6 * np.linalg.norm(b)   # true residual
