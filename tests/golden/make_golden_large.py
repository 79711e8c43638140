"""Reference-pinned goldens for the BASELINE configurations C2-C4 (and the
3D jump family used to study C5), made by running the UNMODIFIED reference
(``mvamg`` from /root/reference/pkg/src) in this container:

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden_large.py c3 [--save DIR]

For config ``cfg`` it builds the repo's generator output (problems.CONFIGS /
problems.jump_3d -- the reference has no C2-C5 generators), runs
``MultiVectorAMG().fit(A)`` (estimator.py:94-136) and ``solve(b)``
(estimator.py:138-145) with the reference's defaults, and writes
``tests/golden/<cfg>_ref.json``: SHA-256 of every level's A_k and P_k (CSR
arrays normalised to int64 indptr/indices, float64 data), sizes, nnz, the PCG
iteration count, the residual history, a digest of x, the reference's fit
and solve seconds on one core, and diagnostics (max diagonal per level,
max |P_k'P_k - I|, condition of the coarsest level).  The hierarchies are far
too large to commit; ``--save DIR`` keeps them as npz for offline study.
"""

import argparse
import json
import os
import sys
import time

import numpy as np
import scipy.sparse as sp

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.environ.get("MVAMG_REF", "/root/reference/pkg/src"))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

from mvamg.estimator import MultiVectorAMG  # noqa: E402

from _digest import coarsest_condition, csr_digest, diagnostics, hierarchy_record, vec_digest  # noqa: E402

from paper_1907_04417_b200 import problems  # noqa: E402


def workload(cfg):
    """(A, b, description) exactly as bench.py / the GPU tests build them."""
    if cfg in problems.CONFIGS:
        A = problems.CONFIGS[cfg]["build"]()
        b = problems.elasticity_rhs(A) if cfg == "c4" else problems.rhs_uniform(A.shape[0], 0)
        return A, b, problems.CONFIGS[cfg]["desc"]
    if cfg.startswith("j"):  # jNNN: 3D jump coefficient on NNN^3 (the C3/C5 family)
        g = int(cfg[1:])
        A = problems.jump_3d(g, 16, 1)
        return A, problems.rhs_uniform(A.shape[0], 0), f"3D jump 7-point FV {g}^3 (C3/C5 family)"
    raise SystemExit(f"unknown config {cfg!r}")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cfg")
    ap.add_argument("--save", default=None, help="directory for the full hierarchy (npz)")
    ap.add_argument("--no-solve", action="store_true")
    args = ap.parse_args()
    cfg = args.cfg.lower()
    A, b, desc = workload(cfg)
    rec = {"config": cfg, "workload": desc, "n": int(A.shape[0]), "nnz": int(A.nnz),
           "A_digest": csr_digest(A), "b_digest": vec_digest(b),
           "reference": "mvamg (unmodified, /root/reference/pkg/src) MultiVectorAMG() defaults",
           "host": {"cpu_count": os.cpu_count(), "openblas_threads": os.environ.get("OPENBLAS_NUM_THREADS")}}
    t0 = time.perf_counter()
    est = MultiVectorAMG().fit(A)
    rec["fit_s"] = time.perf_counter() - t0
    print(f"[{cfg}] fit {rec['fit_s']:.1f} s", flush=True)
    mats = list(est.hierarchy_.matrices)
    pros = list(est.hierarchy_.prolongator_matrices)
    rec.update(hierarchy_record(mats, pros))
    rec["bootstrap_stages"] = int(est.composite_.n_components) if est.composite_ is not None else 0
    rec["stage_rho"] = [float(s.rho) for s in est.composite_.stage_records] if est.composite_ is not None else []
    rec["smooth_vector_sha256"] = [vec_digest(v) for v in est.smooth_vectors_]
    rec["diagnostics"] = diagnostics(mats, pros)
    if args.save:
        os.makedirs(args.save, exist_ok=True)
        d = {"b": b}
        for k, M in enumerate(mats):
            M = sp.csr_matrix(M)
            d[f"A{k}_indptr"], d[f"A{k}_indices"], d[f"A{k}_data"] = M.indptr, M.indices, M.data
            d[f"A{k}_shape"] = np.asarray(M.shape)
        for k, P in enumerate(pros):
            P = sp.csr_matrix(P)
            d[f"P{k}_indptr"], d[f"P{k}_indices"], d[f"P{k}_data"] = P.indptr, P.indices, P.data
            d[f"P{k}_shape"] = np.asarray(P.shape)
        d["nlev"] = np.int64(len(mats))
        np.savez(os.path.join(args.save, f"{cfg}_ref_hierarchy.npz"), **d)
    out = os.path.join(HERE, f"{cfg}_ref.json")
    json.dump(rec, open(out, "w"), indent=1)
    if not args.no_solve:
        est.solve(b, rtol=1e-6)  # warm-up (numba JIT)
        t0 = time.perf_counter()
        x, rep = est.solve(b, rtol=1e-6)
        rec["solve_s"] = time.perf_counter() - t0
        rec["nit"] = int(rep.iterations)
        rec["converged"] = bool(rep.converged)
        rec["final_relres"] = float(rep.final_relative_residual)
        rec["residual_history"] = [float(v) for v in rep.residual_history]
        rec["x_sha256"] = vec_digest(x)
        rec["x_norm"] = float(np.linalg.norm(x))
        rec["x_head"] = [float(v) for v in x[:8]]
        print(f"[{cfg}] solve {rec['solve_s']:.2f} s nit {rec['nit']}", flush=True)
        json.dump(rec, open(out, "w"), indent=1)
    rec["coarsest"] = coarsest_condition(sp.csr_matrix(mats[-1]))
    json.dump(rec, open(out, "w"), indent=1)
    print(f"[{cfg}] done: levels {rec['levels']} coarsest {rec['coarsest']}", flush=True)


if __name__ == "__main__":
    main()
