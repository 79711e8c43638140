"""Fit a BASELINE workload on the box with this repo's setup and record the
same digests tests/golden/make_golden_large.py records for the unmodified
reference (tests/golden/<cfg>_ref.json), then solve it on the GPU (H1) and
compare with the reference's record when one is committed.

    python tools/fit_record.py c3 [j160 ...] [--out gpurun_out] [--no-solve]

Writes <out>/fit_<cfg>.json.  Diagnostics per level: diagonal range,
Gershgorin bound, max |P'P - I| and the largest prolongator column norm
(multi-vector blocks are orthonormal by construction, multivector.py:181-212)
and, for a coarsest level of at most 12k rows, its spectrum.
"""

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))

from _digest import coarsest_condition, diagnostics, hierarchy_record, vec_digest  # noqa: E402

from paper_1907_04417_b200 import problems  # noqa: E402


def workload(cfg):
    if cfg in problems.CONFIGS:
        A = problems.CONFIGS[cfg]["build"]()
        b = problems.elasticity_rhs(A) if cfg == "c4" else problems.rhs_uniform(A.shape[0], 0)
        return A, b
    g = int(cfg[1:])
    A = problems.jump_3d(g, 16, 1)
    return A, problems.rhs_uniform(A.shape[0], 0)


def compare(rec, ref):
    """Structural identity and value closeness against the reference record."""
    out = {"levels_equal": rec["levels"] == ref["levels"],
           "nnz_equal": rec["nnz_levels"] == ref["nnz_levels"] and rec["nnz_P"] == ref.get("nnz_P")}
    if "A_pattern" in ref:
        out["A_pattern_equal"] = [a == b for a, b in zip(rec["A_pattern"], ref["A_pattern"])]
        out["P_pattern_equal"] = [a == b for a, b in zip(rec["P_pattern"], ref["P_pattern"])]
        out["A_moment_rel"] = [max(abs(x - y) / max(abs(y), 1e-300) for x, y in zip(a, b))
                               for a, b in zip(rec["A_moments"], ref["A_moments"])]
        out["P_moment_rel"] = [max(abs(x - y) / max(abs(y), 1e-300) for x, y in zip(a, b))
                               for a, b in zip(rec["P_moments"], ref["P_moments"])]
    out["A_sha_equal"] = [a == b for a, b in zip(rec["A_sha256"], ref["A_sha256"])]
    out["P_sha_equal"] = [a == b for a, b in zip(rec["P_sha256"], ref["P_sha256"])]
    if "nit" in rec and "nit" in ref:
        out["nit"] = [rec["nit"], ref["nit"]]
        h, hr = np.asarray(rec["residual_history"]), np.asarray(ref["residual_history"])
        m = min(h.shape[0], hr.shape[0])
        out["history_rel_max"] = float(np.max(np.abs(h[:m] - hr[:m]) / np.abs(hr[:m])))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cfgs", nargs="+")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out"))
    ap.add_argument("--no-solve", action="store_true")
    args = ap.parse_args()
    os.makedirs(args.out, exist_ok=True)
    from paper_1907_04417_b200.estimator import MultiVectorAMG

    for cfg in args.cfgs:
        A, b = workload(cfg)
        t0 = time.perf_counter()
        est = MultiVectorAMG().fit(A)
        rec = {"config": cfg, "fit_s": time.perf_counter() - t0}
        mats = list(est.hierarchy_.matrices)
        pros = list(est.hierarchy_.prolongator_matrices)
        rec.update(hierarchy_record(mats, pros))
        rec["bootstrap_stages"] = int(est.composite_.n_components)
        rec["stage_rho"] = [float(s.rho) for s in est.composite_.stage_records]
        rec["smooth_vector_sha256"] = [vec_digest(v) for v in est.smooth_vectors_]
        rec["diagnostics"] = diagnostics(mats, pros)
        print(f"[{cfg}] fit {rec['fit_s']:.1f} s levels {rec['levels']}", flush=True)
        if not args.no_solve:
            try:
                est.solve(b)
                t0 = time.perf_counter()
                x, rep = est.solve(b)
                rec["solve_s"] = time.perf_counter() - t0
                rec["nit"] = int(rep.iterations)
                rec["converged"] = bool(rep.converged)
                rec["residual_history"] = [float(v) for v in rep.residual_history]
                rec["x_norm"] = float(np.linalg.norm(x))
            except Exception as exc:  # record the failure (C5: NotSpdError) and keep going
                rec["solve_error"] = f"{type(exc).__name__}: {exc}"
        rec["coarsest"] = coarsest_condition(mats[-1])
        ref_path = os.path.join(ROOT, "tests", "golden", f"{cfg}_ref.json")
        if os.path.exists(ref_path):
            rec["vs_reference"] = compare(rec, json.load(open(ref_path)))
        json.dump(rec, open(os.path.join(args.out, f"fit_{cfg}.json"), "w"), indent=1)
        print(f"[{cfg}] nit {rec.get('nit')} {rec.get('solve_error', '')} coarsest {rec['coarsest']}", flush=True)
        print(json.dumps({"diag": [(d['level'], d['diag_max'], d.get('ptp_minus_i_max'), d.get('p_col_norm_max'))
                                   for d in rec['diagnostics']]}), flush=True)
        del est
        import torch

        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
