"""Fit the same problem repeatedly and fingerprint the hierarchies (setup must
be deterministic).  Variants force the coarse-sweep choices.

  python tools/fit_determinism.py [ne] [reps]
"""
import hashlib
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_1907_04417_b200 import GpuConfig, problems  # noqa: E402
from paper_1907_04417_b200.estimator import MultiVectorAMG  # noqa: E402

ne = int(sys.argv[1]) if len(sys.argv) > 1 else 128
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
A = problems.elasticity_q1(ne)
b = problems.elasticity_rhs(A)


def fingerprint(est):
    h = hashlib.sha1()
    for M in est.hierarchy_.matrices:
        h.update(M.indptr.tobytes()); h.update(M.indices.tobytes()); h.update(M.data.tobytes())
    for w in est.smooth_vectors_:
        h.update(np.asarray(w).tobytes())
    return h.hexdigest()[:12]


variants = [("default", GpuConfig()), ("rows", GpuConfig(force_row_gs=True)),
            ("levels", GpuConfig(autotune_gs=False)), ("no-graphs", GpuConfig(graphs=False))]
for name, cfg in variants:
    for r in range(reps):
        t = time.time()
        est = MultiVectorAMG(config=cfg).fit(A)
        x, rep = est.solve(b)
        print(f"{name} rep {r}: {fingerprint(est)} stages {est.composite_.n_components} "
              f"levels {est.hierarchy_.sizes()} nit {rep.iterations} ({time.time() - t:.1f}s)", flush=True)
