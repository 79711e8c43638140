"""Time MultiVectorAMG().fit + one solve for a config on the GPU box."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_1907_04417_b200 import problems  # noqa: E402
from paper_1907_04417_b200.estimator import MultiVectorAMG  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
t = time.time()
A = problems.CONFIGS[cfg]["build"]()
print(f"{cfg}: build {time.time() - t:.1f}s n={A.shape[0]} nnz={A.nnz}", flush=True)
t = time.time()
est = MultiVectorAMG().fit(A)
print(f"fit {time.time() - t:.1f}s stages={est.composite_.n_components} "
      f"rho={[round(r.rho, 3) for r in est.composite_.stage_records]} levels={est.hierarchy_.sizes()} "
      f"opc={est.operator_complexity_:.3f}", flush=True)
b = problems.rhs_uniform(A.shape[0], 0)
for _ in range(2):
    t = time.time()
    x, rep = est.solve(b)
    print(f"solve {time.time() - t:.3f}s nit={rep.iterations} relres={rep.final_relative_residual:.2e}", flush=True)
