"""PCG iteration counts on a fitted config: CPU oracle (the reference's
recipe) against the GPU cycle in exact and tolerance-parity modes.

  python tools/parity_nit.py c4
"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import bench  # noqa: E402
from oracle.oracle import OracleOperator, oracle_pcg  # noqa: E402
from paper_1907_04417_b200 import GpuConfig, GpuMultigridOperator, pcg  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
mats, pros, b, desc, info = bench.load_workload(name)
print(name, "levels", [M.shape[0] for M in mats], flush=True)
t = time.time()
ref = OracleOperator(mats, pros)
_, hist, nit, conv = oracle_pcg(ref, b)
print(f"oracle: nit {nit} conv {conv} ({time.time() - t:.0f}s)", flush=True)
z_ref = ref.apply(b)
for label, cfg in (("exact", GpuConfig(exact_gs=True)), ("relaxed", GpuConfig())):
    op = GpuMultigridOperator(mats, pros, config=cfg)
    z = op.apply(b)
    x, rep = pcg(mats[0], b, precond=op, rtol=1e-6)
    m = min(len(hist), len(rep.residual_history))
    herr = np.max(np.abs(rep.residual_history[:m] - hist[:m]) / hist[:m])
    print(f"{label}: cycle rel {np.max(np.abs(z - z_ref)) / np.max(np.abs(z_ref)):.2e}  nit {rep.iterations}  "
          f"hist rel (first {m}) {herr:.2e}", flush=True)
    for k in (10, 50, 100, 150, 198):
        if k < m:
            print(f"    it {k}: gpu {rep.residual_history[k]:.6e} oracle {hist[k]:.6e}")
