"""Debug driver for the C5 (3D jump 320^3) solve: fit once (hierarchy cached
in /tmp as a pickle), then compare one V-cycle application across schedules
and against the CPU oracle.

  python tools/c5_debug.py [grid]
"""
import os
import pickle
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1907_04417_b200 import problems  # noqa: E402
from paper_1907_04417_b200.cycles import GpuMultigridOperator  # noqa: E402
from paper_1907_04417_b200.device import GpuConfig  # noqa: E402
from paper_1907_04417_b200.estimator import MultiVectorAMG  # noqa: E402

g = int(sys.argv[1]) if len(sys.argv) > 1 else 320
path = f"/tmp/jump3d_{g}.pkl"
if os.path.exists(path):
    with open(path, "rb") as f:
        mats, pros, b = pickle.load(f)
    print("loaded cached hierarchy", flush=True)
else:
    A = problems.jump_3d(g, 16, 1)
    b = problems.rhs_uniform(A.shape[0], 0)
    t = time.time()
    est = MultiVectorAMG().fit(A)
    print(f"fit {time.time() - t:.0f}s", flush=True)
    mats, pros = list(est.hierarchy_.matrices), list(est.hierarchy_.prolongator_matrices)
    with open(path, "wb") as f:
        pickle.dump((mats, pros, b), f, protocol=4)
print("levels", [M.shape[0] for M in mats], "nnz", [M.nnz for M in mats], flush=True)
for k, M in enumerate(mats):
    d = M.diagonal()
    print(f"  level {k}: min diag {d.min():.3e} max {d.max():.3e} sym {abs(M - M.T).max():.2e}", flush=True)
for name, cfg in (("exact", GpuConfig(exact_gs=True)), ("relaxed", GpuConfig())):
    op = GpuMultigridOperator(mats, pros, config=cfg)
    z = op.apply(b)
    rz = float(np.dot(b, z))
    print(f"{name}: r'z = {rz:.6e}  |z| = {np.linalg.norm(z):.3e} finite={np.all(np.isfinite(z))}", flush=True)
    for k, lv in enumerate(op.level_dev):
        kinds = [key for key in ("gs", "levels", "rows", "scan", "mega") if lv.get(key)]
        print(f"    level {k}: {kinds}", flush=True)
    del op
    torch.cuda.empty_cache()
