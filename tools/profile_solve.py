"""One PCG solve of a bench workload between cudaProfilerStart/Stop, for ncu
with --profile-from-start off (the fit's kernels stay unprofiled).

  ncu --profile-from-start off ... python tools/profile_solve.py c2 [solve|gs0|rows1]
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1907_04417_b200 import GpuMultigridOperator  # noqa: E402
from paper_1907_04417_b200.krylov import pcg  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
what = sys.argv[2] if len(sys.argv) > 2 else "solve"
mats, pros, b, info = bench.load_workload(cfg)
op = GpuMultigridOperator(mats, pros)
x, rep = pcg(mats[0], b, precond=op, rtol=1e-6)  # warm-up (graphs captured)
torch.cuda.synchronize()
lv = op.level_dev
n0 = mats[0].shape[0]
r = torch.from_numpy(np.asarray(b)).cuda()
xn = torch.empty(n0, dtype=torch.float64, device="cuda")
ws = torch.zeros(8, dtype=torch.int32, device="cuda")
torch.cuda.profiler.start()
if what == "solve":
    x, rep = pcg(mats[0], b, precond=op, rtol=1e-6)
elif what == "gs0":
    lv[0]["gs"].sweep(0, r, None, xn, ws)
elif what.startswith("rows"):
    k = int(what[4:])
    rw = lv[k]["rows"][0]
    n = mats[k].shape[0]
    rk = torch.randn(n, dtype=torch.float64, device="cuda")
    xk = torch.empty(n, dtype=torch.float64, device="cuda")
    rw.sweep(rk, None, xk, ws)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print(f"{cfg} {what} done: nit={rep.iterations}", flush=True)
