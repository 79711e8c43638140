"""One piece of a bench workload's H1 solve between cudaProfilerStart/Stop, for
ncu with --profile-from-start off (the fit's and warm-up's kernels stay
unprofiled).

  ncu --profile-from-start off ... python tools/profile_solve.py c3 [what]
  what: solve (one PCG solve) | fwdK / bwdK (level K's forward-from-zero /
        backward-from-x_old sweep, whatever schedule it runs) | cycle
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1907_04417_b200 import GpuMultigridOperator  # noqa: E402
from paper_1907_04417_b200.device import stream_handle  # noqa: E402
from paper_1907_04417_b200.krylov import pcg  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
what = sys.argv[2] if len(sys.argv) > 2 else "solve"
mats, pros, b, info = bench.load_workload(cfg)
op = GpuMultigridOperator(mats, pros)
x, rep = pcg(mats[0], b, precond=op, rtol=1e-6)  # warm-up (graphs captured)
torch.cuda.synchronize()
s = stream_handle()
fn = None
if what in ("fwd", "bwd") or what[:3] in ("fwd", "bwd"):
    k = int(what[3:] or 0)
    nk = mats[k].shape[0]
    bk = torch.from_numpy(np.random.default_rng(k).uniform(-1, 1, nk)).cuda()
    xo = torch.from_numpy(np.random.default_rng(100 + k).uniform(-1, 1, nk)).cuda()
    xn = torch.empty(nk, dtype=torch.float64, device="cuda")
    ws = torch.zeros(8, dtype=torch.int32, device="cuda")
    f, bw, fname, bname = bench._level_sweeps(op, k, bk, xo, xn, ws, s)
    fn = f if what.startswith("fwd") else bw
    fn()  # warm-up
elif what == "cycle":
    r = torch.from_numpy(np.asarray(b)).cuda()
    fn = lambda: op.apply_device(r)  # noqa: E731
    fn()
torch.cuda.synchronize()
torch.cuda.profiler.start()
if what == "solve":
    x, rep = pcg(mats[0], b, precond=op, rtol=1e-6)
else:
    fn()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print(f"{cfg} {what} done: nit={rep.iterations}", flush=True)
