"""Per-round clock64 trace of the lean GS kernel's first warp (diagnostics, GPU).

Builds a separate .so with -DMVAMG_LEAN_TRACE=1 (scratch/), runs one forward
sweep of a Q1 grid and prints the distribution of round durations and the
share of chunk-start overhead.
  python tools/lean_trace.py [grid]
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
so = os.path.join(ROOT, "scratch", "libmvamg_trace.so")
if not os.environ.get("MVAMG_LIB"):
    sys.path.insert(0, ROOT)
    from paper_1907_04417_b200 import _lib as L0
    os.makedirs(os.path.dirname(so), exist_ok=True)
    subprocess.run(["nvcc", *L0.NVCC_FLAGS, "-DMVAMG_LEAN_TRACE=1", "-o", so, L0.SRC], check=True)
    os.environ["MVAMG_LIB"] = so
    os.execv(sys.executable, [sys.executable] + sys.argv)

import numpy as np  # noqa: E402
import torch  # noqa: E402

sys.path.insert(0, ROOT)
from paper_1907_04417_b200 import _lib, problems  # noqa: E402
from paper_1907_04417_b200.device import DeviceGsPlan, ptr  # noqa: E402

g = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
A = problems.anisotropic_q1(g)
n = A.shape[0]
K = int(sys.argv[2]) if len(sys.argv) > 2 else 1
from paper_1907_04417_b200.device import GpuConfig  # noqa: E402
gp = DeviceGsPlan(A, GpuConfig(lean_rows_per_round=K))
print(f"plan: tiles={gp.plan.ntiles} thr={gp.plan.threads} lean_C={gp.plan.lean_C} R={gp.plan.R} D={gp.plan.D}")
b = torch.randn(n, dtype=torch.float64, device="cuda")
xn = torch.empty(n, dtype=torch.float64, device="cuda")
ws = torch.zeros(8, dtype=torch.int32, device="cuda")
tr = torch.zeros(16384 + 8192 + 4096, dtype=torch.int64, device="cuda")
if K > 1:
    L = _lib.load()
    for _ in range(3):
        gp.sweep(0, b, None, xn, ws)
    L.mvamg_gs_set_trace(ptr(tr))
    gp.sweep(0, b, None, xn, ws)
    torch.cuda.synchronize()
    L.mvamg_gs_set_trace(None)
    t = tr.cpu().numpy()[:16384].reshape(-1, 2)
    ends = t[:, 1]
    nr = int(np.count_nonzero(ends))
    d = np.diff(ends[:nr])
    print(f"K={K} rounds traced {nr}: round cycles p50 {np.median(d):.0f} mean {d.mean():.0f}; spins per round "
          f"p50 {np.median(t[:nr, 0]):.0f} mean {t[:nr, 0].mean():.1f}")
    print("first 30 deltas", d[:30].tolist())
    print("first 30 spins", t[:30, 0].tolist())
    sys.exit(0)
L = _lib.load()
for _ in range(3):
    gp.sweep(0, b, None, xn, ws)
L.mvamg_gs_set_trace(ptr(tr))
gp.sweep(0, b, None, xn, ws)
torch.cuda.synchronize()
L.mvamg_gs_set_trace(None)
tt = tr.cpu().numpy()
ends = tt[:16384].reshape(-1, 2)[:, 1]
nr = int(np.count_nonzero(ends))
ends = ends[:nr]
spins = tt[16384 + 8192:16384 + 8192 + 4096][:nr]
d = np.diff(ends)
print(f"warp {os.environ.get('MVAMG_GS_DEBUG', '0')}>>8: rounds {nr}, round cycles p10 {np.percentile(d, 10):.0f} "
      f"p50 {np.median(d):.0f} p90 {np.percentile(d, 90):.0f} mean {d.mean():.0f}; total {ends[-1] - ends[0]} cycles; "
      f"rounds with spins {np.count_nonzero(spins)}, spins total {spins.sum()}")
print("first 40 deltas", d[:40].tolist())
print("mid 40 deltas", d[nr // 2:nr // 2 + 40].tolist())
