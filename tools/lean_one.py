"""One lean GS sweep of a Q1 grid (for ncu captures).  python tools/lean_one.py [grid] [K]"""
import sys

import torch

sys.path.insert(0, ".")
from paper_1907_04417_b200 import problems  # noqa: E402
from paper_1907_04417_b200.device import DeviceGsPlan, GpuConfig  # noqa: E402

g = int(sys.argv[1]) if len(sys.argv) > 1 else 256
K = int(sys.argv[2]) if len(sys.argv) > 2 else 1
A = problems.anisotropic_q1(g)
gp = DeviceGsPlan(A, GpuConfig(lean_rows_per_round=K))
n = A.shape[0]
b = torch.randn(n, dtype=torch.float64, device="cuda")
xn = torch.empty(n, dtype=torch.float64, device="cuda")
ws = torch.zeros(8, dtype=torch.int32, device="cuda")
for _ in range(3):
    gp.sweep(0, b, None, xn, ws)
torch.cuda.synchronize()
print("ok", gp.plan.lean_C, gp.plan.R, gp.plan.D)
