"""Time the lean wavefront sweep on a config's fine operator with its tiles
launched as thread-block clusters of 0 (off), 2, 4, 8 CTAs.

  python tools/lean_cluster.py [c2] [clusters ...]
"""
import sys

import torch

sys.path.insert(0, ".")
from paper_1907_04417_b200 import problems  # noqa: E402
from paper_1907_04417_b200.device import DeviceGsPlan, GpuConfig, time_sweep  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
cls = [int(k) for k in sys.argv[2:]] or [0, 2, 4, 8]
import os
ring = tuple(int(x) for x in os.environ["LEAN_RING"].split(",")) if os.environ.get("LEAN_RING") else None
A = problems.CONFIGS[name]["build"]()
n = A.shape[0]
g = torch.Generator(device="cuda").manual_seed(0)
b = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
xo = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
xn = torch.empty(n, dtype=torch.float64, device="cuda")
ws = torch.zeros(8, dtype=torch.int32, device="cuda")
ref = {}
for cl in cls:
    gp = DeviceGsPlan(A, GpuConfig(lean_cluster=cl, lean_ring=ring))
    t0 = time_sweep(lambda: gp.sweep(0, b, None, xn, ws), reps=5)
    y0 = xn.clone()
    t2 = time_sweep(lambda: gp.sweep(1, b, xo, xn, ws), reps=5)
    y2 = xn.clone()
    same = ""
    if ref:
        same = f" same-bits fwd {bool(torch.equal(y0, ref[0]))} bwd {bool(torch.equal(y2, ref[2]))}"
    else:
        ref = {0: y0, 2: y2}
    print(f"{name} ring {gp.plan.R},{gp.plan.D} cluster {cl}: tiles={gp.plan.ntiles} fwd {t0 * 1e6:.0f} us bwd {t2 * 1e6:.0f} us "
          f"timeout={int(ws[1].item())}{same}", flush=True)
