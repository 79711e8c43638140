"""Time the chain-scan GS sweep against the wavefront (lean) sweep on a
config's fine operator (no setup needed).

  python tools/scan_probe.py [c2|c3|c1] [modes...]
"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1907_04417_b200 import problems  # noqa: E402
from paper_1907_04417_b200.device import DeviceGsPlan, GpuConfig, time_sweep  # noqa: E402
from paper_1907_04417_b200.gs_scan import DeviceGsScan, plan_scan  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
modes = [int(m) for m in sys.argv[2:]] or [0, 3]
A = problems.CONFIGS[name]["build"]() if name != "c1" else problems.poisson_2d(128)
n = A.shape[0]
g = torch.Generator(device="cuda").manual_seed(0)
b = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
xo = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
xn = torch.empty(n, dtype=torch.float64, device="cuda")
ws = torch.zeros(8, dtype=torch.int32, device="cuda")
gp = DeviceGsPlan(A, GpuConfig())
for m in modes:
    t0 = time.time()
    p = plan_scan(A, m)
    tp = time.time() - t0
    if p is None:
        print(f"mode {m}: no scan plan")
        continue
    sc = DeviceGsScan(A, m, plan=p)
    import os
    if os.environ.get("SCAN_SINGLE"):
        p1 = plan_scan(A, m, GpuConfig(scan_cluster=0))
        sc1 = DeviceGsScan(A, m, plan=p1)
        t1 = time_sweep(lambda: sc1.sweep(b, xo if m % 2 else None, xn, ws), reps=5)
        print(f"  single-CTA scan {t1 * 1e6:.0f} us")
    xold = xo if m % 2 else None
    t_scan = time_sweep(lambda: sc.sweep(b, xold, xn, ws), reps=5)
    t_wave = time_sweep(lambda: gp.sweep(0 if m < 2 else 1, b, xold, xn, ws), reps=5)
    print(f"{name} mode {m}: n={n} chains={p.nchains} W={p.W} K={p.K} warps={p.threads // 32} S={p.S} "
          f"cluster={p.cluster} depth={p.depth} plan {tp:.1f}s | scan {t_scan * 1e6:.0f} us ({t_scan * 1e6 / max(1, p.depth):.3f} us/step)"
          f" | wave {t_wave * 1e6:.0f} us | timeout={int(ws[1].item())}", flush=True)
