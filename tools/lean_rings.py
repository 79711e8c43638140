"""Time the lean wavefront sweep on a config's fine operator for several ring
sizes (GpuConfig.ring_bytes picks the (R, D) chunking).

  python tools/lean_rings.py [c2] [ring_kb ...]
"""
import sys

import torch

sys.path.insert(0, ".")
from paper_1907_04417_b200 import problems  # noqa: E402
from paper_1907_04417_b200.device import DeviceGsPlan, GpuConfig, time_sweep  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
kbs = [int(k) for k in sys.argv[2:]] or [48, 72]
A = problems.CONFIGS[name]["build"]()
n = A.shape[0]
g = torch.Generator(device="cuda").manual_seed(0)
b = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
xo = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
xn = torch.empty(n, dtype=torch.float64, device="cuda")
ws = torch.zeros(8, dtype=torch.int32, device="cuda")
for kb in kbs:
    gp = DeviceGsPlan(A, GpuConfig(ring_bytes=kb * 1024))
    p = gp.plan
    t0 = time_sweep(lambda: gp.sweep(0, b, None, xn, ws), reps=5)
    t2 = time_sweep(lambda: gp.sweep(1, b, xo, xn, ws), reps=5)
    print(f"{name} ring {kb} KB: R={p.R} D={p.D} tiles={p.ntiles} threads={p.threads} fwd {t0 * 1e6:.0f} us "
          f"bwd {t2 * 1e6:.0f} us", flush=True)
