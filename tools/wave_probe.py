"""Time the lean wavefront GS sweep on Q1 / 5-point grids under several tilings."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1907_04417_b200 as mv  # noqa: E402
from paper_1907_04417_b200 import problems  # noqa: E402
from paper_1907_04417_b200.device import DeviceGsPlan  # noqa: E402

stream = torch.cuda.current_stream()


def run(A, name, **kw):
    cfg = mv.GpuConfig(**kw)
    t = time.time()
    gp = DeviceGsPlan(A, cfg)
    gp.mode(0)
    tb = time.time() - t
    n = A.shape[0]
    b = torch.randn(n, dtype=torch.float64, device="cuda")
    xn = torch.empty(n, dtype=torch.float64, device="cuda")
    ws = torch.zeros(8, dtype=torch.int32, device="cuda")
    for _ in range(2):
        gp.sweep(0, b, None, xn, ws)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(3):
        gp.sweep(0, b, None, xn, ws)
    e1.record(stream)
    e1.synchronize()
    ms = e0.elapsed_time(e1) / 3
    p = gp.plan
    print(f"{name:10s} {str(kw):60s} chains={p.nchains} tiles={p.ntiles} thr={p.threads} C={p.lean_C} R={p.R} D={p.D} "
          f"depth={p.depth} | {ms * 1e3:9.1f} us  {ms * 1e6 / p.depth:7.0f} ns/level  (plan {tb:.1f}s)", flush=True)


for g in (256, 1024):
    A = problems.anisotropic_q1(g)
    for kw in (dict(), dict(ring_bytes=80 * 1024), dict(max_threads=64, ring_bytes=24576)):
        run(A, f"q1_{g}", **kw)
A = problems.poisson_2d(512)
for kw in (dict(), dict(max_threads=32)):
    run(A, "p5_512", **kw)
