"""Hop latency of the dataflow GS row sweep on pure dependency chains (GPU).

Lower-bidiagonal-coupled 1D Laplacian (depth n) and a few bands: per-level time
= one publish -> poll -> compute -> publish hop; plus iterations per row.
"""
import sys

import numpy as np
import scipy.sparse as sp
import torch

sys.path.insert(0, ".")
from paper_1907_04417_b200 import _lib  # noqa: E402
from paper_1907_04417_b200.device import DeviceGsRows, GpuConfig, ptr  # noqa: E402

L = _lib.load()


def banded(n, w):
    """SPD band matrix: row i couples to i-1..i-w (depth n for forward sweeps)."""
    offs = list(range(-w, w + 1))
    diags = [np.full(n - abs(o), -1.0 if o else 2.0 * w + 1.0) for o in offs]
    return sp.diags(diags, offs, format="csr")


for name, A, cfgkw in [("lap1d_4096", banded(4096, 1), {}), ("band4_4096", banded(4096, 4), {}),
                       ("band16_2048", banded(2048, 16), {}), ("band30_2048", banded(2048, 30), {}),
                       ("lap1d_4096_T32", banded(4096, 1), dict(row_gs_threads=32))]:
    n = A.shape[0]
    for mode in (0, 2):
        rw = DeviceGsRows(A, mode, GpuConfig(**cfgkw))
        b = torch.randn(n, dtype=torch.float64, device="cuda")
        xo = torch.randn(n, dtype=torch.float64, device="cuda") if mode == 2 else None
        xn = torch.empty(n, dtype=torch.float64, device="cuda")
        ws = torch.zeros(8, dtype=torch.int32, device="cuda")
        for _ in range(3):
            rw.sweep(b, xo, xn, ws)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            rw.sweep(b, xo, xn, ws)
        e1.record()
        e1.synchronize()
        t_us = e0.elapsed_time(e1) / 5 * 1e3
        tr = torch.zeros(2 * n, dtype=torch.int64, device="cuda")
        L.mvamg_gs_set_trace(ptr(tr))
        rw.sweep(b, xo, xn, ws)
        torch.cuda.synchronize()
        L.mvamg_gs_set_trace(None)
        t = tr.cpu().numpy()
        its = t[n:]
        print(f"{name} mode={mode} nlev={rw.nlev} T={rw.threads} ctas={rw.ctas}: {t_us:.0f}us "
              f"{t_us * 1e3 / rw.nlev:.0f} ns/level | iterations/row p50 {np.median(its):.0f} "
              f"p90 {np.percentile(its, 90):.0f} max {its.max()}", flush=True)
