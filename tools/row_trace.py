"""Per-row publish timestamps of the dataflow GS row sweep (diagnostics, GPU).

  python tools/row_trace.py [scratch/h64.npz]
For each level: sweep time, DAG depth, and the distribution of each row's
delay between its last input being published and its own publish.
"""
import ctypes
import sys

import numpy as np
import scipy.sparse as sp
import torch

sys.path.insert(0, ".")
from paper_1907_04417_b200 import _lib  # noqa: E402
from paper_1907_04417_b200.device import DeviceGsRows, GpuConfig, ptr  # noqa: E402

path = sys.argv[1] if len(sys.argv) > 1 else "scratch/h64.npz"
z = np.load(path)
L = _lib.load()
ks = sorted(int(k[1:]) for k in z.files if k.startswith("n"))
for k in ks:
    n = int(z[f"n{k}"])
    M = sp.csr_matrix((z[f"v{k}"], z[f"ix{k}"], z[f"ip{k}"]), shape=(n, n))
    for mode in (0, 2):
        rw = DeviceGsRows(M, mode, GpuConfig())
        b = torch.randn(n, dtype=torch.float64, device="cuda")
        xo = torch.randn(n, dtype=torch.float64, device="cuda") if mode == 2 else None
        xn = torch.empty(n, dtype=torch.float64, device="cuda")
        ws = torch.zeros(8, dtype=torch.int32, device="cuda")
        tr = torch.zeros(2 * n, dtype=torch.int64, device="cuda")
        for _ in range(3):
            rw.sweep(b, xo, xn, ws)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            rw.sweep(b, xo, xn, ws)
        e1.record()
        e1.synchronize()
        t_us = e0.elapsed_time(e1) / 10 * 1e3
        L.mvamg_gs_set_trace(ptr(tr))
        rw.sweep(b, xo, xn, ws)
        torch.cuda.synchronize()
        L.mvamg_gs_set_trace(None)
        t = tr.cpu().numpy()
        perm = rw.perm.cpu().numpy()
        prog = t[n:]
        tf = t[:n][perm]  # per row
        t0 = tf.min()
        ip, ix = M.indptr, M.indices
        lat, last = [], np.zeros(n)
        for i in range(n):
            c = ix[ip[i]:ip[i + 1]]
            c = c[c < i] if mode == 0 else c[c > i]
            if len(c):
                last[i] = tf[c].max()
                lat.append(tf[i] - last[i])
        lat = np.array(lat)
        # position of the latest input within the row's CSR-order entry list
        posl = []
        for i in range(0, n, max(1, n // 2000)):
            c = ix[ip[i]:ip[i + 1]]
            c = c[c < i] if mode == 0 else c[c > i]
            if len(c):
                posl.append(int(np.argmax(tf[c])) / max(1, len(c) - 1))
        print(f"level {k} n={n} mode={mode} nlev={rw.nlev} T={rw.threads} ctas={rw.ctas} sweep {t_us:.0f}us "
              f"span {(tf.max() - t0) / 1e3:.0f}us per-level {(tf.max() - t0) / rw.nlev:.0f}ns | delay after last "
              f"input ns: p10 {np.percentile(lat, 10):.0f} p50 {np.percentile(lat, 50):.0f} p90 "
              f"{np.percentile(lat, 90):.0f} max {lat.max():.0f} | latest-input pos (0=first,1=last) mean "
              f"{np.mean(posl):.2f} | progress iterations p50 {np.median(prog):.0f} p90 {np.percentile(prog, 90):.0f}",
              flush=True)
