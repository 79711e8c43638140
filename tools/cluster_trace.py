"""Per-row trace of the cluster dataflow sweep on one CTA (clock64 is per SM):
publish clock, poll iterations, tile start / staged clocks (diagnostics, GPU).

  python tools/cluster_trace.py scratch/c3_coarse.npz level=7 mode=0 wpc=2
"""
import sys

import numpy as np
import scipy.sparse as sp
import torch

sys.path.insert(0, ".")
from paper_1907_04417_b200 import _lib  # noqa: E402
from paper_1907_04417_b200.device import DeviceGsCluster, GpuConfig, ptr  # noqa: E402

kw = dict(a.split("=") for a in sys.argv[2:])
z = np.load(sys.argv[1])
k = int(kw.get("level", 7))
mode = int(kw.get("mode", 0))
n = int(z[f"n{k}"])
M = sp.csr_matrix((z[f"v{k}"], z[f"ix{k}"], z[f"ip{k}"]), shape=(n, n))
cl = DeviceGsCluster(M, mode, GpuConfig(), ncta=int(kw.get("ncta", 1)), wpc=int(kw.get("wpc", 2)))
b = torch.randn(n, dtype=torch.float64, device="cuda")
xo = torch.randn(n, dtype=torch.float64, device="cuda") if mode == 2 else None
xn = torch.empty(n, dtype=torch.float64, device="cuda")
ws = torch.zeros(8, dtype=torch.int32, device="cuda")
for _ in range(3):
    cl.sweep(b, xo, xn, ws)
tr = torch.zeros(3 * n, dtype=torch.int64, device="cuda")
L = _lib.load()
L.mvamg_gs_set_trace(ptr(tr))
cl.sweep(b, xo, xn, ws)
torch.cuda.synchronize()
L.mvamg_gs_set_trace(None)
t0, pub, t_early = tr.cpu().numpy().reshape(3, n)   # by q
base = t0.min()
print(f"level {k} n={n} mode {mode} depth {cl.nlev} cluster {cl.ncta}x{cl.wpc}; total {pub.max() - base} cycles = "
      f"{(pub.max() - base) / cl.nlev:.0f} cycles/level")
dur = pub - t0
for nm, x0, x1 in (("header+early", t0, t_early), ("tree+late+tail", t_early, pub)):
    d = x1 - x0
    print(f"  {nm:15s} p10 {np.percentile(d, 10):6.0f} p50 {np.median(d):6.0f} p90 {np.percentile(d, 90):6.0f}")
gap = t0[1:] - pub[:-1]
wptr = cl.wptr.cpu().numpy()
mask = np.ones(n - 1, bool); mask[wptr[1:-1][wptr[1:-1] > 0] - 1] = False
print(f"  gap publish -> next row's start (same worker) p10 {np.percentile(gap[mask], 10):.0f} p50 "
      f"{np.median(gap[mask]):.0f} p90 {np.percentile(gap[mask], 90):.0f}")
print(f"row time (start -> publish) cycles: p10 {np.percentile(dur, 10):.0f} p50 {np.median(dur):.0f} p90 "
      f"{np.percentile(dur, 90):.0f} max {dur.max()}")
# delay between a row's last input being published and its own publish (same SM clock only with ncta=1)
ip, ix = M.indptr, M.indices
perm = cl.perm.cpu().numpy()
lat = []
for i in range(n):
    c = ix[ip[i]:ip[i + 1]]
    c = c[c < i] if mode == 0 else c[c > i]
    if len(c):
        lat.append(pub[perm[i]] - pub[perm[c]].max())
lat = np.array(lat)
print(f"publish - last input's publish, cycles: p10 {np.percentile(lat, 10):.0f} p50 {np.median(lat):.0f} p90 "
      f"{np.percentile(lat, 90):.0f} max {lat.max()}")
wptr = cl.wptr.cpu().numpy()
print(f"rows whose latest input is on their own CTA: {cl.local_late} of {n}; rows per worker min {np.diff(wptr).min()} "
      f"max {np.diff(wptr).max()}; slots per CTA {cl.slots}")
