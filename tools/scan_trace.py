"""Per-segment timeline of the chain-scan sweep (globaltimer stamps):
where a segment step's time goes, and the line-to-line lag.

  python tools/scan_trace.py [c2|c1] [mode] [cluster]
"""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1907_04417_b200 import _lib, problems  # noqa: E402
from paper_1907_04417_b200.device import GpuConfig, ptr  # noqa: E402
from paper_1907_04417_b200.gs_scan import DeviceGsScan, plan_scan  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
m = int(sys.argv[2]) if len(sys.argv) > 2 else 0
cl = int(sys.argv[3]) if len(sys.argv) > 3 else 8
A = problems.CONFIGS[name]["build"]() if name != "c1" else problems.poisson_2d(128)
n = A.shape[0]
p = plan_scan(A, m, GpuConfig(scan_cluster=cl))
sc = DeviceGsScan(A, m, plan=p)
b = torch.randn(n, dtype=torch.float64, device="cuda")
xo = torch.randn(n, dtype=torch.float64, device="cuda")
xn = torch.empty(n, dtype=torch.float64, device="cuda")
ws = torch.zeros(8, dtype=torch.int32, device="cuda")
nseg = int(p.seg_ptr[-1])
tr = torch.zeros(4 * nseg, dtype=torch.int64, device="cuda")
L = _lib.load()
sc.sweep(b, xo if m % 2 else None, xn, ws)
L.mvamg_gs_scan_set_trace(ptr(tr))
sc.sweep(b, xo if m % 2 else None, xn, ws)
torch.cuda.synchronize()
L.mvamg_gs_scan_set_trace(None)
t = tr.cpu().numpy().reshape(nseg, 4).astype(np.int64)
if not np.any(t > 0):
    print("no trace (kernel without instrumentation)")
    sys.exit(0)
t -= t[t > 0].min()
print(f"{name} mode {m} cluster {p.cluster}: total {t.max() / 1e3:.0f} us over {nseg} segments, depth {p.depth}")
d = np.diff(t, axis=1)
print("mean ns: stage-wait {:.0f}  fix+deps-wait {:.0f}  compute+publish {:.0f}".format(*d.mean(axis=0)))
print("median ns:", np.median(d, axis=0))
seg_ptr = p.seg_ptr
# line-to-line lag: start of segment 0 of chain L minus that of chain L-1
starts = t[seg_ptr[:-1], 0]
ends = t[seg_ptr[1:] - 1, 3]
print("chain start lag (ns) median", np.median(np.diff(starts)), "chain duration median", np.median(ends - starts))
for c in (0, 1, 2):
    g = seg_ptr[c]
    print("chain", c, "t0 per seg (us):", (t[g:seg_ptr[c + 1], 0] / 1e3).round(2)[:12])
    print("chain", c, "stage-wait/deps/compute ns:", np.diff(t[g:g + 6], axis=1).tolist())
mid = len(seg_ptr) // 2
g0 = seg_ptr[mid]
print("chain", mid, "per-segment step ns:", np.diff(t[g0:seg_ptr[mid + 1], 0])[:12])
print("chain", mid, "raw (t0..t3) first 4 segs:\n", t[g0:g0 + 4])
