"""Per-stage / per-batch timeline of one streamed GS sweep (gs_stream_kernel)
on a level of a bench workload, from the kernel's clock64 trace
(mvamg_gs_stream_set_trace):

  python tools/stream_trace.py c3 5 [fwd|bwd]
Prints cycles spent waiting for stages vs per batch (by rows in the batch)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1907_04417_b200 import GpuMultigridOperator, _lib  # noqa: E402
from paper_1907_04417_b200.device import ptr, stream_handle  # noqa: E402

cfg, k = sys.argv[1], int(sys.argv[2])
which = sys.argv[3] if len(sys.argv) > 3 else "fwd"
mats, pros, b, info = bench.load_workload(cfg)
op = GpuMultigridOperator(mats, pros)
nk = mats[k].shape[0]
bk = torch.from_numpy(np.random.default_rng(k).uniform(-1, 1, nk)).cuda()
xo = torch.from_numpy(np.random.default_rng(100 + k).uniform(-1, 1, nk)).cuda()
xn = torch.empty(nk, dtype=torch.float64, device="cuda")
ws = torch.zeros(8, dtype=torch.int32, device="cuda")
f, bw, fname, bname = bench._level_sweeps(op, k, bk, xo, xn, ws, stream_handle())
fn = f if which == "fwd" else bw
cap = 1 << 20
tr = torch.zeros(cap, dtype=torch.int64, device="cuda")
L = _lib.load()
fn()
torch.cuda.synchronize()
L.mvamg_gs_stream_set_trace(ptr(tr), cap)
fn()
torch.cuda.synchronize()
L.mvamg_gs_stream_set_trace(None, 0)
t = tr.cpu().numpy()
m = int(t[0])
ev = t[1:m].reshape(-1, 2)
tags, clk = ev[:, 0], ev[:, 1]
lv = op.level_dev[k]
plans = lv.get("stream") or {}
print(f"{cfg} level {k} {which} ({fname if which == 'fwd' else bname}) plans "
      f"{ {m_: (p.ncta, p.group, p.nstages, p.nslots, p.slot, p.nlev) for m_, p in plans.items()} }")
# events per batch: -4 (row done), -5 (next fetched), rn (after barrier)
ib = np.flatnonzero(tags >= 0)
comp, fet, bar = [], [], []
prev = clk[0]
for i in ib:
    if i >= 2 and tags[i - 1] == -5 and tags[i - 2] == -4:
        comp.append(clk[i - 2] - prev)
        fet.append(clk[i - 1] - clk[i - 2])
        bar.append(clk[i] - clk[i - 1])
    prev = clk[i]
comp, fet, bar = map(np.asarray, (comp, fet, bar))
rows = tags[ib]
tot = clk[-1] - clk[0]
print(f"total {tot} cycles, {len(ib)} batches ({tot / max(1, len(ib)):.0f} per batch), rows per batch {rows.mean():.1f}")
def seg(a_, b_):
    ia = np.flatnonzero(tags[:-1] == a_)
    ia = ia[tags[ia + 1] == b_]
    return (clk[ia + 1] - clk[ia]).mean() if len(ia) else float("nan")


print(f"  thread 0 per batch: compute {comp.mean():.0f}  fetch-next {fet.mean():.0f}  barrier {bar.mean():.0f}  "
      f"(medians {np.median(comp):.0f} / {np.median(fet):.0f} / {np.median(bar):.0f})")
