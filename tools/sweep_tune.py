"""Time one level's forward / backward sweeps of a bench workload under several
GpuConfig variants (device time, CUDA events, 20 reps each):

  python tools/sweep_tune.py c3 0 "ring_bytes=24576" "ring_bytes=16384" ...
  python tools/sweep_tune.py c3 1 "row_gs_threads=64" "row_gs_ctas=296" ...
Each variant is a comma-separated list of GpuConfig fields (python literals)."""
import ast
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1907_04417_b200 import GpuMultigridOperator  # noqa: E402
from paper_1907_04417_b200.device import GpuConfig, stream_handle  # noqa: E402

cfg_name, k = sys.argv[1], int(sys.argv[2])
variants = [""] + sys.argv[3:]
mats, pros, b, info = bench.load_workload(cfg_name)
nk = mats[k].shape[0]
bk = torch.from_numpy(np.random.default_rng(k).uniform(-1, 1, nk)).cuda()
xo = torch.from_numpy(np.random.default_rng(100 + k).uniform(-1, 1, nk)).cuda()
xn = torch.empty(nk, dtype=torch.float64, device="cuda")
ws = torch.zeros(8, dtype=torch.int32, device="cuda")
s = stream_handle()
stream = torch.cuda.current_stream()
for v in variants:
    kw = {}
    for part in filter(None, v.split(";")):
        key, val = part.split("=", 1)
        kw[key.strip()] = ast.literal_eval(val.strip())
    try:
        if k == 0:  # the fine level's wavefront plan alone (no coarse levels to build)
            from types import SimpleNamespace

            from paper_1907_04417_b200.device import DeviceGsPlan

            gp = DeviceGsPlan(mats[0], GpuConfig(**kw))
            op = SimpleNamespace(level_dev=[dict(gs=gp)])
        else:
            op = GpuMultigridOperator(mats, pros, config=GpuConfig(**kw))
        f, bw, fname, bname = bench._level_sweeps(op, k, bk, xo, xn, ws, s)
        tf = bench._event_time(f, 20, stream) * 1e6
        tb = bench._event_time(bw, 20, stream) * 1e6
        p = op.level_dev[k].get("gs")
        extra = ""
        if p is not None:
            extra = (f"tiles {p.plan.ntiles} threads {p.plan.threads} window {p.plan.window} "
                     f"ring R{p.plan.R}xD{p.plan.D} blocked {getattr(p.plan, 'chain_order', None) is not None}")
        print(f"level {k} [{v or 'default'}]: fwd {tf:.1f} us ({fname})  bwd {tb:.1f} us ({bname})  {extra}", flush=True)
        del op
    except Exception as exc:
        print(f"level {k} [{v}]: {type(exc).__name__}: {exc}", flush=True)
