"""Time the fine level's wavefront sweeps (gs_lean_kernel) of a bench configuration under GpuConfig
variants -- only A0 is built, no hierarchy fit (GPU).

  python tools/fine_tune.py c5 "" "ring_bytes=16384" "ring_bytes=8192;lean_wpos=32"
"""
import ast
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1907_04417_b200 import problems  # noqa: E402
from paper_1907_04417_b200.device import DeviceGsPlan, GpuConfig, stream_handle  # noqa: E402

name = sys.argv[1]
A = problems.CONFIGS[name]["build"]()
n = A.shape[0]
b = torch.from_numpy(np.random.default_rng(0).uniform(-1, 1, n)).cuda()
xo = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, n)).cuda()
xn = torch.empty(n, dtype=torch.float64, device="cuda")
wk = torch.empty(n, dtype=torch.float64, device="cuda")
ws = torch.zeros(8, dtype=torch.int32, device="cuda")
s = stream_handle()
ref = {}
for v in sys.argv[2:] or [""]:
    kw = {}
    for part in filter(None, v.split(";")):
        key, val = part.split("=", 1)
        kw[key.strip()] = ast.literal_eval(val.strip())
    try:
        gp = DeviceGsPlan(A, GpuConfig(**kw))
        out = []
        for d, xold in ((0, None), (1, xo)):
            fn = lambda: gp.sweep(d, b, xold, xn, ws, s, work=wk)  # noqa: E731
            for _ in range(3):
                fn()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10):
                fn()
            e1.record()
            e1.synchronize()
            assert int(ws[1].item()) == 0, "timeout"
            x = xn.clone()
            same = "" if d not in ref else (" same bits" if torch.equal(ref[d], x) else " BITS DIFFER")
            ref.setdefault(d, x)
            out.append(f"{'fwd' if d == 0 else 'bwd'} {e0.elapsed_time(e1) / 10 * 1e3:.0f} us{same}")
        p = gp.plan
        print(f"{name} level 0 [{v or 'default'}]: {' | '.join(out)} | tiles {p.ntiles} threads {p.threads} window "
              f"{p.window} wpos {getattr(p, 'wpos', None)} ring R{p.R}xD{p.D} C{p.lean_C}", flush=True)
        del gp
    except Exception as exc:  # noqa: BLE001
        print(f"{name} level 0 [{v}]: {type(exc).__name__}: {exc}", flush=True)
