"""Compare GS sweep schedules on the coarse levels of a fitted config (GPU).

  python tools/coarse_probe.py c2 [ctas ...]
Per coarse level: level-set (cluster) sweep vs the dataflow row sweep at a few
resident-CTA counts, mode 0 (fwd from 0) and folded backward; checks bits agree.
"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1907_04417_b200 import problems  # noqa: E402
from paper_1907_04417_b200.device import DeviceGsLevels, DeviceGsRows, GpuConfig  # noqa: E402
from paper_1907_04417_b200.estimator import MultiVectorAMG  # noqa: E402

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "c2"
ctas_list = [int(x) for x in sys.argv[2:]] or [0, 32, 74, 148, 296]
A = problems.CONFIGS[cfg_name]["build"]()
t = time.time()
est = MultiVectorAMG().fit(A)
print(f"{cfg_name}: fit {time.time() - t:.1f}s levels={est.hierarchy_.sizes()}", flush=True)
stream = torch.cuda.current_stream()


def timeit(f, reps=5):
    for _ in range(2):
        f()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        f()
    e1.record(stream)
    e1.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


mats = est.hierarchy_.matrices
for k in range(1, len(mats) - 1):
    M = mats[k]
    n = M.shape[0]
    g = torch.Generator(device="cuda").manual_seed(k)
    bb = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
    xo = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
    ws = torch.zeros(8, dtype=torch.int32, device="cuda")
    out = []
    ref = {}
    try:
        lv0 = DeviceGsLevels(M, 0)
        lv2 = DeviceGsLevels(M, 2)
        xa = torch.empty(n, dtype=torch.float64, device="cuda")
        xb = torch.empty(n, dtype=torch.float64, device="cuda")
        out.append(f"levels[c={lv0.ncta} nlev={lv0.nlev}] f0 {timeit(lambda: lv0.sweep(bb, None, xa, ws)):.0f}us "
                   f"bfold {timeit(lambda: lv2.sweep(bb, xo, xb, ws, fold=True)):.0f}us")
        torch.cuda.synchronize()
        ref = {0: xa.clone(), 2: xb.clone()}
    except ValueError as e:
        out.append(f"levels n/a ({e})")
    t0 = time.time()
    rw0 = DeviceGsRows(M, 0)
    rw2 = DeviceGsRows(M, 2)
    tb = time.time() - t0
    out.append(f"rows[nlev={rw0.nlev} slots={rw0.nslots} auto_ctas={rw0.ctas} build {tb:.1f}s]")
    for c in ctas_list:
        for rw in (rw0, rw2):
            rw.ctas = c if c > 0 else rw.ctas
        ya = torch.empty(n, dtype=torch.float64, device="cuda")
        yb = torch.empty(n, dtype=torch.float64, device="cuda")
        ws.zero_()
        t0_ = timeit(lambda: rw0.sweep(bb, None, ya, ws))
        t2_ = timeit(lambda: rw2.sweep(bb, xo, yb, ws))
        torch.cuda.synchronize()
        ok = ""
        if ref:
            ok = "ok" if (torch.equal(ya, ref[0]) and torch.equal(yb, ref[2])) else "MISMATCH"
        st = int(ws[1].item())
        out.append(f"ctas={rw0.ctas}: f0 {t0_:.0f}us bfold {t2_:.0f}us {ok}{' TIMEOUT' if st else ''}")
    print(f"  level {k}: n={n} nnz/row={M.nnz / n:.1f} | " + " | ".join(out), flush=True)
op = est.operator_
r = torch.randn(A.shape[0], dtype=torch.float64, device="cuda")
print(f"  V-cycle (default schedules) {timeit(lambda: op.apply_device(r)) / 1e3:.2f} ms", flush=True)
b = problems.rhs_uniform(A.shape[0], 0)
for _ in range(2):
    t = time.time()
    x, rep = est.solve(b)
    print(f"solve {time.time() - t:.3f}s nit={rep.iterations} relres={rep.final_relative_residual:.2e}", flush=True)
