"""Time MultiVectorAMG().fit + one solve for a config on the GPU box."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_1907_04417_b200 import problems  # noqa: E402
from paper_1907_04417_b200.estimator import MultiVectorAMG  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
t = time.time()
A = problems.CONFIGS[cfg]["build"]()
print(f"{cfg}: build {time.time() - t:.1f}s n={A.shape[0]} nnz={A.nnz}", flush=True)
t = time.time()
est = MultiVectorAMG().fit(A)
print(f"fit {time.time() - t:.1f}s stages={est.composite_.n_components} "
      f"rho={[round(r.rho, 3) for r in est.composite_.stage_records]} levels={est.hierarchy_.sizes()} "
      f"opc={est.operator_complexity_:.3f}", flush=True)
for k, lv in enumerate(est.operator_.level_dev):
    M = est.hierarchy_.matrices[k]
    if lv.get("levels") and lv.get("rows"):
        how = ("autotuned: " + ", ".join(f"mode{m}=level-set(c={s.ncta})" for m, s in lv["levels"].items()) + ", "
               + ", ".join(f"mode{m}=rows" for m in lv["rows"]))
    elif lv.get("levels"):
        s0 = next(iter(lv["levels"].values()))
        how = f"level-set cluster={s0.ncta} nlev={s0.nlev} thr={s0.threads}"
    elif lv.get("rows"):
        s0 = next(iter(lv["rows"].values()))
        how = f"row sweep nlev={s0.nlev} thr={s0.threads} ctas={s0.ctas}"
    else:
        pl = lv["plan"]
        how = f"wavefront lean_C={pl.lean_C} tiles={pl.ntiles} thr={pl.threads} depth={pl.depth}"
    print(f"  level {k}: n={M.shape[0]} nnz/row={M.nnz / M.shape[0]:.1f} {how}", flush=True)
import torch  # noqa: E402
stream = torch.cuda.current_stream()
for k, lv in enumerate(est.operator_.level_dev):
    n = est.hierarchy_.matrices[k].shape[0]
    bb = torch.randn(n, dtype=torch.float64, device="cuda")
    xo = torch.randn(n, dtype=torch.float64, device="cuda")
    xn = torch.empty(n, dtype=torch.float64, device="cuda")
    ws = torch.zeros(8, dtype=torch.int32, device="cuda")
    if lv.get("levels") or lv.get("rows"):
        fns = {}
        for m, s in (lv.get("levels") or {}).items():
            fns[m] = lambda s=s, m=m: s.sweep(bb, None if m % 2 == 0 else xo, xn, ws)
            if m == 2:
                fns[3] = lambda s=s: s.sweep(bb, xo, xn, ws, fold=True)
        for m, s in (lv.get("rows") or {}).items():
            fns[m] = lambda s=s, m=m: s.sweep(bb, None if m % 2 == 0 else xo, xn, ws)
            if m == 2:
                fns[3] = lambda s=s: s.sweep(bb, xo, xn, ws)
    else:
        gp = lv["gs"]
        fns = {0: lambda: gp.sweep(0, bb, None, xn, ws), 2: lambda: gp.sweep(1, bb, xo, xn, ws)}
    out = []
    for m, f in sorted(fns.items()):
        for _ in range(2):
            f()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(5):
            f()
        e1.record(stream); e1.synchronize()
        out.append(f"mode{m} {e0.elapsed_time(e1) / 5 * 1e3:.0f}us")
    print(f"  sweep level {k}: " + " ".join(out), flush=True)
t = time.time()
for _ in range(5):
    est.operator_.apply_device(torch.randn(A.shape[0], dtype=torch.float64, device="cuda"))
torch.cuda.synchronize()
print(f"  V-cycle {(time.time() - t) / 5 * 1e3:.2f} ms", flush=True)
b = problems.rhs_uniform(A.shape[0], 0)
for _ in range(2):
    t = time.time()
    x, rep = est.solve(b)
    print(f"solve {time.time() - t:.3f}s nit={rep.iterations} relres={rep.final_relative_residual:.2e}", flush=True)
