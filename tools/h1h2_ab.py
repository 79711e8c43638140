"""A/B of GpuConfig variants on a bench workload: H1 PCG solve (V-cycle) and
H2 PCG solve (symmetrized composite of the bootstrap K-cycles), device time.

  python tools/h1h2_ab.py c3 "" "stream_gs=False" "stream_max_rows=1024"   [--h1: skip H2]
Each variant: semicolon-separated GpuConfig fields (python literals)."""
import ast
import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_1907_04417_b200 as mv  # noqa: E402
from paper_1907_04417_b200.krylov import pcg  # noqa: E402

h1_only = "--h1" in sys.argv
argv = [a for a in sys.argv if a != "--h1"]
cfg_name = argv[1]
variants = argv[2:] or [""]
mats, pros, b, info = bench.load_workload(cfg_name)
comps = info["components"]


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        out = fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps, out


for v in variants:
    kw = {}
    for part in filter(None, v.split(";")):
        key, val = part.split("=", 1)
        kw[key.strip()] = ast.literal_eval(val.strip())
    cfg = mv.GpuConfig(**kw)
    op = mv.GpuMultigridOperator(mats, pros, config=cfg)
    t1, (_, r1) = timed(lambda: pcg(mats[0], b, precond=op, rtol=1e-6), 5)
    if h1_only:
        print(f"[{v or 'default'}] H1 {t1 * 1e3:.1f} ms (nit {r1.iterations})", flush=True)
        del op
        continue
    ops = [mv.GpuMultigridOperator(m, p, cycle=mv.CycleSpec("K", 2), config=cfg) for m, p in comps]
    pc = mv.GpuCompositePreconditioner(mv.GpuComposite(ops))
    t2, (_, r2) = timed(lambda: pcg(mats[0], b, precond=pc, rtol=1e-6), 2)
    print(f"[{v or 'default'}] H1 {t1 * 1e3:.1f} ms (nit {r1.iterations})  H2 {t2 * 1e3:.1f} ms (nit {r2.iterations})",
          flush=True)
    del op, ops, pc
