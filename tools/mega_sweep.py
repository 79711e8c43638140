"""Sweep GpuConfig.mega_max_rows (0 = off) for H1 solves and H2 applications.

  python tools/mega_sweep.py c3 0 256 1024 4096
"""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1907_04417_b200 import problems  # noqa: E402
from paper_1907_04417_b200.composite import GpuComposite, GpuCompositePreconditioner  # noqa: E402
from paper_1907_04417_b200.cycles import GpuMultigridOperator  # noqa: E402
from paper_1907_04417_b200.device import GpuConfig  # noqa: E402
from paper_1907_04417_b200.estimator import MultiVectorAMG  # noqa: E402
from paper_1907_04417_b200.krylov import pcg  # noqa: E402

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "c3"
thr = [int(x) for x in sys.argv[2:]] or [0, 256, 1024, 4096]
A = problems.CONFIGS[cfg_name]["build"]()
b = problems.rhs_uniform(A.shape[0], 0)
est = MultiVectorAMG().fit(A)
comps = [c.operator for c in est.composite_.components]
r = torch.randn(A.shape[0], dtype=torch.float64, device="cuda")
for t in thr:
    cfg = GpuConfig(coarse_mega=t > 0, mega_max_rows=max(t, 1))
    h1 = GpuMultigridOperator(est.hierarchy_.matrices, est.hierarchy_.prolongator_matrices, config=cfg)
    ops = [GpuMultigridOperator(o.matrices, o.prolongators, cycle=o.cycle, config=cfg) for o in comps]
    pc = GpuCompositePreconditioner(GpuComposite(ops))
    for _ in range(2):
        torch.cuda.synchronize()
        t0 = time.time()
        x, rep = pcg(A, b, precond=h1, rtol=1e-6)
        torch.cuda.synchronize()
        th1 = time.time() - t0
    for _ in range(2):
        pc.apply_device(r)
    torch.cuda.synchronize()
    t0 = time.time()
    for _ in range(3):
        pc.apply_device(r)
    torch.cuda.synchronize()
    th2 = (time.time() - t0) / 3
    print(f"mega_max_rows={t}: H1 k0={h1.mega_k0} solve {th1:.3f}s nit={rep.iterations} | H2 k0s="
          f"{[o.mega_k0 for o in ops]} application {th2 * 1e3:.1f} ms", flush=True)
