"""H2 solve on the GPU: PCG preconditioned by the symmetrized multiplicative
composite of the fitted bootstrap components (K-cycles), vs the H1 V-cycle.

  python tools/h2_bench.py c2
"""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1907_04417_b200 import problems  # noqa: E402
from paper_1907_04417_b200.composite import GpuCompositePreconditioner, gpu_composite_of  # noqa: E402
from paper_1907_04417_b200.estimator import MultiVectorAMG  # noqa: E402
from paper_1907_04417_b200.krylov import pcg  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
A = problems.CONFIGS[cfg]["build"]()
b = problems.rhs_uniform(A.shape[0], 0)
t = time.time()
est = MultiVectorAMG().fit(A)
print(f"{cfg}: fit {time.time() - t:.1f}s components={est.composite_.n_components}", flush=True)
gc = gpu_composite_of(est.composite_)
pc = GpuCompositePreconditioner(gc)
for name, prec in (("H1 V-cycle", est.operator_), ("H2 composite", pc)):
    for _ in range(2):
        torch.cuda.synchronize()
        t = time.time()
        x, rep = pcg(A, b, precond=prec, rtol=1e-6)
        torch.cuda.synchronize()
        dt = time.time() - t
    print(f"{name}: {dt:.3f}s nit={rep.iterations} relres={rep.final_relative_residual:.2e}", flush=True)
r = torch.randn(A.shape[0], dtype=torch.float64, device="cuda")
for _ in range(2):
    pc.apply_device(r)
torch.cuda.synchronize()
t = time.time()
for _ in range(5):
    pc.apply_device(r)
torch.cuda.synchronize()
print(f"one H2 application {(time.time() - t) / 5 * 1e3:.2f} ms", flush=True)
import ctypes  # noqa: E402

from paper_1907_04417_b200 import _lib  # noqa: E402

L = _lib.load()
cnt = ctypes.c_longlong()
L.mvamg_kernel_launches(None, 1)
pc.apply_device(r)
torch.cuda.synchronize()
L.mvamg_kernel_launches(ctypes.byref(cnt), 1)
print(f"kernels per H2 application: {cnt.value}", flush=True)
for i, op in enumerate(gc.operators[:2]):
    print(f"component {i}: levels {[M.shape[0] for M in op.matrices]} nnz/row "
          f"{[round(M.nnz / M.shape[0], 1) for M in op.matrices]}", flush=True)
    for k, lv in enumerate(op.level_dev):
        kind = "levels" if lv.get("levels") else ("rows" if lv.get("rows") else "wavefront")
        print(f"   level {k}: {kind}", flush=True)
