"""One small sweep of every GS kernel variant plus one V-cycle, K-cycle and
composite application -- the workload for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck):

  compute-sanitizer --tool racecheck python tools/sanitize_gs.py

Each sweep is also checked against the CPU oracle -- bit for bit for the
exact-order schedules, within 1e-12 for the tolerance-mode ones ("-G") -- so a
run that the sanitizer passes is a correct run too."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from _fixtures import golden, hierarchy, laplacian_2d, laplacian_3d, random_spd_csr  # noqa: E402
from oracle.oracle import oracle_gs  # noqa: E402

import paper_1907_04417_b200 as mv  # noqa: E402
from paper_1907_04417_b200.device import (DeviceGsCluster, DeviceGsLevels, DeviceGsPlan, DeviceGsRows,  # noqa: E402
                                          DeviceGsStream, GpuConfig, to_device)

rng = np.random.default_rng(0)
cases = [("lap2d", laplacian_2d(24).tocsr()), ("lap3d", laplacian_3d(8).tocsr()),
         ("rand", random_spd_csr(300, density=0.03, seed=1))]
ok = True


def dev(a):
    return to_device(np.asarray(a, dtype=np.float64))


for name, A in cases:
    n = A.shape[0]
    b, x0 = rng.standard_normal(n), rng.standard_normal(n)
    ws = torch.zeros(8, dtype=torch.int32, device="cuda")
    for direction in ("forward", "backward"):
        want = x0.copy()
        oracle_gs(A, b, want, direction)
        want0 = np.zeros(n)
        oracle_gs(A, b, want0, direction)
        d = 0 if direction == "forward" else 1
        runs = []
        for cfg in (GpuConfig(exact_gs=True), GpuConfig(exact_gs=True, generic_gs=True)):
            gp = DeviceGsPlan(A, cfg)
            runs.append((f"wavefront{'-generic' if cfg.generic_gs else ''}", lambda xn, gp=gp: gp.sweep(d, dev(b), dev(x0), xn, ws), want))
        lv = DeviceGsLevels(A, 2 * d + 1, GpuConfig(exact_gs=True))
        runs.append(("level-set", lambda xn, lv=lv: lv.sweep(dev(b), dev(x0), xn, ws), want))
        rw = DeviceGsRows(A, 2 * d + 1, GpuConfig(exact_gs=True))
        runs.append(("row", lambda xn, rw=rw: rw.sweep(dev(b), dev(x0), xn, ws), want))
        st = DeviceGsStream(A, 2 * d + 1, GpuConfig(exact_gs=True))
        runs.append(("stream", lambda xn, st=st: st.sweep(dev(b), dev(x0), xn, ws), want))
        st0 = DeviceGsStream(A, 2 * d, GpuConfig(exact_gs=False))
        runs.append(("stream-G", lambda xn, st=st0: st.sweep(dev(b), None, xn, ws), want0))
        # cluster / grid dataflow sweeps (tolerance mode: fixed tree + ordered tail, within rounding of the oracle)
        for what, kw in (("cluster", dict(ncta=4, wpc=4)), ("cluster-16", dict(ncta=16, wpc=8)),
                         ("grid", dict(grid=True, ncta=37, wpc=5))):
            c1 = DeviceGsCluster(A, 2 * d + 1, GpuConfig(), **kw)
            runs.append((f"{what}-G", lambda xn, c1=c1: c1.sweep(dev(b), dev(x0), xn, ws), want))
            c0 = DeviceGsCluster(A, 2 * d, GpuConfig(), **kw)
            runs.append((f"{what}-zero-G", lambda xn, c0=c0: c0.sweep(dev(b), None, xn, ws), want0))
        for what, fn, ref in runs:
            xn = torch.empty(n, dtype=torch.float64, device="cuda")
            fn(xn)
            torch.cuda.synchronize()
            got = xn.cpu().numpy()
            good = (np.array_equal(got, ref) if not what.endswith("-G") else
                    np.max(np.abs(got - ref)) <= 1e-12 * np.max(np.abs(ref)))
            ok &= bool(good)
            print(f"{name:6s} {direction:8s} {what:18s} {'ok' if good else 'MISMATCH'}", flush=True)

d = golden("c1")
mats, pros = hierarchy(d, "mv")
for cfg in (GpuConfig(), GpuConfig(exact_gs=True)):
    op = mv.GpuMultigridOperator(mats, pros, config=cfg)
    z = op.apply(d["b"])
    e = float(np.max(np.abs(z - d["apply_b"])) / np.max(np.abs(d["apply_b"])))
    ok &= e <= 1e-10
    print(f"V-cycle exact_gs={cfg.exact_gs}: rel {e:.2e}", flush=True)
comps = [hierarchy(d, f"c{c}", fine=mats[0]) for c in range(int(d["n_comp"]))]
ops = [mv.GpuMultigridOperator(m, p, cycle=mv.CycleSpec("K", 2)) for m, p in comps]
c = mv.GpuComposite(ops)
y = c.apply_symmetrized(d["x4"])
e = float(np.max(np.abs(y - d["comp_x4"])) / np.max(np.abs(d["comp_x4"])))
ok &= e <= 1e-9
print(f"composite: rel {e:.2e}", flush=True)
print("ALL OK" if ok else "FAILURES", flush=True)
sys.exit(0 if ok else 1)
