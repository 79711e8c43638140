"""Cluster dataflow GS sweep (gs_cluster.cuh) against the row / streamed sweeps
on the coarse levels of a hierarchy dump (GPU).

  python tools/dump_levels.py c3 scratch/c3_coarse.npz
  python tools/cluster_bench.py scratch/c3_coarse.npz [levels=1,2,3] [grid=1] [small=1] [sleeps=0,50]

Per level and sweep (forward from x=0, folded backward from x_old): CUDA-event
times of the row / streamed schedule and of the cluster sweep (default shape,
or a grid of cluster sizes / worker warps / poll back-offs with grid=1), its
error against the oracle's serial sweep and a run-to-run identity check."""
import sys

import numpy as np
import scipy.sparse as sp
import torch

sys.path.insert(0, ".")
from paper_1907_04417_b200.device import (DeviceGsCluster, DeviceGsRows, DeviceGsStream, GpuConfig,  # noqa: E402
                                          cluster_shape)  # noqa: F401
from oracle.oracle import oracle_gs  # noqa: E402


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


def main():
    path = sys.argv[1]
    kw = dict(a.split("=") for a in sys.argv[2:])
    z = np.load(path)
    ks = sorted(int(k[1:]) for k in z.files if k.startswith("n"))
    if "levels" in kw:
        ks = [int(x) for x in kw["levels"].split(",")]
    grid = kw.get("grid", "0") == "1"
    for k in ks:
        n = int(z[f"n{k}"])
        M = sp.csr_matrix((z[f"v{k}"], z[f"ix{k}"], z[f"ip{k}"]), shape=(n, n))
        g = torch.Generator(device="cuda").manual_seed(k)
        b = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
        xo = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
        xn = torch.empty(n, dtype=torch.float64, device="cuda")
        ws = torch.zeros(8, dtype=torch.int32, device="cuda")
        bh, xoh = b.cpu().numpy(), xo.cpu().numpy()
        ref = {0: oracle_gs(M, bh, np.zeros(n), "forward"), 2: oracle_gs(M, bh, xoh, "backward")}
        for mode in (0, 2):
            xold = xo if mode == 2 else None
            cfg = GpuConfig()
            rows = DeviceGsRows(M, mode, cfg)
            t_rows = timed(lambda: rows.sweep(b, xold, xn, ws))
            line = f"level {k} n={n} mode {mode}: row sweep {t_rows:.1f} us"
            if n <= cfg.stream_max_rows:
                st = DeviceGsStream(M, mode, cfg)
                t_st = timed(lambda: st.sweep(b, xold, xn, ws, fold=(mode == 2)))
                line += f" | stream {t_st:.1f} us"
            print(line, flush=True)
            rows.sweep(b, xold, xn, ws)
            torch.cuda.synchronize()
            x_rows = xn.cpu().numpy().copy()
            shapes = [None]
            sleeps = [cfg.cluster_sleep_ns]
            if grid:
                if kw.get("small", "0") == "1":
                    shapes = [(False, c, w) for c in (1, 2, 4, 8, 16) for w in (4, 8, 16, 32)]
                else:
                    shapes = ([(False, c, w) for c in (16,) for w in (16, 32)] +
                              [(True, c, w) for c in (74, 148) for w in (8, 16, 32)])
                sleeps = [0]
            if "sleeps" in kw:
                sleeps = [int(x) for x in kw["sleeps"].split(",")]
            best = None
            for shape in shapes:
                try:
                    cl = (DeviceGsCluster(M, mode, cfg) if shape is None else
                          DeviceGsCluster(M, mode, cfg, grid=shape[0], ncta=shape[1], wpc=shape[2]))
                except ValueError:
                    continue
                shape = (cl.ncta, cl.wpc, int(cl.grid))
                for sl in sleeps:
                    cl.sleep_ns = sl
                    xn.fill_(0.0)
                    cl.sweep(b, xold, xn, ws)
                    torch.cuda.synchronize()
                    assert int(ws[1].item()) == 0, "timeout"
                    x1 = xn.clone()
                    cl.sweep(b, xold, xn, ws)
                    torch.cuda.synchronize()
                    assert torch.equal(x1, xn), "not reproducible"
                    err = np.max(np.abs(xn.cpu().numpy() - ref[mode])) / np.max(np.abs(ref[mode]))
                    dr = np.max(np.abs(xn.cpu().numpy() - x_rows)) / np.max(np.abs(ref[mode]))
                    t = timed(lambda: cl.sweep(b, xold, xn, ws))
                    if best is None or t < best[0]:
                        best = (t, shape, sl)
                    print(f"   cluster {shape[0]:2d} x {shape[1]:2d} warps grid {shape[2]} sleep {sl:3d}: {t:7.1f} us "
                          f"({t * 1e3 / cl.nlev:.0f} ns/level) rel err vs serial {err:.1e} vs row sweep {dr:.1e}",
                          flush=True)
                del cl
            if best:
                print(f"   best {best[1]} sleep {best[2]}: {best[0]:.1f} us = {t_rows / best[0]:.2f}x the row sweep",
                      flush=True)


if __name__ == "__main__":
    main()
