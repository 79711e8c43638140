"""Per-level GS sweep timing (CUDA events) for a bench workload: warm (L2-hot)
and cold (after a 256 MiB L2 flush).  Prints one line per level."""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1907_04417_b200 as mv  # noqa: E402
from paper_1907_04417_b200 import _lib  # noqa: E402
from paper_1907_04417_b200.device import ptr, stream_handle  # noqa: E402


def load(cfg):
    if cfg.startswith("lap1d"):
        import scipy.sparse as sp
        n = int(cfg[5:] or 4096)
        A = sp.diags([-np.ones(n - 1), 2 * np.ones(n), -np.ones(n - 1)], [-1, 0, 1]).tocsr()
        return [A, sp.eye(1).tocsr()], [sp.csr_matrix(np.ones((n, 1)))], np.ones(n), "lap1d"
    return bench.load_workload(cfg)


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c1"
    kw = dict(a.split("=") for a in sys.argv[2:])
    conf = mv.GpuConfig(**{k: (v == "1" if k == "generic_gs" else int(v)) for k, v in kw.items()})
    mats, pros, b, desc = load(cfg)
    op = mv.GpuMultigridOperator(mats, pros, config=conf)
    L = _lib.load()
    s = stream_handle()
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    stream = torch.cuda.current_stream()
    for k, lv in enumerate(op.level_dev):
        A = mats[k]
        if lv.get("levels") is not None:
            import torch as _t
            n = A.shape[0]
            bb = _t.randn(n, dtype=_t.float64, device="cuda")
            xo = _t.randn(n, dtype=_t.float64, device="cuda")
            xn = _t.empty(n, dtype=_t.float64, device="cuda")
            ws = _t.zeros(8, dtype=_t.int32, device="cuda")
            res = {}
            modes = dict(lv["levels"])
            if 2 in modes:
                modes[3] = modes[2]
            for m, s in sorted(modes.items()):
                def once():
                    s.sweep(bb, None if m % 2 == 0 else xo, xn, ws, fold=(m == 3))
                for _ in range(3):
                    once()
                for mode in ("warm", "cold"):
                    tot = 0.0
                    for _ in range(20):
                        if mode == "cold":
                            flush.fill_(1.0)
                        e0 = _t.cuda.Event(enable_timing=True); e1 = _t.cuda.Event(enable_timing=True)
                        e0.record(stream); once(); e1.record(stream); e1.synchronize()
                        tot += e0.elapsed_time(e1)
                    res[(m, mode)] = tot / 20 * 1e3
            desc = " | ".join(f"mode{m} warm {res[(m,'warm')]:.1f}us cold {res[(m,'cold')]:.1f}us" for m in sorted(modes))
            s0 = next(iter(lv["levels"].values()))
            print(f"level {k}: n={n} nnz={A.nnz} LEVEL-SET nlev={s0.nlev} thr={s0.threads} | {desc} | "
                  f"{res[(0,'warm')]*1e3/s0.nlev:.0f} ns/level", flush=True)
            continue
        n = A.shape[0]
        plan = lv["plan"]
        dA = lv["A"]
        bb = torch.randn(n, dtype=torch.float64, device="cuda")
        xo = torch.randn(n, dtype=torch.float64, device="cuda")
        xn = torch.empty(n, dtype=torch.float64, device="cuda")
        ws = torch.zeros(8, dtype=torch.int32, device="cuda")
        wk = torch.empty(n, dtype=torch.float64, device="cuda")
        res = {}
        gp = lv["gs"]
        for direction, zero in ((0, 1), (1, 0)):
            def once():
                gp.sweep(direction, bb, None if zero else xo, xn, ws, s, work=wk)
            for _ in range(3):
                once()
            for mode in ("warm", "cold"):
                tot = 0.0
                for _ in range(20):
                    if mode == "cold":
                        flush.fill_(1.0)
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                    once()
                    e1.record(stream)
                    e1.synchronize()
                    tot += e0.elapsed_time(e1)
                res[(direction, mode)] = tot / 20 * 1e3
            assert int(ws[1].item()) == 0
        # one traced forward sweep
        trace = torch.zeros(16 * 148 * 8 * 8, dtype=torch.int64, device="cuda")
        L.mvamg_gs_set_trace(ptr(trace))
        gp.sweep(0, bb, None, xn, ws, s)
        torch.cuda.synchronize()
        L.mvamg_gs_set_trace(None)
        tr = trace.view(-1, 16).cpu().numpy()
        tr = tr[tr[:, 6] > 0]
        rounds, spins, span = tr[:, 0].sum(), tr[:, 1].sum(), tr[:, 5].sum()
        ph = tr[:, 8:16].sum(axis=0) / max(rounds, 1)
        if ph.sum() > 0:
            print("  phases/round: wait %.0f hdr %.0f gather %.0f sum %.0f div+pub %.0f chunkend %.0f . issue %.0f" %
                  (ph[0], ph[1], ph[2], ph[3], ph[4], ph[5], ph[7]))
        print(f"  trace fwd: warps={len(tr)} rounds/warp={rounds/len(tr):.0f} spins/round={spins/max(rounds,1):.2f} "
              f"span/warp={span/len(tr):.0f}cyc cyc/round={span/max(rounds,1):.0f}", flush=True)
        print(f"level {k}: n={n} nnz={A.nnz} chains={plan.nchains} tiles={plan.ntiles} thr={plan.threads} C={plan.lean_C} R={plan.R} D={plan.D} "
              f"win={plan.window} depth={plan.depth} | fwd warm {res[(0,'warm')]:.1f}us cold {res[(0,'cold')]:.1f}us"
              f" | bwd warm {res[(1,'warm')]:.1f}us cold {res[(1,'cold')]:.1f}us | "
              f"fwd warm {res[(0,'warm')]*1e3/max(plan.depth,1):.0f} ns/level", flush=True)


if __name__ == "__main__":
    main()
