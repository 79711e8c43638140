import sys
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import numpy as np, torch
from _fixtures import golden, hierarchy
from paper_1907_04417_b200.device import DeviceGsLevels, GpuConfig, time_sweep
mats, pros = hierarchy(golden("c1"), "mv")
for k in (1, 2):
    A = mats[k]
    n = A.shape[0]
    for m in (0,):
        for cfg in (GpuConfig(), GpuConfig(level_reg=False), GpuConfig(exact_gs=True)):
            lv = DeviceGsLevels(A, m, cfg)
            b = torch.randn(n, dtype=torch.float64, device="cuda")
            xn = torch.empty(n, dtype=torch.float64, device="cuda")
            ws = torch.zeros(8, dtype=torch.int32, device="cuda")
            t = time_sweep(lambda: lv.sweep(b, None, xn, ws), reps=20)
            print(k, m, "reg", lv.reg, "group", lv.group, "threads", lv.threads, "nlev", lv.nlev, "maxrows", lv.max_rows,
                  "maxents", lv.max_ents, f"{t*1e6:.1f} us {t*1e6/lv.nlev:.2f} us/level", flush=True)
