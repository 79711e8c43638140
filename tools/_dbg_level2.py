import sys
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import numpy as np, torch, scipy.sparse as sp
from _fixtures import laplacian_1d
from paper_1907_04417_b200.device import DeviceGsLevels, GpuConfig, time_sweep
for name, A in (("diag500", sp.diags(np.full(500, 2.0)).tocsr()), ("lap1d_500", laplacian_1d(500)),
                ("lap1d_2000", laplacian_1d(2000))):
    n = A.shape[0]
    for cfg in (GpuConfig(), GpuConfig(level_reg=False), GpuConfig(exact_gs=True)):
        lv = DeviceGsLevels(A, 0, cfg)
        b = torch.randn(n, dtype=torch.float64, device="cuda")
        xn = torch.empty(n, dtype=torch.float64, device="cuda")
        ws = torch.zeros(8, dtype=torch.int32, device="cuda")
        t = time_sweep(lambda: lv.sweep(b, None, xn, ws), reps=20)
        print(name, "reg", lv.reg, "group", lv.group, "threads", lv.threads, "nlev", lv.nlev,
              f"{t*1e6:.1f} us {t*1e6/lv.nlev:.3f} us/level", flush=True)
