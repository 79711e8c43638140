"""Run the batched local SVD kernel once on C2-shaped aggregate blocks
(23,499 aggregates of 8-64 rows, k = 5 smooth-vector columns) for ncu:

  ncu --set full -k regex:jacobi_svd python tools/svd_probe.py
"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_1907_04417_b200.setup import _jacobi_svd_device  # noqa: E402

rng = np.random.default_rng(3)
sizes = rng.integers(8, 65, 23499)
rp = np.zeros(sizes.shape[0] + 1, dtype=np.int32)
np.cumsum(sizes, out=rp[1:])
x = np.arange(rp[-1]) / rp[-1]
local = np.ascontiguousarray(np.stack([np.cos(np.pi * (j + 1) * x) + 1e-3 * rng.standard_normal(x.shape)
                                       for j in range(5)], axis=1))
_jacobi_svd_device(rp, local, 5)
t0 = time.perf_counter()
code, U, sig, failed = _jacobi_svd_device(rp, local, 5)
print(f"blocks={sizes.shape[0]} rows={rp[-1]} code={code} {1e3 * (time.perf_counter() - t0):.2f} ms (with copies)")
