"""Write the coarse-level matrices of a bench workload's hierarchy (hierarchy cache, or fitted here) to one
npz -- the input of tools/cluster_bench.py, cluster_trace.py and row_trace.py.

  python tools/dump_levels.py c3 scratch/c3_coarse.npz      # keys n{k}, ip{k}, ix{k}, v{k}, k >= 1
"""
import os
import sys

import numpy as np
import scipy.sparse as sp

sys.path.insert(0, ".")
import bench  # noqa: E402

name, out = sys.argv[1], sys.argv[2]
mats = bench.load_workload(name, setup=os.environ.get("MVAMG_SETUP", "gpu"))[0]
d = {}
for k, A in enumerate(mats):
    if k == 0:
        continue
    A = sp.csr_matrix(A)
    d[f"n{k}"] = A.shape[0]
    d[f"ip{k}"] = A.indptr.astype(np.int32)
    d[f"ix{k}"] = A.indices.astype(np.int32)
    d[f"v{k}"] = A.data
os.makedirs(os.path.dirname(os.path.abspath(out)), exist_ok=True)
np.savez(out, **d)
print(out, {k: int(v) for k, v in d.items() if k.startswith("n")})
