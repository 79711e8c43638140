"""Is the coarsest-level dense inverse the reason the C5 V-cycle diverges?
Fits (or loads the /tmp cache of tools/c5_debug.py), then on the host:
accuracy of inv = lu_solve(LU, I) on A_L, and r'z of the oracle cycle (LU
solve) against the GPU cycle (inverse GEMV)."""
import os
import pickle
import sys
import time

import numpy as np
import scipy.linalg

sys.path.insert(0, ".")
from paper_1907_04417_b200 import problems  # noqa: E402
from paper_1907_04417_b200.estimator import MultiVectorAMG  # noqa: E402

g = int(sys.argv[1]) if len(sys.argv) > 1 else 320
path = f"/tmp/jump3d_{g}.pkl"
if os.path.exists(path):
    with open(path, "rb") as f:
        mats, pros, b = pickle.load(f)
else:
    A = problems.jump_3d(g, 16, 1)
    b = problems.rhs_uniform(A.shape[0], 0)
    t = time.time()
    est = MultiVectorAMG().fit(A)
    print(f"fit {time.time() - t:.0f}s", flush=True)
    mats, pros = list(est.hierarchy_.matrices), list(est.hierarchy_.prolongator_matrices)
    with open(path, "wb") as f:
        pickle.dump((mats, pros, b), f, protocol=4)
Ac = mats[-1].toarray()
n = Ac.shape[0]
lu = scipy.linalg.lu_factor(Ac)
inv = scipy.linalg.lu_solve(lu, np.eye(n))
rng = np.random.default_rng(0)
v = rng.standard_normal(n)
f = Ac @ v
e_inv = np.linalg.norm(inv @ f - v) / np.linalg.norm(v)
e_lu = np.linalg.norm(scipy.linalg.lu_solve(lu, f) - v) / np.linalg.norm(v)
print(f"coarsest n={n}: cond~{np.linalg.cond(Ac):.2e}  inverse err {e_inv:.2e}  lu_solve err {e_lu:.2e}", flush=True)
# refinement with the inverse
x = inv @ f
for k in range(4):
    x = x + inv @ (f - Ac @ x)
    print(f"  refinement {k + 1}: err {np.linalg.norm(x - v) / np.linalg.norm(v):.2e}", flush=True)
sys.path.insert(0, "tests")
from oracle.oracle import OracleOperator  # noqa: E402
op = OracleOperator(mats, pros)
t = time.time()
z = op.apply(b)
print(f"oracle cycle ({time.time() - t:.1f}s): r'z = {np.dot(b, z):.6e} |z| = {np.linalg.norm(z):.3e}", flush=True)
