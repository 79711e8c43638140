"""Repeat the device Galerkin product many times on several operand shapes
and check every result is identical (hunting intermittent faults)."""
import sys
import time

import numpy as np
import scipy.sparse as sp

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from _galerkin_cases import aggregation_case, cancellation_case, overflow_case  # noqa: E402
from paper_1907_04417_b200 import problems  # noqa: E402
from paper_1907_04417_b200.device import galerkin_product_device  # noqa: E402
from paper_1907_04417_b200.setup import galerkin_product  # noqa: E402


def block_p(n, agg, nsv, seed):
    rng = np.random.default_rng(seed)
    aid = np.arange(n) // agg
    na = aid.max() + 1
    return sp.csr_matrix((rng.standard_normal(n * nsv), (np.repeat(np.arange(n), nsv),
                                                         (aid[:, None] * nsv + np.arange(nsv)).ravel())),
                         shape=(n, na * nsv))


reps = int(sys.argv[1]) if len(sys.argv) > 1 else 100
Ael = problems.elasticity_q1(96)
cases = [("elast_block", block_p(Ael.shape[0], 16, 4, 1), Ael), ("overflow", *overflow_case()),
         ("agg", *aggregation_case()), ("cancel", *cancellation_case(1)),
         ("jump", block_p(problems.jump_3d(24, 8, 1).shape[0], 27, 5, 2), problems.jump_3d(24, 8, 1))]
for name, P, A in cases:
    ref = galerkin_product(P, A)
    t = time.time()
    for r in range(reps):
        G = galerkin_product_device(P, A)
        ok = (np.array_equal(G.indptr, ref.indptr) and np.array_equal(G.indices, ref.indices)
              and np.array_equal(G.data, ref.data))
        if not ok:
            print(f"{name}: MISMATCH at rep {r}", flush=True)
            break
    print(f"{name}: {reps} reps ok={ok} ({time.time() - t:.1f}s)", flush=True)
