"""Time the device Galerkin product (csrc/galerkin.cuh) against the reference's
scipy recipe on C2's fine operator with a block prolongator of the reference's
shape (8x8 aggregates, 5 vectors), and check the result bit for bit.

  python tools/galerkin_bench.py [--grid 1024] [--reps 3]
"""
import argparse
import os
import sys
import time

import numpy as np
import scipy.sparse as sp

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1907_04417_b200 import problems  # noqa: E402
from paper_1907_04417_b200.device import galerkin_product_device  # noqa: E402
from paper_1907_04417_b200.setup import galerkin_product  # noqa: E402


def block_p(g, agg=8, nsv=5, seed=0):
    rng = np.random.default_rng(seed)
    n = g * g
    ii, jj = np.divmod(np.arange(n), g)
    aid = (ii // agg) * (g // agg) + jj // agg
    return sp.csr_matrix((rng.standard_normal(n * nsv), (np.repeat(np.arange(n), nsv),
                                                         (aid[:, None] * nsv + np.arange(nsv)).ravel())),
                         shape=(n, (g // agg) ** 2 * nsv))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", type=int, default=1024)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    A = problems.anisotropic_q1(a.grid)
    P = block_p(a.grid)
    G = galerkin_product_device(P, A)
    for _ in range(a.reps):
        t = {}
        G = galerkin_product_device(P, A, timing=t)
        print("device", {k: round(v, 3) for k, v in t.items()})
    t0 = time.perf_counter()
    H = galerkin_product(P, A)
    print(f"scipy {1e3 * (time.perf_counter() - t0):.1f} ms")
    same = np.array_equal(G.indptr, H.indptr) and np.array_equal(G.indices, H.indices) and \
        np.array_equal(G.data, H.data)
    print("bit_exact", same, "nnz", G.nnz)


if __name__ == "__main__":
    main()
