"""CPU-only setup (fit) -- TEST INFRASTRUCTURE ONLY.

bench.py's ``--impl reference`` arm must time the reference's CPU solve on a
hierarchy built without this repo's GPU library (libmvamg_b200.so is never
loaded in that process).  The reference itself cannot travel to the GPU box,
so this module runs the reference's setup algorithm on the host:

  bootstrap loop        pkg/src/mvamg/bootstrap.py:144-198 (restated below)
  test phase            pkg/src/mvamg/bootstrap.py:116-141 (restated below),
                        the symmetrized composite on the oracle's K-cycles
  a_norm                pkg/src/mvamg/sparse.py:69-82
  greedy matching       pkg/src/mvamg/matching.py:106-122 + _kernels.py:41-61
                        (oracle or_greedy_accept)
  local Jacobi SVD      pkg/src/mvamg/svd.py:17-55 + _kernels.py:64-121
                        (oracle or_jacobi_svd_batch)
  pairwise / multi-vector levels, Galerkin products: the numpy/scipy pieces of
  paper_1907_04417_b200/setup.py (bit-exact with the reference on its own
  inputs, tests/test_setup.py), with the scipy Galerkin recipe.

Only bench.py (reference arm / cpu_baseline) and tests/ import this file.
"""

import time

import numpy as np

from oracle.oracle import OracleOperator, lib, oracle_composite, oracle_dot, oracle_spmv, _ptr

from paper_1907_04417_b200 import setup as S
from paper_1907_04417_b200.exceptions import CoarseningStagnationError, NotSpdError


def host_matching(A, w, weight_floor=S.WEIGHT_FLOOR):
    """edge weights (matching.py:78-103) + the greedy (matching.py:106-122)."""
    i, j, c = S.edge_weights(A, w)
    keep = c > weight_floor
    ei, ej, ec = i[keep], j[keep], c[keep]
    order = np.lexsort((ej, ei, -ec))
    ei = np.ascontiguousarray(ei[order], dtype=np.int64)
    ej = np.ascontiguousarray(ej[order], dtype=np.int64)
    n = A.shape[0]
    partner = np.empty(max(1, n), dtype=np.int64)
    pi = np.empty(max(1, ei.shape[0]), dtype=np.int64)
    pj = np.empty(max(1, ei.shape[0]), dtype=np.int64)
    k = int(lib().or_greedy_accept(ei.shape[0], _ptr(ei), _ptr(ej), n, _ptr(partner), _ptr(pi), _ptr(pj)))
    pairs = np.stack([pi[:k], pj[:k]], axis=1) if k else np.empty((0, 2), dtype=np.int64)
    return pairs, np.flatnonzero(partner[:n] < 0).astype(np.int64)


def host_svd(rp, local, nv):
    """Batched jacobi_svd of the stacked aggregate blocks; (code, U, sigma, failed)."""
    import ctypes

    n_agg = rp.shape[0] - 1
    U = np.empty_like(local)
    sig = np.empty((n_agg, nv))
    failed = ctypes.c_int(-1)
    st = lib().or_jacobi_svd_batch(n_agg, _ptr(rp), nv, _ptr(np.ascontiguousarray(local)), S.SVD_MAX_SWEEPS,
                                   S.SVD_PAIR_TOL, _ptr(U), _ptr(sig), ctypes.byref(failed))
    return (0 if st == 0 else 3), U, sig, failed.value   # 3 = E_NOT_SPD: SvdConvergenceError


def a_norm(A, x):
    """sqrt(x' A x) with the reference's clamp / raise (sparse.py:69-82)."""
    Ax = oracle_spmv(A, x)
    quad = oracle_dot(x, Ax)
    if quad < 0.0:
        scale = float(np.sqrt(oracle_dot(x, x)) * np.sqrt(oracle_dot(Ax, Ax)))
        if quad < -1e-10 * max(scale, np.finfo(np.float64).tiny):
            raise NotSpdError(f"negative quadratic form x'Ax = {quad:.3e}; matrix is not SPD")
        quad = 0.0
    return float(np.sqrt(quad))


def test_phase(ops, A, nu, rng):
    """bootstrap.py:116-141 on the oracle composite: (rho, w or None)."""
    x = rng.uniform(-1.0, 1.0, size=A.shape[0])
    anorms = [a_norm(A, x)]
    for _ in range(nu):
        x = oracle_composite(ops, x)
        anorms.append(a_norm(A, x))
        if anorms[-1] == 0.0:
            break
    if anorms[-1] == 0.0:
        return 0.0, None
    return float(anorms[-1] / anorms[-2]), x / anorms[-1]


def fit_host(A, nsv=5, merge_levels=3, svd_tol=0.1, rho_des=0.8, maxstage=15, nu=15, steps_per_level=2,
             min_coarse_size=40, max_levels=20, seed=0, inner_fcg_iters=2, log=None):
    """MultiVectorAMG(...).fit(A) (estimator.py:94-136) on host cores only.
    Returns (matrices, prolongators, info)."""
    t0 = time.perf_counter()
    A = S.as_csr(A)
    n = A.shape[0]
    params = S.CoarseningParams(steps_per_level=steps_per_level, max_levels=max_levels,
                                min_coarse_size=min_coarse_size)
    w0 = np.ones(n)
    build = dict(product=S.galerkin_product, matcher=host_matching)
    if nsv == 1:
        pairwise, vectors, stages = S.build_pairwise_hierarchy(A, w0, params, **build), [w0], []
        hiers = []
    else:
        min_stages, maxstage = nsv - 1, max(maxstage, nsv - 1)
        rng = np.random.default_rng(seed)
        comps, hiers, vecs, stages = [], [], [w0], []
        rho, stage, stagnated_before = 1.0, 1, False
        while (rho >= rho_des or stage <= min_stages) and stage <= maxstage:
            try:
                hier = S.build_pairwise_hierarchy(A, vecs[-1], params, **build)
            except CoarseningStagnationError:
                if stagnated_before or not comps:
                    raise
                stagnated_before = True
                _, w_new = test_phase(comps, A, nu, rng)
                if w_new is None:
                    break
                vecs.append(w_new)
                continue
            stagnated_before = False
            hiers.append(hier)
            comps.append(OracleOperator(hier.matrices, hier.prolongators, cycle="K", inner_fcg_iters=inner_fcg_iters))
            rho, w_new = test_phase(comps, A, nu, rng)
            stages.append(rho)
            if log:
                log(f"stage {stage}: rho {rho:.4f} levels {hier.sizes()} ({time.perf_counter() - t0:.0f} s)")
            if w_new is None:
                break
            vecs.append(w_new)
            stage += 1
        n_use = min(nsv, len(comps) + 1)
        pairwise, vectors = hiers[n_use - 2], vecs[:n_use]
        del comps
    mvh = S.build_multivector_hierarchy(A, pairwise, vectors, merge_levels=merge_levels, tol=svd_tol,
                                        min_coarse_size=min_coarse_size, product=S.galerkin_product,
                                        svd=host_svd)
    info = {"fit_s": time.perf_counter() - t0, "bootstrap_stages": len(stages), "stage_rho": stages,
            "setup": "CPU-only (oracle/host_setup.py)",
            "components": [(list(h.matrices), list(h.prolongators)) for h in hiers]}
    return list(mvh.matrices), list(mvh.prolongator_matrices), info
