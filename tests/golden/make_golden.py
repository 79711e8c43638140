"""Generate the golden fixtures the parity tests pin against.

Runs the UNMODIFIED reference package (``mvamg`` from /root/reference/pkg/src,
read-only) in this container and records its inputs and outputs on the hot
path: the config-1 multi-vector V-cycle hierarchy, the bootstrap composite of
K-cycle components, and the outputs of ``MultigridOperator.apply`` /
``error_propagation`` / ``pcg`` / ``apply_composite_symmetrized`` /
``test_phase`` on seeded vectors.  The reference cannot travel to the GPU box,
so the fixtures are committed; this script is how they were made:

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py

Reference call sites: estimator.py:94-145 (fit/solve), cycles.py:150-184
(cycle, error propagation), krylov.py:28-107 (pcg/fcg), bootstrap.py:98-141
(composite, test phase), _kernels.py:15-38 (GS sweeps).
"""

import os
import sys

import numpy as np
import scipy.sparse as sp

sys.path.insert(0, os.environ.get("MVAMG_REF", "/root/reference/pkg/src"))

from mvamg import _kernels  # noqa: E402
from mvamg.bootstrap import apply_composite_symmetrized, test_phase  # noqa: E402
from mvamg.cycles import CycleSpec, MultigridOperator  # noqa: E402
from mvamg.estimator import MultiVectorAMG  # noqa: E402
from mvamg.krylov import pcg  # noqa: E402
from mvamg.pairwise import CoarseningParams, build_pairwise_hierarchy  # noqa: E402
from mvamg.problems import AnisotropySpec, assemble_diffusion_stiffness, generate_anisotropic_2d  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def put_csr(d, key, M):
    M = sp.csr_matrix(M)
    d[key + "_indptr"] = M.indptr.astype(np.int32)
    d[key + "_indices"] = M.indices.astype(np.int32)
    d[key + "_data"] = M.data.astype(np.float64)
    d[key + "_shape"] = np.asarray(M.shape, dtype=np.int64)


def put_hierarchy(d, prefix, op):
    d[prefix + "_nlev"] = np.int64(op.n_levels)
    for k, A in enumerate(op.matrices):
        if k > 0 or not (prefix[0] == "c" and prefix[1:].isdigit()):
            put_csr(d, f"{prefix}_A{k}", A)
    for k, P in enumerate(op.prolongators):
        put_csr(d, f"{prefix}_P{k}", P)


def composite_pcg(A, b, ops, rtol=1e-6, itmax=1000):
    """PCG preconditioned by the symmetrized multiplicative composite
    (1..r then r..1, x <- x + B_i(r - A x))."""

    def bsym(r):
        x = np.zeros_like(r)
        for op in list(ops) + list(reversed(ops)):
            x = x + op.apply(r - A @ x)
        return x

    return pcg(A, b, bsym, rtol=rtol, itmax=itmax)


def make_c1():
    d = {}
    A = assemble_diffusion_stiffness(np.eye(2), 128)
    est = MultiVectorAMG().fit(A)
    op = est.operator_
    n = A.shape[0]
    put_hierarchy(d, "mv", op)
    b = np.random.default_rng(0).uniform(-1.0, 1.0, n)
    d["b"] = b
    d["apply_b"] = op.apply(b)
    r1 = np.random.default_rng(1).standard_normal(n)
    d["r1"] = r1
    d["apply_r1"] = op.apply(r1)
    x2 = np.random.default_rng(2).standard_normal(n)
    d["x2"] = x2
    d["errprop_x2"] = op.error_propagation(x2)
    # bit-exact kernel goldens on the finest level
    A0 = op.matrices[0]
    d["spmv_A0_r1"] = A0 @ r1
    xf = np.zeros(n)
    _kernels.gs_forward(A0.indptr, A0.indices, A0.data, op.diagonals[0], b, xf)
    d["gsf_A0_b"] = xf
    xb = x2.copy()
    _kernels.gs_backward(A0.indptr, A0.indices, A0.data, op.diagonals[0], b, xb)
    d["gsb_A0_b_x2"] = xb
    for k in range(op.n_levels - 1):
        t = np.random.default_rng(10 + k).standard_normal(op.matrices[k].shape[0])
        d[f"restrict_in{k}"] = t
        d[f"restrict_out{k}"] = op.restrictions[k] @ t
        xc = np.random.default_rng(20 + k).standard_normal(op.matrices[k + 1].shape[0])
        d[f"prolong_in{k}"] = xc
        d[f"prolong_out{k}"] = op.prolongators[k] @ xc
    x, rep = est.solve(b, rtol=1e-6)
    d["pcg_x"] = x
    d["pcg_hist"] = rep.residual_history
    d["pcg_nit"] = np.int64(rep.iterations)
    d["rho_est"] = np.float64(est.estimate_convergence_factor())
    # smooth vectors (setup parity, later rows)
    d["smooth_vectors"] = np.stack(est.smooth_vectors_)
    # composite of K-cycle components (H2)
    comp = est.composite_
    d["n_comp"] = np.int64(comp.n_components)
    for c, component in enumerate(comp.components):
        put_hierarchy(d, f"c{c}", component.operator)
    ops = [c.operator for c in comp.components]
    r3 = np.random.default_rng(3).standard_normal(n)
    d["r3"] = r3
    d["kapply_c0_r3"] = ops[0].apply(r3)
    d["kapply_c3_r3"] = ops[-1].apply(r3)
    d["kerr_c1_r3"] = ops[1].error_propagation(r3)
    x4 = np.random.default_rng(4).uniform(-1.0, 1.0, n)
    d["x4"] = x4
    d["comp_x4"] = apply_composite_symmetrized(comp, x4)
    rep_t, w = test_phase(comp, A, 15, np.random.default_rng(5))
    d["testphase_anorms"] = rep_t.per_iteration_anorms
    d["testphase_w"] = w
    xh2, reph2 = composite_pcg(A, b, ops)
    d["h2pcg_x"] = xh2
    d["h2pcg_hist"] = reph2.residual_history
    d["h2pcg_nit"] = np.int64(reph2.iterations)
    # V-cycle components variant of H2 (strictly linear)
    vops = [MultigridOperator(c.hierarchy.matrices, c.hierarchy.prolongators, cycle=CycleSpec("V"))
            for c in comp.components]
    xh2v, reph2v = composite_pcg(A, b, vops)
    d["h2vpcg_hist"] = reph2v.residual_history
    d["h2vpcg_nit"] = np.int64(reph2v.iterations)
    np.savez_compressed(os.path.join(HERE, "c1.npz"), **d)
    print("c1:", rep.iterations, "its; H2:", reph2.iterations, "; H2-V:", reph2v.iterations,
          "; sizes", [M.shape[0] for M in op.matrices])


def laplacian_2d(grid):
    T = sp.diags([-np.ones(grid - 1), 2 * np.ones(grid), -np.ones(grid - 1)], [-1, 0, 1]).tocsr()
    eye = sp.eye(grid, format="csr")
    return (sp.kron(eye, T) + sp.kron(T, eye)).tocsr()


def make_small():
    d = {}
    # pairwise hierarchy on a 16x16 Laplacian (test_cycles.py:153-170 shape)
    A = laplacian_2d(16)
    h = build_pairwise_hierarchy(A, np.ones(A.shape[0]), CoarseningParams(min_coarse_size=8))
    v = MultigridOperator(h.matrices, h.prolongators, cycle=CycleSpec("V"))
    k2 = MultigridOperator(h.matrices, h.prolongators, cycle=CycleSpec("K", inner_fcg_iters=2))
    k1 = MultigridOperator(h.matrices, h.prolongators, cycle=CycleSpec("K", inner_fcg_iters=1))
    put_hierarchy(d, "lap16", v)
    r = np.random.default_rng(5).standard_normal(A.shape[0])
    d["lap16_r"] = r
    d["lap16_v"] = v.apply(r)
    d["lap16_k2"] = k2.apply(r)
    d["lap16_k1"] = k1.apply(r)
    x, rep = pcg(A, r, v.apply, rtol=1e-10)
    d["lap16_pcg_hist"] = rep.residual_history
    # anisotropic rotated (non-M-matrix) ANI2 32^2 two-level hierarchy
    A2 = generate_anisotropic_2d(AnisotropySpec(0.001, np.pi / 8, 32))
    h2 = build_pairwise_hierarchy(A2, np.ones(A2.shape[0]), CoarseningParams(min_coarse_size=40))
    v2 = MultigridOperator(h2.matrices, h2.prolongators, cycle=CycleSpec("V"))
    put_hierarchy(d, "ani2", v2)
    r2 = np.random.default_rng(6).standard_normal(A2.shape[0])
    d["ani2_r"] = r2
    d["ani2_v"] = v2.apply(r2)
    d["ani2_e"] = v2.error_propagation(r2)
    x, rep = pcg(A2, np.ones(A2.shape[0]), v2.apply, rtol=1e-8)
    d["ani2_pcg_hist"] = rep.residual_history
    d["ani2_pcg_x"] = x
    np.savez_compressed(os.path.join(HERE, "small.npz"), **d)
    print("small: lap16 levels", h.sizes(), "ani2 levels", h2.sizes())


if __name__ == "__main__":
    make_small()
    make_c1()
