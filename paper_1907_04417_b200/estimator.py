"""MultiVectorAMG facade on the GPU -- mirror of pkg/src/mvamg/estimator.py:24-156.

fit(A) runs the setup (bootstrap with GPU test phases, then the single
multi-vector hierarchy) and uploads the V-cycle to the device; solve(b) runs
PCG fully on the device; aspreconditioner() / estimate_convergence_factor()
keep the reference's semantics.
"""

import numpy as np

from .composite import DeviceANorm
from .cycles import CycleSpec, GpuMultigridOperator
from .device import GpuConfig, to_device
from .krylov import pcg
from .setup import (BootstrapParams, CoarseningParams, bootstrap_run, build_multivector_hierarchy, coarse_product,
                    build_pairwise_hierarchy, operator_complexity)


def _check_operator(A):
    """pkg/src/mvamg/validation.py:10-26: square, finite, exactly symmetric, positive diagonal."""
    from .device import as_csr
    from .exceptions import NotSpdError

    A = as_csr(A)
    if A.shape[0] != A.shape[1]:
        raise ValueError(f"operator must be square, got {A.shape[0]}x{A.shape[1]}")
    if A.nnz and not np.all(np.isfinite(A.data)):
        raise ValueError("operator contains NaN or Inf entries")
    if (A != A.T).nnz != 0:
        raise NotSpdError("operator is not symmetric")
    if (A.diagonal() <= 0.0).any():
        raise NotSpdError("operator diagonal must be strictly positive")
    return A


def _check_vector(x, n=None, name="vector"):
    x = np.asarray(x, dtype=np.float64)
    if x.ndim != 1:
        raise ValueError(f"{name} must be 1-d, got shape {x.shape}")
    if n is not None and x.shape[0] != n:
        raise ValueError(f"{name} has length {x.shape[0]}, expected {n}")
    if not np.all(np.isfinite(x)):
        raise ValueError(f"{name} contains NaN or Inf entries")
    return x



def _device_svd(config):
    """Whether the multi-vector setup runs its local SVDs on the GPU."""
    return (config or GpuConfig()).device_svd

class MultiVectorAMG:
    """AMG preconditioner folding adaptively generated smooth vectors into one
    aggregation hierarchy (parameters as pkg/src/mvamg/estimator.py:61-85)."""

    _params = ("nsv", "merge_levels", "svd_tol", "rho_des", "maxstage", "nu", "steps_per_level",
               "min_coarse_size", "max_levels", "seed", "workers")

    def __init__(self, nsv=5, merge_levels=3, svd_tol=0.1, rho_des=0.8, maxstage=15, nu=15,
                 steps_per_level=2, min_coarse_size=40, max_levels=20, seed=0, workers=1, config=None):
        self.nsv = nsv
        self.merge_levels = merge_levels
        self.svd_tol = svd_tol
        self.rho_des = rho_des
        self.maxstage = maxstage
        self.nu = nu
        self.steps_per_level = steps_per_level
        self.min_coarse_size = min_coarse_size
        self.max_levels = max_levels
        self.seed = seed
        self.workers = workers
        self.config = config

    def get_params(self, deep=True):
        return {k: getattr(self, k) for k in self._params}

    def set_params(self, **kw):
        for k, v in kw.items():
            if k not in self._params:
                raise ValueError(f"unknown parameter {k!r}")
            setattr(self, k, v)
        return self

    def _coarsening(self):
        return CoarseningParams(steps_per_level=self.steps_per_level, max_levels=self.max_levels,
                                min_coarse_size=self.min_coarse_size)

    def fit(self, A, y=None):
        if self.nsv < 1:
            raise ValueError("nsv must be >= 1")
        A = _check_operator(A)
        w0 = np.ones(A.shape[0])
        if self.nsv == 1:
            from .device import GpuConfig

            pairwise = build_pairwise_hierarchy(A, w0, self._coarsening(), product=coarse_product(self.config),
                                                device_matching=(self.config or GpuConfig()).device_matching)
            self.composite_ = None
            vectors = [w0]
        else:
            params = BootstrapParams(rho_des=self.rho_des, maxstage=max(self.maxstage, self.nsv - 1), nu=self.nu,
                                     rng_seed=self.seed, min_stages=self.nsv - 1, coarsening=self._coarsening())
            self.composite_ = bootstrap_run(A, w0, params, config=self.config)
            n_use = min(self.nsv, self.composite_.n_components + 1)
            pairwise = self.composite_.components[n_use - 2].hierarchy
            vectors = self.composite_.smooth_vectors[:n_use]
        self.hierarchy_ = build_multivector_hierarchy(A, pairwise, vectors, merge_levels=self.merge_levels,
                                                      tol=self.svd_tol, min_coarse_size=self.min_coarse_size,
                                                      product=coarse_product(self.config),
                                                      device_svd=_device_svd(self.config))
        self.operator_ = GpuMultigridOperator(self.hierarchy_.matrices, self.hierarchy_.prolongator_matrices,
                                              cycle=CycleSpec("V"), config=self.config)
        self.smooth_vectors_ = vectors
        self.matrix_ = A
        self.n_levels_ = self.hierarchy_.nl
        self.operator_complexity_ = operator_complexity(self.hierarchy_.matrices)
        sizes = self.hierarchy_.sizes()
        self.coarsening_factor_ = float(np.mean([sizes[k - 1] / sizes[k] for k in range(1, len(sizes))])) \
            if len(sizes) > 1 else 1.0
        return self

    def _fitted(self):
        if not hasattr(self, "operator_"):
            raise RuntimeError("MultiVectorAMG instance is not fitted yet; call fit first")

    def solve(self, b, rtol=1e-6, itmax=1000, x0=None):
        """PCG with the fitted V-cycle (estimator.py:138-145), on the device."""
        self._fitted()
        b = _check_vector(b, n=self.matrix_.shape[0], name="right-hand side")
        return pcg(self.matrix_, b, self.operator_, rtol=rtol, itmax=itmax, x0=x0)

    def aspreconditioner(self):
        self._fitted()
        return self.operator_.as_linear_operator()

    def estimate_convergence_factor(self, applications=10, seed=None):
        """Last-ratio energy-norm estimate of the V-cycle's error propagation
        (pkg/src/mvamg/bench.py:103-116), iterations on the device."""
        self._fitted()
        seed = self.seed + 1 if seed is None else seed
        rng = np.random.default_rng(seed)
        x = to_device(rng.uniform(-1.0, 1.0, size=self.matrix_.shape[0]))
        norm = DeviceANorm(self.operator_._dA[0])
        prev, ratio = norm(x), 0.0
        for _ in range(applications):
            x = self.operator_.error_propagation_device(x)
            cur = norm(x)
            if cur == 0.0:
                return 0.0
            ratio, prev = cur / prev, cur
        self.operator_._status("estimate_convergence_factor")
        return float(ratio)
