"""Device-resident multigrid operator -- drop-in for the reference's
``MultigridOperator`` (pkg/src/mvamg/cycles.py:100-190).

Same constructor (matrices, prolongators, cycle, pre_smoother, post_smoother),
same validation and exceptions, same duck-typed surface (.apply, __call__,
.error_propagation, .as_linear_operator, .n_levels, .shape, .matrices,
.prolongators, .restrictions, .diagonals).  The hierarchy is uploaded once to
HBM; each application runs one V- or K-cycle in libmvamg_b200.so.
"""

import ctypes
import dataclasses
from dataclasses import dataclass

import numpy as np
import scipy.linalg
import scipy.sparse.linalg as spla

from . import _lib
from .device import (DeviceCSR, DeviceGsCluster, DeviceGsLevels, DeviceGsPlan, DeviceGsRows, DeviceGsStream, GpuConfig,
                     as_csr,
                     stream_ctas,
                     autotune_coarse_gs,
                     level_gs_fits, ptr, row_gs_fits,
                     stream_handle, to_device, torch_cuda)
from .exceptions import NotSpdError

GS_FORWARD = "gauss_seidel_forward"
GS_BACKWARD = "gauss_seidel_backward"
WEIGHTED_JACOBI = "weighted_jacobi"
_KIND = {GS_FORWARD: _lib.GS_FORWARD, GS_BACKWARD: _lib.GS_BACKWARD, WEIGHTED_JACOBI: _lib.WEIGHTED_JACOBI}


@dataclass(frozen=True)
class SmootherSpec:
    """Mirror of cycles.py:28-40."""

    kind: str = GS_FORWARD
    sweeps: int = 1
    omega: float = 1.0

    def __post_init__(self):
        if self.kind not in (GS_FORWARD, GS_BACKWARD, WEIGHTED_JACOBI):
            raise ValueError(f"unknown smoother kind {self.kind!r}")
        if self.kind == WEIGHTED_JACOBI and not 0.0 < self.omega < 2.0:
            raise ValueError("weighted Jacobi requires omega in (0, 2)")
        if self.sweeps < 0:
            raise ValueError("sweeps must be >= 0")


@dataclass(frozen=True)
class CycleSpec:
    """Mirror of cycles.py:43-52."""

    kind: str = "V"
    inner_fcg_iters: int = 2

    def __post_init__(self):
        if self.kind not in ("V", "K"):
            raise ValueError(f"unknown cycle kind {self.kind!r}")
        if self.inner_fcg_iters < 0:
            raise ValueError("inner_fcg_iters must be >= 0")


def _checked_diagonal(A):
    d = A.diagonal()
    if np.any(d == 0.0):
        raise NotSpdError("zero diagonal entry; Gauss-Seidel/Jacobi undefined")
    return d


def coarse_pinv(Ac, rtol):
    """Truncated-eigen pseudo-inverse of a symmetric dense matrix: eigenvalues
    at or below rtol * lambda_max are dropped (row-major float64)."""
    w, Q = np.linalg.eigh(Ac)
    keep = w > rtol * w[-1]
    return np.ascontiguousarray((Q[:, keep] / w[keep]) @ Q[:, keep].T)


class GpuMultigridOperator:
    """Prepared B^{-1} on the GPU for a hierarchy of (matrices, prolongators)."""

    def __init__(self, matrices, prolongators, cycle=None, pre_smoother=None, post_smoother=None,
                 config=None):
        if len(matrices) != len(prolongators) + 1:
            raise ValueError("need exactly one prolongator per coarse level")
        self.matrices = [as_csr(A) for A in matrices]
        self.prolongators = [as_csr(P) for P in prolongators]
        self.restrictions = [P.T.tocsr() for P in self.prolongators]
        for R in self.restrictions:
            R.sort_indices()
        for k, P in enumerate(self.prolongators):
            if P.shape[0] != self.matrices[k].shape[0] or P.shape[1] != self.matrices[k + 1].shape[0]:
                raise ValueError(f"prolongator {k} does not chain the level dimensions")
        self.cycle = cycle or CycleSpec()
        self.pre_smoother = pre_smoother or SmootherSpec(GS_FORWARD)
        self.post_smoother = post_smoother or SmootherSpec(GS_BACKWARD)
        for spec in (self.pre_smoother, self.post_smoother):
            if spec.kind not in _KIND:
                raise ValueError(f"unknown smoother kind {spec.kind!r}")
        if self.cycle.kind not in ("V", "K"):
            raise ValueError(f"unknown cycle kind {self.cycle.kind!r}")
        self.diagonals = [_checked_diagonal(A) for A in self.matrices[:-1]]
        self.config = config or GpuConfig()
        self._h = None
        self._upload()

    @classmethod
    def from_reference(cls, op, config=None):
        """Wrap an existing reference MultigridOperator (duck-typed)."""
        return cls(op.matrices, op.prolongators, cycle=op.cycle, pre_smoother=op.pre_smoother,
                   post_smoother=op.post_smoother, config=config)

    def _gs_modes(self):
        """GS record modes the cycle needs (0 fwd from x=0, 1 fwd, 2 bwd)."""
        modes = set()
        for spec, first_zero in ((self.pre_smoother, True), (self.post_smoother, False)):
            if spec.kind == WEIGHTED_JACOBI or spec.sweeps == 0:
                continue
            if spec.kind == GS_BACKWARD:
                modes.add(2)
            else:
                modes.add(0 if first_zero else 1)
                if first_zero and spec.sweeps > 1:
                    modes.add(1)
        return sorted(modes)

    def _gs_level_modes(self):
        """Level-set sweep modes the cycle needs (0 fwd x=0, 1 fwd, 2 bwd x=0, 3 bwd)."""
        modes = set()
        for spec, first_zero in ((self.pre_smoother, True), (self.post_smoother, False)):
            if spec.kind == WEIGHTED_JACOBI or spec.sweeps == 0:
                continue
            if spec.kind == GS_BACKWARD:
                modes.add(2)  # from x_old: folded upper neighbours + the zero-guess schedule
            elif first_zero:
                modes.add(0)
                if spec.sweeps > 1:
                    modes.add(1)
            else:
                modes.add(1)
        return sorted(modes)

    def _gs_cluster_modes(self, A):
        """Cluster / grid plans the cycle needs for level matrix A (0 fwd x=0, 1 fwd, 2 bwd x=0 -- with
        x_old the folded backward sweep --, 3 bwd).  A backward sweep from x_old runs as its own mode-3
        plan (x_old entries read in the kernel) up to config.cluster_fused_fold_rows rows, else folded."""
        modes = set()
        for spec, first_zero in ((self.pre_smoother, True), (self.post_smoother, False)):
            if spec.kind == WEIGHTED_JACOBI or spec.sweeps == 0:
                continue
            if spec.kind == GS_BACKWARD:
                if first_zero:
                    modes.add(2)
                if not first_zero or spec.sweeps > 1:
                    modes.add(3 if A.shape[0] <= self.config.cluster_fused_fold_rows else 2)
            else:
                modes.add(0 if first_zero else 1)
                if first_zero and spec.sweeps > 1:
                    modes.add(1)
        return sorted(modes)

    def _gs_stream_modes(self, A):
        """Stream plans the cycle needs for level matrix A: {mode: plan mode}
        (a backward sweep from x_old that does not fit with b in shared memory
        runs the folded mode-2 plan); None when a needed mode cannot stream."""
        need = {}
        for spec, first_zero in ((self.pre_smoother, True), (self.post_smoother, False)):
            if spec.kind == WEIGHTED_JACOBI or spec.sweeps == 0:
                continue
            base = 0 if spec.kind == GS_FORWARD else 2
            for m in ({base + (0 if first_zero else 1)} | ({base + 1} if spec.sweeps > 1 else set())):
                if stream_ctas(A, m, self.config):
                    need[m] = m
                elif m == 3 and stream_ctas(A, 2, self.config):
                    need[m] = 2
                else:
                    return None
        return need

    def _init_plain(self, A):
        """Single-level handle used only for its matrix (pcg with precond=None)."""
        self.matrices = [as_csr(A)]
        self.prolongators, self.restrictions, self.diagonals = [], [], []
        self.cycle = CycleSpec()
        self.pre_smoother = SmootherSpec(GS_FORWARD)
        self.post_smoother = SmootherSpec(GS_BACKWARD)
        self.config = GpuConfig()
        self._h = None
        self._upload(plain=True)

    # ---- upload ------------------------------------------------------------
    def _upload(self, plain=False):
        torch = torch_cuda()
        L = _lib.load()
        nl = len(self.matrices)
        h = ctypes.c_void_p()
        pre, post = self.pre_smoother, self.post_smoother
        _lib.check(L.mvamg_hierarchy_create(
            ctypes.byref(h), nl, _lib.CYCLE_V if self.cycle.kind == "V" else _lib.CYCLE_K,
            int(self.cycle.inner_fcg_iters), _KIND[pre.kind], int(pre.sweeps), float(pre.omega),
            _KIND[post.kind], int(post.sweeps), float(post.omega)), "hierarchy_create")
        self._h = h
        self._keep = []
        self.gs_plans = []
        self.level_dev = []
        self._dA = []
        cfg = self.config
        for k, A in enumerate(self.matrices):
            dA = DeviceCSR(A)
            self._dA.append(dA)
            if k < nl - 1:
                dd = to_device(self.diagonals[k], np.float64)
                self._keep.append(dd)
                # streamed sweeps on the V-cycle's levels (C3 H1: 1.15-1.3x the level-set kernel); the K-cycle
                # components of H2 stay on the level-set kernel (C3 H2 solve 2.22 s vs 2.43 s streamed)
                if (k >= 1 and cfg.cluster_gs and not cfg.exact_gs and not cfg.generic_gs and not cfg.force_level_gs
                        and not cfg.force_row_gs and A.shape[0] <= cfg.cluster_max_rows):
                    # cluster dataflow sweeps: x in one thread-block cluster's distributed shared memory
                    try:
                        plans = {m: DeviceGsCluster(A, m, cfg) for m in self._gs_cluster_modes(A)}
                    except ValueError:
                        plans = None
                    if plans is not None:
                        self.gs_plans.append(None)
                        self.level_dev.append(dict(A=dA, gs=None, plan=None, levels=None, rows=None, cluster=plans))
                        _lib.check(L.mvamg_hierarchy_set_level(h, k, dA.n, dA.nnz, *dA.ptrs(), ptr(dd),
                                                               None, 0, None, None, None, 32, 0, 0), "set_level")
                        for m, cp in plans.items():
                            _lib.check(L.mvamg_hierarchy_set_gs_cluster(h, k, m, *cp.args()), "set_gs_cluster")
                        continue
                smodes = (self._gs_stream_modes(A) if cfg.stream_gs and self.cycle.kind == "V" and not cfg.generic_gs
                          and not cfg.force_level_gs and not cfg.force_row_gs else None)
                if smodes:
                    # streamed level-set sweeps on one SM (x, b in shared memory)
                    plans = {pm: DeviceGsStream(A, pm, cfg) for pm in set(smodes.values())}
                    self.gs_plans.append(None)
                    self.level_dev.append(dict(A=dA, gs=None, plan=None, levels=None, rows=None, stream=plans))
                    _lib.check(L.mvamg_hierarchy_set_level(h, k, dA.n, dA.nnz, *dA.ptrs(), ptr(dd),
                                                           None, 0, None, None, None, 32, 0, 0), "set_level")
                    for pm, sp in plans.items():
                        _lib.check(L.mvamg_hierarchy_set_gs_stream(h, k, pm, *sp.args()), "set_gs_stream")
                    continue
                if (k >= 1 and self.config.autotune_gs and not self.config.generic_gs
                        and not self.config.force_level_gs and not self.config.force_row_gs
                        and A.shape[0] <= self.config.level_gs_max_rows):
                    # coarse level: the faster of the row and level-set sweeps, per mode
                    pick = autotune_coarse_gs(A, self._gs_level_modes(), self.config)
                    self.gs_plans.append(None)
                    lv = dict(A=dA, gs=None, plan=None, levels=None, rows=None)
                    _lib.check(L.mvamg_hierarchy_set_level(h, k, dA.n, dA.nnz, *dA.ptrs(), ptr(dd),
                                                           None, 0, None, None, None, 32, 0, 0), "set_level")
                    for m, s in pick.items():
                        if isinstance(s, DeviceGsRows):
                            lv["rows"] = lv["rows"] or {}
                            lv["rows"][m] = s
                            _lib.check(L.mvamg_hierarchy_set_gs_rows(h, k, m, *s.hierarchy_args()), "set_gs_rows")
                        else:
                            lv["levels"] = lv["levels"] or {}
                            lv["levels"][m] = s
                            _lib.check(L.mvamg_hierarchy_set_gs_levels(h, k, m, *s.args()), "set_gs_levels")
                    self.level_dev.append(lv)
                    continue
                if row_gs_fits(A, k, self.config):
                    # dataflow row sweeps over the whole GPU; no wavefront schedule needed
                    rows = {m: DeviceGsRows(A, m, self.config) for m in self._gs_level_modes()}
                    self.gs_plans.append(None)
                    self.level_dev.append(dict(A=dA, gs=None, plan=None, levels=None, rows=rows))
                    _lib.check(L.mvamg_hierarchy_set_level(h, k, dA.n, dA.nnz, *dA.ptrs(), ptr(dd),
                                                           None, 0, None, None, None, 32, 0, 0), "set_level")
                    for m, s in rows.items():
                        _lib.check(L.mvamg_hierarchy_set_gs_rows(h, k, m, *s.hierarchy_args()), "set_gs_rows")
                    continue
                small = None
                if level_gs_fits(A, self.config):
                    try:
                        small = {m: DeviceGsLevels(A, m, self.config) for m in self._gs_level_modes()}
                    except ValueError:
                        small = None
                if small is not None:
                    # single-CTA level-set sweeps; no wavefront schedule needed
                    self.gs_plans.append(None)
                    self.level_dev.append(dict(A=dA, gs=None, plan=None, levels=small))
                    _lib.check(L.mvamg_hierarchy_set_level(h, k, dA.n, dA.nnz, *dA.ptrs(), ptr(dd),
                                                           None, 0, None, None, None, 32, 0, 0), "set_level")
                    for m, s in small.items():
                        _lib.check(L.mvamg_hierarchy_set_gs_levels(h, k, m, *s.args()), "set_gs_levels")
                    continue
                gp = DeviceGsPlan(A, self.config)
                if (not self.config.generic_gs and gp.plan.nchains > 0
                        and A.shape[0] / gp.plan.nchains < self.config.min_chain_rows):
                    # no chain structure for the wavefront: the grid-form dataflow sweep (tolerance mode;
                    # C4's fine level, 525k rows of 2 interleaved dofs: 4x the row sweep), else row sweeps
                    plans = None
                    if cfg.cluster_gs and not cfg.exact_gs and not cfg.force_row_gs and A.shape[0] <= cfg.cluster_max_rows:
                        try:
                            plans = {m: DeviceGsCluster(A, m, cfg, grid=True) for m in self._gs_cluster_modes(A)}
                        except ValueError:
                            plans = None
                    if plans is not None:
                        self.gs_plans.append(None)
                        self.level_dev.append(dict(A=dA, gs=None, plan=None, levels=None, rows=None, cluster=plans))
                        _lib.check(L.mvamg_hierarchy_set_level(h, k, dA.n, dA.nnz, *dA.ptrs(), ptr(dd),
                                                               None, 0, None, None, None, 32, 0, 0), "set_level")
                        for m, cp in plans.items():
                            _lib.check(L.mvamg_hierarchy_set_gs_cluster(h, k, m, *cp.args()), "set_gs_cluster")
                        continue
                    rows = {m: DeviceGsRows(A, m, self.config) for m in self._gs_level_modes()}
                    self.gs_plans.append(None)
                    self.level_dev.append(dict(A=dA, gs=None, plan=None, levels=None, rows=rows))
                    _lib.check(L.mvamg_hierarchy_set_level(h, k, dA.n, dA.nnz, *dA.ptrs(), ptr(dd),
                                                           None, 0, None, None, None, 32, 0, 0), "set_level")
                    for m, s in rows.items():
                        _lib.check(L.mvamg_hierarchy_set_gs_rows(h, k, m, *s.hierarchy_args()), "set_gs_rows")
                    continue
                self.gs_plans.append(gp.plan)
                self.level_dev.append(dict(A=dA, gs=gp, plan=gp.plan, levels=None))
                _lib.check(L.mvamg_hierarchy_set_level(h, k, dA.n, dA.nnz, *dA.ptrs(), ptr(dd),
                                                       None, gp.plan.ntiles, ptr(gp.chain_ptr),
                                                       ptr(gp.tile_ptr), ptr(gp.chain_order), gp.plan.threads,
                                                       gp.plan.window, gp.plan.wpos), "set_level")
                for m in self._gs_modes():
                    sch = gp.mode(m)
                    _lib.check(L.mvamg_hierarchy_set_gs_schedule(
                        h, k, m, ptr(sch["rec"]), ptr(sch["round_off"]), ptr(sch["tbase"]),
                        ptr(sch["tile_wbase"]), ptr(sch["perm"]), ptr(sch["tperm"]), sch["R"], sch["D"],
                        sch["lean_C"], sch["slot_words"], sch["rec_words_max"]), "set_gs_schedule")
            else:
                _lib.check(L.mvamg_hierarchy_set_level(h, k, dA.n, dA.nnz, *dA.ptrs(), None, None, 0,
                                                       None, None, None, 32, 0, 0), "set_level")
        for k, (P, R) in enumerate(zip(self.prolongators, self.restrictions)):
            dP, dR = DeviceCSR(P), DeviceCSR(R)
            self._keep += [dP, dR]
            _lib.check(L.mvamg_hierarchy_set_transfer(h, k, *dP.ptrs(), *dR.ptrs()), "set_transfer")
        # Coarsest: the reference LU-factors A_L once (cycles.py:88-97); apply
        # it as a dense inverse built from those same factors (one GEMV/visit).
        if plain:
            self.coarse_lu = None
            self._inv = to_device(np.zeros(1), np.float64)  # never applied (no cycle)
        else:
            self._inv = to_device(self._coarse_inverse(), np.float64)
        _lib.check(L.mvamg_hierarchy_set_coarse(h, ptr(self._inv)), "set_coarse")
        nbytes = ctypes.c_longlong()
        _lib.check(L.mvamg_hierarchy_workspace_bytes(h, ctypes.byref(nbytes)), "workspace_bytes")
        self._ws = torch.empty(max(8, nbytes.value), dtype=torch.uint8, device="cuda")
        _lib.check(L.mvamg_hierarchy_bind_workspace(h, ptr(self._ws), stream_handle()), "bind_workspace")
        _lib.check(L.mvamg_hierarchy_set_graphs(h, int(bool(self.config.graphs))), "set_graphs")

    def _coarse_inverse(self):
        """Dense coarsest operator applied by one GEMV per visit: the inverse
        from the reference's own LU factors (cycles.py:88-97), or with
        config.coarse_pinv_rtol > 0 the truncated-eigen pseudo-inverse."""
        Ac = self.matrices[-1].toarray()
        rtol = float(self.config.coarse_pinv_rtol)
        if rtol > 0.0:
            self.coarse_lu = None
            return coarse_pinv(Ac, rtol)
        self.coarse_lu = scipy.linalg.lu_factor(Ac)
        return np.ascontiguousarray(scipy.linalg.lu_solve(self.coarse_lu, np.eye(Ac.shape[0])))

    def set_coarse_pinv(self, rtol):
        """Switch the coarsest solve in place (same device buffer, so captured
        graphs stay valid): rtol > 0 pseudo-inverse, 0 the LU inverse."""
        torch = torch_cuda()
        self.config = dataclasses.replace(self.config, coarse_pinv_rtol=float(rtol))
        self._inv.copy_(torch.from_numpy(self._coarse_inverse()).reshape(self._inv.shape))
        torch.cuda.synchronize()

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                _lib.load().mvamg_hierarchy_destroy(h)
            except Exception:
                pass
            self._h = None

    # ---- reference surface -------------------------------------------------
    @property
    def n_levels(self):
        return len(self.matrices)

    @property
    def shape(self):
        n = self.matrices[0].shape[0]
        return (n, n)

    @property
    def handle(self):
        return self._h

    def _status(self, what):
        st = ctypes.c_int()
        _lib.check(_lib.load().mvamg_hierarchy_status(self._h, ctypes.byref(st), 1), what)
        _lib.raise_status(st.value, what)

    def apply_device(self, r):
        """z = B^{-1} r for a CUDA float64 tensor r (stays on the device)."""
        torch = torch_cuda()
        z = torch.empty_like(r)
        _lib.check(_lib.load().mvamg_cycle_apply(self._h, ptr(r), ptr(z), stream_handle()), "cycle_apply")
        return z

    def apply(self, r):
        """z approximating B^{-1} r (one cycle) -- cycles.py:174-179."""
        r = np.asarray(r, dtype=np.float64)
        if r.shape[0] != self.matrices[0].shape[0]:
            raise ValueError("residual length does not match the hierarchy")
        z = self.apply_device(to_device(r)).cpu().numpy()
        self._status("apply")
        return z

    __call__ = apply

    def error_propagation_device(self, x):
        torch = torch_cuda()
        e = torch.empty_like(x)
        _lib.check(_lib.load().mvamg_error_propagation(self._h, ptr(x), ptr(e), stream_handle()),
                   "error_propagation")
        return e

    def error_propagation(self, x):
        """(I - B^{-1} A) x for the finest-level matrix -- cycles.py:181-184."""
        x = np.asarray(x, dtype=np.float64)
        if x.shape[0] != self.matrices[0].shape[0]:
            raise ValueError("vector length does not match the hierarchy")
        e = self.error_propagation_device(to_device(x)).cpu().numpy()
        self._status("error_propagation")
        return e

    def as_linear_operator(self):
        return spla.LinearOperator(self.shape, matvec=self.apply, dtype=np.float64)
