"""Multiplicative composite of cycles on the GPU (the H2 path).

* apply_composite_symmetrized(composite, x) -- drop-in for
  pkg/src/mvamg/bootstrap.py:98-113: x <- E_1..E_r E_r..E_1 x with
  E_i = I - B_i A, each B_i a (K-)cycle.
* GpuCompositePreconditioner -- Bsym as a PCG preconditioner (the paper's
  original bootstrap-AMG solve; not present in the reference, built on its
  operator API as in SURVEY.md section 0).
* test_phase / a_norm -- the bootstrap probe (bootstrap.py:116-141,
  sparse.py:69-82) driving the composite on the device.
"""

import ctypes

import numpy as np

from . import _lib
from .bootstrap_types import TestReport
from .device import DeviceCSR, ptr, stream_handle, to_device, torch_cuda
from .exceptions import NotSpdError


class GpuComposite:
    """Ordered GPU cycles B_1..B_r sharing the finest matrix A."""

    def __init__(self, operators):
        from .cycles import GpuMultigridOperator

        operators = list(operators)
        if not operators:
            raise ValueError("composite has no components")
        for op in operators:
            if not isinstance(op, GpuMultigridOperator):
                raise TypeError("GpuComposite components must be GpuMultigridOperator")
        n = operators[0].shape[0]
        if any(op.shape[0] != n for op in operators):
            raise ValueError("composite components differ in size")
        self.operators = operators
        self.owner = operators[0]
        L = _lib.load()
        arr = (ctypes.c_void_p * len(operators))(*[op.handle.value for op in operators])
        h = ctypes.c_void_p()
        _lib.check(L.mvamg_composite_create(ctypes.byref(h), len(operators), arr), "composite_create")
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                _lib.load().mvamg_composite_destroy(h)
            except Exception:
                pass
            self._h = None

    @property
    def handle(self):
        return self._h

    @property
    def n_components(self):
        return len(self.operators)

    def _status(self, what):
        for op in self.operators:
            op._status(what)

    def apply_symmetrized_device(self, x):
        y = x.clone()
        _lib.check(_lib.load().mvamg_composite_apply_symmetrized(self._h, ptr(y), stream_handle()),
                   "composite_apply")
        return y

    def apply_symmetrized(self, x):
        x = np.asarray(x, dtype=np.float64)
        y = self.apply_symmetrized_device(to_device(x)).cpu().numpy()
        self._status("apply_composite_symmetrized")
        return y

    def as_preconditioner(self):
        return GpuCompositePreconditioner(self)


class GpuCompositePreconditioner:
    """z = Bsym r with x = 0; for i in 1..r, r..1: x += B_i (r - A x)."""

    def __init__(self, composite):
        self.composite = composite
        self.owner = composite.owner
        self.handle = composite.handle
        self.shape = composite.owner.shape

    def apply_device(self, r):
        torch = torch_cuda()
        z = torch.empty_like(r)
        _lib.check(_lib.load().mvamg_composite_precond(self.handle, ptr(r), ptr(z), stream_handle()),
                   "composite_precond")
        return z

    def __call__(self, r):
        r = np.asarray(r, dtype=np.float64)
        z = self.apply_device(to_device(r)).cpu().numpy()
        self.composite._status("composite_precond")
        return z

    apply = __call__


def gpu_composite_of(composite):
    """GpuComposite for a GpuComposite or a reference-style object with
    ``.components[i].operator`` GPU operators (cached on the object)."""
    if isinstance(composite, GpuComposite):
        return composite
    comps = getattr(composite, "components", None)
    if comps is None:
        raise TypeError("expected a GpuComposite or an object with .components")
    if len(comps) == 0:
        raise ValueError("composite has no components")
    ops = [c.operator for c in comps]
    key = tuple(id(o) for o in ops)
    cached = getattr(composite, "_gpu_composite", None)
    if cached is not None and cached[0] == key:
        return cached[1]
    gc = GpuComposite(ops)
    try:
        composite._gpu_composite = (key, gc)
    except AttributeError:
        pass
    return gc


def apply_composite_symmetrized(composite, x):
    """One application of the symmetrized multiplicative error operator
    (bootstrap.py:98-113): component 1 first, up to r twice, back down."""
    return gpu_composite_of(composite).apply_symmetrized(x)


class DeviceANorm:
    """sqrt(x'Ax) with the reference's clamp/raise rule (sparse.py:69-82)."""

    def __init__(self, A):
        torch = torch_cuda()
        self.dA = A if isinstance(A, DeviceCSR) else DeviceCSR(A)
        L = _lib.load()
        self._ws = torch.zeros(L.mvamg_dot_ws_bytes(), dtype=torch.uint8, device="cuda")
        self._res = torch.empty(3, dtype=torch.float64, device="cuda")
        self._ax = torch.empty(self.dA.n, dtype=torch.float64, device="cuda")

    def __call__(self, x):
        L = _lib.load()
        s = stream_handle()
        n = self.dA.n
        _lib.check(L.mvamg_csr_spmv_f64(n, *self.dA.ptrs(), ptr(x), ptr(self._ax), s), "spmv")
        r = self._res
        _lib.check(L.mvamg_dot_f64(n, ptr(x), ptr(self._ax), ptr(r[0:1]), ptr(self._ws), s), "dot")
        quad = float(r[0].item())
        if quad < 0.0:
            _lib.check(L.mvamg_dot_f64(n, ptr(x), ptr(x), ptr(r[1:2]), ptr(self._ws), s), "dot")
            _lib.check(L.mvamg_dot_f64(n, ptr(self._ax), ptr(self._ax), ptr(r[2:3]), ptr(self._ws), s), "dot")
            scale = float(np.sqrt(r[1].item()) * np.sqrt(r[2].item()))
            if quad < -1e-10 * max(scale, np.finfo(np.float64).tiny):
                raise NotSpdError(f"negative quadratic form x'Ax = {quad:.3e}; matrix is not SPD")
            quad = 0.0
        return float(np.sqrt(quad))


def a_norm(A, x):
    """Energy norm sqrt(x' A x) on the device (sparse.py:69-82)."""
    return DeviceANorm(A)(to_device(np.asarray(x, dtype=np.float64)))


def test_phase(composite, A, nu, rng):
    """Bootstrap probe on A x = 0 (bootstrap.py:116-141), composite on device."""
    if nu < 2:
        raise ValueError("nu must be >= 2")
    if isinstance(rng, (int, np.integer)):
        rng = np.random.default_rng(rng)
    gc = gpu_composite_of(composite)
    x = rng.uniform(-1.0, 1.0, size=A.shape[0])
    norm = DeviceANorm(gc.owner._dA[0])
    xd = to_device(x)
    anorms = [norm(xd)]
    for _ in range(nu):
        xd = gc.apply_symmetrized_device(xd)
        anorms.append(norm(xd))
        if anorms[-1] == 0.0:
            break
    gc._status("test_phase")
    anorms = np.asarray(anorms)
    stage = gc.n_components
    if anorms[-1] == 0.0:
        return TestReport(stage, 0.0, 0.0, anorms), None
    rho = float(anorms[-1] / anorms[-2])
    rho_geo = float((anorms[-1] / anorms[0]) ** (1.0 / (len(anorms) - 1)))
    return TestReport(stage, rho, rho_geo, anorms), xd.cpu().numpy() / anorms[-1]
