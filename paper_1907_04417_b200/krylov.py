"""Preconditioned CG on the GPU -- drop-in for pkg/src/mvamg/krylov.py:28-72.

``pcg(A, b, precond, rtol, itmax, x0, callback)`` keeps the reference's
signature, return value ``(x, SolveReport)`` and exceptions.  When ``precond``
is one of this package's device operators (a GpuMultigridOperator, its bound
``apply``, a GpuComposite preconditioner) or None, and ``x0``/``callback`` are
unset, the whole iteration runs in libmvamg_b200.so with the scalars on the
device (one host round trip per iteration for the stop test).  Otherwise a
device-vector PCG loop drives the same kernels and calls the foreign
preconditioner through host memory.
"""

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .device import DeviceCSR, as_csr, ptr, stream_handle, to_device, torch_cuda
from .exceptions import NotSpdError


@dataclass
class SolveReport:
    """Mirror of krylov.py:10-15."""

    iterations: int
    final_relative_residual: float
    converged: bool
    residual_history: np.ndarray  # length iterations + 1


def _same_matrix(A, B):
    if A is B:
        return True
    A = as_csr(A)
    if A.shape != B.shape or A.nnz != B.nnz:
        return False
    return (np.array_equal(A.indptr, B.indptr) and np.array_equal(A.indices, B.indices)
            and np.array_equal(A.data, B.data))


def _device_precond(precond):
    """Return (owner_operator, pc_kind, composite) if precond is ours."""
    from .composite import GpuCompositePreconditioner
    from .cycles import GpuMultigridOperator

    if precond is None:
        return None, _lib.PC_NONE, None
    if isinstance(precond, GpuMultigridOperator):
        return precond, _lib.PC_CYCLE, None
    owner = getattr(precond, "__self__", None)
    if isinstance(owner, GpuMultigridOperator) and getattr(precond, "__name__", "") in ("apply", "__call__"):
        return owner, _lib.PC_CYCLE, None
    if isinstance(precond, GpuCompositePreconditioner):
        return precond.owner, _lib.PC_COMPOSITE, precond
    if isinstance(owner, GpuCompositePreconditioner):
        return owner.owner, _lib.PC_COMPOSITE, owner
    return None, None, None


class _PlainMatrixOwner:
    """A one-level device hierarchy used only for its matrix (precond=None)."""

    _cache = {}

    @classmethod
    def get(cls, A):
        from .cycles import GpuMultigridOperator

        key = id(A)
        hit = cls._cache.get(key)
        if hit is not None and hit[0] is A:
            return hit[1]
        op = GpuMultigridOperator.__new__(GpuMultigridOperator)
        # minimal single-level hierarchy; its coarse inverse is a 1x1 dummy
        op._init_plain(A)
        cls._cache = {key: (A, op)}
        return op


def pcg_device(owner, b, pc_kind, composite=None, rtol=1e-6, itmax=1000):
    """Run PCG fully on the device for host/numpy b; returns (x, SolveReport)."""
    b = np.ascontiguousarray(b, dtype=np.float64)
    n = b.shape[0]
    x = np.empty(n)
    hist = np.zeros(itmax + 1)
    nit, conv, st = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    comp = composite.handle if composite is not None else None
    _lib.check(_lib.load().mvamg_pcg_solve_host(
        owner.handle, pc_kind, comp, b.ctypes.data_as(ctypes.c_void_p),
        x.ctypes.data_as(ctypes.c_void_p), float(rtol), int(itmax),
        hist.ctypes.data_as(ctypes.c_void_p), ctypes.byref(nit), ctypes.byref(conv),
        ctypes.byref(st), stream_handle()), "pcg")
    _lib.raise_status(st.value, "pcg")
    k = nit.value
    hist = hist[: k + 1].copy()
    r0 = hist[0]
    if r0 == 0.0:
        return x, SolveReport(0, 0.0, True, hist)
    return x, SolveReport(k, float(hist[-1] / r0), bool(conv.value), hist)


def pcg(A, b, precond=None, rtol=1e-6, itmax=1000, x0=None, callback=None):
    """Preconditioned CG on SPD A, stopping at ||r|| <= rtol * ||r0|| (krylov.py:28-72)."""
    b = np.asarray(b, dtype=np.float64)
    owner, pc_kind, comp = _device_precond(precond)
    x0_zero = x0 is None or not np.any(np.asarray(x0))
    if pc_kind is not None and x0_zero and callback is None:
        if owner is None:
            owner = _PlainMatrixOwner.get(A)
        if _same_matrix(A, owner.matrices[0]):
            return pcg_device(owner, b, pc_kind, comp, rtol, itmax)
    return _pcg_loop(A, b, precond, rtol, itmax, x0, callback)


def _pcg_loop(A, b, precond, rtol, itmax, x0, callback):
    """Device-vector PCG for the general call forms (x0, callback, foreign
    preconditioner).  SpMV and dots run in libmvamg_b200.so; a foreign
    preconditioner callable is invoked on host copies of r."""
    torch = torch_cuda()
    L = _lib.load()
    s = stream_handle()
    dA = DeviceCSR(A)
    n = dA.n
    ws = torch.empty(L.mvamg_dot_ws_bytes(), dtype=torch.uint8, device="cuda")
    ws.zero_()
    res = torch.empty(1, dtype=torch.float64, device="cuda")

    def dot(u, v):
        _lib.check(L.mvamg_dot_f64(n, ptr(u), ptr(v), ptr(res), ptr(ws), s), "dot")
        return float(res.item())

    def spmv(u, out):
        _lib.check(L.mvamg_csr_spmv_f64(n, *dA.ptrs(), ptr(u), ptr(out), s), "spmv")
        return out

    owner, pc_kind, comp = _device_precond(precond)
    if pc_kind == _lib.PC_CYCLE:
        M = owner.apply_device
    elif pc_kind == _lib.PC_COMPOSITE:
        M = comp.apply_device
    elif precond is None:
        M = lambda r: r.clone()  # noqa: E731
    else:
        f = precond if callable(precond) else getattr(precond, "matvec", None)
        if f is None:
            raise TypeError("preconditioner must be callable, have .matvec, or be None")
        M = lambda r: to_device(np.asarray(f(r.cpu().numpy()), dtype=np.float64))  # noqa: E731

    bd = to_device(b)
    x = torch.zeros(n, dtype=torch.float64, device="cuda") if x0 is None else to_device(np.array(x0, dtype=np.float64))
    if x0 is not None and bool(torch.any(x != 0)):
        r = torch.empty_like(bd)
        _lib.check(L.mvamg_csr_residual_f64(n, *dA.ptrs(), ptr(bd), ptr(x), ptr(r), s), "residual")
    else:
        r = bd.clone()
    r0 = float(np.sqrt(dot(r, r)))
    history = [r0]
    if r0 == 0.0:
        return x.cpu().numpy(), SolveReport(0, 0.0, True, np.asarray(history))
    z = M(r)
    rz = dot(r, z)
    if rz <= 0.0:
        raise NotSpdError(f"preconditioner breakdown: r'z = {rz:.3e}")
    p = z.clone()
    q = torch.empty_like(p)
    converged = False
    k = 0
    while k < itmax:
        spmv(p, q)
        pq = dot(p, q)
        if pq <= 0.0:
            raise NotSpdError(f"CG breakdown: p'Ap = {pq:.3e}")
        alpha = rz / pq
        x += alpha * p
        r -= alpha * q
        k += 1
        history.append(float(np.sqrt(dot(r, r))))
        if callback is not None:
            callback(x.cpu().numpy())
        if history[-1] <= rtol * r0:
            converged = True
            break
        z = M(r)
        rz_next = dot(r, z)
        if rz_next <= 0.0:
            raise NotSpdError(f"preconditioner breakdown: r'z = {rz_next:.3e}")
        p = z + (rz_next / rz) * p
        rz = rz_next
    return x.cpu().numpy(), SolveReport(k, history[-1] / r0, converged, np.asarray(history))
