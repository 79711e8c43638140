"""ctypes wrapper around liboracle (mvamg_oracle.c) -- TEST INFRASTRUCTURE ONLY.

Restates, on the CPU, the reference solve path of arXiv 1907.04417's `mvamg`:
  * OracleOperator        ~ cycles.py:100-190 MultigridOperator (V / K cycles,
                            GS / weighted-Jacobi smoothers, LU coarse solve)
  * oracle_pcg            ~ krylov.py:28-72 pcg (x0 = 0)
  * oracle_composite      ~ bootstrap.py:98-113 apply_composite_symmetrized
  * oracle_gs / oracle_spmv ~ _kernels.py:15-38, sparse.py:30-40
Pinned against the reference's own outputs by tests/test_oracle_golden.py.
Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg) may use it.
"""

import ctypes
import os
import subprocess

import numpy as np
import scipy.linalg
import scipy.sparse as sp

HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

_I = ctypes.c_int
_D = ctypes.c_double
_P = ctypes.c_void_p

KIND = {"gauss_seidel_forward": 0, "gauss_seidel_backward": 1, "weighted_jacobi": 2}


def build():
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(HERE, "libmvamg_oracle.so")
        if not os.path.exists(path):
            build()
        L = ctypes.CDLL(path)
        L.or_hier_new.restype = _P
        L.or_hier_new.argtypes = [_I, _I, _I, _I, _I, _D, _I, _I, _D]
        L.or_hier_set_level.argtypes = [_P, _I, _I, _P, _P, _P, _P]
        L.or_hier_set_transfer.argtypes = [_P, _I, _I, _I, _P, _P, _P, _P, _P, _P]
        L.or_hier_set_coarse.argtypes = [_P, _P, _P]
        L.or_hier_set_coarse_inverse.argtypes = [_P, _P]
        L.or_hier_alloc.argtypes = [_P]
        L.or_hier_destroy.argtypes = [_P]
        L.or_apply.argtypes = [_P, _P, _P]
        L.or_apply.restype = _I
        L.or_composite.argtypes = [_P, _I, _P, _P, _P]
        L.or_composite.restype = _I
        L.or_pcg_h.argtypes = [_P, _P, _I, _P, _I, _D, _I, _P, _P, _P, _P, _P]
        L.or_pcg_h.restype = _I
        L.or_spmv.argtypes = [_I, _P, _P, _P, _P, _P]
        L.or_gs.argtypes = [_I, _I, _P, _P, _P, _P, _P, _P]
        L.or_dot.argtypes = [_I, _P, _P]
        L.or_dot.restype = _D
        L.or_set_threads.argtypes = [_I]
        L.or_set_threads.restype = _I
        L.or_greedy_accept.argtypes = [ctypes.c_longlong, _P, _P, _I, _P, _P, _P]
        L.or_greedy_accept.restype = ctypes.c_longlong
        L.or_jacobi_svd_batch.argtypes = [_I, _P, _I, _P, _I, _D, _P, _P, ctypes.POINTER(_I)]
        L.or_jacobi_svd_batch.restype = _I
        _LIB = L
    return _LIB


def _ptr(a):
    return a.ctypes.data_as(_P)


def _csr(M):
    M = sp.csr_matrix(M)
    M.sum_duplicates()
    M.sort_indices()
    return (M, np.ascontiguousarray(M.indptr, dtype=np.int32),
            np.ascontiguousarray(M.indices, dtype=np.int32),
            np.ascontiguousarray(M.data, dtype=np.float64))


def set_threads(t=0):
    """Host threads for the oracle's SpMVs, vector updates, dots and batched
    SVDs (0: keep the OpenMP default).  Results do not depend on it; the GS
    sweeps are serial.  Returns the thread count in effect."""
    return int(lib().or_set_threads(int(t)))


def oracle_dot(x, y):
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    return float(lib().or_dot(x.shape[0], _ptr(x), _ptr(y)))


def oracle_spmv(A, x):
    M, ip, ix, v = _csr(A)
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.empty(M.shape[0])
    lib().or_spmv(M.shape[0], _ptr(ip), _ptr(ix), _ptr(v), _ptr(x), _ptr(y))
    return y


def oracle_gs(A, b, x, direction="forward"):
    """In-place lexicographic GS sweep (_kernels.py:15-38); returns x."""
    M, ip, ix, v = _csr(A)
    d = np.ascontiguousarray(M.diagonal())
    b = np.ascontiguousarray(b, dtype=np.float64)
    assert x.dtype == np.float64 and x.flags.c_contiguous
    lib().or_gs(0 if direction == "forward" else 1, M.shape[0], _ptr(ip), _ptr(ix), _ptr(v),
                _ptr(d), _ptr(b), _ptr(x))
    return x


class OracleOperator:
    """CPU restatement of MultigridOperator (cycles.py:100-190)."""

    def __init__(self, matrices, prolongators, cycle="V", inner_fcg_iters=2,
                 pre=("gauss_seidel_forward", 1, 1.0), post=("gauss_seidel_backward", 1, 1.0),
                 coarse_pinv_rtol=0.0):
        """coarse_pinv_rtol > 0: the stated C5 deviation -- the coarsest level
        is solved with the truncated-eigen pseudo-inverse (eigenvalues at or
        below rtol * lambda_max dropped) instead of the reference's LU."""
        L = lib()
        self._keep = []
        self.nlev = len(matrices)
        self.n = matrices[0].shape[0]
        self.h = L.or_hier_new(self.nlev, 0 if cycle == "V" else 1, int(inner_fcg_iters),
                               KIND[pre[0]], int(pre[1]), float(pre[2]),
                               KIND[post[0]], int(post[1]), float(post[2]))
        self.matrices = []
        for k, A in enumerate(matrices):
            M, ip, ix, v = _csr(A)
            d = np.ascontiguousarray(M.diagonal())
            self._keep += [ip, ix, v, d]
            self.matrices.append(M)
            L.or_hier_set_level(self.h, k, M.shape[0], _ptr(ip), _ptr(ix), _ptr(v), _ptr(d))
        for k, P in enumerate(prolongators):
            Pm, pip, pix, pv = _csr(P)
            Rm, rip, rix, rv = _csr(Pm.T.tocsr())
            self._keep += [pip, pix, pv, rip, rix, rv]
            L.or_hier_set_transfer(self.h, k, Pm.shape[0], Pm.shape[1], _ptr(pip), _ptr(pix),
                                   _ptr(pv), _ptr(rip), _ptr(rix), _ptr(rv))
        if coarse_pinv_rtol > 0.0:
            w, Q = np.linalg.eigh(self.matrices[-1].toarray())
            keep = w > coarse_pinv_rtol * w[-1]
            inv = np.ascontiguousarray((Q[:, keep] / w[keep]) @ Q[:, keep].T)
            self._keep.append(inv)
            L.or_hier_set_coarse_inverse(self.h, _ptr(inv))
        else:
            lu, piv = scipy.linalg.lu_factor(self.matrices[-1].toarray())
            lu = np.ascontiguousarray(lu)
            piv = np.ascontiguousarray(piv, dtype=np.int32)
            self._keep += [lu, piv]
            L.or_hier_set_coarse(self.h, _ptr(lu), _ptr(piv))
        L.or_hier_alloc(self.h)

    def __del__(self):
        if getattr(self, "h", None):
            lib().or_hier_destroy(self.h)
            self.h = None

    def apply(self, r):
        r = np.ascontiguousarray(r, dtype=np.float64)
        z = np.empty_like(r)
        st = lib().or_apply(self.h, _ptr(r), _ptr(z))
        if st:
            raise ArithmeticError(f"oracle breakdown {st}")
        return z

    __call__ = apply

    def error_propagation(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        return x - self.apply(self.matrices[0] @ x)


def oracle_composite(ops, x):
    """apply_composite_symmetrized (bootstrap.py:98-113) over OracleOperators."""
    x = np.array(x, dtype=np.float64, copy=True)
    arr = (_P * len(ops))(*[o.h for o in ops])
    t1 = np.empty_like(x)
    t2 = np.empty_like(x)
    st = lib().or_composite(arr, len(ops), _ptr(x), _ptr(t1), _ptr(t2))
    if st:
        raise ArithmeticError(f"oracle breakdown {st}")
    return x


def oracle_pcg(owner, b, precond="cycle", ops=None, rtol=1e-6, itmax=1000):
    """pcg (krylov.py:28-72) with x0 = 0 on owner's finest matrix.

    precond: "none", "cycle" (owner's cycle) or "composite" (symmetrized
    multiplicative composite of ``ops``).  Returns (x, hist, nit, converged).
    """
    b = np.ascontiguousarray(b, dtype=np.float64)
    n = b.shape[0]
    kind = {"none": 0, "cycle": 1, "composite": 2}[precond]
    ops = ops if ops is not None else [owner]
    arr = (_P * len(ops))(*[o.h for o in ops])
    x = np.empty(n)
    hist = np.zeros(itmax + 1)
    nit = ctypes.c_int(0)
    conv = ctypes.c_int(0)
    work = np.empty(6 * n)
    st = lib().or_pcg_h(owner.h, _ptr(b), kind, arr, len(ops), float(rtol), int(itmax), _ptr(x),
                        _ptr(hist), ctypes.byref(nit), ctypes.byref(conv), _ptr(work))
    if st:
        raise ArithmeticError(f"oracle PCG breakdown {st}")
    return x, hist[: nit.value + 1].copy(), nit.value, bool(conv.value)


def oracle_galerkin(P, A):
    """galerkin_product(P, A) (sparse.py:50-66) restated in C: (G + G')/2 with
    G = P'(A P), scipy csr_matmat summation order, exact zeros dropped."""
    Am, aip, aix, av = _csr(A)
    Pm, pip, pix, pv = _csr(P)
    if Pm.shape[0] != Am.shape[0] or Am.shape[0] != Am.shape[1]:
        raise ValueError("dimension mismatch")
    L = lib()
    L.or_galerkin.restype = _I
    L.or_galerkin.argtypes = [_I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P]
    L.or_free.argtypes = [_P]
    n, nc = Pm.shape
    oip, oix, ov = _P(), _P(), _P()
    nnz = L.or_galerkin(n, nc, _ptr(aip), _ptr(aix), _ptr(av), _ptr(pip), _ptr(pix), _ptr(pv),
                        ctypes.byref(oip), ctypes.byref(oix), ctypes.byref(ov))
    ip = np.ctypeslib.as_array(ctypes.cast(oip, ctypes.POINTER(_I)), (nc + 1,)).copy()
    ix = np.ctypeslib.as_array(ctypes.cast(oix, ctypes.POINTER(_I)), (max(nnz, 1),))[:nnz].copy()
    v = np.ctypeslib.as_array(ctypes.cast(ov, ctypes.POINTER(_D)), (max(nnz, 1),))[:nnz].copy()
    for p in (oip, oix, ov):
        L.or_free(p)
    return sp.csr_matrix((v, ix, ip), shape=(nc, nc))
