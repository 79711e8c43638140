"""Device buffers (PyTorch-owned) and host-side preparation of CSR operands.

PyTorch is used only for allocation, lifetime and the current CUDA stream; all
arithmetic on the solve path runs in libmvamg_b200.so.
"""

import ctypes
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from . import _lib
from .exceptions import DeviceError


def torch_cuda():
    import torch

    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device: the mvamg B200 path has no CPU fallback")
    return torch


def stream_handle():
    torch = torch_cuda()
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def as_csr(A):
    """Canonical float64 CSR (sorted, summed) -- pkg/src/mvamg/sparse.py:13-27."""
    if not sp.issparse(A):
        A = np.asarray(A)
        if A.ndim != 2:
            raise ValueError(f"expected a 2-d operator, got shape {A.shape}")
        A = sp.csr_matrix(A)
    A = A.tocsr().astype(np.float64, copy=False)
    A.sum_duplicates()
    A.sort_indices()
    return A


def to_device(a, dtype=None):
    torch = torch_cuda()
    t = torch.from_numpy(np.ascontiguousarray(a if dtype is None else np.asarray(a, dtype=dtype)))
    return t.to("cuda", non_blocking=False)


def ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


@dataclass
class GpuConfig:
    """B200 knobs that the reference does not have (kept apart from its specs).

    max_chain   : longest dependency chain one thread walks in a GS sweep
    max_threads : chains (threads) per GS tile / CTA
    max_window  : rows of a tile kept in the shared-memory window (8 B each)
    graphs      : capture cycles / PCG half-iterations into CUDA graphs
    """

    max_chain: int = 4096
    max_threads: int = 128
    max_window: int = 24576
    graphs: bool = True


class DeviceCSR:
    """A CSR matrix resident in HBM (int32 indptr/indices, fp64 data)."""

    def __init__(self, A):
        A = as_csr(A)
        if A.nnz >= 2**31:
            raise ValueError("int32 indices: nnz must be < 2^31")
        self.host = A
        self.shape = A.shape
        self.n = A.shape[0]
        self.nnz = A.nnz
        self.indptr = to_device(A.indptr, np.int32)
        self.indices = to_device(A.indices, np.int32)
        self.data = to_device(A.data, np.float64)

    def ptrs(self):
        return ptr(self.indptr), ptr(self.indices), ptr(self.data)


@dataclass
class GsPlanHost:
    nchains: int
    ntiles: int
    threads: int
    window: int
    depth: int
    chain_ptr: np.ndarray
    tile_ptr: np.ndarray


def gs_analyse(A, cfg=None):
    """Chain/tile schedule of a CSR matrix for the sync-free GS sweep (host)."""
    cfg = cfg or GpuConfig()
    A = as_csr(A)
    L = _lib.load()
    ip = np.ascontiguousarray(A.indptr, dtype=np.int32)
    ix = np.ascontiguousarray(A.indices, dtype=np.int32)
    nch, nt, thr, win, dep = (ctypes.c_int() for _ in range(5))
    n = A.shape[0]
    c_ip = ip.ctypes.data_as(ctypes.c_void_p)
    c_ix = ix.ctypes.data_as(ctypes.c_void_p)
    _lib.check(L.mvamg_gs_analyse(n, c_ip, c_ix, cfg.max_chain, cfg.max_threads, cfg.max_window,
                                  ctypes.byref(nch), ctypes.byref(nt), None, None, None, None,
                                  None), "gs_analyse")
    cp = np.empty(nch.value + 1, dtype=np.int32)
    tp = np.empty(nt.value + 1, dtype=np.int32)
    _lib.check(L.mvamg_gs_analyse(n, c_ip, c_ix, cfg.max_chain, cfg.max_threads, cfg.max_window,
                                  ctypes.byref(nch), ctypes.byref(nt),
                                  cp.ctypes.data_as(ctypes.c_void_p),
                                  tp.ctypes.data_as(ctypes.c_void_p), ctypes.byref(thr),
                                  ctypes.byref(win), ctypes.byref(dep)), "gs_analyse")
    return GsPlanHost(nch.value, nt.value, max(32, thr.value), win.value, dep.value, cp, tp)
