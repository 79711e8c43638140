"""ctypes binding of libmvamg_b200.so (include/mvamg_b200.h).

There is deliberately no CPU fallback: if the shared object is missing or no
CUDA device is present, every entry point raises DeviceError.
"""

import ctypes
import os
import subprocess

from .exceptions import DeviceError, NotSpdError

PKG = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(PKG)
# MVAMG_LIB: load a diagnostic build instead (e.g. the round-trace build of tools/lean_trace.py)
SO_PATH = os.environ.get("MVAMG_LIB") or os.path.join(PKG, "libmvamg_b200.so")
SRC = os.path.join(PKG, "csrc", "mvamg_b200.cu")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-fmad=false", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-ffp-contract=off", "-shared",
]

E_ARG, E_CUDA, E_NOT_SPD, E_TIMEOUT, E_STATE = 1, 2, 3, 4, 5
ST_RZ, ST_PQ, ST_FCG, ST_GS_TIMEOUT = 1, 2, 4, 8
GS_FORWARD, GS_BACKWARD, WEIGHTED_JACOBI = 0, 1, 2
CYCLE_V, CYCLE_K = 0, 1
PC_NONE, PC_CYCLE, PC_COMPOSITE = 0, 1, 2

_I, _D, _P, _LL = ctypes.c_int, ctypes.c_double, ctypes.c_void_p, ctypes.c_longlong
_PI = ctypes.POINTER(ctypes.c_int)

# (name, restype, argtypes) -- keep in sync with include/mvamg_b200.h
SIGNATURES = [
    ("mvamg_version", _I, []),
    ("mvamg_last_error", ctypes.c_char_p, []),
    ("mvamg_kernel_launches", _I, [ctypes.POINTER(_LL), _I]),
    ("mvamg_gs_set_trace", _I, [_P]),
    ("mvamg_gs_analyse", _I, [_I, _P, _P, _I, _I, _I, _PI, _PI, _P, _P, _PI, _PI, _PI, _P]),
    ("mvamg_csr_spmv_f64", _I, [_I, _P, _P, _P, _P, _P, _P]),
    ("mvamg_csr_residual_f64", _I, [_I, _P, _P, _P, _P, _P, _P, _P]),
    ("mvamg_csr_spmv_mode_f64", _I, [_I, _I, _I, _P, _P, _P, _P, _P, _P, _P]),
    ("mvamg_csr_spmv_add_f64", _I, [_I, _P, _P, _P, _P, _P, _P]),
    ("mvamg_gs_schedule", _I, [_I, _P, _P, _P, _I, _P, _P, _I, _I, _I, _I, _I, ctypes.POINTER(_LL), _PI, _PI,
                               _PI, _P, _P, _P, _P, _P, _P, _I]),
    ("mvamg_gs_sweep_f64", _I, [_I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _I, _P, _P,
                                _P, _I, _I, _I, _P, _P, _P, _P, _P]),
    ("mvamg_gs_levels", _I, [_I, _P, _P, _P, _I, _I, _I, _I, _PI, ctypes.POINTER(_LL), _PI, _PI, _PI, _P, _P,
                             _P, _P, _P]),
    ("mvamg_gs_level_sweep_f64", _I, [_I, _I, _P, _P, _P, _I, _I, _I, _I, _I, _I, _I, _P, _P, _P, _P, _P, _P,
                                      _P, _P, _P, _P, _P]),
    ("mvamg_gs_rows", _I, [_I, _P, _P, _P, _I, _I, ctypes.POINTER(_LL), _PI, _P, _P, _P, _P, _P, _P, _P, _P,
                           _P, _I, _I]),
    ("mvamg_gs_row_sweep_ext_f64", _I, [_I, _I, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I, _I, _I,
                                        _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    ("mvamg_ipc_handle", _I, [_P, _P]),
    ("mvamg_ipc_open", _I, [_P, ctypes.POINTER(_P)]),
    ("mvamg_ipc_close", _I, [_P]),
    ("mvamg_gs_row_sweep_f64", _I, [_I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I, _I, _I, _P,
                                    _P, _P, _P, _P, _P]),
    ("mvamg_gs_cluster_plan", _I, [_I, _P, _P, _P, _I, _I, _I, _I, _I, ctypes.POINTER(_LL), _PI, _PI, _PI, _P, _P,
                                   _P, _P, _P]),
    ("mvamg_gs_cluster_sweep_f64", _I, [_I, _I, _P, _P, _P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _I, _P, _P, _P, _P,
                                        _P, _P]),
    ("mvamg_hierarchy_set_gs_cluster", _I, [_P, _I, _I, _P, _P, _P, _P, _I, _I, _I, _I, _I, _I, _P]),
    ("mvamg_gs_stream_plan", _I, [_I, _P, _P, _P, _I, _I, _I, ctypes.POINTER(_LL), _PI, _PI, _P, _P]),
    ("mvamg_gs_stream_sweep_f64", _I, [_I, _I, _I, _I, _I, _I, _I, _P, _P, _P, _P, _P, _P]),
    ("mvamg_gs_stream_sweep_folded_f64", _I, [_I, _P, _P, _P, _I, _I, _I, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P]),
    ("mvamg_gs_stream_set_trace", _I, [_P, _I]),
    ("mvamg_set_spmv_stream", _I, [_I]),
    ("mvamg_comm_unique_id", _I, [_P]),
    ("mvamg_comm_init", _I, [ctypes.POINTER(_P), _I, _I, _P]),
    ("mvamg_comm_destroy", _I, [_P]),
    ("mvamg_halo_exchange", _I, [_P, _I, _P, _P, _P, _I, _P, _P, _P, _P]),
    ("mvamg_allreduce_sum_f64", _I, [_P, _P, _LL, _P]),
    ("mvamg_hierarchy_set_gs_stream", _I, [_P, _I, _I, _I, _I, _I, _I, _I, _P, _P, _P]),
    ("mvamg_greedy_match", _I, [_LL, _P, _P, _I, _P, _P, _P, ctypes.POINTER(_LL)]),
    ("mvamg_jacobi_svd_batch", _I, [_I, _P, _I, _P, _I, _D, _P, _P, _PI]),
    ("mvamg_gs_level_sweep_folded_f64", _I, [_I, _P, _P, _P, _I, _I, _I, _I, _I, _I, _I, _P, _P, _P, _P, _P,
                                             _P, _P, _P, _P, _P, _P]),
    ("mvamg_dense_gemv_f64", _I, [_I, _P, _P, _P, _P]),
    ("mvamg_dot_f64", _I, [_I, _P, _P, _P, _P, _P]),
    ("mvamg_dot_ws_bytes", _I, []),
    ("mvamg_hierarchy_create", _I, [ctypes.POINTER(_P), _I, _I, _I, _I, _I, _D, _I, _I, _D]),
    ("mvamg_hierarchy_destroy", _I, [_P]),
    ("mvamg_hierarchy_set_level", _I, [_P, _I, _I, _I, _P, _P, _P, _P, _P, _I, _P, _P, _P, _I, _I, _I]),
    ("mvamg_hierarchy_set_gs_schedule", _I, [_P, _I, _I, _P, _P, _P, _P, _P, _P, _I, _I, _I, _I, _I]),
    ("mvamg_hierarchy_set_gs_levels", _I, [_P, _I, _I, _I, _I, _I, _I, _I, _I, _I, _P, _P, _P, _P, _P, _P]),
    ("mvamg_hierarchy_set_gs_rows", _I, [_P, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I, _I, _I, _P]),
    ("mvamg_hierarchy_set_transfer", _I, [_P, _I, _P, _P, _P, _P, _P, _P]),
    ("mvamg_hierarchy_set_coarse", _I, [_P, _P]),
    ("mvamg_hierarchy_workspace_bytes", _I, [_P, ctypes.POINTER(_LL)]),
    ("mvamg_hierarchy_bind_workspace", _I, [_P, _P, _P]),
    ("mvamg_hierarchy_set_graphs", _I, [_P, _I]),
    ("mvamg_cycle_apply", _I, [_P, _P, _P, _P]),
    ("mvamg_error_propagation", _I, [_P, _P, _P, _P]),
    ("mvamg_hierarchy_status", _I, [_P, _PI, _I]),
    ("mvamg_pcg_solve", _I, [_P, _I, _P, _P, _P, _D, _I, _P, _PI, _PI, _PI, _P]),
    ("mvamg_pcg_solve_host", _I, [_P, _I, _P, _P, _P, _D, _I, _P, _PI, _PI, _PI, _P]),
    ("mvamg_composite_create", _I, [ctypes.POINTER(_P), _I, _P]),
    ("mvamg_composite_destroy", _I, [_P]),
    ("mvamg_composite_apply_symmetrized", _I, [_P, _P, _P]),
    ("mvamg_composite_precond", _I, [_P, _P, _P, _P]),
    ("mvamg_galerkin_f64", _I, [_I, _I, _P, _P, _P, _P, _P, _P, ctypes.POINTER(_P), ctypes.POINTER(_LL), _P, _P]),
    ("mvamg_spmat_copy", _I, [_P, _P, _P, _P, _P]),
    ("mvamg_spmat_destroy", _I, [_P]),
    ("mvamg_greedy_match_device", _I, [_I, _P, _P, _P, _P, _P, _D, _P, _PI, _P]),
    ("mvamg_jacobi_svd_batch_device", _I, [_I, _P, _I, _P, _I, _D, _P, _P, _PI, _P]),
    ("mvamg_gather_f64", _I, [_I, _P, _P, _P, _P]),
    ("mvamg_scatter_f64", _I, [_I, _P, _P, _P, _P]),
    ("mvamg_axpy_f64", _I, [_I, _D, _P, _P, _P]),
    ("mvamg_xpby_f64", _I, [_I, _P, _D, _P, _P]),
]

_lib = None


def build(force=False, verbose=False):
    """Compile libmvamg_b200.so in-tree for sm_100a (nvcc cross-compiles; no GPU needed)."""
    csrc = os.path.join(PKG, "csrc")
    srcs = [os.path.join(csrc, f) for f in sorted(os.listdir(csrc)) if f.endswith((".cu", ".cuh", ".h"))]
    srcs.append(os.path.join(REPO, "include", "mvamg_b200.h"))
    if not force and os.path.exists(SO_PATH):
        so_t = os.path.getmtime(SO_PATH)
        if all(os.path.getmtime(s) <= so_t for s in srcs):
            return SO_PATH
    cmd = ["nvcc", *NVCC_FLAGS, "-o", SO_PATH, SRC, "-ldl"]
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    return SO_PATH


def load():
    """Load the shared object (no GPU needed just to load)."""
    global _lib
    if _lib is None:
        if not os.path.exists(SO_PATH):
            raise DeviceError(f"{SO_PATH} is missing: run __graft_entry__.build() first")
        L = ctypes.CDLL(SO_PATH)
        for name, res, args in SIGNATURES:
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(code, what=""):
    if code == 0:
        return
    msg = load().mvamg_last_error().decode(errors="replace")
    if code == E_ARG:
        raise ValueError(f"{what}: {msg}")
    if code == E_NOT_SPD:
        raise NotSpdError(f"{what}: {msg}")
    raise DeviceError(f"{what}: error {code}: {msg}")


def raise_status(status, what=""):
    """Map device status bits to the reference's exceptions (krylov.py:46-47,54-55,101-102)."""
    if not status:
        return
    if status & ST_GS_TIMEOUT:
        raise DeviceError(f"{what}: Gauss-Seidel dependency wait timed out")
    if status & ST_PQ:
        raise NotSpdError(f"{what}: CG breakdown: p'Ap <= 0")
    if status & ST_RZ:
        raise NotSpdError(f"{what}: preconditioner breakdown: r'z <= 0")
    if status & ST_FCG:
        raise NotSpdError(f"{what}: FCG breakdown: p'Ap <= 0")
    raise DeviceError(f"{what}: status {status}")
