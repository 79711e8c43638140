"""CPU-side checks of the C ABI: the library loads, exports every symbol the
public header declares, and its host-side GS schedule analysis is correct.
No compute calls that need a GPU."""

import ctypes
import os
import re

import numpy as np
import pytest
import scipy.sparse as sp

from _fixtures import c1_fine, laplacian_1d, laplacian_2d, laplacian_3d, random_spd_csr

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "mvamg_b200.h")).read()
    return sorted(set(re.findall(r"\b(mvamg_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_header_symbols():
    from paper_1907_04417_b200 import _lib

    L = _lib.load()
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(L, s), s
    bound = {name for name, _, _ in _lib.SIGNATURES}
    assert bound == set(syms)


def test_version():
    from paper_1907_04417_b200 import _lib

    assert _lib.load().mvamg_version() == 1


def _plan(A, **kw):
    from paper_1907_04417_b200 import GpuConfig, gs_analyse

    return gs_analyse(A, GpuConfig(**kw))


def _check_plan(A, plan, max_threads, max_window):
    A = sp.csr_matrix(A)
    n = A.shape[0]
    cp, tp = plan.chain_ptr, plan.tile_ptr
    assert cp[0] == 0 and cp[-1] == n and np.all(np.diff(cp) > 0)
    assert tp[0] == 0 and tp[-1] == plan.nchains and np.all(np.diff(tp) > 0)
    # within a chain every row couples to its predecessor
    for c in range(plan.nchains):
        for i in range(cp[c] + 1, cp[c + 1]):
            assert A[i, i - 1] != 0 or (i - 1) in A.indices[A.indptr[i]:A.indptr[i + 1]]
    assert np.max(np.diff(tp)) <= max_threads
    assert plan.threads % 32 == 0 and plan.threads >= np.max(np.diff(tp))


def test_gs_plan_1d_single_chain():
    A = laplacian_1d(100)
    p = _plan(A)
    assert p.nchains == 1 and p.ntiles == 1 and p.depth == 100


def test_gs_plan_diagonal_all_singletons():
    A = sp.diags(np.arange(1.0, 11.0)).tocsr()
    p = _plan(A)
    assert p.nchains == 10 and p.depth == 1


def test_gs_plan_grid_lines():
    g = 32
    A = laplacian_2d(g)
    p = _plan(A, max_threads=8, max_window=32 * g)
    assert p.nchains == g  # one chain per grid line
    assert p.depth == 2 * g - 1  # 5-point level-set depth
    _check_plan(A, p, 8, 32 * g)


def test_gs_plan_3d_depth():
    g = 12
    A = laplacian_3d(g)
    p = _plan(A)
    assert p.depth == 3 * g - 2
    _check_plan(A, p, 128, 24576)


@pytest.mark.parametrize("seed", range(4))
def test_gs_plan_random(seed):
    A = random_spd_csr(300, density=0.03, seed=seed)
    p = _plan(A, max_chain=7, max_threads=32, max_window=320)
    assert np.max(np.diff(p.chain_ptr)) <= 7
    _check_plan(A, p, 32, 320)


def test_gs_plan_c1_fine():
    A = c1_fine()
    p = _plan(A)
    assert p.depth == 255  # C1 fine-level depth


def test_no_cpu_fallback():
    """Without a GPU the device operator must fail loudly, not fall back."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1907_04417_b200 import DeviceError, GpuMultigridOperator

    A = laplacian_2d(4)
    with pytest.raises(DeviceError):
        GpuMultigridOperator([A], [])


def test_setup_device_kernels_no_cpu_fallback():
    """The setup's device matching and device SVD fail loudly without a GPU
    (the host restatements run only when the GpuConfig asks for them)."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1907_04417_b200 import DeviceError
    from paper_1907_04417_b200.setup import _jacobi_svd_device, greedy_matching_device

    with pytest.raises(DeviceError):
        _jacobi_svd_device(np.array([0, 2], dtype=np.int32), np.ones((2, 3)), 3)
    A = laplacian_2d(4)
    with pytest.raises(DeviceError):
        greedy_matching_device(A, np.ones(A.shape[0]))
