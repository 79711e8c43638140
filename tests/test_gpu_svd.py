"""GPU: the batched local SVD of the multi-vector setup (csrc/svd.cuh,
mvamg_jacobi_svd_batch_device) bit for bit against the host restatement
mvamg_jacobi_svd_batch (pkg/src/mvamg/svd.py:17-55, _kernels.py:64-121),
which tests/test_setup.py pins to the reference's hierarchies."""

import ctypes

import numpy as np
import pytest

from paper_1907_04417_b200 import _lib, problems
from paper_1907_04417_b200.setup import SVD_MAX_SWEEPS, SVD_PAIR_TOL, _jacobi_svd_device

pytestmark = pytest.mark.gpu


def _host(rp, local, k, sweeps=SVD_MAX_SWEEPS):
    nblk = rp.shape[0] - 1
    U, sig = np.empty_like(local), np.empty((nblk, k))
    failed = ctypes.c_int(-1)
    vp = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    code = _lib.load().mvamg_jacobi_svd_batch(nblk, vp(rp), k, vp(local), sweeps, SVD_PAIR_TOL, vp(U), vp(sig),
                                              ctypes.byref(failed))
    return code, U, sig, failed.value


def _device(rp, local, k, sweeps=SVD_MAX_SWEEPS):
    from paper_1907_04417_b200.device import ptr, stream_handle, to_device, torch_cuda

    torch = torch_cuda()
    nblk = rp.shape[0] - 1
    d_rp, d_a = to_device(rp, np.int32), to_device(local, np.float64)
    d_u = torch.empty(max(1, local.size), dtype=torch.float64, device="cuda")
    d_s = torch.empty(max(1, nblk * k), dtype=torch.float64, device="cuda")
    failed = ctypes.c_int(-1)
    code = _lib.load().mvamg_jacobi_svd_batch_device(nblk, ptr(d_rp), k, ptr(d_a), sweeps, SVD_PAIR_TOL, ptr(d_u),
                                                     ptr(d_s), ctypes.byref(failed), stream_handle())
    U = d_u.cpu().numpy()[:local.size].reshape(local.shape)
    return code, U, d_s.cpu().numpy()[:nblk * k].reshape(nblk, k), failed.value


def _blocks(rng, k, nblk):
    sizes = rng.integers(1, 65, nblk)
    rp = np.zeros(nblk + 1, dtype=np.int32)
    np.cumsum(sizes, out=rp[1:])
    local = rng.standard_normal((int(rp[-1]), k))
    for b in range(nblk):  # special blocks: zero, rank one, duplicate columns, tiny / huge scale, smooth
        r0, r1 = rp[b], rp[b + 1]
        kind = b % 7
        if kind == 0:
            local[r0:r1] = 0.0
        elif kind == 1:
            local[r0:r1] = np.outer(rng.standard_normal(r1 - r0), rng.standard_normal(k))
        elif kind == 2 and k > 1:
            local[r0:r1, 1] = local[r0:r1, 0]
        elif kind == 3:
            local[r0:r1] *= 1e-150
        elif kind == 4:
            local[r0:r1] *= 1e150
        elif kind == 5:
            local[r0:r1] = np.cos(np.outer(np.arange(r1 - r0), np.arange(1, k + 1)) / 40.0)
    return rp, np.ascontiguousarray(local)


def same_bits(a, b):
    return np.array_equal(np.ascontiguousarray(a).view(np.int64), np.ascontiguousarray(b).view(np.int64))


@pytest.mark.parametrize("k", [1, 2, 3, 5, 8, 16])
def test_device_svd_bit_identical(k):
    rng = np.random.default_rng(100 + k)
    rp, local = _blocks(rng, k, 3000)
    ch, Uh, sh, _ = _host(rp, local, k)
    cd, Ud, sd, _ = _device(rp, local, k)
    assert ch == cd == 0
    assert same_bits(Uh, Ud)
    assert same_bits(sh, sd)


def test_device_svd_nonconvergence_reports_first_block():
    """With one sweep allowed, the first block that needs a rotation fails,
    on both paths (SvdConvergenceError carries that aggregate id)."""
    rng = np.random.default_rng(7)
    k = 4
    rp = np.arange(0, 9 * 10, 10, dtype=np.int32)  # 8 blocks of 10 rows
    local = np.zeros((80, k))
    local[30:40] = rng.standard_normal((10, k))
    local[60:70] = rng.standard_normal((10, k))
    ch, _, _, fh = _host(rp, local, k, sweeps=1)
    cd, _, _, fd = _device(rp, local, k, sweeps=1)
    assert ch == cd == _lib.E_NOT_SPD
    assert fh == fd == 3


def test_device_svd_rejects_bad_arguments():
    rp = np.array([0, 2], dtype=np.int32)
    code, *_ = _device(rp, np.ones((2, 17)), 17)
    assert code == _lib.E_ARG
    code, *_ = _device(np.array([0, 2, 2], dtype=np.int32), np.ones((2, 3)), 3)  # empty block
    assert code == _lib.E_ARG


def test_device_svd_on_fit_blocks():
    """The blocks the setup actually factors (C2-size aggregates of the fine
    level with five cosine-like smooth vectors) via the setup's own helper."""
    n = 256 * 256
    rng = np.random.default_rng(3)
    sizes = rng.integers(8, 65, n // 30)
    rp = np.zeros(sizes.shape[0] + 1, dtype=np.int32)
    np.cumsum(sizes, out=rp[1:])
    x = np.arange(rp[-1]) / rp[-1]
    local = np.ascontiguousarray(np.stack([np.cos(np.pi * (j + 1) * x) + 1e-3 * rng.standard_normal(x.shape)
                                           for j in range(5)], axis=1))
    ch, Uh, sh, _ = _host(rp, local, 5)
    cd, Ud, sd, _ = _jacobi_svd_device(rp, local, 5)
    assert ch == cd == 0
    assert same_bits(Uh, Ud) and same_bits(sh, sd)


def test_fit_with_device_svd_is_identical():
    """A whole fit with the device SVD gives the same hierarchy, bit for bit,
    as with the host SVD (elasticity 64^2)."""
    import paper_1907_04417_b200 as mv

    A = problems.elasticity_q1(64)
    e1 = mv.MultiVectorAMG(config=mv.GpuConfig(device_svd=True)).fit(A)
    e0 = mv.MultiVectorAMG(config=mv.GpuConfig(device_svd=False)).fit(A)
    assert len(e0.hierarchy_.matrices) == len(e1.hierarchy_.matrices)
    for M0, M1 in zip(e0.hierarchy_.matrices, e1.hierarchy_.matrices):
        assert M0.shape == M1.shape and np.array_equal(M0.indptr, M1.indptr)
        assert np.array_equal(M0.indices, M1.indices) and same_bits(M0.data, M1.data)
    for P0, P1 in zip(e0.hierarchy_.prolongator_matrices, e1.hierarchy_.prolongator_matrices):
        assert np.array_equal(P0.indices, P1.indices) and same_bits(P0.data, P1.data)
