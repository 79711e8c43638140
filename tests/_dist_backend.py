"""Test-only arithmetic backend for paper_1907_04417_b200.distributed: the CPU
oracle (oracle/) on torch CPU tensors, so the row-partitioned algorithm (plans,
relays, halos, gather / broadcast) runs under gloo without a GPU.  The product
backend is distributed.DeviceBackend; this file lives in tests/ only."""

import numpy as np
import torch

from oracle.oracle import OracleOperator, oracle_gs, oracle_spmv


class OracleBackend:
    def vec(self, n):
        return torch.zeros(n, dtype=torch.float64)

    def index(self, a):
        return torch.as_tensor(np.asarray(a, dtype=np.int64)) if len(a) else None

    def from_host(self, a):
        return torch.from_numpy(np.array(a, dtype=np.float64))

    def to_host(self, t):
        return t.numpy().copy()

    def mat(self, M):
        return M if M.shape[0] > 0 else None

    def spmv(self, M, x, y):
        if M is not None:
            y.numpy()[:] = oracle_spmv(M, x.numpy())

    def residual(self, M, b, x, r):
        if M is None or M.nnz == 0 or x.numel() == 0:
            r.copy_(b)
            return
        r.numpy()[:] = b.numpy() - oracle_spmv(M, x.numpy())

    def spmv_add(self, M, x, y):
        if M is not None:
            y.numpy()[:] = y.numpy() + oracle_spmv(M, x.numpy())

    def gather(self, idx, src, dst):
        if idx is not None:
            dst.numpy()[:] = src.numpy()[idx.numpy()]

    def scatter(self, idx, src, dst):
        if idx is not None:
            dst.numpy()[idx.numpy()] = src.numpy()

    def dot(self, x, y):
        return float(np.dot(x.numpy(), y.numpy()))

    def axpy(self, alpha, x, y):
        y.numpy()[:] = y.numpy() + alpha * x.numpy()

    def xpby(self, x, beta, y):
        y.numpy()[:] = x.numpy() + beta * y.numpy()

    def smoother(self, A):
        return A if A.shape[0] else None

    def gs(self, A, direction, b, x_old, x_new):
        x = np.zeros(A.shape[0]) if x_old is None else np.array(x_old.numpy(), copy=True)
        oracle_gs(A, np.ascontiguousarray(b.numpy()), x, "forward" if direction == 0 else "backward")
        x_new.numpy()[:] = x

    def coarse(self, mats, pros):
        return OracleOperator(mats, pros)

    def coarse_apply(self, op, rc, out):
        out.numpy()[:] = op.apply(rc.numpy())
