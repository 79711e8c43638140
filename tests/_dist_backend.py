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


# ---- pipelined sweeps (DistributedVCycle.pipelined) emulated on the CPU ----
# Every rank's extended x lives in POSIX shared memory; a rank's sweep walks its
# own rows in sweep order, polls a ghost input until its owner (another process,
# concurrently) has stored it, and stores each final value into its own x and
# into the peers that read it -- the protocol of mvamg_gs_row_sweep_ext_f64,
# with the same arithmetic as the serial loop (_kernels.py:15-38).
import time  # noqa: E402
from multiprocessing import shared_memory  # noqa: E402

SENTINEL = np.int64(-1)


class PipelinedOracleBackend(OracleBackend):
    def __init__(self, tag):
        self.tag = tag
        self._shm = []

    def pipe_ok(self, comm):
        return True

    def pipe_plan(self, M_ext, row_range, mode, mirror_rows):
        return {"M": M_ext, "range": row_range, "mode": mode, "mirror": mirror_rows}

    def pipe_share(self, comm, n):
        name = f"mvamg_{self.tag}_{comm.rank}"
        shm = shared_memory.SharedMemory(name=name, create=True, size=max(8, 8 * n))
        self._shm.append(shm)
        comm.barrier()
        peers = []
        for q in range(comm.size):
            if q == comm.rank:
                peers.append(np.ndarray((max(1, n),), dtype=np.float64, buffer=shm.buf))
            else:
                other = shared_memory.SharedMemory(name=f"mvamg_{self.tag}_{q}")
                self._shm.append(other)
                peers.append(np.ndarray((other.size // 8,), dtype=np.float64, buffer=other.buf))
        xp = torch.from_numpy(peers[comm.rank][:n])
        return xp, peers

    def fill_sentinel(self, t):
        t.numpy().view(np.int64)[:] = SENTINEL

    def pipe_sweep(self, plan, b_own, x_old_ext, x_ext, peers):
        M, (lo, hi), mode, mirror = plan["M"], plan["range"], plan["mode"], plan["mirror"]
        x = x_ext.numpy()
        xi64 = x.view(np.int64)
        b = b_own.numpy()
        xo = None if x_old_ext is None else x_old_ext.numpy()
        ip, ix, v = M.indptr, M.indices, M.data
        fwd = mode == 0
        rows = range(lo, hi) if fwd else range(hi - 1, lo - 1, -1)
        for i in rows:
            s = float(b[i - lo])
            d = 0.0
            for k in range(ip[i], ip[i + 1]):
                j = int(ix[k])
                if j == i:
                    d = float(v[k])
                    continue
                if (j < i) != fwd:             # the other side: x_old (backward from x_old) or zero
                    if xo is not None and not fwd and j < i:
                        s = s - float(v[k]) * float(xo[j])
                    continue
                while xi64[j] == SENTINEL:     # a ghost (or own row) not final yet
                    time.sleep(0)
                s = s - float(v[k]) * float(x[j])
            xv = s / d
            for q, slot in mirror.get(i - lo, ()):
                peers[q][slot] = xv
            x[i] = xv

    def close(self):
        for shm in self._shm:
            shm.close()
        for shm in self._shm[:1]:
            shm.unlink()
