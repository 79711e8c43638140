"""Row-partitioned solve across GPUs: one process per GPU.

The finest level A_0 is split into contiguous row blocks balanced by nonzeros.
Coarse levels are gathered to rank 0, as SURVEY 8(e) specifies.  One V-cycle
application on rank r (pkg/src/mvamg/cycles.py:150-179 with the default
smoothers) runs as follows.

1. Forward GS from x = 0 over the own rows.  Pipelined (one GPU per rank):
   every rank launches its sweep at once over its extended layout
   [lower ghosts | own rows | upper ghosts]; its kernel polls a ghost input
   until the owner's kernel -- running concurrently on the neighbour GPU --
   stores the final value straight into this rank's extended x over NVLink
   (CUDA IPC pointers, mirror tables built here; the value's NaN sentinel is
   its own ready flag, as between the tiles of one GPU).  The sweep is one
   wavefront across the GPUs: a slab starts as soon as the first rows it
   needs from the slab below are final, not when that slab is done, so the
   critical path is the global DAG depth plus one hop per slab boundary
   (C5 at N GPUs: 958 levels + (N - 1) hops) instead of the relay's sum of
   the slabs' depths (N (40 + 319 + 319) levels at N = 8).  Fallback (ranks
   sharing a GPU, or a backend without it): a relay in rank order -- rank r
   receives the final lower ghosts, folds them into the right-hand side and
   sweeps its block with the single-GPU kernels.
2. t = r - A x through the x halo (ghosts before and after the own rows, in
   global column order, so each row's sum keeps the scipy CSR order).
3. Restriction.  Each aggregate belongs to the rank owning its smallest
   member.  The owner receives the remote members' t values (restriction
   halo) and forms its rows of R t in CSR order.
4. The owned coarse values are gathered to rank 0.  Rank 0 runs the V-cycle
   of levels 1..L (a GpuMultigridOperator) and broadcasts x_c.
5. x += P x_c on the own rows.
6. Backward GS from x: pipelined as 1 in the other direction (the old lower
   neighbours, own and ghost, folded into the right-hand side first, in CSR
   order); or relayed in reverse rank order (old lower ghosts and new upper
   ghosts folded into the right-hand side).

`dist_pcg` is krylov.py:28-72 over distributed vectors.  q = A p uses the halo
SpMV; two allreduces per iteration (p'q, then r'r and r'z together).

Parity (north star): at one rank the result is bit-identical to the
single-GPU path.  The pipelined sweeps keep both the dependency order and
every row's CSR summation order, so a V-cycle at any rank count is
bit-identical to one GPU (tests/test_distributed.py emulates it across
processes on the CPU; tests/test_gpu_distributed.py runs the kernel rank by
rank on one GPU).  The relay rounds the folded upper ghosts of the backward
sweep differently (cycle within 1e-10).  Dots are summed across ranks:
PCG histories within 1e-10, iteration count equal or +-1.

Scaling.  SpMV, restriction, prolongation and the vector updates shard.  The
exact-order sweeps cannot: their critical path is the DAG depth (DESIGN.md
(e)); the pipelined wavefront keeps it at one GPU's depth plus the hops.

Communication goes through `Comm`, a thin wrapper over torch.distributed.
NCCL moves device buffers directly.  Other backends (gloo: the CPU tests and
the one-GPU multi-process test) stage through host memory.  Arithmetic goes
through a backend object; the product backend is `DeviceBackend`
(libmvamg_b200.so kernels).  The CPU tests inject their own backend from
tests/ (the oracle).  This module has no CPU arithmetic path.
"""

from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp

from .device import as_csr
from .exceptions import NotSpdError
from .krylov import SolveReport


# ------------------------------------------------------------------- plans ---
@dataclass
class RowPartition:
    """Contiguous row blocks: rank r owns rows offsets[r]:offsets[r+1]."""

    offsets: np.ndarray

    @property
    def nranks(self):
        return self.offsets.shape[0] - 1

    @classmethod
    def balanced(cls, A, nranks):
        """Blocks with about nnz(A)/nranks nonzeros each, at least one row each."""
        A = as_csr(A)
        n = A.shape[0]
        if nranks < 1 or n < nranks:
            raise ValueError(f"cannot split {n} rows over {nranks} ranks")
        targets = A.nnz * np.arange(1, nranks) / nranks
        cuts = np.searchsorted(A.indptr, targets, side="left").astype(np.int64)
        off = np.concatenate([[0], cuts, [n]]).astype(np.int64)
        for r in range(1, nranks):  # at least one row per rank, monotone
            off[r] = min(max(off[r], off[r - 1] + 1), n - (nranks - r))
        return cls(off)

    def owner(self, idx):
        return np.searchsorted(self.offsets, np.asarray(idx), side="right") - 1

    def block(self, r):
        return int(self.offsets[r]), int(self.offsets[r + 1])


@dataclass
class Halo:
    """Extended layout [lower ghosts | own rows | upper ghosts] of one rank.

    The ghosts are sorted global indices, so extended positions follow global
    order.  recv[q] is the slice of the ghost array that rank q fills;
    send[q] lists the local indices of own rows that rank q needs."""

    rank: int
    lo: int
    hi: int
    ghosts: np.ndarray
    n_lower: int
    recv: dict = field(default_factory=dict)
    send: dict = field(default_factory=dict)

    @property
    def n_own(self):
        return self.hi - self.lo

    @property
    def n_ghost(self):
        return self.ghosts.shape[0]

    def ext_index(self, cols):
        """Global column -> extended position (columns must be own or ghosts)."""
        cols = np.asarray(cols, dtype=np.int64)
        out = np.empty(cols.shape[0], dtype=np.int64)
        own = (cols >= self.lo) & (cols < self.hi)
        out[own] = self.n_lower + cols[own] - self.lo
        g = np.searchsorted(self.ghosts, cols[~own])
        if g.size and (np.any(g >= self.n_ghost) or np.any(self.ghosts[np.minimum(g, self.n_ghost - 1)]
                                                            != cols[~own])):
            raise ValueError("column is neither owned nor a ghost")
        out[~own] = np.where(g < self.n_lower, g, g + self.n_own)
        return out


def make_halo(part, rank, needed):
    """Halo of `rank` given needed[q] = sorted global columns rank q reads
    (own columns included or not -- they are filtered)."""
    lo, hi = part.block(rank)
    mine = np.asarray(needed[rank], dtype=np.int64)
    ghosts = np.unique(mine[(mine < lo) | (mine >= hi)])
    h = Halo(rank, lo, hi, ghosts, int(np.searchsorted(ghosts, lo)))
    own_of = part.owner(ghosts)
    for q in range(part.nranks):
        if q == rank:
            continue
        idx = np.nonzero(own_of == q)[0]
        if idx.size:
            h.recv[q] = slice(int(idx[0]), int(idx[-1]) + 1)  # contiguous: ghosts sorted, blocks contiguous
        qn = np.asarray(needed[q], dtype=np.int64)
        qlo, qhi = part.block(q)
        want = np.unique(qn[(qn >= lo) & (qn < hi) & ((qn < qlo) | (qn >= qhi))])
        if want.size:
            h.send[q] = (want - lo).astype(np.int32)
    return h


def _remap(M, halo):
    """Rows of M (already restricted to what this rank forms) with columns in
    the extended layout of `halo`; column order (hence CSR sum order) kept."""
    M = sp.csr_matrix(M)
    cols = halo.ext_index(M.indices)
    return sp.csr_matrix((M.data, cols, M.indptr), shape=(M.shape[0], halo.n_own + halo.n_ghost))


@dataclass
class RankPlan:
    """Everything rank r needs for the fine level (host CSR, built once)."""

    part: RowPartition
    rank: int
    xhalo: Halo                 # SpMV / GS ghosts of x
    thalo: Halo                 # restriction ghosts of t
    A_ext: object               # own rows of A_0 over the x extended layout
    A_own: object               # square own block (GS)
    A_lg: object                # own rows x lower ghosts (fold)
    A_ug: object                # own rows x upper ghosts (fold)
    R_ext: object               # owned aggregates' rows of R_0 over the t extended layout
    coarse_own: np.ndarray      # global coarse indices of the owned aggregates (R_ext's rows)
    coarse_counts: np.ndarray   # owned aggregates per rank (rank 0 gathers)
    coarse_lists: list          # per rank: global coarse indices, in the order they are sent
    P_own: object               # own rows of P_0 (n_own x n_1)
    n: int
    nc: int
    M_ext: object = None        # pipelined sweeps: n_ext x n_ext, own rows over the extended layout, ghost rows empty
    mirror_fwd: dict = None     # own local row -> [(peer, ext slot)]: peers reading it as a lower ghost
    mirror_bwd: dict = None     # ... as an upper ghost


def plan_rank(A, P, part, rank):
    """Host plan of one rank from the global fine operator A_0 and P_0."""
    A = as_csr(A)
    P = as_csr(P)
    n, nc = P.shape
    if A.shape != (n, n):
        raise ValueError("P rows must match A")
    R = P.T.tocsr()
    R.sort_indices()
    nr = part.nranks
    need_x = [np.unique(A.indices[A.indptr[part.offsets[q]]:A.indptr[part.offsets[q + 1]]]) for q in range(nr)]
    # aggregate c belongs to the rank owning its smallest member (R rows are sorted)
    rlen = np.diff(R.indptr)
    first = np.where(rlen > 0, R.indices[np.minimum(R.indptr[:-1], max(R.nnz - 1, 0))], 0)
    cown = part.owner(first)
    lists = [np.nonzero(cown == q)[0] for q in range(nr)]
    need_t = [np.unique(R[rows].indices) for rows in lists]
    xh = make_halo(part, rank, need_x)
    th = make_halo(part, rank, need_t)
    lo, hi = part.block(rank)
    Ar = A[lo:hi]
    A_ext = _remap(Ar, xh)
    A_own = Ar[:, lo:hi].tocsr()
    A_lg = Ar[:, xh.ghosts[:xh.n_lower]].tocsr()
    A_ug = Ar[:, xh.ghosts[xh.n_lower:]].tocsr()
    for M in (A_own, A_lg, A_ug):
        M.sort_indices()
    R_ext = _remap(R[lists[rank]], th)
    pl = RankPlan(part, rank, xh, th, A_ext, A_own, A_lg, A_ug, R_ext, lists[rank],
                  np.array([len(x) for x in lists]), lists, P[lo:hi].tocsr(), n, nc)
    # pipelined sweeps: the own rows as rows [n_lower, n_lower + n_own) of a square
    # matrix over the extended layout (ghost rows empty; global order kept, so a
    # row's CSR order and its lower / upper split are the single-GPU ones), and for
    # every own row the peers that read it as a ghost, with its slot in their layout
    n_ext = xh.n_own + xh.n_ghost
    ip = np.zeros(n_ext + 1, dtype=np.int64)
    ip[xh.n_lower + 1:xh.n_lower + xh.n_own + 1] = np.diff(A_ext.indptr)
    np.cumsum(ip, out=ip)
    pl.M_ext = sp.csr_matrix((A_ext.data, A_ext.indices, ip), shape=(n_ext, n_ext))
    pl.mirror_fwd, pl.mirror_bwd = {}, {}
    for q in range(nr):
        if q == rank:
            continue
        hq = make_halo(part, q, need_x)
        sel = np.nonzero((hq.ghosts >= lo) & (hq.ghosts < hi))[0]
        for g in sel:
            own = int(hq.ghosts[g] - lo)
            if g < hq.n_lower:   # q reads it as a lower ghost: the forward sweep feeds q
                pl.mirror_fwd.setdefault(own, []).append((q, int(g)))
            else:                # an upper ghost of q: the backward sweep feeds q
                pl.mirror_bwd.setdefault(own, []).append((q, int(g) + hq.n_own))
    return pl


# -------------------------------------------------------------------- comm ---
class Comm:
    """Point-to-point and collectives of the row-partitioned solve over
    torch.distributed (NCCL: device buffers directly; other backends: staged
    through host memory).  world_size 1 needs no process group."""

    def __init__(self, group=None, direct=None):
        """direct: hand the arithmetic's tensors to the backend as they are (NCCL
        with device buffers; default) or stage them through host memory (other
        backends with device buffers).  The CPU tests use direct=True with gloo
        and host tensors to run the NCCL code path."""
        import torch.distributed as dist

        self.dist = dist if dist.is_available() and dist.is_initialized() else None
        self.group = group
        if self.dist is None:
            self.rank, self.size, self.nccl = 0, 1, False
        else:
            self.rank = dist.get_rank(group)
            self.size = dist.get_world_size(group)
            self.nccl = dist.get_backend(group) == "nccl"
        self.direct = self.nccl if direct is None else bool(direct)

    def _stage(self, t):
        return t if self.direct else t.detach().to("cpu")

    def sendrecv(self, sends, recvs):
        """sends: [(peer, tensor)], recvs: [(peer, tensor)] -- one batch."""
        if not sends and not recvs:
            return
        dist = self.dist
        ops, back = [], []
        for q, t in sends:
            ops.append(dist.P2POp(dist.isend, self._stage(t).contiguous(), q, self.group))
        for q, t in recvs:
            buf = t if self.direct else t.new_empty(t.shape, device="cpu")
            ops.append(dist.P2POp(dist.irecv, buf, q, self.group))
            back.append((t, buf))
        for req in dist.batch_isend_irecv(ops):
            req.wait()
        for t, buf in back:
            if buf is not t:
                t.copy_(buf)

    def allreduce(self, values):
        """Sum of a short host float list over the ranks."""
        if self.size == 1:
            return [float(v) for v in values]
        import torch

        dev = "cuda" if self.nccl else "cpu"
        t = torch.tensor(values, dtype=torch.float64, device=dev)
        self.dist.all_reduce(t, group=self.group)
        return [float(v) for v in t.cpu().tolist()]

    def broadcast(self, t, root=0):
        if self.size == 1:
            return
        if self.direct:
            self.dist.broadcast(t, root, group=self.group)
        else:
            buf = t.detach().to("cpu")
            self.dist.broadcast(buf, root, group=self.group)
            t.copy_(buf)

    def barrier(self):
        if self.size > 1:
            self.dist.barrier(group=self.group)


# ----------------------------------------------------------------- backend ---
class DeviceBackend:
    """The product arithmetic: libmvamg_b200.so kernels on torch-owned buffers."""

    def __init__(self, config=None):
        from .device import GpuConfig, torch_cuda

        self.torch = torch_cuda()
        self.cfg = config or GpuConfig()
        from . import _lib

        self.L = _lib.load()
        self._lib = _lib
        self._ws = self.torch.zeros(8, dtype=self.torch.int32, device="cuda")
        self._dot_ws = self.torch.empty(self.L.mvamg_dot_ws_bytes(), dtype=self.torch.uint8, device="cuda")
        self._dot_out = self.torch.empty(1, dtype=self.torch.float64, device="cuda")

    # buffers
    def vec(self, n):
        return self.torch.zeros(n, dtype=self.torch.float64, device="cuda")

    def index(self, a):
        from .device import to_device

        return to_device(np.asarray(a, dtype=np.int32)) if len(a) else None

    def from_host(self, a):
        from .device import to_device

        return to_device(np.asarray(a, dtype=np.float64))

    def to_host(self, t):
        return t.detach().cpu().numpy()

    # operators
    def mat(self, M):
        from .device import DeviceCSR

        return DeviceCSR(M) if M.shape[0] > 0 else None

    def _s(self):
        from .device import stream_handle

        return stream_handle()

    def spmv(self, M, x, y):
        from .device import ptr

        if M is not None:
            self._lib.check(self.L.mvamg_csr_spmv_f64(M.n, *M.ptrs(), ptr(x), ptr(y), self._s()), "spmv")

    def residual(self, M, b, x, r):
        """r = b - M x (M None or empty: r = b)."""
        from .device import ptr

        if M is None or M.nnz == 0 or x.numel() == 0:
            if r.data_ptr() != b.data_ptr():
                r.copy_(b)
            return
        self._lib.check(self.L.mvamg_csr_residual_f64(M.n, *M.ptrs(), ptr(b), ptr(x), ptr(r), self._s()),
                        "residual")

    def spmv_add(self, M, x, y):
        from .device import ptr

        if M is not None:
            self._lib.check(self.L.mvamg_csr_spmv_add_f64(M.n, *M.ptrs(), ptr(x), ptr(y), self._s()), "spmv_add")

    def gather(self, idx, src, dst):
        from .device import ptr

        if idx is not None:
            self._lib.check(self.L.mvamg_gather_f64(idx.numel(), ptr(idx), ptr(src), ptr(dst), self._s()), "gather")

    def scatter(self, idx, src, dst):
        from .device import ptr

        if idx is not None:
            self._lib.check(self.L.mvamg_scatter_f64(idx.numel(), ptr(idx), ptr(src), ptr(dst), self._s()),
                            "scatter")

    def dot(self, x, y):
        from .device import ptr

        self._lib.check(self.L.mvamg_dot_f64(x.numel(), ptr(x), ptr(y), ptr(self._dot_out), ptr(self._dot_ws),
                                             self._s()), "dot")
        return float(self._dot_out.item())

    def axpy(self, alpha, x, y):
        from .device import ptr

        self._lib.check(self.L.mvamg_axpy_f64(x.numel(), float(alpha), ptr(x), ptr(y), self._s()), "axpy")

    def xpby(self, x, beta, y):
        from .device import ptr

        self._lib.check(self.L.mvamg_xpby_f64(x.numel(), ptr(x), float(beta), ptr(y), self._s()), "xpby")

    # smoother on the own block: the single-GPU planner's choice for a fine level
    def smoother(self, A):
        from .device import DeviceGsPlan, DeviceGsRows

        if A.shape[0] == 0:
            return None
        gp = DeviceGsPlan(A, self.cfg)
        if gp.plan.nchains > 0 and A.shape[0] / gp.plan.nchains < self.cfg.min_chain_rows:
            return ("rows", {0: DeviceGsRows(A, 0, self.cfg), 2: DeviceGsRows(A, 2, self.cfg)})
        return ("wave", gp)

    def gs(self, sm, direction, b, x_old, x_new):
        """x_new = one exact-order GS sweep of the own block (forward from 0 when x_old is None)."""
        kind, obj = sm
        if kind == "wave":
            obj.sweep(direction, b, x_old, x_new, self._ws)
        else:
            obj[0 if direction == 0 else 2].sweep(b, x_old, x_new, self._ws)

    # pipelined fine-level sweeps across the ranks (DistributedVCycle.pipelined)
    def pipe_ok(self, comm):
        """Only with one GPU per rank (NCCL): ranks whose kernels poll each other
        must not share a GPU (one could hold every SM while the other waits)."""
        return comm.nccl

    def pipe_plan(self, M_ext, row_range, mode, mirror_rows):
        """Row schedule of the own rows over the extended layout plus the
        position-indexed mirror table (peer << 24 | slot) of mvamg_gs_row_sweep_ext_f64."""
        from .device import DeviceGsRows, to_device

        rows = DeviceGsRows(M_ext, mode, self.cfg, row_range=row_range)
        lo = row_range[0]
        rowid = rows.rowid.cpu().numpy()[:rows.n]
        ptr_, dst = [0], []
        for i in rowid:
            for q, slot in mirror_rows.get(int(i) - lo, ()):
                if slot >= (1 << 24) or q >= 256:
                    raise ValueError("pipelined sweep: mirror slot / peer out of range")
                dst.append((q << 24) | slot)
            ptr_.append(len(dst))
        return {"rows": rows, "mptr": to_device(np.asarray(ptr_, dtype=np.int32)),
                "mdst": to_device(np.asarray(dst or [0], dtype=np.uint32).view(np.int32))}

    def pipe_share(self, comm, n):
        """This rank's extended x for the pipelined sweeps and a device array of
        every rank's (CUDA IPC: the peers' kernels store into it over NVLink)."""
        import ctypes

        torch = self.torch
        xp = torch.empty(max(1, n), dtype=torch.float64, device="cuda")
        handle = ctypes.create_string_buffer(64)
        self._lib.check(self.L.mvamg_ipc_handle(ctypes.c_void_p(xp.data_ptr()), handle), "ipc_handle")
        handles = [handle.raw]
        if comm.size > 1:
            handles = [None] * comm.size
            comm.dist.all_gather_object(handles, handle.raw, group=comm.group)
        ptrs = []
        self._ipc_open = []
        for q, h in enumerate(handles):
            if q == comm.rank:
                ptrs.append(xp.data_ptr())
                continue
            p = ctypes.c_void_p()
            self._lib.check(self.L.mvamg_ipc_open(ctypes.create_string_buffer(h, 64), ctypes.byref(p)), "ipc_open")
            self._ipc_open.append(p)
            ptrs.append(p.value)
        peers = torch.tensor(ptrs, dtype=torch.int64, device="cuda")
        return xp[:n], peers

    def fill_sentinel(self, t):
        t.view(self.torch.int64).fill_(-1)  # all-ones: the NaN no arithmetic produces (not-yet-final)
        self.torch.cuda.synchronize()       # executed, not just queued, before the ranks synchronise

    def pipe_sweep(self, plan, b_own, x_old_ext, x_ext, peers):
        from .device import ptr  # noqa: F401

        plan["rows"].sweep_ext(b_own, x_old_ext, x_ext, plan["mptr"], plan["mdst"], peers, self._ws, self._s())
        self.torch.cuda.synchronize()
        st = int(self._ws[1].item())
        if st:
            self._ws.zero_()  # the relay's kernels share this status word
            raise RuntimeError(f"pipelined GS sweep: status {st} (timeout waiting on a ghost)")

    def coarse(self, mats, pros):
        from .cycles import CycleSpec, GpuMultigridOperator

        return GpuMultigridOperator(mats, pros, cycle=CycleSpec("V"), config=self.cfg)

    def coarse_apply(self, op, rc, out):
        out.copy_(op.apply_device(rc))


# --------------------------------------------------------------- operator ---
class DistributedVCycle:
    """One rank's share of the row-partitioned V-cycle (module docstring)."""

    def __init__(self, matrices, prolongators, comm=None, backend=None, part=None, pipelined=None):
        """pipelined (default: whenever there are several ranks and the backend
        supports it): the fine-level sweeps run as one wavefront across the
        ranks -- every rank sweeps its rows at once, polling its ghost inputs,
        which their owners store into its extended x the moment they are final
        (mvamg_gs_row_sweep_ext_f64) -- instead of the rank-by-rank relay.  Both
        keep the serial loop's dependency order; the pipelined sweep also keeps
        every row's CSR summation order, so the cycle is bit-identical to one GPU."""
        self.comm = comm or Comm()
        self.be = backend or DeviceBackend()
        mats = [as_csr(M) for M in matrices]
        pros = [as_csr(P) for P in prolongators]
        if len(mats) < 2:
            raise ValueError("the row-partitioned cycle needs at least two levels")
        if len(pros) != len(mats) - 1:
            raise ValueError("need one prolongator per coarse level")
        d = mats[0].diagonal()
        if np.any(d == 0.0):
            raise NotSpdError("zero diagonal entry in level 0")
        self.part = part or RowPartition.balanced(mats[0], self.comm.size)
        if self.part.nranks != self.comm.size:
            raise ValueError("partition / communicator size mismatch")
        r = self.comm.rank
        self.plan = pl = plan_rank(mats[0], pros[0], self.part, r)
        be = self.be
        self.n_own = pl.xhalo.n_own
        self.A_ext, self.A_own, self.A_lg, self.A_ug = (be.mat(pl.A_ext), be.mat(pl.A_own), be.mat(pl.A_lg),
                                                        be.mat(pl.A_ug))
        self.R_ext, self.P_own = be.mat(pl.R_ext), be.mat(pl.P_own)
        self.sm = be.smoother(pl.A_own)
        xh, th = pl.xhalo, pl.thalo
        self.x_send = {q: be.index(i) for q, i in xh.send.items()}
        self.t_send = {q: be.index(i) for q, i in th.send.items()}
        self.coarse_idx = [be.index(c) for c in pl.coarse_lists] if r == 0 else None
        self.coarse_op = be.coarse(mats[1:], pros[1:]) if r == 0 else None
        n_own, nc = self.n_own, pl.nc
        self.xe = be.vec(xh.n_own + xh.n_ghost)        # x in the extended layout
        self.te = be.vec(th.n_own + th.n_ghost)        # t in the extended layout
        self.x_new = be.vec(n_own)
        self.b_fold = be.vec(n_own)
        self.rc_own = be.vec(len(pl.coarse_own))
        self.rc = be.vec(nc)
        self.xc = be.vec(nc)
        self.pe = be.vec(xh.n_own + xh.n_ghost)        # PCG direction, extended
        self._bufs = {}
        if pipelined is None:
            pipelined = self.comm.size > 1 and hasattr(be, "pipe_plan") and be.pipe_ok(self.comm)
        self.pipelined = bool(pipelined)
        if self.pipelined:
            lo_e, hi_e = xh.n_lower, xh.n_lower + xh.n_own
            self.pipe_fwd = be.pipe_plan(pl.M_ext, (lo_e, hi_e), 0, pl.mirror_fwd)
            self.pipe_bwd = be.pipe_plan(pl.M_ext, (lo_e, hi_e), 2, pl.mirror_bwd)
            # the pipelined sweeps' extended x, which the peers store into, and theirs
            self.xp, self.peers = be.pipe_share(self.comm, xh.n_own + xh.n_ghost)

    # ---- halo exchanges --------------------------------------------------
    def _buf(self, key, n):
        t = self._bufs.get(key)
        if t is None or t.numel() != n:
            t = self._bufs[key] = self.be.vec(n)
        return t

    def _xsl(self, halo, ext):
        lo = halo.n_lower
        return ext[lo:lo + halo.n_own]

    def _ghost(self, halo, ext, q):
        """View of ext holding the ghosts rank q sends (recv slice, shifted past own rows if upper)."""
        s = halo.recv[q]
        if s.start >= halo.n_lower:
            return ext[s.start + halo.n_own:s.stop + halo.n_own]
        return ext[s.start:s.stop]

    def exchange(self, halo, ext, send_idx, peers_to=None, peers_from=None):
        """Fill ext's ghosts from the owners; send own values to the ranks in
        peers_to (default: all) and receive from peers_from (default: all)."""
        own = self._xsl(halo, ext)
        sends, recvs = [], []
        for q, idx in send_idx.items():
            if peers_to is not None and q not in peers_to:
                continue
            buf = self._buf(("s", id(halo), q), idx.numel())
            self.be.gather(idx, own, buf)
            sends.append((q, buf))
        for q in halo.recv:
            if peers_from is not None and q not in peers_from:
                continue
            recvs.append((q, self._ghost(halo, ext, q)))
        self.comm.sendrecv(sends, recvs)

    # ---- one application ------------------------------------------------
    def apply(self, r_own, z_own):
        """z_own = this rank's rows of B r (one V-cycle, default smoothers)."""
        be, pl, comm = self.be, self.plan, self.comm
        rank, nr = comm.rank, comm.size
        xh, th = pl.xhalo, pl.thalo
        xe = self.xe
        x_own = self._xsl(xh, xe)
        lower = xe[:xh.n_lower]
        upper = xe[xh.n_lower + xh.n_own:]
        # 1. forward GS from x = 0: one wavefront across the ranks, or relayed in rank order
        if self.pipelined and self._pipe_sweep(self.pipe_fwd, r_own, None):
            self._xsl(xh, xe).copy_(self._xsl(xh, self.xp))
        else:
            self.exchange(xh, xe, self.x_send, peers_to=(), peers_from=range(rank))
            be.residual(self.A_lg, r_own, lower, self.b_fold)
            be.gs(self.sm, 0, self.b_fold, None, x_own)
            self.exchange(xh, xe, self.x_send, peers_to=range(rank + 1, nr), peers_from=())
        # 2. t = r - A x over the full x halo
        self.exchange(xh, xe, self.x_send)
        t_own = self._xsl(th, self.te)
        be.residual(self.A_ext, r_own, xe, t_own)
        # 3. restriction of the owned aggregates (remote members via the t halo)
        self.exchange(th, self.te, self.t_send)
        be.spmv(self.R_ext, self.te, self.rc_own)
        # 4. gather to rank 0, coarse V-cycle there, broadcast the correction
        if rank == 0:
            be.scatter(self.coarse_idx[0], self.rc_own, self.rc)
            recvs = []
            for q in range(1, nr):
                if pl.coarse_counts[q]:
                    recvs.append((q, self._buf(("rc", q), int(pl.coarse_counts[q]))))
            comm.sendrecv([], recvs)
            for q, buf in recvs:
                be.scatter(self.coarse_idx[q], buf, self.rc)
            be.coarse_apply(self.coarse_op, self.rc, self.xc)
        elif self.rc_own.numel():
            comm.sendrecv([(0, self.rc_own)], [])
        comm.broadcast(self.xc, 0)
        # 5. x += P x_c on the own rows
        be.spmv_add(self.P_own, self.xc, x_own)
        # 6. backward GS from x: one wavefront across the ranks, or relayed in reverse rank order
        self.exchange(xh, xe, self.x_send)                   # old values of every ghost
        if self.pipelined and self._pipe_sweep(self.pipe_bwd, r_own, xe):
            x_own.copy_(self._xsl(xh, self.xp))
            z_own.copy_(x_own)
            return z_own
        self.exchange(xh, xe, self.x_send, peers_to=(), peers_from=range(rank + 1, nr))
        be.residual(self.A_lg, r_own, lower, self.b_fold)
        be.residual(self.A_ug, self.b_fold, upper, self.b_fold)
        be.gs(self.sm, 1, self.b_fold, x_own, self.x_new)
        x_own.copy_(self.x_new)
        self.exchange(xh, xe, self.x_send, peers_to=range(rank), peers_from=())
        z_own.copy_(x_own)
        return z_own

    def _pipe_sweep(self, plan, b_own, x_old_ext):
        """Reset the shared extended x to the sentinel, synchronise the ranks (no
        peer may store a value before the reset), then sweep: every rank's kernel
        polls its ghosts while its peers' kernels are still running.  Returns
        False -- on every rank, and for the rest of the run -- if any rank's sweep
        failed (a ghost never arrived before the kernel's spin limit: peer
        stores not visible on this system); the caller then relays instead."""
        self.be.fill_sentinel(self.xp)
        self.comm.barrier()
        failed = 0.0
        try:
            self.be.pipe_sweep(plan, b_own, x_old_ext, self.xp, self.peers)
        except RuntimeError as exc:
            failed, self.pipe_error = 1.0, str(exc)
        failed, = self.comm.allreduce([failed])  # also: every peer's stores into this rank's x are done
        if failed:
            self.pipelined = False
            return False
        return True

    # ---- distributed operator pieces for PCG ---------------------------------
    def matvec(self, p_own, q_own):
        """q = A p on the own rows (halo exchange of p)."""
        pe = self.pe
        self._xsl(self.plan.xhalo, pe).copy_(p_own)
        self.exchange(self.plan.xhalo, pe, self.x_send)
        self.be.spmv(self.A_ext, pe, q_own)
        return q_own


def dist_pcg(op, b_own, rtol=1e-6, itmax=1000):
    """pcg (pkg/src/mvamg/krylov.py:28-72) with x0 = 0 over row-partitioned
    vectors; every rank returns its own rows of x and the same SolveReport.

    Two allreduces per iteration: p'q, then [r'r, r'z] together -- the
    preconditioner is applied to the updated residual before the stop test, so
    the two dots travel in one message (the iterates and the history are those
    of the reference's loop; a converged solve pays one extra application)."""
    be, comm = op.be, op.comm
    n = b_own.numel()
    x = be.vec(n)
    r = be.vec(n)
    r.copy_(b_own)
    z, p, q = be.vec(n), be.vec(n), be.vec(n)
    rr0, = comm.allreduce([be.dot(r, r)])
    nr0 = float(np.sqrt(rr0))
    hist = [nr0]
    if nr0 == 0.0:
        return x, SolveReport(0, 0.0, True, np.array(hist))
    op.apply(r, z)
    rz, = comm.allreduce([be.dot(r, z)])
    if rz <= 0.0:
        raise NotSpdError("preconditioner breakdown: r'z <= 0")
    p.copy_(z)
    converged = False
    it = 0
    while it < itmax:
        op.matvec(p, q)
        pq, = comm.allreduce([be.dot(p, q)])
        if pq <= 0.0:
            raise NotSpdError("CG breakdown: p'Ap <= 0")
        alpha = rz / pq
        be.axpy(alpha, p, x)
        be.axpy(-alpha, q, r)
        it += 1
        op.apply(r, z)  # before the stop test: r'r and r'z share one allreduce
        rr, rz_new = comm.allreduce([be.dot(r, r), be.dot(r, z)])
        nrm = float(np.sqrt(rr))
        hist.append(nrm)
        if nrm <= rtol * nr0:
            converged = True
            break
        if rz_new <= 0.0:
            raise NotSpdError("preconditioner breakdown: r'z <= 0")
        be.xpby(z, rz_new / rz, p)
        rz = rz_new
    return x, SolveReport(it, hist[-1] / nr0, converged, np.array(hist))


@dataclass
class DistributedSolver:
    """MultiVectorAMG.solve (estimator.py:138-145) over row-partitioned GPUs:
    each rank passes the global b (or its rows) and gets the global x back."""

    matrices: list
    prolongators: list
    comm: object = None
    backend: object = None

    def __post_init__(self):
        self.op = DistributedVCycle(self.matrices, self.prolongators, self.comm, self.backend)
        self.comm = self.op.comm

    def own_rows(self, v):
        lo, hi = self.op.part.block(self.comm.rank)
        return np.asarray(v)[lo:hi]

    def solve(self, b, rtol=1e-6, itmax=1000):
        be = self.op.be
        b = np.asarray(b, dtype=np.float64)
        if b.shape[0] == self.op.plan.n:
            b = self.own_rows(b)
        x_own, rep = dist_pcg(self.op, be.from_host(b), rtol=rtol, itmax=itmax)
        return be.to_host(x_own), rep
