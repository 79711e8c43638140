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
    max_threads: int = 256
    max_window: int = 1 << 20
    graphs: bool = True
    smem_budget: int = 220 * 1024   # bytes of shared memory per GS CTA (window + rings)
    ring_bytes: int = 48 * 1024     # TMA ring size per warp (D slots of R rounds)
    rounds_in_flight: int = 16      # rounds of records the ring keeps ahead (generic kernel)
    generic_gs: bool = False        # force the generic GS kernel (tests / diagnostics)
    level_gs_max_rows: int = 393216 # levels up to this size may use the cluster level-set sweep
    max_cluster: int = 16           # CTAs per thread-block cluster for level-set sweeps
    level_stage_bytes: int = 32768  # minimum staging buffer per level (else a larger cluster)
    force_level_gs: bool = False    # use it for every small level (tests / diagnostics)
    smem_limit: int = 227 * 1024 - 1024
    lean_rows_per_round: int = 1    # K rows of a lane's chain per round in the lean GS kernel (1 or 4;
                                    # 4 is bit-exact but slower on grid problems, see gs_sweep.cuh)
    row_gs_min_rows: int = 10000    # coarse levels at least this large use the dataflow row sweep
    row_gs_threads: int = 128       # threads per CTA of the row sweep
    row_gs_ctas: int = 0            # resident CTAs of the row sweep (0 = auto)
    device_galerkin: bool = True    # setup forms P'AP with the device kernel (bit-identical to scipy's)
    device_matching: bool = True    # setup matches with the device kernel (identical pairs and order)
    device_svd: bool = True         # setup's local SVDs on the device kernel (bit-identical U, sigma)
    level_gs_small_rows: int = 2000  # tolerance parity: coarse levels up to this size use the level-set sweep
    lean_ring: tuple = None         # (R, D) of the lean kernel's record ring, overriding ring_bytes
    lean_cluster: int = 0           # wavefront tiles as thread-block clusters of this many CTAs (0: off);
                                    # boundary values of the previous tile come over DSMEM, not L2
    level_reg: bool = False         # (with exact_gs False) single-CTA level sweeps with register-prefetched
                                    # entries (gs_level_reg_kernel; measured slower than the staged kernel)
    exact_gs: bool = False          # True: every GS kernel keeps the CSR-order subtractions (bit-exact with
                                    # the serial sweep); False: level-set sweeps sum long rows over several
                                    # lanes (same row order, parity within rounding -- north star: 1e-10)
    row_gs_smem: int = 96 * 1024    # staged entry slices per row-sweep tile (halve threads above)
    force_row_gs: bool = False      # use the row sweep for every coarse level (tests / diagnostics)
    autotune_gs: bool = True        # coarse levels: time row and level-set sweeps once, keep the faster per mode
    min_chain_rows: float = 8.0     # a level whose wavefront chains average fewer rows uses the row sweep
                                    # (e.g. interleaved multi-dof systems, where row i rarely couples to i-1)
    lean_small_ring_tiles: int = 148  # lean sweeps with at least this many tiles use the (4, 2) TMA ring (0: never)
    lean_many_tiles: int = 1184     # ... and with this many one-warp tiles a modular window of 16 positions
    lean_wpos: int = 64             # lean sweeps: one-warp tiles with a window of this many positions per chain
                                    # (power of two; 0: the whole chain, which caps tiles per SM and chain length)
    block_chains: bool = True       # 3-D grid lines: tiles of 2-D blocks of lines (chain_block_order), so a
                                    # line's z-neighbour is mostly in the same tile's shared window
    stream_gs: bool = True          # levels whose x (and b) fit one SM's shared memory: the streamed level-set
                                    # sweep (gs_stream.cuh: TMA ring of level packets), before any other schedule
    stream_slot_bytes: int = 65536  # largest ring slot of the streamed sweep (four slots fill the free smem)
    stream_entries_per_cta: int = 1 << 30  # entries a sweep streams per SM before it spreads over a cluster
                                    # (clusters measured slower than the row sweep on C3: off by default)
    stream_max_rows: int = 4096     # levels up to this size stream (C3: 1.3-1.9x the level-set / row sweeps
                                    # at <= 1.8k rows, equal at 5k)
    cluster_gs: bool = True         # (tolerance parity) coarse levels whose x fits one thread-block cluster's
                                    # shared memory: the cluster dataflow sweep (gs_cluster.cuh), before any other
    cluster_max_rows: int = 4000000  # ... up to this size (what decides is whether a CTA's x slice and page rings
                                    # fit its shared memory)
    cluster_full_rows: int = 1000   # cluster form: 16 CTAs from this size up, cluster_small_ctas below
    cluster_small_ctas: int = 8
    cluster_grid_rows: int = 10000  # above: the grid form (ordinary CTAs over the whole GPU, early inputs through L2;
                                    # C3: 2-3x the row sweep at 53k and 160k rows, level with the cluster form at 16k)
    cluster_grid_ctas: int = 0      # CTAs of the grid form (0: one per SM)
    cluster_min_warps: int = 8      # worker warps per CTA, at least
    cluster_max_warps: int = 32     # ... and at most
    cluster_fused_fold_rows: int = 300000  # levels up to this size sweep backward from x_old with a mode-3 plan
                                    # (x_old entries read inside the kernel) instead of the fold kernel + the
                                    # zero-guess plan (C3: H1 70.6 -> 67.8 ms with every level fused)
    cluster_page_bytes: int = 2048  # page of row records a worker warp streams per TMA bulk copy (doubled while
                                    # a row's record does not fit)
    cluster_sleep_ns: int = 0       # back-off (ns) of a worker warp whose poll found nothing new
    coarse_pinv_rtol: float = 0.0   # 0: the coarsest inverse from the reference's LU factors (cycles.py:88-97);
                                    # > 0: the stated C5 deviation -- truncated-eigen pseudo-inverse dropping
                                    # eigenvalues <= rtol * lambda_max (a numerically singular A_L)


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


LEAN_RINGS = ((8, 3), (8, 2), (4, 4), (2, 8), (1, 8))  # (R, D) pairs the lean kernel is built for


def _row_counts(A):
    """Per-row counts of strictly lower / strictly upper stored entries."""
    n = A.shape[0]
    rows = np.repeat(np.arange(n), np.diff(A.indptr))
    lo = np.bincount(rows[A.indices < rows], minlength=n)
    up = np.bincount(rows[A.indices > rows], minlength=n)
    return lo, up


LEAN_K_RINGS = ((2, 3), (2, 2))  # (R, D) of the K = 4 rows-per-round lean kernel


def _gs_ring(A, cfg):
    """Ring plan (lean_C, R, D, slot_words, S) for matrix A.

    The lean kernel (lean_C > 0) serves sweeps whose rows have <= 8 dependent
    entries: uniform records of S = 3 + 2C words, slots of R rounds of records
    plus R x 32 right-hand-side values.  Otherwise the generic kernel, S bounded
    by the longest row.  Aims for many rounds in flight within cfg.ring_bytes."""
    lo, up = _row_counts(A)
    cmax = int(max(lo.max(initial=0), up.max(initial=0)))
    if cmax <= 8 and not cfg.generic_gs:
        C = 2 if cmax <= 2 else (4 if cmax <= 4 else 8)
        S = 3 + 2 * C
        K = int(cfg.lean_rows_per_round)
        if K == 4 and C <= 4:
            for R, D in LEAN_K_RINGS:
                slot = R * 32 * K * (S + 1)
                if D * slot * 8 <= cfg.ring_bytes:
                    return C | (K << 8), R, D, slot, S
            R, D = LEAN_K_RINGS[-1]
            return C | (K << 8), R, D, R * 32 * K * (S + 1), S
        if cfg.lean_ring is not None:  # explicit (R, D) (diagnostics / clustered tiles)
            R, D = cfg.lean_ring
            return C, R, D, R * 32 * (S + 1), S
        for R, D in LEAN_RINGS:
            slot = R * 32 * (S + 1)
            if D * slot * 8 <= cfg.ring_bytes:
                return C, R, D, slot, S
        R, D = LEAN_RINGS[-1]
        return C, R, D, R * 32 * (S + 1), S
    nnz_row = np.diff(A.indptr)
    maxcnt = int(nnz_row.max()) if nnz_row.size else 1
    S = 3 + 2 * max(maxcnt - 1, 0)
    per_round = (32 * S + 32) * 8
    best = (1, 2)
    for R in (8, 4, 2, 1):
        for D in (8, 4, 2):
            if R * D * per_round <= cfg.ring_bytes and R * D <= cfg.rounds_in_flight:
                if R * D > best[0] * best[1] or (R * D == best[0] * best[1] and D > best[1]):
                    best = (R, D)
    R, D = best
    return 0, R, D, R * (32 * S + 32), S


def chain_block_order(A, chain_ptr, T):
    """Processing order of the chains for 2-D blocked tiles, or None.

    The chains of a natural ordering of a 3-D grid problem are its x-lines,
    numbered c = y + G z; line (y, z) depends on lines (y-1, z) and (y, z-1).
    Consecutive chains per tile (the natural order) put every z-neighbour in
    another tile, so the sweep's critical path crosses ~G tiles through L2.
    Blocks of by x bz lines per tile (T = by * bz chains; within a tile z-major
    pairs of y-runs per warp) keep both neighbours in the tile's shared window
    for all but the block faces: ~G/by + G/bz cross-tile hops.  Detected from
    the chain-to-chain dependence offsets (1 and a dominant G > 1); every
    input still lies in an earlier block (tiles run in order), which
    mvamg_gs_schedule verifies.  None when there is no such structure."""
    nch = chain_ptr.shape[0] - 1
    if nch < 4 * T or T < 32:
        return None
    n = A.shape[0]
    chain_of = np.repeat(np.arange(nch, dtype=np.int64), np.diff(chain_ptr))
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(A.indptr))
    lo = A.indices < rows
    d = chain_of[rows[lo]] - chain_of[A.indices[lo]]
    d = d[d > 1]
    if d.size == 0:
        return None
    vals, cnt = np.unique(d, return_counts=True)
    G = int(vals[np.argmax(cnt)])
    if cnt.max() < 0.9 * d.size or nch % G or G < 8:
        return None
    Z = nch // G
    bz = 1
    while bz * bz * 2 < T:
        bz *= 2
    by = T // bz
    if by < 8 or Z < 2 * bz:
        return None
    order = []
    for z0 in range(0, Z, bz):
        for y0 in range(0, G, by):
            zz = np.arange(z0, min(z0 + bz, Z))
            yy = np.arange(y0, min(y0 + by, G))
            order.append((yy[None, :] + G * zz[:, None]).ravel())
    return np.ascontiguousarray(np.concatenate(order), dtype=np.int32)


def gs_analyse(A, cfg=None):
    """Chain/tile schedule of a CSR matrix for the exact-order GS sweep (host).

    Warps per tile and the shared window (position-major slots) are sized so
    that window + per-warp rings + mbarriers fit cfg.smem_budget."""
    cfg = cfg or GpuConfig()
    A = as_csr(A)
    L = _lib.load()
    ip = np.ascontiguousarray(A.indptr, dtype=np.int32)
    ix = np.ascontiguousarray(A.indices, dtype=np.int32)
    n = A.shape[0]
    C, R, D, slot, S = _gs_ring(A, cfg)
    ring_warp = D * (slot * 8 + 8)
    c_ip = ip.ctypes.data_as(ctypes.c_void_p)
    c_ix = ix.ctypes.data_as(ctypes.c_void_p)
    nch, nt, thr, win, dep = (ctypes.c_int() for _ in range(5))
    # natural chain length (longest run of rows coupled to their predecessor,
    # e.g. a grid line): keep chains whole and pick the widest tile whose
    # position-major window still fits; split chains only if one warp cannot hold them
    _lib.check(L.mvamg_gs_analyse(n, c_ip, c_ix, min(cfg.max_chain, 1 << 30), 1, 1 << 30, ctypes.byref(nch),
                                  ctypes.byref(nt), None, None, None, None, None, None), "gs_analyse")
    cp0 = np.empty(nch.value + 1, dtype=np.int32)
    tp0 = np.empty(nt.value + 1, dtype=np.int32)
    _lib.check(L.mvamg_gs_analyse(n, c_ip, c_ix, min(cfg.max_chain, 1 << 30), 1, 1 << 30, ctypes.byref(nch),
                                  ctypes.byref(nt), cp0.ctypes.data_as(ctypes.c_void_p),
                                  tp0.ctypes.data_as(ctypes.c_void_p), None, None, None, None), "gs_analyse")
    lmax = int(np.diff(cp0).max()) if nch.value else 1
    T, slots, max_chain = 32, 0, 1
    for T_ in (256, 128, 64, 32):
        if T_ > max(32, cfg.max_threads):
            continue
        s_ = min((cfg.smem_budget - (T_ // 32) * ring_warp) // 8 - 2, cfg.max_window)
        if s_ >= T_ * lmax or T_ == 32:
            T, slots = T_, s_
            break
    if slots < 32:
        raise ValueError(f"GS ring of {ring_warp} bytes per warp does not fit shared memory")
    T = min(T, max(1, cfg.max_threads))
    max_chain = max(1, min(cfg.max_chain, lmax, slots // max(32, (T + 31) // 32 * 32)))
    # lean sweeps with a modular window: one-warp tiles of whole chains whose shared
    # window keeps lean_wpos positions per chain (32 x wpos slots), so several tiles
    # share an SM -- the window no longer caps the chain length or the tile count
    # (only where the whole-chain window already forces tiles of at most one warp: C2 1.21 ->
    # 1.08 ms, C5 5.5 -> 2.6 ms per sweep; C3's two-warp tiles of 8 x 8 lines stay faster)
    wpos = 0
    if (C > 0 and cfg.lean_wpos > 0 and not cfg.generic_gs and not cfg.lean_cluster and lmax > cfg.lean_wpos
            and T <= 32):
        wpos = int(cfg.lean_wpos)
        T, slots, max_chain = 32, 1 << 30, max(1, min(cfg.max_chain, lmax))
    order = None
    if cfg.block_chains and not cfg.lean_cluster:
        _lib.check(L.mvamg_gs_analyse(n, c_ip, c_ix, max_chain, T, slots, ctypes.byref(nch),
                                      ctypes.byref(nt), None, None, None, None, None, None), "gs_analyse")
        cpn = np.empty(nch.value + 1, dtype=np.int32)
        tpn = np.empty(nt.value + 1, dtype=np.int32)
        _lib.check(L.mvamg_gs_analyse(n, c_ip, c_ix, max_chain, T, slots, ctypes.byref(nch), ctypes.byref(nt),
                                      cpn.ctypes.data_as(ctypes.c_void_p), tpn.ctypes.data_as(ctypes.c_void_p),
                                      None, None, None, None), "gs_analyse")
        order = chain_block_order(A, cpn, T)
    vo = order.ctypes.data_as(ctypes.c_void_p) if order is not None else None
    _lib.check(L.mvamg_gs_analyse(n, c_ip, c_ix, max_chain, T, slots, ctypes.byref(nch),
                                  ctypes.byref(nt), None, None, None, None, None, vo), "gs_analyse")
    cp = np.empty(nch.value + 1, dtype=np.int32)
    tp = np.empty(nt.value + 1, dtype=np.int32)
    _lib.check(L.mvamg_gs_analyse(n, c_ip, c_ix, max_chain, T, slots, ctypes.byref(nch),
                                  ctypes.byref(nt), cp.ctypes.data_as(ctypes.c_void_p),
                                  tp.ctypes.data_as(ctypes.c_void_p), ctypes.byref(thr),
                                  ctypes.byref(win), ctypes.byref(dep), vo), "gs_analyse")
    plan = GsPlanHost(nch.value, nt.value, max(32, thr.value), max(win.value, 1), dep.value, cp, tp)
    plan.chain_order = order
    plan.wpos = wpos
    if wpos:
        plan.window = 32 * wpos
    plan.lean_C, plan.R, plan.D = C, R, D
    plan.smem_budget = cfg.smem_budget
    return plan


@dataclass
class GsScheduleHost:
    rec: np.ndarray        # uint64 words, round-major records
    round_off: np.ndarray  # int32, nrounds + 1
    tbase: np.ndarray      # int32, nwarps + 1
    tile_wbase: np.ndarray # int32, ntiles + 1
    perm: np.ndarray       # int32, n
    nrounds: int
    max_S: int


def gs_schedule(A, plan, mode, R=None, uniform_S=0, K=1):
    """Static round schedule of one GS sweep mode (0 forward from x=0, 1 forward, 2 backward)."""
    A = as_csr(A)
    L = _lib.load()
    n = A.shape[0]
    ip = np.ascontiguousarray(A.indptr, dtype=np.int32)
    ix = np.ascontiguousarray(A.indices, dtype=np.int32)
    v = np.ascontiguousarray(A.data, dtype=np.float64)
    cp = np.ascontiguousarray(plan.chain_ptr, dtype=np.int32)
    tp = np.ascontiguousarray(plan.tile_ptr, dtype=np.int32)
    vp = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    nw, nr, nwarps, smax = ctypes.c_longlong(), ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    args = (n, vp(ip), vp(ix), vp(v), plan.ntiles, vp(cp), vp(tp), plan.window, int(mode),
            int(R or plan.R), int(uniform_S), int(K), ctypes.byref(nw), ctypes.byref(nr), ctypes.byref(nwarps),
            ctypes.byref(smax))
    order = getattr(plan, "chain_order", None)
    vo = vp(np.ascontiguousarray(order, dtype=np.int32)) if order is not None else None
    wpos = int(getattr(plan, "wpos", 0))
    _lib.check(L.mvamg_gs_schedule(*args, None, None, None, None, None, vo, wpos), "gs_schedule")
    rec = np.zeros(max(2, nw.value), dtype=np.uint64)
    round_off = np.empty(nr.value + 1, dtype=np.int32)
    tbase = np.empty(nwarps.value + 1, dtype=np.int32)
    tile_wbase = np.empty(plan.ntiles + 1, dtype=np.int32)
    perm = np.empty(max(1, n), dtype=np.int32)
    _lib.check(L.mvamg_gs_schedule(*args, vp(rec), vp(round_off), vp(tbase), vp(tile_wbase), vp(perm), vo, wpos),
               "gs_schedule")
    return GsScheduleHost(rec, round_off, tbase, tile_wbase, perm, nr.value, smax.value)


class DeviceGsPlan:
    """Schedule of one matrix on the device: chains/tiles plus, per sweep mode
    (built on demand), the round-major records and the rhs buffer."""

    def __init__(self, A, cfg=None, plan=None):
        self.A = as_csr(A)
        self.cfg = cfg or GpuConfig()
        self._csr = None
        self._set_plan(plan or gs_analyse(self.A, self.cfg))
        if plan is None:
            self._tune_for_many_tiles()

    def _set_plan(self, plan):
        self.plan = plan
        self.chain_ptr = to_device(plan.chain_ptr, np.int32)
        self.tile_ptr = to_device(plan.tile_ptr, np.int32)
        order = getattr(plan, "chain_order", None)
        self.chain_order = to_device(order, np.int32) if order is not None else None
        self.modes = {}

    def _tune_for_many_tiles(self):
        """Lean sweeps with (many) more tiles than the GPU holds at once are bound by the tiles resident
        per SM, i.e. by each tile's shared memory, not by a tile's latency: halve the TMA ring to (R, D) =
        (4, 2) from one tile per SM up (C3: 325 / 353 -> 305 / 327 us), and with >= cfg.lean_many_tiles
        one-warp tiles also cut the modular window to 16 positions (C5: 2.56 / 2.67 -> 1.97 / 2.08 ms per
        sweep; same bits).  A window too short for the matrix's reads fails the schedule's check
        (ValueError): then the standard plan stays."""
        import dataclasses

        p, cfg = self.plan, self.cfg
        if not (p.lean_C > 0 and (p.lean_C >> 8) <= 1 and cfg.lean_ring is None and not cfg.lean_cluster
                and not cfg.generic_gs and (p.R, p.D) == (8, 2) and p.ntiles >= cfg.lean_small_ring_tiles > 0):
            return
        wpos = int(getattr(p, "wpos", 0))
        many = wpos > 16 and p.ntiles >= cfg.lean_many_tiles > 0
        cfg2 = dataclasses.replace(cfg, lean_ring=(4, 2), lean_wpos=16 if many else cfg.lean_wpos,
                                   max_threads=p.threads)  # the smaller ring must not widen the tiles
        base = p
        try:
            self._set_plan(gs_analyse(self.A, cfg2))
            if (self.plan.threads, self.plan.ntiles) != (base.threads, base.ntiles):
                raise ValueError("tile shape changed")
            if many:  # the shorter window must pass the schedule's read-before-overwrite check
                for m in (0, 2):
                    self.mode(m)
        except ValueError:
            self._set_plan(base)

    def mode(self, m):
        """Device schedule dict for mode m."""
        if m not in self.modes:
            import torch

            p = self.plan
            if p.lean_C > 0 and m != 1:
                C, K = p.lean_C & 0xFF, max(1, p.lean_C >> 8)
                S = 3 + 2 * C
                R, D = p.R, p.D
                # thread-block-cluster tiles: sources in the previous tile of the same
                # cluster are read over DSMEM (GpuConfig.lean_cluster; needs >= 2 tiles)
                cl = int(self.cfg.lean_cluster) if (self.cfg.lean_cluster > 1 and p.ntiles > 1 and K == 1) else 0
                h = gs_schedule(self.A, p, m, R=R, uniform_S=S, K=K | (cl << 8))
                rec_words_max = R * 32 * K * S
                slot_words = rec_words_max + R * 32 * K
                lean = p.lean_C | (cl << 16)
            else:
                # generic kernel: pick the deepest ring that fits beside the window
                h = gs_schedule(self.A, p, m, R=1)
                S = h.max_S
                avail = p.smem_budget - 8 * ((p.window + 1) & ~1)
                R, D = 1, 2
                for R_, D_ in ((8, 4), (4, 4), (4, 2), (2, 4), (2, 2), (1, 4), (1, 2)):
                    if (p.threads // 32) * D_ * (R_ * (32 * S + 32) + 1) * 8 <= avail:
                        R, D = R_, D_
                        break
                if R > 1:
                    h = gs_schedule(self.A, p, m, R=R)
                    S = h.max_S
                rec_words_max = R * 32 * S
                slot_words = rec_words_max + R * 32
                slot_words += slot_words & 1
                lean = 0
            self.modes[m] = dict(
                rec=to_device(h.rec.view(np.int64)), round_off=to_device(h.round_off),
                tbase=to_device(h.tbase), tile_wbase=to_device(h.tile_wbase), perm=to_device(h.perm),
                tperm=torch.empty(max(32, 32 * h.nrounds * max(1, lean >> 8)), dtype=torch.float64,
                                  device="cuda"),
                R=R, D=D, lean_C=lean, slot_words=slot_words, rec_words_max=rec_words_max,
                nrounds=h.nrounds, max_S=h.max_S)
        return self.modes[m]

    def nbytes(self, m):
        s = self.mode(m)
        return s["rec"].numel() * 8 + s["round_off"].numel() * 4 + s["perm"].numel() * 4

    def sweep(self, direction, b, x_old, x_new, ws, stream=None, work=None):
        """x_new = one GS sweep (direction 0 fwd / 1 bwd) from x_old (None: zero)."""
        m = (0 if x_old is None else 1) if direction == 0 else 2
        sch = self.mode(m)
        p = self.plan
        if self._csr is None:
            self._csr = DeviceCSR(self.A)
        _lib.check(_lib.load().mvamg_gs_sweep_f64(
            direction, self.A.shape[0], *self._csr.ptrs(), ptr(sch["rec"]), ptr(sch["round_off"]),
            ptr(sch["tbase"]), ptr(sch["tile_wbase"]), ptr(sch["perm"]), ptr(sch["tperm"]), sch["R"],
            sch["D"], sch["lean_C"], sch["slot_words"], sch["rec_words_max"], p.ntiles, ptr(self.chain_ptr), ptr(self.tile_ptr),
            ptr(self.chain_order), p.threads, p.window, int(getattr(p, "wpos", 0)), ptr(b), ptr(x_old), ptr(x_new),
            ptr(ws), stream or stream_handle()),
            "gs_sweep")


LEVEL_ROW_DTYPE = np.dtype([("row", "<i4"), ("estart", "<i4"), ("cnt", "<i4"), ("pad", "<i4"),
                            ("diag", "<f8"), ("rdiag", "<f8")])
LEVEL_ENT_DTYPE = np.dtype([("coef", "<f8"), ("src", "<i4"), ("pad", "<i4")])


class DeviceGsLevels:
    """Level-set GS schedule of one small / mid-size matrix and sweep mode (0 fwd
    from x=0, 1 fwd, 2 bwd from x=0, 3 bwd) on one thread-block cluster of 1..16
    CTAs (the smallest cluster whose shared memory holds x), on the device."""

    def __init__(self, A, mode, cfg=None):
        import torch

        cfg = cfg or GpuConfig()
        A = as_csr(A)
        L = _lib.load()
        n = A.shape[0]
        ip = np.ascontiguousarray(A.indptr, dtype=np.int32)
        ix = np.ascontiguousarray(A.indices, dtype=np.int32)
        v = np.ascontiguousarray(A.data, dtype=np.float64)
        vp = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
        nlev, mr, me, rpc = ctypes.c_int(), ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        ne = ctypes.c_longlong()
        chosen = None
        # tolerance parity, x fits one CTA: the register-prefetch kernel needs
        # no staging buffers, so levels are not split (caps 0 = unlimited)
        reg_ents = 512 * 8  # kRegThreads x kRegEnts of gs_level_reg_kernel: entries per sub-level
        self.reg = (not cfg.exact_gs and cfg.level_reg and n > 0
                    and 8 * (n + 2) + 8 * reg_ents + 1024 <= cfg.smem_limit)
        if self.reg:
            _lib.check(L.mvamg_gs_levels(n, vp(ip), vp(ix), vp(v), int(mode), 1, 0, reg_ents,
                                         ctypes.byref(nlev), ctypes.byref(ne), ctypes.byref(mr), ctypes.byref(me),
                                         ctypes.byref(rpc), None, None, None, None, None), "gs_levels")
            chosen = (1, 0, reg_ents)
            if 8 * (n + 2 + me.value + nlev.value) + 1024 > cfg.smem_limit:
                self.reg, chosen = False, None
        for ncta in (1, 2, 4, 8, 16):
            if chosen is not None:
                break
            if ncta > cfg.max_cluster:
                break
            rpc_ = -(-n // ncta)
            room = cfg.smem_limit - 8 * ((rpc_ + 1) & ~1)
            per_buf = room // 3
            if per_buf < cfg.level_stage_bytes and not (ncta == cfg.max_cluster or ncta == 16):
                continue
            row_cap = min(1024, max(32, per_buf // 160))
            ent_cap = (per_buf - row_cap * 40 - 32) // 16
            _lib.check(L.mvamg_gs_levels(n, vp(ip), vp(ix), vp(v), int(mode), ncta, row_cap, ent_cap,
                                         ctypes.byref(nlev), ctypes.byref(ne), ctypes.byref(mr), ctypes.byref(me),
                                         ctypes.byref(rpc), None, None, None, None, None), "gs_levels")
            if self._smem(rpc.value, max(1, mr.value), max(1, me.value)) <= cfg.smem_limit:
                chosen = (ncta, row_cap, ent_cap)
                break
        if chosen is None:
            raise ValueError("level-set GS schedule does not fit a thread-block cluster")
        ncta, row_cap, ent_cap = chosen
        lev_ptr = np.empty(ncta * (nlev.value + 1), dtype=np.int32)
        lev_eptr = np.empty(ncta * (nlev.value + 1), dtype=np.int32)
        rows = np.zeros(max(1, n), dtype=LEVEL_ROW_DTYPE)
        ents = np.zeros(max(1, ne.value), dtype=LEVEL_ENT_DTYPE)
        perm = np.empty(max(1, n), dtype=np.int32)
        _lib.check(L.mvamg_gs_levels(n, vp(ip), vp(ix), vp(v), int(mode), ncta, row_cap, ent_cap,
                                     ctypes.byref(nlev), ctypes.byref(ne), ctypes.byref(mr), ctypes.byref(me),
                                     ctypes.byref(rpc), vp(lev_ptr), vp(lev_eptr), vp(rows), vp(ents), vp(perm)),
                   "gs_levels")
        self.n, self.mode, self.ncta, self.rows_per_cta = n, mode, ncta, rpc.value
        self.nlev, self.max_rows, self.max_ents = nlev.value, max(1, mr.value), max(1, me.value)
        # lanes per row: 1 keeps the CSR-order subtractions (bit-exact); otherwise
        # about 8 entries per lane, summed by a shuffle tree (tolerance parity)
        avg = A.nnz / max(1, n)
        self.group = 1 if cfg.exact_gs else int(min(16, max(1, 1 << int(np.ceil(np.log2(max(1.0, avg / 8)))))))
        if self.reg and self.group == 1:
            self.group = 2
        self.threads = int(min(1024, max(64, (self.max_rows * self.group + 31) // 32 * 32)))
        if self.reg:  # fixed block (kRegThreads); every thread holds <= 8 of a level's entries
            self.threads = 512
        self.lev_ptr = to_device(lev_ptr)
        self.lev_eptr = to_device(lev_eptr)
        self.rows = to_device(rows.view(np.uint8))
        self.ents = to_device(ents.view(np.uint8))
        self.perm = to_device(perm)
        self.tperm = torch.empty(max(2, n + 2), dtype=torch.float64, device="cuda")
        self._csr = DeviceCSR(A)

    @staticmethod
    def _smem(rpc, max_rows, max_ents):
        xw = (rpc + 1) & ~1
        buf = max_rows * 32 + max_ents * 16 + ((max_rows + 2) * 8 + 15) // 16 * 16
        return xw * 8 + 3 * buf

    def smem_bytes(self):
        return self._smem(self.rows_per_cta, self.max_rows, self.max_ents)

    def args(self):
        return (self.ncta, self.rows_per_cta, self.nlev, self.max_rows, self.max_ents, self.threads,
                self.group | (0x100 if self.reg else 0),
                ptr(self.lev_ptr), ptr(self.lev_eptr), ptr(self.rows), ptr(self.ents), ptr(self.perm),
                ptr(self.tperm))

    def sweep(self, b, x_old, x_new, ws, stream=None, fold=False):
        if fold:  # backward from x_old with this (mode 2) schedule
            _lib.check(_lib.load().mvamg_gs_level_sweep_folded_f64(
                self.n, *self._csr.ptrs(), *self.args(), ptr(b), ptr(x_old), ptr(x_new), ptr(ws),
                stream or stream_handle()), "gs_level_sweep_folded")
            return
        _lib.check(_lib.load().mvamg_gs_level_sweep_f64(
            0 if self.mode < 2 else 1, self.n, *self._csr.ptrs(), *self.args(), ptr(b), ptr(x_old),
            ptr(x_new), ptr(ws), stream or stream_handle()), "gs_level_sweep")


def stream_ctas(A, mode, cfg=None):
    """CTAs (1 or a cluster of 2..16) of a streamed sweep of A in `mode`, or 0
    when none fits.  One SM streams up to ~200k entries per sweep in step with
    its DAG levels; larger levels spread their rows over a cluster (x sliced
    across the CTAs' shared memory, remote entries read over DSMEM; zero-guess
    modes only -- a backward sweep from x_old then runs folded)."""
    cfg = cfg or GpuConfig()
    n = A.shape[0]
    if n > cfg.stream_max_rows:
        return 0
    reads = (A.nnz - n) if mode & 1 else (A.nnz - n) / 2
    want = 1
    while want < 16 and reads / want > cfg.stream_entries_per_cta:
        want *= 2
    if mode & 1 and want > 1:
        return 0
    tries = (1,) if mode & 1 else ((want, 16) if want < 16 else (16,))
    for c in tries:
        R = -(-n // c)
        xw = (R + 1) & ~1
        if xw * 8 * (2 if mode & 1 else 1) + 4 * 8192 <= cfg.smem_limit and (c == 1 or c <= cfg.max_cluster):
            return c
    return 0


def stream_group(A, mode, exact):
    """Lanes per row of the streamed sweep: 1 (bit-exact CSR order) in exact
    mode, else about 8-16 entries per lane."""
    if exact:
        return 1
    n = A.shape[0]
    avg = (A.nnz - n) / max(1, n) / (1 if mode & 1 else 2)
    for g, lim in ((1, 6), (2, 16), (4, 40)):
        if avg < lim:
            return g
    return 8


class DeviceGsStream:
    """Streamed level-set GS plan (gs_stream.cuh) of one matrix and sweep mode
    (0 fwd from x=0, 1 fwd, 2 bwd from x=0 -- also the folded backward sweep
    from x_old --, 3 bwd), on the device: one SM or a thread-block cluster, x
    in shared memory, the level packets streamed through a ring of TMA bulk
    copies."""

    def __init__(self, A, mode, cfg=None, group=None, ncta=None):
        import torch

        cfg = cfg or GpuConfig()
        A = as_csr(A)
        n = A.shape[0]
        ncta = stream_ctas(A, mode, cfg) if ncta is None else int(ncta)
        if ncta < 1:
            raise ValueError("gs stream: the level does not fit one SM or cluster")
        R = -(-n // ncta) if ncta > 1 else n
        xw = (R + 1) & ~1
        budget = cfg.smem_limit - xw * 8 * (2 if mode & 1 else 1)
        # four slots of up to stream_slot_bytes: big slots carry many DAG levels per stage
        slot = max(4096, min(int(cfg.stream_slot_bytes), (budget // 4) & ~127))
        nslots = min(8, budget // slot)
        if nslots < 2:
            raise ValueError("gs stream: no room for the ring")
        L = _lib.load()
        ip = np.ascontiguousarray(A.indptr, dtype=np.int32)
        ix = np.ascontiguousarray(A.indices, dtype=np.int32)
        v = np.ascontiguousarray(A.data, dtype=np.float64)
        vp = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
        nb, ns, nl = ctypes.c_longlong(), ctypes.c_int(), ctypes.c_int()
        _lib.check(L.mvamg_gs_stream_plan(n, vp(ip), vp(ix), vp(v), int(mode), slot, ncta, ctypes.byref(nb),
                                          ctypes.byref(ns), ctypes.byref(nl), None, None), "gs_stream_plan")
        blob = np.zeros(max(16, nb.value), dtype=np.uint8)
        off = np.zeros(ns.value * ncta + 1, dtype=np.int64)
        _lib.check(L.mvamg_gs_stream_plan(n, vp(ip), vp(ix), vp(v), int(mode), slot, ncta, ctypes.byref(nb),
                                          ctypes.byref(ns), ctypes.byref(nl), vp(blob), vp(off)), "gs_stream_plan")
        self.n, self.mode, self.nstages, self.nslots, self.slot, self.ncta = n, mode, ns.value, nslots, slot, ncta
        self.nlev, self.nbytes = nl.value, nb.value
        self.group = int(group) if group is not None else stream_group(A, mode, cfg.exact_gs)
        self.blob = to_device(blob)
        self.stage_off = to_device(off)
        self.tfold = torch.empty(max(2, n), dtype=torch.float64, device="cuda") if mode == 2 else None
        self._csr = DeviceCSR(A)

    def args(self):
        return (self.nstages, self.nslots, self.slot, self.group, self.ncta, ptr(self.blob), ptr(self.stage_off),
                ptr(self.tfold))

    def sweep(self, b, x_old, x_new, ws=None, stream=None, fold=False):
        """One sweep; fold (mode-2 plan, x_old given): backward from x_old."""
        L = _lib.load()
        s = stream or stream_handle()
        if fold:
            _lib.check(L.mvamg_gs_stream_sweep_folded_f64(
                self.n, *self._csr.ptrs(), self.nstages, self.nslots, self.slot, self.group, self.ncta,
                ptr(self.blob), ptr(self.stage_off), ptr(self.tfold), ptr(b), ptr(x_old), ptr(x_new), ptr(ws), s),
                "gs_stream_sweep_folded")
            return
        _lib.check(L.mvamg_gs_stream_sweep_f64(self.n, self.mode, self.nstages, self.nslots, self.slot,
                                               self.group, self.ncta, ptr(self.blob), ptr(self.stage_off), ptr(b),
                                               ptr(x_old), ptr(x_new), s), "gs_stream_sweep")


def cluster_shape(n, nlev, cfg=None, grid=None):
    """(grid, ncta, wpc) of the cluster dataflow sweep of a level with n rows.
    One warp sweeps one row at a time (~1,200 cycles each), so the sweep wants
    many worker warps -- measured on C3's levels (tools/cluster_bench.py).
    Cluster form (x in distributed shared memory) up to cfg.cluster_grid_rows
    rows: 16 CTAs from ~1k rows up, 8 to 32 warps each, about 15 rows per warp.
    Above, the grid form: one CTA per SM, early inputs through L2."""
    cfg = cfg or GpuConfig()
    if n < 1:
        return None
    if grid is None:
        grid = n > cfg.cluster_grid_rows
    if grid:
        ncta = max(1, min(cfg.cluster_grid_ctas or _num_sms(), -(-n // 256)))
    else:
        ncta = 16 if n >= cfg.cluster_full_rows else max(1, cfg.cluster_small_ctas)
        ncta = max(1, min(ncta, cfg.max_cluster))
    wpc = int(min(cfg.cluster_max_warps, max(cfg.cluster_min_warps, -(-n // (15 * ncta)))))
    return bool(grid), ncta, wpc


_NUM_SMS = {}


def _num_sms():
    """SMs of the current CUDA device (the grid form runs one CTA on each)."""
    torch = torch_cuda()
    dev = torch.cuda.current_device()
    if dev not in _NUM_SMS:
        _NUM_SMS[dev] = torch.cuda.get_device_properties(dev).multi_processor_count
    return _NUM_SMS[dev]


def cluster_smem(slots, wpc, page_bytes):
    """Shared memory per CTA of the cluster sweep: x slice, page rings, mbarriers."""
    return ((slots * 8 + 127) & ~127) + wpc * 2 * (page_bytes + 8)


class DeviceGsCluster:
    """Cluster dataflow GS plan (gs_cluster_kernel, mvamg_gs_cluster_plan) of one
    matrix and sweep mode (0 fwd from x=0, 1 fwd, 2 bwd from x=0 -- also the
    folded backward sweep from x_old --, 3 bwd), on the device."""

    def __init__(self, A, mode, cfg=None, ncta=None, wpc=None, sleep_ns=None, grid=None):
        import torch

        cfg = cfg or GpuConfig()
        A = as_csr(A)
        L = _lib.load()
        n = A.shape[0]
        ip = np.ascontiguousarray(A.indptr, dtype=np.int32)
        ix = np.ascontiguousarray(A.indices, dtype=np.int32)
        v = np.ascontiguousarray(A.data, dtype=np.float64)
        vp = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
        npg, nlev, slots, hits = ctypes.c_longlong(), ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        page = int(cfg.cluster_page_bytes)

        def plan(c, w, *out):
            return L.mvamg_gs_cluster_plan(n, vp(ip), vp(ix), vp(v), int(mode), int(bool(grid)), int(c), int(w), page,
                                           ctypes.byref(npg), ctypes.byref(nlev), ctypes.byref(slots),
                                           ctypes.byref(hits), *out)

        while plan(ncta or 1, wpc or 1, *([None] * 5)) != 0:  # a row too long for the page: larger pages
            page *= 2
            if page > 16384:
                raise ValueError("gs cluster: a row's record exceeds the largest page")
        if ncta is None or wpc is None:
            shape = cluster_shape(n, nlev.value, cfg, grid)
            if shape is None:
                raise ValueError("gs cluster: the level's x does not fit one thread-block cluster")
            grid, ncta, wpc = shape[0], (ncta or shape[1]), (wpc or shape[2])
        grid = bool(grid)
        _lib.check(plan(ncta, wpc, *([None] * 5)), "gs_cluster_plan")
        # worker warps per CTA: as many as leave room for their page rings beside the x slice
        # (the slice depends on wpc only through the plan's balance slack: re-plan and re-check)
        while wpc > 1 and cluster_smem(slots.value, wpc, page) > cfg.smem_limit:
            room = cfg.smem_limit - ((slots.value * 8 + 127) & ~127)
            wpc = max(1, min(wpc - 1, room // (2 * (page + 8))))
            _lib.check(plan(ncta, wpc, *([None] * 5)), "gs_cluster_plan")
        if cluster_smem(slots.value, wpc, page) > cfg.smem_limit:
            raise ValueError("gs cluster: x slice and page rings exceed shared memory")
        wptr = np.empty(ncta * wpc + 1, dtype=np.int32)
        wpage = np.empty(ncta * wpc + 1, dtype=np.int32)
        rowid = np.empty(max(1, n), dtype=np.int32)
        perm = np.empty(max(1, n), dtype=np.int32)
        blob = np.zeros(max(1, npg.value) * page, dtype=np.uint8)
        _lib.check(plan(ncta, wpc, vp(wptr), vp(wpage), vp(rowid), vp(perm), vp(blob)), "gs_cluster_plan")
        self.n, self.mode, self.nlev, self.npages, self.page_bytes = n, mode, nlev.value, npg.value, page
        self.ncta, self.wpc, self.slots, self.local_late = int(ncta), int(wpc), slots.value, hits.value
        self.grid = grid
        self.sleep_ns = int(cfg.cluster_sleep_ns if sleep_ns is None else sleep_ns)
        self.wptr, self.wpage, self.blob = to_device(wptr), to_device(wpage), to_device(blob)
        self.rowid, self.perm = to_device(rowid), to_device(perm)
        self.tperm = torch.empty(max(2, n + 2), dtype=torch.float64, device="cuda")
        self._csr = DeviceCSR(A)

    def args(self):
        return (ptr(self.wptr), ptr(self.wpage), ptr(self.blob), ptr(self.perm), int(self.grid), self.ncta, self.wpc,
                self.slots, self.page_bytes, self.sleep_ns, ptr(self.tperm))

    def sweep(self, b, x_old, x_new, ws, stream=None):
        """One sweep; with x_old a mode-2 plan runs the folded backward sweep."""
        _lib.check(_lib.load().mvamg_gs_cluster_sweep_f64(
            self.mode, self.n, *self._csr.ptrs(), *self.args(), ptr(b), ptr(x_old), ptr(x_new), ptr(ws),
            stream or stream_handle()), "gs_cluster_sweep")


class DeviceGsRows:
    """Dataflow GS row schedule (gs_row_kernel) of one matrix and sweep mode
    (0 fwd from x=0, 1 fwd, 2 bwd from x=0 -- also the folded backward sweep
    from x_old --, 3 bwd), on the device."""

    def __init__(self, A, mode, cfg=None, row_range=None):
        """row_range (lo, hi): only those rows are swept (the own rows of a
        row-partitioned level over its extended layout; the others are ghost
        inputs, mvamg_gs_row_sweep_ext_f64)."""
        import torch

        cfg = cfg or GpuConfig()
        A = as_csr(A)
        L = _lib.load()
        n_all = A.shape[0]
        lo, hi = row_range if row_range is not None else (-1, -1)
        n = n_all if row_range is None else hi - lo
        self.row_range = row_range
        ip = np.ascontiguousarray(A.indptr, dtype=np.int32)
        ix = np.ascontiguousarray(A.indices, dtype=np.int32)
        v = np.ascontiguousarray(A.data, dtype=np.float64)
        vp = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
        ns, nlev = ctypes.c_longlong(), ctypes.c_int()
        order = 0 if cfg.exact_gs else 1  # 1: entries by input level (tolerance parity)
        self.order = order
        _lib.check(L.mvamg_gs_rows(n_all, vp(ip), vp(ix), vp(v), int(mode), order, ctypes.byref(ns),
                                   ctypes.byref(nlev), None, None, None, None, None, None, None, None, None,
                                   lo, hi), "gs_rows")
        nw = -(-n // 32)
        rowid = np.empty(max(1, n), dtype=np.int32)
        cnt = np.empty(max(1, n), dtype=np.int32)
        crit = np.empty(max(1, n), dtype=np.int32)
        dg = np.empty(max(1, n), dtype=np.float64)
        rdg = np.empty(max(1, n), dtype=np.float64)
        perm = np.empty(max(1, n_all), dtype=np.int32)
        wofs = np.empty(nw + 1, dtype=np.int32)
        coef = np.empty(max(32, 32 * ns.value), dtype=np.float64)
        src = np.empty(max(32, 32 * ns.value), dtype=np.int32)
        _lib.check(L.mvamg_gs_rows(n_all, vp(ip), vp(ix), vp(v), int(mode), order, ctypes.byref(ns),
                                   ctypes.byref(nlev), vp(rowid), vp(cnt), vp(crit), vp(dg), vp(rdg), vp(perm),
                                   vp(wofs), vp(coef), vp(src), lo, hi),
                   "gs_rows")
        self.n, self.mode, self.nlev, self.nslots = n, mode, nlev.value, ns.value
        self.n_all = n_all
        # threads per tile: the configured width, halved while the widest
        # tile's staged slices (384 B per slice row) exceed the budget
        T = int(cfg.row_gs_threads)
        while True:
            nwb = T // 32
            ends = np.minimum(np.arange(0, nw + nwb, nwb), nw)
            mts = int(np.diff(wofs[ends]).max(initial=0))
            if 384 * mts <= cfg.row_gs_smem or T == 32:
                break
            T //= 2
        if 384 * mts > cfg.smem_limit:
            raise ValueError("gs rows: a warp's entry slices exceed shared memory")
        self.threads, self.max_tile_slots = T, mts
        if cfg.row_gs_ctas > 0:
            self.ctas = int(cfg.row_gs_ctas)
        else:  # keep ~16 levels of rows in flight: enough to cover the dependency latency, few idle pollers
            per_level = n / max(1, self.nlev)
            self.ctas = int(min(4 * 148, max(8, np.ceil(16 * per_level / self.threads))))
        self.rowid, self.cnt, self.dg, self.rdg = to_device(rowid), to_device(cnt), to_device(dg), to_device(rdg)
        self.crit = to_device(crit)
        self.perm, self.wofs, self.coef, self.src = to_device(perm), to_device(wofs), to_device(coef), to_device(src)
        self.tperm = torch.empty(max(2, n + 2), dtype=torch.float64, device="cuda")
        self._csr = DeviceCSR(A)

    def sweep_ext(self, b_own, x_old_ext, x_ext, mirror_ptr, mirror_dst, peers, ws, stream=None):
        """Pipelined sweep of the own rows (row_range) over the extended layout
        (mvamg_gs_row_sweep_ext_f64); x_ext's own and ghost slots must hold the
        sentinel when the ranks start."""
        lo, hi = self.row_range
        _lib.check(_lib.load().mvamg_gs_row_sweep_ext_f64(
            self.mode, self.n_all, lo, hi, *self._csr.ptrs(), ptr(self.rowid), ptr(self.cnt), ptr(self.crit),
            ptr(self.dg), ptr(self.rdg), ptr(self.wofs), ptr(self.coef), ptr(self.src), self.threads, self.ctas,
            self.max_tile_slots, ptr(self.tperm), ptr(b_own), ptr(x_old_ext), ptr(x_ext), ptr(mirror_ptr),
            ptr(mirror_dst), ptr(peers), ptr(ws), stream or stream_handle()), "gs_row_sweep_ext")

    def args(self):
        return (ptr(self.rowid), ptr(self.cnt), ptr(self.crit), ptr(self.dg), ptr(self.rdg), ptr(self.perm),
                ptr(self.wofs), ptr(self.coef), ptr(self.src), self.threads, self.ctas, self.max_tile_slots,
                ptr(self.tperm))

    def hierarchy_args(self):
        return self.args()

    def sweep(self, b, x_old, x_new, ws, stream=None):
        """One sweep; with x_old a mode-2 schedule runs the folded backward sweep."""
        _lib.check(_lib.load().mvamg_gs_row_sweep_f64(
            self.mode, self.n, *self._csr.ptrs(), *self.args(), ptr(b), ptr(x_old), ptr(x_new), ptr(ws),
            stream or stream_handle()), "gs_row_sweep")


def time_sweep(fn, reps=3):
    """Device time (s) of fn() -- one GS sweep -- after one warm-up launch.
    (Direct launches: for very short sweeps this includes the host issue rate,
    the same for every candidate the autotune compares.)"""
    torch = torch_cuda()
    fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps * 1e-3


def autotune_coarse_gs(A, modes, cfg):
    """For a coarse level: per sweep mode, the faster of the dataflow row sweep
    and the level-set sweep, timed once on the device ({mode: schedule}).
    Mode 2 is timed as the folded backward sweep it runs in a cycle.

    Only in exact mode: there every schedule gives the same bits.  With
    tolerance parity the two kernels round differently, so a timing-based pick
    could make two runs of the same problem differ.  There the choice is by
    size: the single-CTA level-set sweep up to cfg.level_gs_small_rows rows
    (faster on every C2/C3/composite level that small), the row sweep above."""
    torch = torch_cuda()
    n = A.shape[0]
    if not cfg.exact_gs:
        if n <= cfg.level_gs_small_rows:
            try:
                return {m: DeviceGsLevels(A, m, cfg) for m in modes}
            except ValueError:
                pass
        return {m: DeviceGsRows(A, m, cfg) for m in modes}
    rows = {m: DeviceGsRows(A, m, cfg) for m in modes}
    try:
        lvls = {m: DeviceGsLevels(A, m, cfg) for m in modes}
    except ValueError:
        return dict(rows)
    g = torch.Generator(device="cuda").manual_seed(0)
    b = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
    xo = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
    xn = torch.empty(n, dtype=torch.float64, device="cuda")
    ws = torch.zeros(8, dtype=torch.int32, device="cuda")
    out = {}
    for m in modes:
        xold = xo if m in (1, 2, 3) else None
        t_rows = time_sweep(lambda: rows[m].sweep(b, xold, xn, ws))
        if m == 2:
            t_lvl = time_sweep(lambda: lvls[m].sweep(b, xo, xn, ws, fold=True))
        else:
            t_lvl = time_sweep(lambda: lvls[m].sweep(b, xold, xn, ws))
        out[m] = rows[m] if t_rows <= t_lvl else lvls[m]
    return out


def row_gs_fits(A, k, cfg):
    """Whether a coarse level (k >= 1) should use the dataflow row sweep."""
    if k == 0 or cfg.generic_gs or cfg.force_level_gs:
        return False
    if cfg.force_row_gs:
        return True
    return A.shape[0] >= cfg.row_gs_min_rows


def level_gs_fits(A, cfg):
    """Whether the small-level single-CTA sweep is the better schedule for A:
    small enough for shared memory, and with rows too long for the lean
    wavefront kernel (the wavefront wins on short-row grid levels)."""
    n = A.shape[0]
    if n > cfg.level_gs_max_rows or cfg.generic_gs:
        return False
    if cfg.force_level_gs:
        return True
    lo, up = _row_counts(as_csr(A))
    return int(max(lo.max(initial=0), up.max(initial=0))) > 8


def galerkin_product_device(P, A, timing=None):
    """galerkin_product(P, A) (pkg/src/mvamg/sparse.py:50-66) on the GPU.

    Same arguments, ValueError on a dimension mismatch, and the same canonical
    CSR bit for bit (csrc/galerkin.cuh restates scipy's summation order).  The
    operands are uploaded, A_c is formed on the device and returned as a scipy
    CSR.  ``timing``: optional dict that receives the device milliseconds of the
    four phases (transpose, A P, P'(A P), symmetrise) and their total."""
    P = as_csr(P)
    A = as_csr(A)
    if P.shape[0] != A.shape[0] or A.shape[0] != A.shape[1]:
        raise ValueError(f"dimension mismatch: P is {P.shape[0]}x{P.shape[1]}, A is {A.shape[0]}x{A.shape[1]}")
    torch = torch_cuda()
    L = _lib.load()
    n, nc = P.shape
    dev = [to_device(a) for a in (A.indptr.astype(np.int32), A.indices.astype(np.int32), A.data,
                                  P.indptr.astype(np.int32), P.indices.astype(np.int32), P.data)]
    h = ctypes.c_void_p()
    nnz = ctypes.c_longlong(0)
    ph = (ctypes.c_float * 4)()
    _lib.check(L.mvamg_galerkin_f64(n, nc, *[ptr(t) for t in dev], ctypes.byref(h), ctypes.byref(nnz), ph,
                                    stream_handle()), "galerkin_product")
    try:
        ip = torch.empty(nc + 1, dtype=torch.int32, device="cuda")
        ix = torch.empty(max(nnz.value, 1), dtype=torch.int32, device="cuda")
        v = torch.empty(max(nnz.value, 1), dtype=torch.float64, device="cuda")
        _lib.check(L.mvamg_spmat_copy(h, ptr(ip), ptr(ix), ptr(v), stream_handle()), "galerkin_product")
        torch.cuda.current_stream().synchronize()
    finally:
        L.mvamg_spmat_destroy(h)
    if timing is not None:
        names = ("transpose_ms", "ap_ms", "ptap_ms", "symmetrize_ms")
        timing.update({k: float(x) for k, x in zip(names, ph)})
        timing["total_ms"] = float(sum(ph))
    k = nnz.value
    return sp.csr_matrix((v.cpu().numpy()[:k], ix.cpu().numpy()[:k], ip.cpu().numpy()), shape=(nc, nc))
