"""Host-side setup of the composite / multi-vector AMG (vectorised restatement).

The north star keeps the reference's Python setup as is; the reference cannot
travel to the GPU box, so this module restates its setup algorithm in
vectorised numpy/scipy (plus two native helpers in libmvamg_b200.so) to build
the hierarchies the solve phase consumes.  The bootstrap's test phase -- the
symmetrized multiplicative composite of K-cycles, i.e. the H2 hot path -- runs
on the GPU through GpuComposite.

Reference algorithm, file:line:
  edge weights          pkg/src/mvamg/matching.py:78-103
  greedy matching       pkg/src/mvamg/matching.py:106-122, _kernels.py:41-61
  pair prolongator      pkg/src/mvamg/pairwise.py:108-159
  pairwise composition  pkg/src/mvamg/pairwise.py:170-210
  pairwise hierarchy    pkg/src/mvamg/pairwise.py:213-243
  aggregate merging     pkg/src/mvamg/multivector.py:125-160
  truncated local SVD   pkg/src/mvamg/multivector.py:181-212, svd.py:17-55
  block prolongator     pkg/src/mvamg/multivector.py:215-259
  multi-vector levels   pkg/src/mvamg/multivector.py:262-321
  bootstrap loop        pkg/src/mvamg/bootstrap.py:144-198
Aggregates are kept as CSR-like (ptr, members) arrays instead of lists of
arrays, so million-row levels stay vectorised.  Given the same inputs the
matchings, aggregates and prolongators come out identical (checked against the
reference's own hierarchies in tests/test_setup.py).
"""

import ctypes
import time
import warnings
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp

from . import _lib
from .device import as_csr
from .exceptions import CoarseningStagnationError, NotSpdError, SvdConvergenceError

WEIGHT_FLOOR = 1e-12
ZERO_ENTRY_PERTURBATION = 1e-8
SVD_MAX_SWEEPS = 60
SVD_PAIR_TOL = 1e-14


# ----------------------------------------------------------------- helpers ---
def galerkin_product(P, A):
    """P' A P symmetrised as (G + G')/2 -- the reference's exact scipy recipe
    (pkg/src/mvamg/sparse.py:50-66), so coarse matrices match bit for bit."""
    if P.shape[0] != A.shape[0] or A.shape[0] != A.shape[1]:
        raise ValueError(f"dimension mismatch: P is {P.shape[0]}x{P.shape[1]}, A is {A.shape[0]}x{A.shape[1]}")
    G = (P.T @ (A @ P)).tocsr()
    G = ((G + G.T) * 0.5).tocsr()
    G.sum_duplicates()
    G.sort_indices()
    return G


@dataclass
class Aggregates:
    """Partition of a level's dofs: aggregate a = members[ptr[a]:ptr[a+1]] (sorted)."""

    ptr: np.ndarray
    members: np.ndarray
    n_prev: int

    @property
    def n_agg(self):
        return self.ptr.shape[0] - 1

    def owner(self):
        own = np.full(self.n_prev, -1, dtype=np.int64)
        own[self.members] = np.repeat(np.arange(self.n_agg), np.diff(self.ptr))
        return own

    def as_lists(self):
        return [self.members[self.ptr[a]:self.ptr[a + 1]] for a in range(self.n_agg)]


def _group(owner, n_groups, n_prev):
    """Aggregates from an owner map (members of a group sorted ascending)."""
    order = np.lexsort((np.arange(owner.shape[0]), owner))
    counts = np.bincount(owner, minlength=n_groups)
    ptr = np.zeros(n_groups + 1, dtype=np.int64)
    np.cumsum(counts, out=ptr[1:])
    return Aggregates(ptr, order.astype(np.int64), n_prev)


def _compose(fine, coarse):
    """Members of each coarse aggregate expanded through the finer aggregates."""
    own_fine = fine.owner()              # fine dof -> fine aggregate
    own_coarse = coarse.owner()          # fine aggregate -> coarse aggregate
    return _group(own_coarse[own_fine], coarse.n_agg, fine.n_prev)


# ---------------------------------------------------------------- matching ---
def edge_weights(A, w):
    """(i, j, c) of every stored pair i < j: c = 1 - 2 a_ij w_i w_j /
    (a_ii w_i^2 + a_jj w_j^2), -inf where the denominator vanishes."""
    w = np.asarray(w, dtype=np.float64)
    if A.shape[0] != A.shape[1] or w.shape[0] != A.shape[0]:
        raise ValueError("A must be square and w of matching length")
    d = A.diagonal()
    if np.any(d == 0.0):
        raise NotSpdError("zero diagonal entry; edge weights are undefined")
    U = sp.triu(A, 1).tocoo()
    i = U.row.astype(np.int64)
    j = U.col.astype(np.int64)
    den = d[i] * w[i] ** 2 + d[j] * w[j] ** 2
    ok = den != 0.0
    c = np.full(i.shape[0], -np.inf)
    c[ok] = 1.0 - 2.0 * U.data[ok] * w[i[ok]] * w[j[ok]] / den[ok]
    return i, j, c


def greedy_matching(i, j, c, n, weight_floor=WEIGHT_FLOOR):
    """Greedy max-product matching: edges by descending weight, ties by (i, j),
    accepted when both ends are free.  Returns (pairs (np x 2), unmatched)."""
    keep = c > weight_floor
    ei, ej, ec = i[keep], j[keep], c[keep]
    order = np.lexsort((ej, ei, -ec))
    ei = np.ascontiguousarray(ei[order], dtype=np.int64)
    ej = np.ascontiguousarray(ej[order], dtype=np.int64)
    partner = np.empty(max(1, n), dtype=np.int64)
    pi = np.empty(max(1, ei.shape[0]), dtype=np.int64)
    pj = np.empty(max(1, ei.shape[0]), dtype=np.int64)
    npairs = ctypes.c_longlong()
    vp = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    _lib.check(_lib.load().mvamg_greedy_match(ei.shape[0], vp(ei), vp(ej), n, vp(partner), vp(pi), vp(pj),
                                              ctypes.byref(npairs)), "greedy_match")
    k = npairs.value
    pairs = np.stack([pi[:k], pj[:k]], axis=1) if k else np.empty((0, 2), dtype=np.int64)
    return pairs, np.flatnonzero(partner[:n] < 0).astype(np.int64)


def greedy_matching_device(A, w, weight_floor=WEIGHT_FLOOR):
    """edge_weights + greedy_matching on the GPU (mvamg_greedy_match_device:
    locally dominant matching, equal to the greedy order's result).  Same
    return value: pairs (i < j) in the greedy's acceptance order (weight
    descending, ties by (i, j)), and the unmatched vertices ascending."""
    from .device import ptr, stream_handle, to_device, torch_cuda

    torch = torch_cuda()
    w = np.asarray(w, dtype=np.float64)
    if A.shape[0] != A.shape[1] or w.shape[0] != A.shape[0]:
        raise ValueError("A must be square and w of matching length")
    d = A.diagonal()
    if np.any(d == 0.0):
        raise NotSpdError("zero diagonal entry; edge weights are undefined")
    n = A.shape[0]
    dev = [to_device(A.indptr, np.int32), to_device(A.indices, np.int32), to_device(A.data, np.float64),
           to_device(d, np.float64), to_device(w, np.float64)]
    partner = torch.empty(max(1, n), dtype=torch.int32, device="cuda")
    rounds = ctypes.c_int()
    _lib.check(_lib.load().mvamg_greedy_match_device(n, *[ptr(t) for t in dev], float(weight_floor), ptr(partner),
                                                     ctypes.byref(rounds), stream_handle()), "greedy_match_device")
    part = partner.cpu().numpy()[:n].astype(np.int64)
    i = np.flatnonzero(part > np.arange(n))
    j = part[i]
    if i.size:
        # weights of the matched pairs, as edge_weights forms them, for the acceptance order
        a = np.asarray(A[i, j]).ravel()
        den = d[i] * w[i] ** 2 + d[j] * w[j] ** 2
        c = 1.0 - 2.0 * a * w[i] * w[j] / den
        order = np.lexsort((j, i, -c))
        pairs = np.stack([i[order], j[order]], axis=1)
    else:
        pairs = np.empty((0, 2), dtype=np.int64)
    return pairs, np.flatnonzero(part < 0).astype(np.int64)


def pair_prolongator(A, w, pairs, unmatched):
    """Coarse prolongator of one pairwise step: matched pairs first (matching
    order), then singletons ascending; returns (P_c, aggregates)."""
    w = np.asarray(w, dtype=np.float64)
    n = A.shape[0]
    d = A.diagonal()
    if np.any(d <= 0.0):
        raise ValueError("matrix diagonal must be positive")
    n_p = pairs.shape[0]
    pi = pairs[:, 0] if n_p else np.empty(0, dtype=np.int64)
    pj = pairs[:, 1] if n_p else np.empty(0, dtype=np.int64)
    wi, wj = w[pi], w[pj]
    scale = np.sqrt(wi ** 2 + wj ** 2)
    if np.any(scale == 0.0):
        raise ValueError("matched pair with w_i = w_j = 0; weights should have excluded it")
    singles = np.sort(unmatched)
    ws = w[singles]
    zero = ws == 0.0
    if np.any(zero):
        winf = float(np.max(np.abs(w)))
        if winf == 0.0:
            raise ValueError("smooth vector is identically zero")
        ws = ws.copy()
        ws[zero] = ZERO_ENTRY_PERTURBATION * winf
    n_s = singles.shape[0]
    rows = np.concatenate([pi, pj, singles])
    cols = np.concatenate([np.arange(n_p), np.arange(n_p), n_p + np.arange(n_s)])
    vals = np.concatenate([wi / scale, wj / scale, np.sign(ws)])
    P = sp.csr_matrix((vals, (rows, cols)), shape=(n, n_p + n_s))
    P.sort_indices()
    own = np.empty(n, dtype=np.int64)
    own[rows] = cols
    return P, _group(own, n_p + n_s, n)


# ---------------------------------------------------------------- pairwise ---
@dataclass
class CoarseningParams:
    steps_per_level: int = 2
    max_levels: int = 20
    min_coarse_size: int = 40
    weight_floor: float = WEIGHT_FLOOR
    min_shrink: float = 0.10


@dataclass
class PairwiseLevel:
    A: sp.csr_matrix
    P: sp.csr_matrix = None
    aggregates: Aggregates = None
    w: np.ndarray = None


@dataclass
class PairwiseHierarchy:
    levels: list
    params: CoarseningParams
    build_seconds: float = 0.0

    @property
    def nl(self):
        return len(self.levels)

    @property
    def matrices(self):
        return [lv.A for lv in self.levels]

    @property
    def prolongators(self):
        return [lv.P for lv in self.levels[1:]]

    def sizes(self):
        return [lv.A.shape[0] for lv in self.levels]


def coarse_product(config=None):
    """The Galerkin product the setup uses: the device kernel
    (device.galerkin_product_device, bit-identical) unless the GpuConfig turns
    it off, in which case the host scipy recipe."""
    from .device import GpuConfig, galerkin_product_device

    return galerkin_product_device if (config or GpuConfig()).device_galerkin else galerkin_product


def pairwise_step(A, w, steps, weight_floor=WEIGHT_FLOOR, product=galerkin_product, device_matching=False,
                  matcher=None):
    """Compose `steps` matching sweeps into one transfer; returns
    (P, A_c, w_c, aggregates, stagnated, steps_done).  matcher(A, w, floor) ->
    (pairs, unmatched) replaces the matching (the CPU-only setup of bench.py's
    reference arm passes the oracle's)."""
    if steps < 1:
        raise ValueError("steps must be >= 1")
    Ak, wk = A, np.asarray(w, dtype=np.float64)
    P, aggs, stagnated, done = None, None, False, 0
    for _ in range(steps):
        if matcher is not None:
            pairs, unmatched = matcher(Ak, wk, weight_floor)
        elif device_matching:
            pairs, unmatched = greedy_matching_device(Ak, wk, weight_floor)
        else:
            i, j, c = edge_weights(Ak, wk)
            pairs, unmatched = greedy_matching(i, j, c, Ak.shape[0], weight_floor)
        if pairs.shape[0] == 0:
            stagnated = True
            break
        Pc, step_aggs = pair_prolongator(Ak, wk, pairs, unmatched)
        aggs = step_aggs if aggs is None else _compose(aggs, step_aggs)
        P = Pc if P is None else (P @ Pc).tocsr()
        Ak = product(Pc, Ak)
        wk = Pc.T @ wk
        done += 1
    if P is None:
        n = A.shape[0]
        signs = np.where(wk >= 0.0, 1.0, -1.0)
        P = sp.csr_matrix((signs, (np.arange(n), np.arange(n))), shape=(n, n))
        aggs = Aggregates(np.arange(n + 1, dtype=np.int64), np.arange(n, dtype=np.int64), n)
        Ak = product(P, A)
        wk = P.T @ np.asarray(w, dtype=np.float64)
    return P, Ak, wk, aggs, stagnated, done


def build_pairwise_hierarchy(A, w, params=None, product=galerkin_product, device_matching=False, matcher=None):
    """Coarsen (A, w) until small; a level shrinking by < min_shrink is
    dropped; no pairs at the finest level raises CoarseningStagnationError."""
    params = params or CoarseningParams()
    A = as_csr(A)
    w = np.asarray(w, dtype=np.float64)
    if A.shape[0] != w.shape[0]:
        raise ValueError("w length must match A")
    t0 = time.perf_counter()
    levels = [PairwiseLevel(A=A, w=w)]
    while levels[-1].A.shape[0] > params.min_coarse_size and len(levels) < params.max_levels:
        cur = levels[-1]
        P, Ac, wc, aggs, stagnated, done = pairwise_step(cur.A, cur.w, params.steps_per_level,
                                                         params.weight_floor, product, device_matching, matcher)
        if done == 0:
            if len(levels) == 1:
                raise CoarseningStagnationError("matching produced no pairs at the finest level", level=0)
            break
        if Ac.shape[0] > (1.0 - params.min_shrink) * cur.A.shape[0]:
            break
        levels.append(PairwiseLevel(A=Ac, P=P, aggregates=aggs, w=wc))
        if stagnated:
            break
    return PairwiseHierarchy(levels, params, time.perf_counter() - t0)


# ------------------------------------------------------------- multivector ---
@dataclass
class BlockProlongator:
    P: sp.csr_matrix
    kept: np.ndarray          # per aggregate
    col_offsets: np.ndarray   # n_agg + 1
    sigma: np.ndarray         # per aggregate singular values (n_agg x nv)


@dataclass
class MultiVectorHierarchy:
    matrices: list
    prolongators: list
    vectors_per_level: list
    aggregate_sets: list
    stalled: bool = False
    build_seconds: float = 0.0
    svd_seconds: float = 0.0

    @property
    def nl(self):
        return len(self.matrices)

    @property
    def prolongator_matrices(self):
        return [bp.P for bp in self.prolongators]

    def sizes(self):
        return [A.shape[0] for A in self.matrices]


def merge_aggregate_levels(hierarchy, merge_levels=3):
    """First `merge_levels` aggregate maps composed into one fine set, then the
    deeper levels untouched (a shallower hierarchy is merged in full)."""
    if merge_levels < 1:
        raise ValueError("merge_levels must be >= 1")
    per = [lv.aggregates for lv in hierarchy.levels[1:]]
    if not per:
        return []
    if len(per) < merge_levels:
        warnings.warn(f"hierarchy has {len(per)} aggregate levels, fewer than merge_levels={merge_levels}; "
                      "merging all of them", stacklevel=2)
        merge_levels = len(per)
    merged = per[0]
    for aggs in per[1:merge_levels]:
        merged = _compose(merged, aggs)
    return [merged] + per[merge_levels:]


def _jacobi_svd_device(rp, local, nv):
    """mvamg_jacobi_svd_batch_device: the batched local SVD on the GPU
    (csrc/svd.cuh), bit-identical to the host mvamg_jacobi_svd_batch."""
    from .device import ptr, stream_handle, to_device, torch_cuda

    torch = torch_cuda()
    n_agg = rp.shape[0] - 1
    d_rp, d_local = to_device(rp, np.int32), to_device(local, np.float64)
    d_u = torch.empty(max(1, local.size), dtype=torch.float64, device="cuda")
    d_sig = torch.empty(max(1, n_agg * nv), dtype=torch.float64, device="cuda")
    failed = ctypes.c_int(-1)
    code = _lib.load().mvamg_jacobi_svd_batch_device(n_agg, ptr(d_rp), nv, ptr(d_local), SVD_MAX_SWEEPS,
                                                     SVD_PAIR_TOL, ptr(d_u), ptr(d_sig), ctypes.byref(failed),
                                                     stream_handle())
    U = d_u.cpu().numpy()[:local.size].reshape(local.shape)
    sig = d_sig.cpu().numpy()[:n_agg * nv].reshape(n_agg, nv)
    return code, U, sig, failed.value


def block_prolongator(aggs, vectors, n_fine, tol=0.1, device_svd=False, svd=None):
    """Per-aggregate truncated SVD bases (one-sided Jacobi), block diagonal.
    device_svd: the SVD runs on the GPU (same U and sigma bit for bit);
    svd(rp, local, nv) -> (code, U, sigma, failed) replaces it (CPU-only setup)."""
    V = np.column_stack([np.asarray(v, dtype=np.float64) for v in vectors])
    if V.shape[0] != aggs.n_prev:
        raise ValueError("vector length does not match the aggregate set")
    nv = V.shape[1]
    sizes = np.diff(aggs.ptr)
    if np.any(sizes < 1):
        raise ValueError("empty aggregate")
    local = np.ascontiguousarray(V[aggs.members])            # stacked blocks, row-major
    rp = np.ascontiguousarray(aggs.ptr, dtype=np.int32)
    if svd is not None:
        code, U, sig, failed_id = svd(rp, local, nv)
    elif device_svd:
        code, U, sig, failed_id = _jacobi_svd_device(rp, local, nv)
    else:
        U = np.empty_like(local)
        sig = np.empty((aggs.n_agg, nv))
        failed = ctypes.c_int(-1)
        vp = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
        code = _lib.load().mvamg_jacobi_svd_batch(aggs.n_agg, vp(rp), nv, vp(local), SVD_MAX_SWEEPS, SVD_PAIR_TOL,
                                                  vp(U), vp(sig), ctypes.byref(failed))
        failed_id = failed.value
    if code == _lib.E_NOT_SPD:
        raise SvdConvergenceError(f"local SVD failed on aggregate {failed_id}", aggregate_id=failed_id)
    _lib.check(code, "jacobi_svd_batch")
    tol_a = tol * sizes / n_fine
    floor = sig[:, 0] * 50.0 * np.maximum(sizes, nv) * np.finfo(np.float64).eps
    kept = np.count_nonzero(sig > np.maximum(tol_a, floor)[:, None], axis=1)
    empty = kept == 0
    kept[empty] = 1
    lead_zero = empty & (sig[:, 0] == 0.0)
    if np.any(lead_zero):  # fully zero local matrix: first coordinate vector
        U[aggs.ptr[:-1][lead_zero], 0] = 1.0
    col_off = np.zeros(aggs.n_agg + 1, dtype=np.int64)
    np.cumsum(kept, out=col_off[1:])
    rep = np.repeat(kept, sizes)                              # kept count of each member's aggregate
    rows = np.repeat(aggs.members, rep)
    within = np.arange(rows.shape[0]) - np.repeat(np.cumsum(rep) - rep, rep)
    agg_of_member = np.repeat(np.arange(aggs.n_agg), sizes)
    cols = np.repeat(col_off[:-1][agg_of_member], rep) + within
    member_pos = np.repeat(np.arange(aggs.members.shape[0]), rep)
    vals = U[member_pos, within]
    P = sp.csr_matrix((vals, (rows, cols)), shape=(aggs.n_prev, int(col_off[-1])))
    P.sort_indices()
    return BlockProlongator(P, kept, col_off, sig)


def build_multivector_hierarchy(A, pairwise, vectors, merge_levels=3, tol=0.1, min_coarse_size=40,
                                product=galerkin_product, device_svd=False, svd=None):
    """The single multi-vector hierarchy from a pairwise substrate and the
    finest-level smooth vectors (pkg/src/mvamg/multivector.py:262-321)."""
    t0 = time.perf_counter()
    A = as_csr(A)
    vectors = [np.asarray(v, dtype=np.float64) for v in vectors]
    if not vectors:
        raise ValueError("at least one smooth vector is required")
    sets = merge_aggregate_levels(pairwise, merge_levels)
    mats, pros, vecs, used = [A], [], [vectors], []
    stalled, svd_s = False, 0.0
    n_fine = A.shape[0]
    for idx, aggs in enumerate(sets):
        if mats[-1].shape[0] <= min_coarse_size:
            break
        ts = time.perf_counter()
        bp = block_prolongator(aggs, vecs[-1], n_fine, tol, device_svd, svd)
        svd_s += time.perf_counter() - ts
        if bp.P.shape[1] >= mats[-1].shape[0]:
            stalled = True
            break
        pros.append(bp)
        used.append(aggs)
        mats.append(product(bp.P, mats[-1]))
        vecs.append([bp.P.T @ v for v in vecs[-1]])
        if idx + 1 < len(sets):  # SVD dofs of an aggregate travel to its parent group
            owner_col = np.repeat(np.arange(bp.kept.shape[0]), bp.kept)
            parent = sets[idx + 1].owner()[owner_col]
            sets[idx + 1] = _group(parent, sets[idx + 1].n_agg, owner_col.shape[0])
    return MultiVectorHierarchy(mats, pros, vecs, used, stalled, time.perf_counter() - t0, svd_s)


# --------------------------------------------------------------- bootstrap ---
@dataclass
class BootstrapParams:
    rho_des: float = 0.8
    maxstage: int = 15
    nu: int = 15
    rng_seed: int = 0
    min_stages: int = 0
    coarsening: CoarseningParams = field(default_factory=CoarseningParams)
    inner_fcg_iters: int = 2

    def __post_init__(self):
        if not 0.0 < self.rho_des < 1.0:
            raise ValueError("rho_des must lie in (0, 1)")
        if self.nu < 2:
            raise ValueError("nu must be >= 2")
        if self.maxstage < 1:
            raise ValueError("maxstage must be >= 1")


@dataclass
class BootstrapComponent:
    hierarchy: PairwiseHierarchy
    cycle: object
    operator: object


@dataclass
class StageRecord:
    stage: int
    rho: float
    nl: int
    opc: float
    build_seconds: float

    def csv_line(self):
        return f"{self.stage},{self.rho:.6e},{self.nl},{self.opc:.6f},{self.build_seconds:.3f}"


@dataclass
class CompositeAMG:
    A: object
    components: list
    smooth_vectors: list
    reports: list = field(default_factory=list)
    stage_records: list = field(default_factory=list)

    @property
    def n_components(self):
        return len(self.components)


def operator_complexity(matrices):
    return float(sum(M.nnz for M in matrices) / matrices[0].nnz)


def bootstrap_run(A, w0=None, params=None, config=None):
    """Adaptive setup loop (pkg/src/mvamg/bootstrap.py:144-198); each stage's
    K-cycle component is a GpuMultigridOperator and the test phase runs the
    symmetrized composite on the GPU."""
    from .composite import GpuComposite, test_phase
    from .cycles import CycleSpec, GpuMultigridOperator

    import dataclasses

    from .device import GpuConfig

    params = params or BootstrapParams()
    # the test phase's smooth vectors steer the next stage's matching: run its
    # K-cycles with the bit-exact sweeps, as the reference's numba loops do, so
    # near-tied matching decisions follow the reference (the solve itself may
    # use tolerance parity)
    config = dataclasses.replace(config or GpuConfig(), exact_gs=True)
    A = as_csr(A)
    w = np.ones(A.shape[0]) if w0 is None else np.asarray(w0, dtype=np.float64)
    rng = np.random.default_rng(params.rng_seed)
    comp = CompositeAMG(A=A, components=[], smooth_vectors=[w])
    rho, stage, stagnated_before = 1.0, 1, False
    while (rho >= params.rho_des or stage <= params.min_stages) and stage <= params.maxstage:
        t0 = time.perf_counter()
        try:
            hier = build_pairwise_hierarchy(A, comp.smooth_vectors[-1], params.coarsening,
                                            product=coarse_product(config),
                                            device_matching=config.device_matching)
        except CoarseningStagnationError:
            if stagnated_before or comp.n_components == 0:
                raise
            stagnated_before = True
            report, w_new = test_phase(GpuComposite([c.operator for c in comp.components]), A, params.nu, rng)
            comp.reports.append(report)
            if w_new is None:
                break
            comp.smooth_vectors.append(w_new)
            continue
        stagnated_before = False
        cycle = CycleSpec("K", inner_fcg_iters=params.inner_fcg_iters)
        op = GpuMultigridOperator(hier.matrices, hier.prolongators, cycle=cycle, config=config)
        comp.components.append(BootstrapComponent(hier, cycle, op))
        report, w_new = test_phase(GpuComposite([c.operator for c in comp.components]), A, params.nu, rng)
        comp.reports.append(report)
        rho = report.rho_estimate
        comp.stage_records.append(StageRecord(stage, rho, hier.nl, operator_complexity(hier.matrices),
                                              time.perf_counter() - t0))
        if w_new is None:
            break
        comp.smooth_vectors.append(w_new)
        stage += 1
    return comp
