"""Chain-scan GS schedule (csrc/gs_scan.cuh) -- host planner and device holder.

Tolerance-parity smoother for levels with chain structure, e.g. grid lines,
selected when GpuConfig.exact_gs is False.  It keeps the reference sweep's
dependency order (pkg/src/mvamg/_kernels.py:15-38) and reassociates each
row's sums (module docstring of gs_scan.cuh).  The planner works in sweep
order: rows are reversed for backward sweeps.  It

- splits the rows into chains (maximal runs where row i couples to row i-1);
- checks that no other in-chain lower entry exists;
- records, per row, the scaled coupling to the chain predecessor and its
  cross-chain sources (chain distance, position);
- records, per 32-row segment, which source segments it has to wait for;
- sizes the shared-memory ring of recent chains.

`plan_scan` returns None when the level does not qualify: no chains, more than
4 cross-chain sources per row, more than 4 source chains per segment, or a
ring that does not fit shared memory.
"""

import ctypes
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from . import _lib
from .device import DeviceCSR, GpuConfig, as_csr, ptr, stream_handle, to_device

MAX_K = 4
MAX_DEPS = 4
ADDR_POS_BITS = 20


@dataclass
class ScanPlan:
    n: int
    mode: int
    nchains: int
    S: int
    ring_len: int
    W: int
    K: int
    threads: int
    seg_ptr: np.ndarray
    chain_start: np.ndarray
    chain_len: np.ndarray
    recv: np.ndarray      # per (segment, vector v, lane): (slope, c0), (c1, c2), ... as double pairs
    addr: np.ndarray      # per (segment, lane): 4 x uint32 (delta << 20 | position), zero cell when unused
    seginfo: np.ndarray   # per segment, 32 B: wait0, wait1, deferred wait, deferred position, its coefficient
    window: int           # > 0: ring slots keep positions mod window (single distance 1)
    cluster: int          # > 1: chains spread over a thread-block cluster of this many CTAs
    rec: np.ndarray       # original row -> record index
    rdiag: np.ndarray     # original row order
    depth: int            # wavefront steps (segment DAG depth)
    deltas: np.ndarray    # distinct source-chain distances (<= 4)
    active: int           # most chains in progress at once in the wavefront

    @property
    def nv(self):
        return (self.K + 2) // 2


MAX_WAITS = 2
SCAN_WINDOW = 256   # positions per ring slot in window mode (8 segments)
STAGES = 3          # staged segments per warp (csrc/gs_scan.cuh kStages)
SCAN_CLUSTER_WARPS = 8  # warps per CTA of the cluster sweep (gs_scan_cluster_kernel: 256 threads)
SEGINFO_DTYPE = np.dtype([("wait0", "<i4"), ("wait1", "<i4"), ("defer", "<i4"), ("defpos", "<i4"),
                          ("defcoef", "<f8"), ("pad", "<f8")])


def plan_scan(A, mode, cfg=None):
    """Chain-scan schedule of A for sweep `mode` (0 fwd from 0, 1 fwd from
    x_old, 2 bwd from 0, 3 bwd from x_old), or None if A does not qualify.

    A segment waits until the source segments of its rows are complete.  One
    exception is the segment's last row, whose sources may reach one segment
    further (the (j+1) neighbour on a 9-point grid).  That single source is
    *deferred*: the row is computed without it, and its term is added when
    the warp starts the next segment, before the segment is published.  Lines
    then lag each other by one segment step instead of two (C2: 1,056 steps
    instead of 2,078)."""
    cfg = cfg or GpuConfig()
    A = as_csr(A)
    n = A.shape[0]
    if n == 0:
        return None
    fwd = mode < 2
    d = A.diagonal()
    if np.any(d == 0.0):
        return None
    if fwd:
        B = A
    else:
        rev = np.arange(n - 1, -1, -1)
        B = sp.csr_matrix(A[rev][:, rev])
        B.sort_indices()
    ip, ix, v = B.indptr.astype(np.int64), B.indices.astype(np.int64), B.data
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(ip))
    dB = d if fwd else d[::-1]
    rdB = 1.0 / dB
    # chains: row i continues the chain of row i-1 when it couples to it
    has_prev = np.zeros(n, dtype=bool)
    has_prev[rows[ix == rows - 1]] = True
    has_prev[0] = False
    heads = np.nonzero(~has_prev)[0]
    nch = heads.shape[0]
    chain_of = np.cumsum(~has_prev) - 1
    clen = np.diff(np.append(heads, n))
    cs_row = heads[chain_of]
    new = ix < rows
    in_chain_other = new & (ix >= cs_row[rows]) & (ix != rows - 1)
    if np.any(in_chain_other):
        return None
    cross = new & (ix < cs_row[rows])
    cr, cc, cv = rows[cross], ix[cross], v[cross]
    src_chain = chain_of[cc]
    delta = chain_of[cr] - src_chain
    pos = cc - heads[src_chain]
    W = int(delta.max()) if delta.size else 0
    deltas = np.unique(delta).astype(np.int32)
    if deltas.shape[0] > MAX_DEPS:
        return None
    per_row = np.bincount(cr, minlength=n)
    K = int(per_row.max()) if per_row.size else 0
    maxlen = int(clen.max())
    if K > MAX_K or maxlen >= (1 << ADDR_POS_BITS) - 1 or W >= 2048:
        return None
    K = max(K, 1)
    NV = (K + 2) // 2
    ring_len = maxlen + 1
    nseg = -(-clen // 32)
    seg_ptr = np.zeros(nch + 1, dtype=np.int64)
    np.cumsum(nseg, out=seg_ptr[1:])
    nsegs = int(seg_ptr[-1])
    rowpos = np.arange(n) - cs_row
    rec_sweep = (seg_ptr[chain_of] + rowpos // 32) * 32 + rowpos % 32
    recv = np.zeros((nsegs, NV, 32, 2))
    seg_r, lane_r = rec_sweep // 32, rec_sweep % 32
    pm = ix == rows - 1
    recv[seg_r[rows[pm]], 0, lane_r[rows[pm]], 0] = -(v[pm] * rdB[rows[pm]])
    addr = np.full((nsegs, 32, 4), maxlen, dtype=np.uint32)  # every slot's last cell stays 0
    seginfo = np.zeros(nsegs, dtype=SEGINFO_DTYPE)
    if cr.size:
        order = np.argsort(cr, kind="stable")
        cr, cc, cv, delta, pos = cr[order], cc[order], cv[order], delta[order], pos[order]
        r = rec_sweep[cr]
        seg, lane = r // 32, r % 32
        own_seg = rowpos[cr] // 32
        src_seg = pos // 32
        late = src_seg > own_seg
        # defer a late source when it is the only late one of its row and the
        # row is its segment's last (its term then reaches no other row)
        nlate = np.bincount(cr[late], minlength=n)
        deferred = late & (lane == 31) & (nlate[cr] == 1)
        keep = ~deferred
        kc = cr[keep]
        start = np.searchsorted(kc, kc, side="left")
        k = np.arange(kc.shape[0]) - start
        slot = k + 1  # slot 0 of the (slope, c0, ...) list is the slope
        recv[seg[keep], slot // 2, lane[keep], slot % 2] = cv[keep] * rdB[kc]
        addr[seg[keep], lane[keep], k] = (delta[keep].astype(np.uint32) << ADDR_POS_BITS) | pos[keep].astype(np.uint32)
        if np.any(deferred):
            gd = seg[deferred]
            seginfo["defer"][gd] = (delta[deferred].astype(np.int64) << 20 | (src_seg[deferred] + 1)).astype(np.int32)
            seginfo["defpos"][gd] = pos[deferred].astype(np.int32)
            seginfo["defcoef"][gd] = cv[deferred] * rdB[cr[deferred]]
        # waits of the kept sources: (delta, segments of the source chain needed)
        need = src_seg[keep] + 1
        key = seg[keep] * 4096 + delta[keep]
        uk, inv = np.unique(key, return_inverse=True)
        mneed = np.zeros(uk.shape[0], dtype=np.int64)
        np.maximum.at(mneed, inv, need)
        useg, udelta = uk // 4096, uk % 4096
        cnt = np.bincount(useg, minlength=nsegs)
        if cnt.max(initial=0) > MAX_WAITS:
            return None
        dstart = np.searchsorted(useg, useg, side="left")
        wslot = np.arange(useg.shape[0]) - dstart
        wv = (udelta.astype(np.int64) << 20 | mneed).astype(np.int32)
        seginfo["wait0"][useg[wslot == 0]] = wv[wslot == 0]
        seginfo["wait1"][useg[wslot == 1]] = wv[wslot == 1]
        dg = seg[deferred]
        depth, active = _segment_schedule(nch, seg_ptr, np.concatenate([useg, dg]),
                                          np.concatenate([udelta, delta[deferred]]),
                                          np.concatenate([mneed, src_seg[deferred] + 1]),
                                          np.concatenate([np.zeros(useg.shape[0], bool), np.ones(dg.shape[0], bool)]))
    else:
        depth, active = int(nseg.max()), nch
    # window mode (every source one chain back): a slot keeps the last WINDOW
    # positions of its chain, producers wait for their reader before reuse
    window = SCAN_WINDOW if (deltas.shape[0] == 1 and deltas[0] == 1 and maxlen > SCAN_WINDOW) else 0
    if window:
        ring_len = window
    # warps: enough for the chains in flight, as many as shared memory allows
    # (ring of S = warps + W + 1 chains, kStages staged segments per warp)
    stage = 256 + NV * 512 + 512 + 32
    threads = 0
    want = int(min(32, max(2, active + 2)))
    for nw in range(want, 0, -1):
        S = nw + W + 1
        if 8 * ((S + 1) & ~1) + 8 * S * ring_len + 128 + nw * STAGES * (stage + 8) <= cfg.smem_limit:
            threads = 32 * nw
            break
    if threads == 0:
        return None
    S = threads // 32 + W + 1
    cluster = 0
    if window and cfg.scan_cluster > 1:
        # chain L on CTA L mod C, NW warps each; a CTA's S slots hold its readers' rings
        cluster, threads = int(cfg.scan_cluster), 32 * SCAN_CLUSTER_WARPS
        S = SCAN_CLUSTER_WARPS + 2
    rec = np.empty(n, dtype=np.int64)
    if fwd:
        rec[:] = rec_sweep
    else:
        rec[n - 1 - np.arange(n)] = rec_sweep
    return ScanPlan(n, mode, nch, S, ring_len, W, K, threads, seg_ptr.astype(np.int32),
                    heads.astype(np.int32), clen.astype(np.int32), recv.ravel(), addr.ravel(), seginfo, window,
                    cluster, rec.astype(np.int32), 1.0 / d, depth, deltas, active)


def _segment_schedule(nch, seg_ptr, useg, udelta, mneed, is_def):
    """Completion step of every segment (one step per segment; a deferred
    source delays only the segment's completion, not its computation):
    (depth, most chains in progress at once).  Chains only wait on earlier
    chains, so one pass over the chains in order suffices."""
    nsegs = int(seg_ptr[-1])
    chain = np.searchsorted(seg_ptr, np.arange(nsegs), side="right") - 1
    done = np.zeros(nsegs, dtype=np.int64)
    src = seg_ptr[chain[useg] - udelta] + mneed - 1   # the source segment that must be complete
    order = np.argsort(useg, kind="stable")
    us, srcs, dfs = useg[order], src[order], is_def[order]
    bounds = np.searchsorted(us, seg_ptr)
    for c in range(nch):
        g0, g1 = seg_ptr[c], seg_ptr[c + 1]
        m = g1 - g0
        ready = np.zeros(m, dtype=np.int64)   # inputs of the computation complete
        fin = np.zeros(m, dtype=np.int64)     # deferred source complete
        e0, e1 = bounds[c], bounds[c + 1]
        if e1 > e0:
            sel, dsel = us[e0:e1] - g0, dfs[e0:e1]
            np.maximum.at(ready, sel[~dsel], done[srcs[e0:e1][~dsel]])
            np.maximum.at(fin, sel[dsel], done[srcs[e0:e1][dsel]])
        t_prev = 0
        for j in range(m):
            t = max(ready[j], t_prev) + 1          # computed one step after inputs and carry
            t = max(t, fin[j])                      # published once the deferred input is there
            done[g0 + j] = t
            t_prev = t
    depth = int(done.max(initial=0))
    start, end = done[seg_ptr[:-1]], done[seg_ptr[1:] - 1]
    ev = np.zeros(depth + 2, dtype=np.int64)
    np.add.at(ev, start, 1)
    np.add.at(ev, end + 1, -1)
    return depth, int(np.cumsum(ev).max(initial=1))


class DeviceGsScan:
    """A ScanPlan on the device plus the sweep launcher."""

    def __init__(self, A, mode, cfg=None, plan=None):
        import torch

        self.plan = p = plan or plan_scan(A, mode, cfg)
        if p is None:
            raise ValueError("level has no chain structure usable by the scan sweep")
        self.mode = mode
        self.seg_ptr, self.chain_start, self.chain_len = (to_device(p.seg_ptr), to_device(p.chain_start),
                                                          to_device(p.chain_len))
        self.recv = to_device(p.recv)
        self.addr = to_device(p.addr.view(np.int32))
        self.seginfo = to_device(p.seginfo.view(np.uint8))
        self.rec, self.rdiag = to_device(p.rec), to_device(p.rdiag)
        self.o0 = torch.zeros(p.seg_ptr[-1] * 32, dtype=torch.float64, device="cuda")
        self._deltas = np.ascontiguousarray(np.append(p.deltas, [0] * 4)[:4], dtype=np.int32)
        self._csr = DeviceCSR(A)

    def args(self):
        p = self.plan
        return (p.nchains, p.S, p.ring_len, int(p.deltas.shape[0]), self._deltas.ctypes.data_as(ctypes.c_void_p),
                p.K, p.threads, p.window | (p.cluster << 16), ptr(self.seg_ptr), ptr(self.chain_start),
                ptr(self.chain_len), ptr(self.recv), ptr(self.addr), ptr(self.seginfo), ptr(self.o0), ptr(self.rec), ptr(self.rdiag))

    def sweep(self, b, x_old, x_new, ws, stream=None):
        mode = self.mode
        _lib.check(_lib.load().mvamg_gs_scan_sweep_f64(
            mode, self.plan.n, *self._csr.ptrs(), *self.args(), ptr(b), ptr(x_old), ptr(x_new), ptr(ws),
            stream or stream_handle()), "gs_scan_sweep")
