// gs_sweep.cuh -- exact-order Gauss-Seidel sweep for sm_100a.
//
// Reference: gs_forward / gs_backward (pkg/src/mvamg/_kernels.py:15-38): for
// i in order, s = b[i]; s -= a_ij * x[j] for j != i in CSR order; x[i] = s / d_i.
// The result of that loop depends only on its dependency DAG (row i reads the
// new x_j of every earlier row j it couples to), so any schedule that respects
// the DAG and keeps each row's CSR-order rounding reproduces it bit for bit.
//
// Schedule (host, mvamg_gs_analyse + mvamg_gs_schedule):
//   chains  -- runs of consecutive rows where row i couples to row i-1 (grid
//              lines of a natural ordering); one chain per lane, so the i-1
//              dependency stays in a register;
//   tiles   -- consecutive chains owned by one CTA, sharing a position-major
//              shared-memory window of published x values;
//   rounds  -- inside a warp, every row gets a static round: one more than its
//              chain predecessor and than every same-warp row it depends on.
//              Lanes therefore run as a skewed systolic wavefront with no
//              intra-warp waiting; a dependency on another warp or tile is
//              polled (the value's NaN sentinel is its own ready flag).
// Data: the host lays each warp's row records out round-major and lane-minor
// (word w of lane L in round r at round_off[r] + 32 w + L), so one elected lane
// streams R rounds at a time into a shared-memory ring with a TMA bulk copy
// (cp.async.bulk + mbarrier) and every lane's read is a conflict-free LDS.  The
// right-hand side is written in the same order by gs_prepare_kernel.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#ifndef MVAMG_GS_PHASES
#define MVAMG_GS_PHASES 0
#endif
#ifndef MVAMG_LEAN_TRACE
#define MVAMG_LEAN_TRACE 0  // diagnostic build: clock64 per round of the first warp into GsArgs::trace
#endif
#if MVAMG_GS_PHASES
#define GS_STAMP(k) do { if (lane == 0) { long long _t = clock64(); ph_acc[k] += _t - ph_last; ph_last = _t; } } while (0)
#else
#define GS_STAMP(k) do {} while (0)
#endif

namespace mvamg {

// Record words (per row, per lane):
//   w0: cnt (bits 0-15, 0xffff = no row this round) | window-only flag (bit 16)
//   w1: diag          w2: RN(1/diag)
//   then cnt entries of 2 words: [coefficient][int code]
// holding, in CSR order, the entries still contributing to the serial loop's
// sum at sweep time: forward sweeps j < i (and from a nonzero guess the upper
// j > i after them); backward sweeps j > i (the upper j < i precede the
// diagonal in CSR order and are folded into the right-hand side by
// gs_prepare_kernel with the same roundings).  Value sources:
//   code & 3 == 0   x_new of the previous row of this chain (a register)
//   code & 3 == 1   the tile's shared window, slot code>>2 (polled)
//   code & 3 == 2   x_new[code>>2] in global memory (another tile, polled)
//   code & 3 == 3   x_old[code>>2] (forward sweep from a nonzero guess)
constexpr unsigned kGsNoRow = 0xffffu;
constexpr long long kGsIdleLimit = 1LL << 22;  // spins on one round before giving up

struct GsArgs {
  int n, ntiles, window;         // window: shared slots per tile
  int slot_words;                // words of one ring slot (R rounds of records + R*32 rhs)
  int rec_words_max;             // words of records in one slot (R * Smax * 32)
  const unsigned long long* rec; // round-major records of all warps
  const int* round_off;          // word offset of every (warp, round); one terminal entry
  const int* tbase;              // first global round of each warp (nwarps + 1)
  const int* tile_wbase;         // first warp of each tile (ntiles + 1)
  const int* chain_ptr;
  const int* tile_ptr;           // tiles: ranges of the chain order
  const int* chain_order;        // processing order of the chains (nullptr: natural order)
  int wmask;                     // window positions mod (wmask + 1) (one-warp tiles; -1: the whole chain)
  const double* tperm;           // right-hand side in (round, lane) order
  const double* xold;
  double* xnew;
  int* ticket;
  int* status;
  long long* trace;              // optional per-warp cycle trace (diagnostics)
  int debug;                     // diagnostics: bit0 = ignore readiness (timing only, wrong results)
};

__device__ __forceinline__ unsigned long long ld_shared_volatile_u64(unsigned saddr) {
  unsigned long long v;
  asm volatile("ld.volatile.shared.b64 %0, [%1];" : "=l"(v) : "r"(saddr));
  return v;
}
__device__ __forceinline__ unsigned long long ld_shared_u64(unsigned saddr) {
  unsigned long long v;
  asm volatile("ld.shared.b64 %0, [%1];" : "=l"(v) : "r"(saddr));
  return v;
}
__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(unsigned dst, const void* src, unsigned bytes, unsigned bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(unsigned bar, unsigned parity) {
  unsigned ok;
  asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
               : "=r"(ok) : "r"(bar), "r"(parity) : "memory");
  return ok != 0;
}

// Value multiplying one record entry (any source).  `win` is the tile's
// shared window; plain (volatile) C++ accesses so the compiler can predicate.
__device__ __forceinline__ unsigned long long gs_src(int code, const volatile unsigned long long* win,
                                                     const double* xnew, const double* xold, double xprev) {
  const int t = code & 3, idx = code >> 2;
  unsigned long long v = (unsigned long long)__double_as_longlong(xprev);
  if (t == 1) v = win[idx];
  if (t == 2) v = ld_relaxed_u64(xnew + idx);
  if (t == 3) v = (unsigned long long)__double_as_longlong(__ldg(xold + idx));
  return v;
}

__device__ __forceinline__ bool gs_published(unsigned long long v) {
  return (unsigned)(v >> 32) != 0xffffffffu;  // the sentinel's high word; arithmetic never makes it
}

// Generic gather of entries [u0, u0+4) of a row (any sources).
__device__ __forceinline__ bool gs_gather4(const GsArgs& a, const volatile unsigned long long* win,
                                           const unsigned long long* rec, int cnt, int u0, double xprev,
                                           double av[4], unsigned long long xb[4]) {
  bool ready = true;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    av[u] = 0.0;
    xb[u] = (unsigned long long)__double_as_longlong(xprev);
    if (u0 + u < cnt) {
      av[u] = __longlong_as_double((long long)rec[32 * (3 + 2 * (u0 + u))]);
      const int code = (int)(unsigned)rec[32 * (4 + 2 * (u0 + u))];
      xb[u] = gs_src(code, win, a.xnew, a.xold, xprev);
    }
    ready &= gs_published(xb[u]);
  }
  return ready;
}

// Fast gather: <= C entries, all sourced from the previous row (code 0) or the
// shared window (code 1).  Straight-line; every load is predicated.
template <int C>
__device__ __forceinline__ bool gs_fast_gather(const volatile unsigned long long* win,
                                               const unsigned long long* rec, int cnt, double xprev,
                                               double av[4], double xv[4]) {
  bool ready = true;
#pragma unroll
  for (int u = 0; u < C; ++u) {
    const bool in = u < cnt;
    const unsigned code = in ? (unsigned)rec[32 * (4 + 2 * u)] : 0u;
    av[u] = in ? __longlong_as_double((long long)rec[32 * (3 + 2 * u)]) : 0.0;
    unsigned long long v = (unsigned long long)__double_as_longlong(xprev);
    if (code & 1u) v = win[code >> 2];
    ready &= gs_published(v);
    xv[u] = __longlong_as_double((long long)v);
  }
  return ready;
}

template <int C>
__device__ __forceinline__ double gs_fast_sum(double s, int cnt, const double av[4], const double xv[4]) {
#pragma unroll
  for (int u = 0; u < C; ++u)
    if (u < cnt) s = __dsub_rn(s, __dmul_rn(av[u], xv[u]));
  return s;
}

template <bool FWD, int R, int D>
__global__ void __launch_bounds__(256, 1) gs_sweep_kernel(GsArgs a) {
  extern __shared__ __align__(16) unsigned long long smem_u64[];
  __shared__ int s_tile;
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps_blk = blockDim.x >> 5;
  volatile unsigned long long* win = smem_u64;                             // window slots
  const int ring_off = ((a.window + 1) & ~1) + warp * D * a.slot_words;    // words
  const unsigned long long* ringp = smem_u64 + ring_off;
  const unsigned sbase = (unsigned)__cvta_generic_to_shared(smem_u64);
  const unsigned ring = sbase + 8u * (unsigned)ring_off;
  const unsigned bars = sbase + 8u * (unsigned)(((a.window + 1) & ~1) + nwarps_blk * D * a.slot_words) +
                        8u * (unsigned)(warp * D);
  if (lane == 0) {
#pragma unroll
    for (int d = 0; d < D; ++d) mbar_init(bars + 8u * d, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  unsigned parity = 0;  // bit d: parity of slot d's next completion
  const bool tracing = a.trace != nullptr;
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) s_tile = atomicAdd(a.ticket, 1);
    __syncthreads();
    const int tk = s_tile;
    if (tk >= a.ntiles) return;
    const int t = FWD ? tk : a.ntiles - 1 - tk;
    const int c0 = a.tile_ptr[t], c1 = a.tile_ptr[t + 1];
    const int TS = ((c1 - c0 + 31) / 32) * 32;  // window slot stride of this tile
    for (int i = threadIdx.x; i < a.window; i += blockDim.x) smem_u64[i] = kSentinel;
    __syncthreads();
    const int w0 = a.tile_wbase[t], nw = a.tile_wbase[t + 1] - w0;
    if (warp < nw) {
      const int g = w0 + warp;
      const int gr_base = a.tbase[g], nr = a.tbase[g + 1] - gr_base, nch = nr / R;
      const int cl = c0 + warp * 32 + lane;  // position in the chain order
      int cs = 0, len = 0;
      if (cl < c1) {
        const int c = a.chain_order ? a.chain_order[cl] : cl;
        cs = a.chain_ptr[c];
        len = a.chain_ptr[c + 1] - cs;
      }
      const int ce = cs + len;
      volatile unsigned long long* wslot = win + (cl - c0);  // + q * TS: this lane's published rows
      // chunk k (rounds [kR, kR+R)) -> slot k % D.  `ko` holds the chunk's round
      // offsets (lane j: round j), loaded a full ring cycle earlier, so issuing
      // never waits on memory.
      auto issue = [&](int k, int ko) {
        const int o0 = __shfl_sync(FULL, ko, 0), o1 = __shfl_sync(FULL, ko, R);
        if (lane == 0) {
          const int d = k % D;
          const int gr0 = gr_base + k * R;
          const unsigned rb = 8u * (unsigned)(o1 - o0), tb = 8u * 32u * R;
          const unsigned dst = ring + 8u * (unsigned)(d * a.slot_words);
          const unsigned bar = bars + 8u * d;
          mbar_expect_tx(bar, rb + tb);
          bulk_g2s(dst, a.rec + o0, rb, bar);
          bulk_g2s(dst + 8u * (unsigned)a.rec_words_max, a.tperm + (size_t)gr0 * 32, tb, bar);
        }
      };
      auto load_offs = [&](int k) { return (k < nch && lane <= R) ? a.round_off[gr_base + k * R + lane] : 0; };
      unsigned pend = 0;  // slots with a copy in flight (uniform across the warp)
      // offsets of chunks k .. k+2D-1 (lane j: round j of the chunk), shifted
      // down one place per chunk so the chunk loop needs no unrolling
      int oq[2 * D];
#pragma unroll
      for (int j = 0; j < 2 * D; ++j) oq[j] = load_offs(j);
#pragma unroll
      for (int d = 0; d < D; ++d) {
        if (d < nch) {
          issue(d, oq[d]);
          pend |= 1u << d;
        }
      }
      int q = 0;
      double xprev = 0.0;
      long long tr_spin = 0, tr_t0 = tracing ? clock64() : 0;
      bool abort = false;
#pragma unroll 1
      for (int k = 0; k < nch && !abort; ++k) {
        const int d = k % D;
        const unsigned long long* slot = ringp + d * a.slot_words;
        if (!(a.debug & 16)) while (!mbar_try_wait(bars + 8u * d, (parity >> d) & 1u)) {}
        parity ^= 1u << d;
        pend &= ~(1u << d);
        const int my_off = oq[0];
        const int o0 = __shfl_sync(FULL, my_off, 0);
        const double* tchunk = reinterpret_cast<const double*>(slot + a.rec_words_max) + lane;
#pragma unroll 1
        for (int rr = 0; rr < R; ++rr) {
          const int ob = __shfl_sync(FULL, my_off, rr), oe = __shfl_sync(FULL, my_off, rr + 1);
          const int cmax = ((oe - ob) / 32 - 3) / 2;  // uniform bound on this round's entries
          const unsigned long long* rec = slot + (ob - o0) + lane;
          const unsigned hw = (unsigned)rec[0];
          const int cnt = (int)(hw & 0xffffu);
          const bool active = cnt != (int)kGsNoRow;
          const int ca = active ? cnt : 0;
          double s = tchunk[rr * 32];
          long long spins = 0;
          const bool fastround = cmax <= 4 && __all_sync(FULL, !active || (hw & 0x10000u));
          if (fastround) {
            double av[4], xv[4];
            for (;;) {
              bool ready;
              if (cmax <= 2) ready = gs_fast_gather<2>(win, rec, ca, xprev, av, xv);
              else ready = gs_fast_gather<4>(win, rec, ca, xprev, av, xv);
              if (__all_sync(FULL, ready) || (a.debug & 1)) break;
              if ((++spins & 255) == 0) {
                bool ab = (*reinterpret_cast<volatile int*>(a.status) & ST_GS_TIMEOUT) != 0;
                if (spins > kGsIdleLimit) {
                  if (lane == 0) atomicOr(a.status, ST_GS_TIMEOUT);
                  ab = true;
                }
                if (__any_sync(FULL, ab)) { abort = true; break; }
              }
            }
            if (abort) break;
            if (cmax <= 2) s = gs_fast_sum<2>(s, ca, av, xv);
            else s = gs_fast_sum<4>(s, ca, av, xv);
          } else {
            double av[4];
            unsigned long long xb[4];
            for (;;) {  // the whole warp waits until every lane's row is ready
              bool ready = true;
              for (int u0 = 4; u0 < ca; u0 += 4) ready &= gs_gather4(a, win, rec, ca, u0, xprev, av, xb);
              ready &= gs_gather4(a, win, rec, ca, 0, xprev, av, xb);
              if (__all_sync(FULL, ready) || (a.debug & 1)) break;
              if ((++spins & 255) == 0) {
                bool ab = (*reinterpret_cast<volatile int*>(a.status) & ST_GS_TIMEOUT) != 0;
                if (spins > kGsIdleLimit) {
                  if (lane == 0) atomicOr(a.status, ST_GS_TIMEOUT);
                  ab = true;
                }
                if (__any_sync(FULL, ab)) { abort = true; break; }
              }
            }
            if (abort) break;
#pragma unroll
            for (int u = 0; u < 4; ++u)
              if (u < ca) s = __dsub_rn(s, __dmul_rn(av[u], __longlong_as_double((long long)xb[u])));
            for (int u0 = 4; u0 < ca; u0 += 4) {
              gs_gather4(a, win, rec, ca, u0, xprev, av, xb);  // published: ready
#pragma unroll
              for (int u = 0; u < 4; ++u)
                if (u0 + u < ca) s = __dsub_rn(s, __dmul_rn(av[u], __longlong_as_double((long long)xb[u])));
            }
          }
          tr_spin += spins;
          if (active) {
            const double xi = (a.debug & 8) ? s * __longlong_as_double((long long)rec[64])
                                            : div_rn_markstein(s, __longlong_as_double((long long)rec[32]),
                                                               __longlong_as_double((long long)rec[64]));
            const int i = FWD ? cs + q : ce - 1 - q;
            if (!(a.debug & 4)) wslot[(q & a.wmask) * TS] = (unsigned long long)__double_as_longlong(xi);
            if (!(a.debug & 2)) a.xnew[i] = xi;
            xprev = xi;
            ++q;
          }
          __syncwarp();
        }
        __syncwarp();
        if (!abort && k + D < nch) {
          issue(k + D, oq[D]);
          pend |= 1u << d;
        }
#pragma unroll
        for (int j = 0; j < 2 * D - 1; ++j) oq[j] = oq[j + 1];
        oq[2 * D - 1] = load_offs(k + 2 * D);
      }
      // an aborted sweep leaves copies in flight: land them before reuse / exit
      for (int d = 0; d < D; ++d) {
        if (pend & (1u << d)) {
          while (!mbar_try_wait(bars + 8u * d, (parity >> d) & 1u)) {}
          parity ^= 1u << d;
        }
      }
      if (tracing && lane == 0) {
        long long* tr = a.trace + 16 * (blockIdx.x * nwarps_blk + warp);
        tr[0] += nr; tr[1] += tr_spin; tr[5] += clock64() - tr_t0; tr[6] += 1;
      }
    }
  }
}


// Lean sweep for the common case (host-verified per level and mode): every row
// has <= C record entries, sourced from the previous row, the shared window or
// another tile's x_new -- no old values -- and every round has the same record
// size S = 3 + 2C (rows padded), so a chunk is a fixed R x 32 x S words and a
// record's position needs no lookup.  Sources are selected branch-free
// (predicated loads), and the R rounds of a chunk are unrolled so the next
// round's record and right-hand-side loads are issued ahead of the current
// round's dependent arithmetic.
// Predicated loads: the destination keeps its value when the predicate is off,
// so a source select is one instruction each and never a branch.
__device__ __forceinline__ void ld_shared_if(unsigned long long& v, bool p, unsigned saddr) {
  asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %1, 0;\n @q ld.volatile.shared.u64 %0, [%2];\n}"
               : "+l"(v) : "r"((unsigned)p), "r"(saddr));
}
__device__ __forceinline__ void ld_global_if(unsigned long long& v, bool p, const void* gaddr) {
  asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %1, 0;\n @q ld.relaxed.gpu.global.u64 %0, [%2];\n}"
               : "+l"(v) : "r"((unsigned)p), "l"(gaddr));
}

template <int C>
__device__ __forceinline__ bool gs_lean_gather(const unsigned long long* rec, int cnt, unsigned wbase,
                                               const double* xnew, double xprev, double av[C],
                                               double xv[C]) {
  bool ready = true;
#pragma unroll
  for (int u = 0; u < C; ++u) {
    const bool in = u < cnt;
    const unsigned code = in ? (unsigned)rec[32 * (4 + 2 * u)] : 0u;
    av[u] = in ? __longlong_as_double((long long)rec[32 * (3 + 2 * u)]) : 0.0;
    const unsigned t = code & 3u, idx = code >> 2;
    unsigned long long v = (unsigned long long)__double_as_longlong(xprev);
    ld_shared_if(v, t == 1u, wbase + 8u * idx);
    ld_global_if(v, t == 2u, xnew + idx);
    ready &= gs_published(v);
    xv[u] = __longlong_as_double((long long)v);
  }
  return ready;
}

// ---- thread-block-cluster tiles (GpuConfig.lean_cluster) ---------------------
// Consecutive tiles (in processing order) run as the CTAs of one cluster.  A
// source row in the previous tile of the same cluster is read from that CTA's
// shared-memory window over DSMEM instead of from x_new through L2; the
// schedule marks such sources with kGsRemote in the code's index (window slot).
constexpr unsigned kGsRemote = 1u << 28;
__device__ __forceinline__ unsigned lean_crank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned lean_cn() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void lean_csync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ unsigned lean_cmap(unsigned saddr, unsigned rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void ld_dsmem_if(unsigned long long& v, bool p, unsigned caddr) {
  asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %1, 0;\n @q ld.relaxed.cluster.shared::cluster.u64 %0, [%2];\n}"
               : "+l"(v) : "r"((unsigned)p), "r"(caddr));
}
// a cross-tile source: x_new through L2, or the previous tile's window over DSMEM
__device__ __forceinline__ void ld_cross_if(unsigned long long& v, bool p, unsigned idx, const double* xnew,
                                            unsigned prev_win) {
  const bool rem = (idx & kGsRemote) != 0u;
  ld_global_if(v, p && !rem, xnew + (idx & (kGsRemote - 1u)));
  ld_dsmem_if(v, p && rem, prev_win + 8u * (idx & (kGsRemote - 1u)));
}

// Records of at most this many entries per row use the half-chunk software
// pipeline of the lean kernel (staging of the next half overlaps the rounds).
#ifndef MVAMG_LEAN_PIPE_C
#define MVAMG_LEAN_PIPE_C 2
#endif

template <bool FWD, int C, int R, int D, int K = 1, bool CLU = false>
__global__ void __launch_bounds__(256, 1) gs_lean_kernel(GsArgs a) {
  constexpr int S = 3 + 2 * C;
  constexpr int RW = R * K * 32 * S;  // record words of one chunk (R rounds of K row slots)
  extern __shared__ __align__(16) unsigned long long smem_u64[];
  __shared__ int s_tile;
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps_blk = blockDim.x >> 5;
  volatile unsigned long long* win = smem_u64;
  const int ring_off = ((a.window + 1) & ~1) + warp * D * a.slot_words;
  const unsigned long long* ringp = smem_u64 + ring_off;
  const unsigned sbase = (unsigned)__cvta_generic_to_shared(smem_u64);
  const unsigned ring = sbase + 8u * (unsigned)ring_off;
  const unsigned bars = sbase + 8u * (unsigned)(((a.window + 1) & ~1) + nwarps_blk * D * a.slot_words) +
                        8u * (unsigned)(warp * D);
  if (lane == 0) {
#pragma unroll
    for (int d = 0; d < D; ++d) mbar_init(bars + 8u * d, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  unsigned parity = 0;
  // CLU: launched as thread-block clusters (a separate instantiation, so the
  // plain kernel keeps its register budget)
  const unsigned crank = CLU ? lean_crank() : 0u, cn = CLU ? lean_cn() : 1u;
  __shared__ int s_blk;
  for (;;) {
    __syncthreads();
    int tk;
    if (cn > 1) {
      // cluster mode: a ticket hands out a block of cn consecutive tiles; the
      // CTA of rank r takes tile block * cn + r.  The barriers also keep every
      // window alive until its readers in the cluster are done with it.
      lean_csync();
      if (threadIdx.x == 0 && crank == 0) s_blk = atomicAdd(a.ticket, 1);
      lean_csync();
      if (threadIdx.x == 0) {
        unsigned v;
        asm volatile("ld.shared::cluster.u32 %0, [%1];"
                     : "=r"(v) : "r"(lean_cmap((unsigned)__cvta_generic_to_shared(&s_blk), 0u)) : "memory");
        s_tile = (int)v * (int)cn + (int)crank;
      }
      __syncthreads();
      tk = s_tile;
      if (tk - (int)crank >= a.ntiles) return;  // the whole cluster is done
    } else {
      if (threadIdx.x == 0) s_tile = atomicAdd(a.ticket, 1);
      __syncthreads();
      tk = s_tile;
      if (tk >= a.ntiles) return;
    }
    const bool idle = tk >= a.ntiles;
    const int t = idle ? 0 : (FWD ? tk : a.ntiles - 1 - tk);
    const int c0 = a.tile_ptr[t], c1 = a.tile_ptr[t + 1];
    const int TS = ((c1 - c0 + 31) / 32) * 32;
    for (int i = threadIdx.x; i < a.window; i += blockDim.x) smem_u64[i] = kSentinel;
    __syncthreads();
    if (cn > 1) lean_csync();  // every window of the cluster is initialised before remote reads
    if (idle) continue;
    const unsigned prev_win = (CLU && cn > 1 && crank > 0) ? lean_cmap(sbase, crank - 1) : 0u;
    (void)prev_win;
    const int w0 = a.tile_wbase[t], nw = a.tile_wbase[t + 1] - w0;
    if (warp >= nw) continue;
    const int g = w0 + warp;
    const int gr_base = a.tbase[g], nch = (a.tbase[g + 1] - gr_base) / R;
    const int cl = c0 + warp * 32 + lane;  // position in the chain order
    int cs = 0, len = 0;
    if (cl < c1) {
      const int c = a.chain_order ? a.chain_order[cl] : cl;
      cs = a.chain_ptr[c];
      len = a.chain_ptr[c + 1] - cs;
    }
    const int ce = cs + len;
    volatile unsigned long long* wslot = win + (cl - c0);
    auto issue = [&](int k) {
      if (lane == 0) {
        const int d = k % D;
        const size_t gr0 = (size_t)gr_base + (size_t)k * R;
        const unsigned dst = ring + 8u * (unsigned)(d * a.slot_words);
        const unsigned bar = bars + 8u * d;
        mbar_expect_tx(bar, 8u * RW + 8u * 32u * R * K);
        bulk_g2s(dst, a.rec + gr0 * 32 * K * S, 8u * RW, bar);
        bulk_g2s(dst + 8u * RW, a.tperm + gr0 * 32 * K, 8u * 32u * R * K, bar);
      }
    };
    int issued = 0, consumed = 0;
    for (; issued < D && issued < nch; ++issued) issue(issued);
    int q = 0;
    double xprev = 0.0;
    bool abort = false;
    // One round: only the dependent part -- fresh window values, products,
    // the CSR-order subtraction chain, the division, the stores.  Absent
    // entries have a zero coefficient in the uniform record and a zero value:
    // s - (+0) == s exactly, so the chain needs no selects.  `tmr`, `ixr`,
    // `gvr` are the round's staged source types / indices / cross-tile values.
#if MVAMG_LEAN_TRACE
    int tr_round = 0;
#endif
    auto run_round = [&](const unsigned long long* slot, int rr, unsigned tmr, const unsigned* ixr,
                         const unsigned long long* gvr) {
      const unsigned long long* rec = slot + rr * 32 * S + lane;
      const double* rhs = reinterpret_cast<const double*>(slot + RW) + lane;
      const bool active = ((unsigned)rec[0] & 0xffffu) != kGsNoRow;
      double av[C], xv[C];
      bool ready = true;
#pragma unroll
      for (int u = 0; u < C; ++u) {
        const unsigned t = (tmr >> (2 * u)) & 3u;
        av[u] = __longlong_as_double((long long)rec[32 * (3 + 2 * u)]);
        unsigned long long v = t == 2u ? gvr[u] : (unsigned long long)__double_as_longlong(xprev);
        ld_shared_if(v, t == 1u, sbase + 8u * ixr[u]);
        ready &= t == 3u || gs_published(v);
        xv[u] = t == 3u ? 0.0 : __longlong_as_double((long long)v);
      }
      if (!__all_sync(FULL, ready)) {
        long long spins = 0;
        do {
#if MVAMG_LEAN_TRACE
          if (a.trace && g == (a.debug >> 8) && lane == 0) a.trace[16384 + 8192 + (tr_round & 4095)] += 1;
#endif
          ready = true;
#pragma unroll
          for (int u = 0; u < C; ++u) {
            const unsigned t = (tmr >> (2 * u)) & 3u;
            unsigned long long v = (unsigned long long)__double_as_longlong(xprev);
            ld_shared_if(v, t == 1u, sbase + 8u * ixr[u]);
            if constexpr (CLU) ld_cross_if(v, t == 2u, ixr[u], a.xnew, prev_win);
            else ld_global_if(v, t == 2u, a.xnew + ixr[u]);
            ready &= t == 3u || gs_published(v);
            xv[u] = t == 3u ? 0.0 : __longlong_as_double((long long)v);
          }
          if ((++spins & 255) == 0) {
            bool ab = (*reinterpret_cast<volatile int*>(a.status) & ST_GS_TIMEOUT) != 0;
            if (spins > kGsIdleLimit) {
              if (lane == 0) atomicOr(a.status, ST_GS_TIMEOUT);
              ab = true;
            }
            if (__any_sync(FULL, ab)) { abort = true; break; }
          }
        } while (!__all_sync(FULL, ready));
        if (abort) return;
      }
      double sacc = rhs[rr * 32];
#pragma unroll
      for (int u = 0; u < C; ++u) sacc = __dsub_rn(sacc, __dmul_rn(av[u], xv[u]));
      if (active) {
        const double xi = div_rn_markstein(sacc, __longlong_as_double((long long)rec[32]),
                                           __longlong_as_double((long long)rec[64]));
        wslot[(q & a.wmask) * TS] = (unsigned long long)__double_as_longlong(xi);
        a.xnew[FWD ? cs + q : ce - 1 - q] = xi;
        xprev = xi;
        ++q;
      }
      __syncwarp();
#if MVAMG_LEAN_TRACE
      if (a.trace && g == (a.debug >> 8) && lane == 0 && tr_round < 8192) a.trace[2 * tr_round + 1] = clock64();
      ++tr_round;
#endif
    };
    // Staging of rounds (independent of the sweep's progress): each entry's
    // source type and index, and the cross-tile values (code 2) requested at
    // once -- one L2 round trip per group of rounds, not per round.
    // Lean records come pre-decoded from mvamg_gs_schedule: the header's
    // bits 16-31 hold every entry's 2-bit source type (absent entries and
    // rows: 3), so staging is loads, shifts and the prefetches.
    auto load_codes = [&](const unsigned long long* slot, int rr, unsigned* code) {
      const unsigned long long* rec = slot + rr * 32 * S + lane;
      code[C] = (unsigned)(rec[0] >> 16);
#pragma unroll
      for (int u = 0; u < C; ++u) code[u] = (unsigned)rec[32 * (4 + 2 * u)];
    };
    auto decode = [&](const unsigned* code, unsigned& tmr, unsigned* ixr, unsigned long long* gvr) {
      tmr = code[C];
#pragma unroll
      for (int u = 0; u < C; ++u) {
        ixr[u] = code[u] >> 2;
        gvr[u] = kSentinel;
        if constexpr (CLU) ld_cross_if(gvr[u], ((tmr >> (2 * u)) & 3u) == 2u, ixr[u], a.xnew, prev_win);
        else ld_global_if(gvr[u], ((tmr >> (2 * u)) & 3u) == 2u, a.xnew + ixr[u]);
      }
    };
    auto wait_chunk = [&](int k) {
      const int d = k % D;
      while (!mbar_try_wait(bars + 8u * d, (parity >> d) & 1u)) {}
      parity ^= 1u << d;
      ++consumed;
    };
    if constexpr (K > 1) {
      // K consecutive rows of each lane's chain per round: every slot's
      // inputs except the chain predecessor come from earlier rounds, so all
      // of them are gathered at the round's start; the K short chains then
      // run back to back with the predecessor in a register.  Opt-in
      // (GpuConfig.lean_rows_per_round): measured slower on Q1 / 5-point
      // grids -- a row still costs ~420 cycles, and a lane can only start a
      // round once the lane above finished its whole round, which doubles
      // the line-to-line skew of the wavefront (tools/lean_trace.py).
#pragma unroll 1
      for (int k = 0; k < nch && !abort; ++k) {
        const unsigned long long* slot = ringp + (k % D) * a.slot_words;
        const double* rhs = reinterpret_cast<const double*>(slot + RW) + lane;
        wait_chunk(k);
        unsigned tmr[R * K], ixr[R * K][C], code[C + 1];
        unsigned long long gvr[R * K][C];
#pragma unroll
        for (int s = 0; s < R * K; ++s) {
          load_codes(slot, s, code);
          decode(code, tmr[s], ixr[s], gvr[s]);
        }
#pragma unroll
        for (int rr = 0; rr < R; ++rr) {
          double xv[K][C];
          bool ready = true;
#pragma unroll
          for (int kk = 0; kk < K; ++kk) {
            const int s = rr * K + kk;
#pragma unroll
            for (int u = 0; u < C; ++u) {
              const unsigned t = (tmr[s] >> (2 * u)) & 3u;
              unsigned long long v = t == 2u ? gvr[s][u] : 0ull;
              ld_shared_if(v, t == 1u, sbase + 8u * ixr[s][u]);
              ready &= t == 0u || t == 3u || gs_published(v);
              xv[kk][u] = __longlong_as_double((long long)v);
            }
          }
#if MVAMG_LEAN_TRACE
          long long nspin = 0;
#endif
          if (!__all_sync(FULL, ready)) {
            long long spins = 0;
            do {
#if MVAMG_LEAN_TRACE
              ++nspin;
#endif
              ready = true;
#pragma unroll
              for (int kk = 0; kk < K; ++kk) {
                const int s = rr * K + kk;
#pragma unroll
                for (int u = 0; u < C; ++u) {
                  const unsigned t = (tmr[s] >> (2 * u)) & 3u;
                  unsigned long long v = 0ull;
                  ld_shared_if(v, t == 1u, sbase + 8u * ixr[s][u]);
                  if constexpr (CLU) ld_cross_if(v, t == 2u, ixr[s][u], a.xnew, prev_win);
                  else ld_global_if(v, t == 2u, a.xnew + ixr[s][u]);
                  ready &= t == 0u || t == 3u || gs_published(v);
                  xv[kk][u] = __longlong_as_double((long long)v);
                }
              }
              if ((++spins & 255) == 0) {
                bool ab = (*reinterpret_cast<volatile int*>(a.status) & ST_GS_TIMEOUT) != 0;
                if (spins > kGsIdleLimit) {
                  if (lane == 0) atomicOr(a.status, ST_GS_TIMEOUT);
                  ab = true;
                }
                if (__any_sync(FULL, ab)) { abort = true; break; }
              }
            } while (!__all_sync(FULL, ready));
            if (abort) break;
          }
          // every slot's record fields before any store: the ring is read
          // through generic pointers the compiler cannot separate from the
          // x_new stores, so loads after a store would be serialised behind it
          double kav[K][C], krb[K], kdg[K], krd[K];
          bool kact[K];
#pragma unroll
          for (int kk = 0; kk < K; ++kk) {
            const int s = rr * K + kk;
            const unsigned long long* rec = slot + s * 32 * S + lane;
            kact[kk] = ((unsigned)rec[0] & 0xffffu) != kGsNoRow;
            krb[kk] = rhs[s * 32];
            kdg[kk] = __longlong_as_double((long long)rec[32]);
            krd[kk] = __longlong_as_double((long long)rec[64]);
#pragma unroll
            for (int u = 0; u < C; ++u) kav[kk][u] = __longlong_as_double((long long)rec[32 * (3 + 2 * u)]);
          }
#pragma unroll
          for (int kk = 0; kk < K; ++kk) {
            const int s = rr * K + kk;
            double sacc = krb[kk];
#pragma unroll
            for (int u = 0; u < C; ++u) {
              const unsigned t = (tmr[s] >> (2 * u)) & 3u;
              const double x = t == 0u ? xprev : xv[kk][u];
              sacc = __dsub_rn(sacc, __dmul_rn(kav[kk][u], x));
            }
            if (kact[kk]) {
              const double xi = div_rn_markstein(sacc, kdg[kk], krd[kk]);
              wslot[(q & a.wmask) * TS] = (unsigned long long)__double_as_longlong(xi);
              a.xnew[FWD ? cs + q : ce - 1 - q] = xi;
              xprev = xi;
              ++q;
            }
          }
          __syncwarp();
#if MVAMG_LEAN_TRACE
          if (a.trace && g == (a.debug >> 8) && lane == 0 && k * R + rr < 8192) {
            a.trace[2 * (k * R + rr) + 1] = clock64();
            a.trace[2 * (k * R + rr)] = nspin;
          }
#endif
        }
        if (abort) break;
        __syncwarp();
        if (k + D < nch) {
          issue(k + D);
          ++issued;
        }
      }
    } else if constexpr (R >= 4 && C <= MVAMG_LEAN_PIPE_C) {
      // Software-pipelined by half chunks (H rounds): while half h runs, the
      // codes of the next half are loaded (before its first round) and decoded
      // with their cross-tile prefetches (after it), so staging latency hides
      // behind the latency-bound rounds.  (Measured: a win for short records,
      // 5-point grids 339 -> 305 ns/level; for C = 4 the extra live state costs
      // more than it hides, so those stage whole chunks below.)
      constexpr int H = R / 2;
      unsigned tmA[H], ixA[H][C], tmB[H], ixB[H][C], raw[H][C + 1];
      unsigned long long gvA[H][C], gvB[H][C];
      if (nch > 0) {
        wait_chunk(0);
#pragma unroll
        for (int h = 0; h < H; ++h) {
          load_codes(ringp, h, raw[h]);
          decode(raw[h], tmA[h], ixA[h], gvA[h]);
        }
      }
#pragma unroll 1
      for (int k = 0; k < nch && !abort; ++k) {
        const unsigned long long* slot = ringp + (k % D) * a.slot_words;
        // half 0 (stage A); stage B = half 1 of this chunk
#pragma unroll
        for (int h = 0; h < H; ++h) load_codes(slot, H + h, raw[h]);
        run_round(slot, 0, tmA[0], ixA[0], gvA[0]);
        if (abort) break;
#pragma unroll
        for (int h = 0; h < H; ++h) decode(raw[h], tmB[h], ixB[h], gvB[h]);
#pragma unroll
        for (int h = 1; h < H; ++h) {
          run_round(slot, h, tmA[h], ixA[h], gvA[h]);
          if (abort) break;
        }
        if (abort) break;
        // half 1 (stage B); stage A = half 0 of the next chunk
        const bool more = k + 1 < nch;
        const unsigned long long* nslot = ringp + ((k + 1) % D) * a.slot_words;
        if (more) {
          wait_chunk(k + 1);
#pragma unroll
          for (int h = 0; h < H; ++h) load_codes(nslot, h, raw[h]);
        }
        run_round(slot, H, tmB[0], ixB[0], gvB[0]);
        if (abort) break;
        if (more) {
#pragma unroll
          for (int h = 0; h < H; ++h) decode(raw[h], tmA[h], ixA[h], gvA[h]);
        }
#pragma unroll
        for (int h = 1; h < H; ++h) {
          run_round(slot, H + h, tmB[h], ixB[h], gvB[h]);
          if (abort) break;
        }
        if (abort) break;
        __syncwarp();
        if (k + D < nch) {
          issue(k + D);
          ++issued;
        }
      }
    } else {
#pragma unroll 1
      for (int k = 0; k < nch && !abort; ++k) {
        const unsigned long long* slot = ringp + (k % D) * a.slot_words;
        wait_chunk(k);
        unsigned tmr[R], ixr[R][C], code[C + 1];
        unsigned long long gvr[R][C];
#pragma unroll
        for (int rr = 0; rr < R; ++rr) {
          load_codes(slot, rr, code);
          decode(code, tmr[rr], ixr[rr], gvr[rr]);
        }
#pragma unroll
        for (int rr = 0; rr < R; ++rr) {
          run_round(slot, rr, tmr[rr], ixr[rr], gvr[rr]);
          if (abort) break;
        }
        if (abort) break;
        __syncwarp();
        if (k + D < nch) {
          issue(k + D);
          ++issued;
        }
      }
    }
    // an aborted sweep leaves copies in flight: land them before reuse / exit
    for (; consumed < issued; ++consumed) {
      const int d = consumed % D;
      while (!mbar_try_wait(bars + 8u * d, (parity >> d) & 1u)) {}
      parity ^= 1u << d;
    }
  }
}

// Per-sweep preparation: the right-hand side in (round, lane) order -- for a
// backward sweep from a nonzero guess t_i = b_i - sum_{j<i} a_ij x_old_j in CSR
// order (exactly the serial loop's partial sum before the diagonal, since the
// j < i entries come first in a sorted row), otherwise t_i = b_i -- plus the
// sentinel fill of x_new and the tile-ticket reset.
__global__ void __launch_bounds__(256) gs_prepare_kernel(int n, const int* __restrict__ ip,
                                                         const int* __restrict__ ix,
                                                         const double* __restrict__ v,
                                                         const double* __restrict__ b,
                                                         const double* __restrict__ xold,
                                                         const int* __restrict__ perm, double* tperm,
                                                         double* xnew, int* ticket, int fold) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double s = __ldg(b + i);
    if (fold) {
      const int k1 = __ldg(ip + i + 1);
      for (int k = __ldg(ip + i); k < k1; ++k) {
        const int j = __ldg(ix + k);
        if (j >= i) break;
        s = __dsub_rn(s, __dmul_rn(__ldg(v + k), __ldg(xold + j)));
      }
    }
    tperm[perm ? __ldg(perm + i) : i] = s;
    reinterpret_cast<unsigned long long*>(xnew)[i] = kSentinel;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *ticket = 0;
}

// gs_prepare_kernel's backward fold with one warp per row (small levels with
// long rows, as spmv_warp_kernel): the lanes form the products of a 32-entry
// chunk of the row's j < i entries at once, then every lane subtracts them in
// CSR order from shuffles -- the same roundings in the same order.
__global__ void __launch_bounds__(256) gs_prepare_fold_warp_kernel(int n, const int* __restrict__ ip,
                                                                   const int* __restrict__ ix,
                                                                   const double* __restrict__ v,
                                                                   const double* __restrict__ b,
                                                                   const double* __restrict__ xold,
                                                                   const int* __restrict__ perm, double* tperm,
                                                                   double* xnew, int* ticket) {
  const int lane = threadIdx.x & 31;
  const int w0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (int i = w0; i < n; i += nw) {
    double s = __ldg(b + i);
    const int k0 = __ldg(ip + i), k1 = __ldg(ip + i + 1);
    for (int c = k0; c < k1; c += 32) {
      const int k = c + lane;
      const int j = k < k1 ? __ldg(ix + k) : 0x7fffffff;
      const bool lower = j < i;
      double pr = 0.0;
      if (lower) pr = __dmul_rn(__ldg(v + k), __ldg(xold + j));
      const int m = __popc(__ballot_sync(0xffffffffu, lower));  // sorted row: the lower entries lead
      for (int t = 0; t < m; ++t) s = __dsub_rn(s, __shfl_sync(0xffffffffu, pr, t));
      if (m < 32) break;
    }
    if (lane == 0) {
      tperm[perm ? __ldg(perm + i) : i] = s;
      reinterpret_cast<unsigned long long*>(xnew)[i] = kSentinel;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *ticket = 0;
}

}  // namespace mvamg

namespace mvamg {

// ---------------------------------------------------------------------------
// Small levels (n <= ~24k rows): one CTA, x resident in shared memory, rows in
// level-set order of the sweep's dependency DAG with one __syncthreads per
// level.  Shared x starts from x_old (or zero), so every entry of a row reads
// x[j] from shared memory: lower neighbours were finished in earlier levels,
// upper neighbours (same sweep, later levels) still hold x_old -- exactly the
// values the serial loop reads.  Each level's rows are contiguous in the
// host-built layout, so the whole CTA stages level l+2 with coalesced cp.async
// while it computes level l.
struct GsLevelRow {  // 32 bytes, level order
  int row, estart, cnt, pad;
  double diag, rdiag;
};
struct GsLevelEntry {  // 16 bytes, CSR order within the row
  double coef;
  int src, pad;
};

struct GsLevelArgs {
  int n, nlev, zero_init;
  int max_rows, max_ents;        // per (CTA, level)
  int rows_per_cta;              // row block owned by each CTA of the cluster
  const int* lev_ptr;            // per CTA: nlev + 1 row offsets (global layout), CTA-major
  const int* lev_eptr;           // per CTA: nlev + 1 entry offsets
  const GsLevelRow* rows;        // n, CTA-major then level order
  const GsLevelEntry* ents;      // entries; src = (owner CTA << 26) | local index
  const double* tperm;           // right-hand side in the rows' layout
  const double* xold;
  double* xnew;
};

__device__ __forceinline__ void cp_async16(unsigned dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned cluster_nctas() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ unsigned map_rank(unsigned saddr, unsigned rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ double ld_dsmem_f64(unsigned caddr) {
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(caddr) : "memory");
  return v;
}

// Small and mid-size levels: x resident in (distributed) shared memory, rows in
// level-set order of the sweep's dependency DAG, one barrier per level (a
// __syncthreads-equivalent cluster barrier across up to 16 CTAs of a thread
// block cluster; a cluster of one CTA is the single-CTA case).  Shared x starts
// from x_old (or zero), so every entry of a row reads x[j] from (distributed)
// shared memory: lower neighbours were finished in earlier levels, upper
// neighbours still hold x_old -- exactly what the serial loop reads.  Each
// (CTA, level) block of rows is contiguous in the host layout and is staged
// two levels ahead with coalesced cp.async.
// G == 1: one thread per row, CSR-order subtractions (bit-exact with the
// serial sweep).  G > 1 (tolerance parity, GpuConfig.exact_gs = False): G lanes
// per row, each summing a strided share of the row's products with FMAs, then
// an xor-shuffle tree; the row is final after cnt/G + log2(G) dependent steps
// instead of cnt.  The level order -- hence the GS dependency order -- is the
// same; only the rounding of each row's sum changes.
template <bool CLUSTER, int G>
__global__ void __launch_bounds__(1024, 1) gs_level_kernel(GsLevelArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const unsigned me = CLUSTER ? cluster_rank() : 0u, ncta = CLUSTER ? cluster_nctas() : 1u;
  double* x = reinterpret_cast<double*>(smem);
  const int xw = (a.rows_per_cta + 1) & ~1;
  const int rows_b = a.max_rows * 32, ents_b = a.max_ents * 16, rhs_b = (a.max_rows + 2) * 8;
  const int buf_b = rows_b + ents_b + ((rhs_b + 15) & ~15);
  unsigned char* bufs = smem + 8 * xw;
  const unsigned xs_local = (unsigned)__cvta_generic_to_shared(x);
  const unsigned bufs_s = (unsigned)__cvta_generic_to_shared(bufs);
  const int T = blockDim.x, tid = threadIdx.x;
  const int base = (int)me * a.rows_per_cta;
  const int nloc = max(0, min(a.rows_per_cta, a.n - base));
  for (int i = tid; i < nloc; i += T) x[i] = a.zero_init ? 0.0 : __ldg(a.xold + base + i);
  const int* lp = a.lev_ptr + (size_t)me * (a.nlev + 1);
  const int* le = a.lev_eptr + (size_t)me * (a.nlev + 1);
  auto stage = [&](int l) {
    if (l < a.nlev) {
      const int b = l % 3;
      const unsigned dst = bufs_s + (unsigned)(b * buf_b);
      const int r0 = __ldg(lp + l), r1 = __ldg(lp + l + 1);
      const int e0 = __ldg(le + l), e1 = __ldg(le + l + 1);
      const char* src = reinterpret_cast<const char*>(a.rows + r0);
      for (int c = tid; c < (r1 - r0) * 2; c += T) cp_async16(dst + 16u * c, src + 16 * c);
      const char* esrc = reinterpret_cast<const char*>(a.ents + e0);
      for (int c = tid; c < e1 - e0; c += T) cp_async16(dst + rows_b + 16u * c, esrc + 16 * c);
      const int t0 = r0 & ~1, t1 = (r1 + 1) & ~1;
      const char* tsrc = reinterpret_cast<const char*>(a.tperm + t0);
      for (int c = tid; c < (t1 - t0) / 2; c += T) cp_async16(dst + rows_b + ents_b + 16u * c, tsrc + 16 * c);
    }
    cp_async_commit();
  };
  stage(0);
  stage(1);
  if (CLUSTER) cluster_sync();  // every CTA's x slice is initialised before anyone reads it
  for (int l = 0; l < a.nlev; ++l) {
    cp_async_wait<1>();
    __syncthreads();
    stage(l + 2);
    const int b = l % 3;
    const unsigned char* bb = bufs + b * buf_b;
    const GsLevelRow* rows = reinterpret_cast<const GsLevelRow*>(bb);
    const GsLevelEntry* ents = reinterpret_cast<const GsLevelEntry*>(bb + rows_b);
    const double* rhs = reinterpret_cast<const double*>(bb + rows_b + ents_b);
    const int r0 = __ldg(lp + l), r1 = __ldg(lp + l + 1);
    const int e0 = __ldg(le + l), toff = r0 & 1;
    if constexpr (G > 1) {
      const int ngroups = T / G, g = tid / G, li = tid % G;
      const int nr = r1 - r0, iters = (nr + ngroups - 1) / ngroups;
      for (int it = 0; it < iters; ++it) {
        const int r = g + it * ngroups;
        const bool act = r < nr;
        double part = 0.0;
        GsLevelRow m;
        if (act) {
          m = rows[r];
          const GsLevelEntry* e = ents + (m.estart - e0);
          for (int k = li; k < m.cnt; k += G) {
            const GsLevelEntry en = e[k];
            double xv;
            if (CLUSTER) {
              const unsigned owner = (unsigned)en.src >> 26, loc = (unsigned)en.src & ((1u << 26) - 1);
              xv = ld_dsmem_f64(map_rank(xs_local + 8u * loc, owner));
            } else {
              xv = x[en.src];
            }
            part = __fma_rn(en.coef, xv, part);
          }
        }
#pragma unroll
        for (int off = G / 2; off > 0; off >>= 1) part = __dadd_rn(part, __shfl_xor_sync(0xffffffffu, part, off));
        if (act && li == 0) x[m.row - base] = div_rn_markstein(__dsub_rn(rhs[toff + r], part), m.diag, m.rdiag);
      }
      if (CLUSTER) cluster_sync();  // level l published cluster-wide
      continue;
    } else {
    for (int r = tid; r < r1 - r0; r += T) {
      const GsLevelRow m = rows[r];
      double s = rhs[toff + r];
      const GsLevelEntry* e = ents + (m.estart - e0);
      // chunks of 8: all loads and products first (independent), then the
      // subtractions in CSR order, one rounding each (bit-exact)
      for (int k0 = 0; k0 < m.cnt; k0 += 8) {
        double p[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          p[u] = 0.0;
          if (k0 + u < m.cnt) {
            const GsLevelEntry en = e[k0 + u];
            double xv;
            if (CLUSTER) {
              const unsigned owner = (unsigned)en.src >> 26, loc = (unsigned)en.src & ((1u << 26) - 1);
              xv = ld_dsmem_f64(map_rank(xs_local + 8u * loc, owner));
            } else {
              xv = x[en.src];
            }
            p[u] = __dmul_rn(en.coef, xv);
          }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (k0 + u < m.cnt) s = __dsub_rn(s, p[u]);
      }
      x[m.row - base] = div_rn_markstein(s, m.diag, m.rdiag);
    }
    if (CLUSTER) cluster_sync();  // level l published cluster-wide
    }
  }
  cp_async_wait<0>();
  __syncthreads();
  for (int i = tid; i < nloc; i += T) a.xnew[base + i] = x[i];
  if (CLUSTER) cluster_sync();  // no CTA leaves while others may still read its slice
  (void)ncta;
}


// Single-CTA level-set sweep, tolerance parity (group G > 1), for levels whose
// x fits in shared memory.  Entries are not staged through shared memory.
// A level runs in two phases.  (1) Every thread forms the products a_ij * x_j
// of up to kRegEnts of the level's entries (a level's entries are contiguous,
// so the loads are coalesced) into a shared product buffer.  Those entries
// were loaded into registers while the previous level computed, so their L2
// latency overlaps it.  (2) G lanes per row sum the row's products with a
// shuffle tree and write x_i.  Sub-levels hold at most blockDim * kRegEnts
// entries (the host splits larger levels).  The first row of each group's
// next level is prefetched the same way.
constexpr int kRegEnts = 8;
constexpr int kRegThreads = 512;

template <int G>
struct LevelRegStage {
  double c[kRegEnts];
  int s[kRegEnts];
  GsLevelRow m;
  double rhs;
  bool has;
};

template <int G>
__device__ __forceinline__ void level_reg_load(const GsLevelArgs& a, const int* lp, const int* le, int l, int tid,
                                               int g, LevelRegStage<G>& st) {
#pragma unroll
  for (int e = 0; e < kRegEnts; ++e) {
    st.c[e] = 0.0;
    st.s[e] = 0;
  }
  st.has = false;
  if (l >= a.nlev) return;
  const int e0 = le[l], e1 = le[l + 1];
#pragma unroll
  for (int e = 0; e < kRegEnts; ++e) {
    const int k = e0 + tid + e * kRegThreads;
    if (k < e1) {
      const GsLevelEntry en = a.ents[k];
      st.c[e] = en.coef;
      st.s[e] = en.src;
    }
  }
  const int p = lp[l] + g;
  if (p < lp[l + 1]) {
    st.m = a.rows[p];
    st.rhs = __ldg(a.tperm + p);
    st.has = true;
  }
}

template <int G>
__device__ __forceinline__ void level_reg_run(const GsLevelArgs& a, const int* lp, const int* le, int l, int tid,
                                              int g, int li, const LevelRegStage<G>& st, double* xsm, double* prod) {
  constexpr int ngroups = kRegThreads / G;
  const int e0 = le[l], ne = le[l + 1] - e0;
  const int r0 = lp[l], r1 = lp[l + 1];
  // phase 1: products of this level's entries (x of earlier levels is final)
#pragma unroll
  for (int e = 0; e < kRegEnts; ++e) {
    const int k = tid + e * kRegThreads;
    if (k < ne) prod[k] = __dmul_rn(st.c[e], xsm[st.s[e]]);
  }
  __syncthreads();
  // phase 2: row sums
  const int iters = (r1 - r0 + ngroups - 1) / ngroups;
  for (int it = 0; it < iters; ++it) {
    GsLevelRow mr;
    double rh = 0.0;
    bool act;
    if (it == 0) {
      mr = st.m;
      rh = st.rhs;
      act = st.has;
    } else {
      const int p = r0 + g + it * ngroups;
      act = p < r1;
      if (act) {
        mr = a.rows[p];
        rh = __ldg(a.tperm + p);
      }
    }
    double part = 0.0;
    if (act)
      for (int k = li; k < mr.cnt; k += G) part = __dadd_rn(part, prod[mr.estart - e0 + k]);
#pragma unroll
    for (int off = G / 2; off > 0; off >>= 1) part = __dadd_rn(part, __shfl_xor_sync(0xffffffffu, part, off));
    if (act && li == 0) xsm[mr.row] = div_rn_markstein(__dsub_rn(rh, part), mr.diag, mr.rdiag);
  }
  __syncthreads();
}

template <int G>
__global__ void __launch_bounds__(kRegThreads, 1) gs_level_reg_kernel(GsLevelArgs a) {
  extern __shared__ __align__(16) double xsm[];
  double* prod = xsm + ((a.n + 1) & ~1);
  // level offsets in shared memory: no L2 round trip at the head of a level
  int* lp = reinterpret_cast<int*>(prod + a.max_ents);
  int* le = lp + a.nlev + 1;
  const int tid = threadIdx.x;
  const int g = tid / G, li = tid % G;
  for (int i = tid; i < a.n; i += kRegThreads) xsm[i] = a.zero_init ? 0.0 : __ldg(a.xold + i);
  for (int i = tid; i <= a.nlev; i += kRegThreads) {
    lp[i] = a.lev_ptr[i];
    le[i] = a.lev_eptr[i];
  }
  __syncthreads();
  // three register stages: level l computes while l + 1 and l + 2 are in flight
  LevelRegStage<G> A, B, C;
  level_reg_load(a, lp, le, 0, tid, g, A);
  level_reg_load(a, lp, le, 1, tid, g, B);
  for (int l = 0; l < a.nlev; l += 3) {
    level_reg_load(a, lp, le, l + 2, tid, g, C);
    level_reg_run(a, lp, le, l, tid, g, li, A, xsm, prod);
    if (l + 1 >= a.nlev) break;
    level_reg_load(a, lp, le, l + 3, tid, g, A);
    level_reg_run(a, lp, le, l + 1, tid, g, li, B, xsm, prod);
    if (l + 2 >= a.nlev) break;
    level_reg_load(a, lp, le, l + 4, tid, g, B);
    level_reg_run(a, lp, le, l + 2, tid, g, li, C, xsm, prod);
  }
  for (int i = tid; i < a.n; i += kRegThreads) a.xnew[i] = xsm[i];
}


// ---------------------------------------------------------------------------
// Mid-size coarse levels (aggregation operators: 20-80 entries per row, DAG
// depth in the hundreds, no chain structure): dataflow, one thread per row,
// rows in topological (level, then longest-first) order handed out to CTAs by
// a ticket so every dependency lies in an earlier or the same ticket (no
// deadlock).  x_new itself is the ready flag (sentinel-filled by
// gs_prepare_kernel).  Each lane advances its row's CSR-order chain as far as
// its inputs are published -- the chain of a row is consumed eagerly while it
// waits, so when its last input lands only the tail is left -- and the warp
// loops until all 32 rows are final, which also makes same-warp dependencies
// safe.  Entries are stored as per-warp ELL slices (entry u of lane l at
// (wofs[w] + u) * 32 + l) so every load instruction is one coalesced segment.
struct GsRowArgs {
  int n, ntiles;
  const int* rowid;     // position -> row
  const int* cnt;       // position -> entries
  const int* crit;      // position -> (c1 | c2 << 16): entry of the latest input, and of one ~2
                        // levels earlier (0xffff = none); a lane waits on c2 before its first scan
  const int* wofs;      // warp -> first slice row (nwarps + 1)
  const double* coef;   // slices
  const int* src;       // slices: row of the value; bit 31 set = x_old (sweep from a nonzero guess)
  const double* dg;     // position -> diagonal
  const double* rdg;    // position -> RN(1 / diagonal)
  const double* tperm;  // position -> right-hand side (folded for backward sweeps from x_old)
  const double* xold;
  double* xnew;
  int* ticket;
  int* status;
  long long* trace;     // diagnostics: per position, %globaltimer when the row was published, then iterations
  int debug;            // > 0: nanosleep after a failed poll (ns)
  // row-partitioned (pipelined) sweeps: each final value is also stored into
  // the peers that read the row as a ghost -- mirror_dst[mirror_ptr[p]..] =
  // peer << 24 | slot, peers[peer] that rank's extended x -- and inputs are
  // polled at system scope (a peer GPU writes them over NVLink)
  const int* mirror_ptr;
  const unsigned* mirror_dst;
  double* const* peers;
  int sys;
};

__device__ __forceinline__ void ld_global_sys_if(unsigned long long& v, bool p, const void* gaddr) {
  asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %1, 0;\n @q ld.relaxed.sys.global.u64 %0, [%2];\n}"
               : "+l"(v) : "r"((unsigned)p), "l"(gaddr));
}
__device__ __forceinline__ void st_relaxed_sys_f64(double* p, double v) {
  asm volatile("st.relaxed.sys.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

__device__ __forceinline__ long long globaltimer_ns() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ void st_relaxed_f64(double* p, double v) {
  asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

// Per tile (blockDim.x consecutive positions) the warps' entry slices are
// staged into shared memory with cp.async.  Each lane then tracks the next 64
// entries of its row from the chain position kc with a done-mask: every
// iteration polls the first 8 still-pending entries (one L2 round trip), turns
// each published one into its product a_k * x_k in place of the coefficient
// (a product is its own rounding, independent of order), and runs the
// CSR-order subtraction chain over the done prefix.  Whichever input lands
// last (the first upper entry of a backward sweep, the last lower entry of a
// forward one), only the dependent subtractions remain when it does.  An
// iteration is ~200 instructions, so a lane re-polls every few hundred cycles.
template <bool OLD>
__global__ void __launch_bounds__(128) gs_row_kernel(GsRowArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int s_tile;
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int T = blockDim.x, nwb = T >> 5;
  const int nwarps = (a.n + 31) >> 5;
  const unsigned sbase = (unsigned)__cvta_generic_to_shared(smem);
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) s_tile = atomicAdd(a.ticket, 1);
    __syncthreads();
    const int tk = s_tile;
    if (tk >= a.ntiles) return;
    // stage the tile's slices: coef (8 B) then src (4 B) per entry
    const int w0 = tk * nwb, w1 = min(w0 + nwb, nwarps);
    const int sl0 = __ldg(a.wofs + w0), sl1 = __ldg(a.wofs + w1);
    const int nsl = sl1 - sl0;
    double* s_coef = reinterpret_cast<double*>(smem);
    int* s_src = reinterpret_cast<int*>(smem + (size_t)nsl * 256);
    {
      const char* gc = reinterpret_cast<const char*>(a.coef + (size_t)sl0 * 32);
      const char* gs = reinterpret_cast<const char*>(a.src + (size_t)sl0 * 32);
      for (int c = threadIdx.x; c < nsl * 16; c += T) cp_async16(sbase + 16u * c, gc + 16 * c);
      const unsigned ss = sbase + (unsigned)nsl * 256u;
      for (int c = threadIdx.x; c < nsl * 8; c += T) cp_async16(ss + 16u * c, gs + 16 * c);
      cp_async_commit();
    }
    const int p = tk * T + threadIdx.x;
    const bool have = p < a.n;
    int i = 0, cnt = 0, kc = 0, wsl = 0;
    double s = 0.0, dg = 1.0, rdg = 1.0;
    if (have) {
      i = __ldg(a.rowid + p);
      cnt = __ldg(a.cnt + p);
      s = __ldg(a.tperm + p);
      dg = __ldg(a.dg + p);
      rdg = __ldg(a.rdg + p);
    }
    if (w0 + warp < w1) wsl = __ldg(a.wofs + w0 + warp) - sl0;
    cp_async_wait<0>();
    __syncthreads();
    double* lc = s_coef + (size_t)wsl * 32 + lane;  // entry e of this lane at lc[32 e]
    const int* ls = s_src + (size_t)wsl * 32 + lane;
    bool done = !have;
    unsigned long long mask = 0;  // bit b: entry kc + b holds its product
    int sc = 4;                   // background cursor (relative to kc), past the fixed slots 1-3
    long long spins = 0, progress = 0;
    for (;;) {
      if (!done) {
        // slot 0 polls the chain's head (the entry blocking it, always
        // pending); slots 1-7 sweep the other pending entries of the 64-entry
        // window so products are formed while the head is awaited
        const int lim = min(cnt - kc, 64);
        int eb[8];
        double cf[8];
        unsigned long long xb[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          // slot 0: the head; slots 1-3: the entries right behind it (the
          // last to be published in a backward sweep, the next needed in a
          // forward one); slots 4-7: a cursor over the rest of the window
          const int b = u < 4 ? u : sc + u - 4;
          const bool v = b < lim && !((mask >> b) & 1ull);
          eb[u] = v ? b : -1;
          int j = 0;
          cf[u] = 0.0;
          if (v) {
            j = ls[32 * (kc + b)];
            cf[u] = lc[32 * (kc + b)];
          }
          const double* src = a.xnew + j;
          if (OLD && j < 0) src = a.xold + (j & 0x7fffffff);
          xb[u] = kSentinel;
          if (a.sys) ld_global_sys_if(xb[u], v, src);
          else ld_global_if(xb[u], v, src);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          if (eb[u] >= 0 && xb[u] != kSentinel) {
            lc[32 * (kc + eb[u])] = __dmul_rn(cf[u], __longlong_as_double((long long)xb[u]));
            mask |= 1ull << eb[u];
          }
        }
        const int m = min(lim, (~mask) ? __ffsll((long long)~mask) - 1 : 64);  // done prefix
        for (int t = 0; t < m; t += 4) {
          double pv[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) pv[q] = (t + q < m) ? lc[32 * (kc + t + q)] : 0.0;
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (t + q < m) s = __dsub_rn(s, pv[q]);
        }
        kc += m;
        mask = (m >= 64) ? 0ull : (mask >> m);
        // after progress, look right behind the new head (where the chain goes
        // next); while blocked, keep sweeping the window
        progress += m > 0;
        sc = m > 0 ? 4 : sc + 4;
        if (sc >= min(cnt - kc, 64)) sc = 4;
        if (kc == cnt) {
          const double xi = div_rn_markstein(s, dg, rdg);
          if (a.mirror_ptr) {  // peers that read this row as a ghost (pipelined row partition)
            const int m1 = __ldg(a.mirror_ptr + p + 1);
            for (int m = __ldg(a.mirror_ptr + p); m < m1; ++m) {
              const unsigned d = __ldg(a.mirror_dst + m);
              st_relaxed_sys_f64(a.peers[d >> 24] + (d & 0xffffffu), xi);
            }
          }
          if (a.sys) st_relaxed_sys_f64(a.xnew + i, xi);
          else st_relaxed_f64(a.xnew + i, xi);
          if (a.trace) {
            a.trace[p] = globaltimer_ns();
            a.trace[a.n + p] = progress;
          }
          done = true;
        }
      }
      if (__all_sync(FULL, done)) break;
      if ((++spins & 1023) == 0) {
        bool ab = (*reinterpret_cast<volatile int*>(a.status) & ST_GS_TIMEOUT) != 0;
        if (spins > kGsIdleLimit) {
          if (lane == 0) atomicOr(a.status, ST_GS_TIMEOUT);
          ab = true;
        }
        if (__any_sync(FULL, ab)) break;
      }
    }
  }
}

}  // namespace mvamg
