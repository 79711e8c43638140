// Gauss-Seidel in the reference's row order for levels without grid structure
// (the coarse levels; a fine level of interleaved dofs): dataflow with one warp
// per row and the critical dependency chain in shared memory.  Cluster form:
// the iterate in the distributed shared memory of ONE thread-block cluster
// (small levels).  Grid form: one CTA per SM, see below.
//
// The serial loop (pkg/src/mvamg/_kernels.py:15-38) makes row i wait for every
// x_new[j] it reads.  gs_row_kernel (gs_sweep.cuh) publishes and polls those
// values through L2: ~1.4 us per dependency level (C3 levels 1-4: depth
// 162-188, so 0.25-0.33 ms per sweep whatever the level's size).  Here the
// iterate lives in the cluster's shared memory -- position p of the
// topological order in a fixed slot of a fixed CTA -- so a row is published by
// one local st.shared and polled with ld.shared (own CTA, ~30 cycles) or
// ld.shared::cluster (a peer's slot): no L2 round trip on the critical path.
//
// Work split (mvamg_gs_cluster_plan): every row of the topological order is
// given to one of the cluster's G = NC x wpc worker warps (worker g = warp *
// NC + cta_rank), which takes its rows in increasing position.  A dependency
// always has a lower position, i.e. belongs to another worker's current or
// earlier row or to an earlier row of the same worker, and all workers are
// co-resident (one cluster): no deadlock.  The plan puts a row on the CTA that
// owns its latest input whenever that CTA's share of the DAG level allows, so
// the poll a row's completion hangs on is mostly a local shared-memory load.
//
// One row at a time per warp, lanes = entries.  The plan orders a row's
// entries by the DAG level at which their inputs become final and splits off
// the last (up to) kClusterLate of them:
//   early entries   one per lane (two chunks of 32 in flight): polled once,
//                   usually landed; lane-local FMAs, then a fixed xor-shuffle tree;
//   late entries    (the last level's inputs, at most kClusterLate, the critical
//                   one last) polled by lane 0 alone in a tight loop -- ld.shared
//                   when the input lives in this CTA, as the plan mostly arranges
//                   -- which then finishes the row: s = (b - early) - a1 x1 - a2 x2 ...,
//                   the division (Markstein) and the publishing stores.
// A sweep from a nonzero guess reads its x_old entries (sorted first) straight
// from global memory in the early phase: no separate fold pass.
// So after a row's last input lands its own value is one (mostly local) load
// plus a few dependent FP64 operations away, and a waiting warp costs one
// lane's polls (DSMEM moves only ~17 B/cycle per SM).
//
// Data: a worker's rows are consumed strictly in order, so the plan packs them
// into that worker's own sequence of fixed-size pages (row records: header,
// coefficients, sources; no record straddles a page) and the warp streams the
// pages through a private ring of shared-memory buffers with TMA bulk copies
// (cp.async.bulk + mbarrier), kClusterRing pages ahead: a row's data is an
// LDS away when its turn comes, never a global-memory round trip.  The right-
// hand sides (written per sweep by gs_prepare_kernel in the same q order) are
// read 32 rows at a time, one per lane, and handed out by shuffle.
//
// Grid form (GRID = true; levels too large or too wide for one cluster): the
// same workers on ordinary CTAs, one per SM over the whole GPU.  Only the
// critical chain stays in shared memory -- a late input owned by the row's own
// CTA is still an ld.shared poll -- while early inputs (a level or more old,
// so latency-tolerant) and the few late inputs of other CTAs are polled in
// x_new through L2 like gs_row_kernel's (gs_prepare_kernel fills it with the
// sentinel).  That removes the cluster's limits -- 16 SMs, and their DSMEM
// request rate (~0.3 remote loads per cycle and SM, which bounds the cluster
// form from ~15k rows up) -- at the price of an L2 round trip per early chunk.
// All CTAs must be resident (grid <= SMs), as for gs_row_kernel.
//
// Rounding: fixed per plan (tree + ordered tail), so results are reproducible
// run to run, but not the serial loop's CSR-order roundings: this kernel
// serves tolerance parity (GpuConfig.exact_gs = False); exact mode keeps the
// CSR-order kernels of gs_sweep.cuh / gs_stream.cuh.
#pragma once
#include "gs_sweep.cuh"

namespace mvamg {

constexpr int kClusterLate = 4;    // late entries per row (lane 0)
constexpr int kClusterRing = 2;    // pages in flight per worker warp
constexpr int kClusterRowHdr = 32; // bytes: int cnt, ne, row, slot; double dg, rdg
constexpr int kClusterPageHdr = 16; // bytes: int nrows, pad

// bytes of one row record: header, cnt coefficients, cnt sources (padded to 16: aligned vector loads)
__host__ __device__ inline int cluster_row_bytes(int cnt) { return (kClusterRowHdr + 12 * cnt + 15) & ~15; }

struct GsClusterArgs {
  int n;                 // rows; q = a row's index in worker-major storage
  int wpc;               // worker warps per CTA
  int slots;             // x slots (8 B) per CTA
  int page_bytes;        // bytes per page (multiple of 128)
  const int* wptr;       // worker -> first q (NC * wpc + 1)
  const int* wpage;      // worker -> first page (NC * wpc + 1)
  const unsigned char* blob;  // pages; sources: cluster form cta << 24 | slot; grid form the row (late entries: bit
                         // 30 | slot when the row's own CTA owns the input); bit 31 | row: an x_old value
  const double* tperm;   // q -> right-hand side (folded for backward sweeps from x_old)
  const double* xold;
  double* xnew;
  int* status;
  long long* trace;      // diagnostics, 3 n: per q clock64 at the row's start, at publish, after the early polls
  int sleep_ns;          // back-off of a warp whose early poll found nothing new
};

__device__ __forceinline__ double lds_f64(unsigned saddr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(saddr));
  return v;
}
__device__ __forceinline__ unsigned lds_u32(unsigned saddr) {
  unsigned v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(saddr));
  return v;
}

// Publishing store and polls: an aligned 8-byte value is written at once and
// is its own ready flag.  The CTA's own slots are polled with ld.volatile.shared
// (LDS, ~30 cycles); other CTAs' with ld.relaxed.cluster.shared::cluster (a
// generic LD.STRONG, a few hundred cycles -- a weak ld.shared::cluster is
// faster but was measured to miss the peer's update for good: it may be served
// from L1).
__device__ __forceinline__ void st_shared_f64(unsigned saddr, double v) {
  asm volatile("st.volatile.shared.f64 [%0], %1;" ::"r"(saddr), "d"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_cluster_u64(unsigned caddr) {
  unsigned long long v;
  asm volatile("ld.relaxed.cluster.shared::cluster.u64 %0, [%1];" : "=l"(v) : "r"(caddr) : "memory");
  return v;
}

template <bool OLD, bool GRID>
__global__ void __launch_bounds__(1024, 1) gs_cluster_kernel(GsClusterArgs a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  constexpr int NB = kClusterRing;
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned NC = GRID ? gridDim.x : cluster_nctas(), cr = GRID ? blockIdx.x : cluster_rank();
  unsigned long long* xs = reinterpret_cast<unsigned long long*>(smem_raw);
  const unsigned xbase = (unsigned)__cvta_generic_to_shared(xs);
  const unsigned xbytes = ((unsigned)a.slots * 8u + 127u) & ~127u;
  const unsigned PAGE = (unsigned)a.page_bytes;
  const unsigned ring = xbase + xbytes + (unsigned)(warp * NB) * PAGE;
  const unsigned bars = xbase + xbytes + (unsigned)(a.wpc * NB) * PAGE + 8u * (unsigned)(warp * NB);
  for (int i = threadIdx.x; i < a.slots; i += blockDim.x) xs[i] = kSentinel;
  if (lane == 0) {
    for (int b = 0; b < NB; ++b) mbar_init(bars + 8u * b, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (GRID) __syncthreads();  // the slice is only ever read by this CTA
  else cluster_sync();        // every slice holds the sentinel before any remote poll
  const int g = warp * (int)NC + (int)cr;
  bool abort = false;
  // a poll that has failed kGsIdleLimit times (or another warp's) ends the sweep with ST_GS_TIMEOUT
  auto timed_out = [&](unsigned& spins) -> bool {
    if ((++spins & 1023u) != 0u) return false;
    if (spins > (unsigned)kGsIdleLimit) atomicOr(a.status, ST_GS_TIMEOUT);
    return (*reinterpret_cast<volatile int*>(a.status) & ST_GS_TIMEOUT) != 0;
  };
  const int q0 = __ldg(a.wptr + g), q1 = __ldg(a.wptr + g + 1);
  const int pg0 = __ldg(a.wpage + g), pg1 = __ldg(a.wpage + g + 1);
  auto fetch = [&](int pg, int b) {  // lane 0: page pg into ring buffer b
    mbar_expect_tx(bars + 8u * b, PAGE);
    bulk_g2s(ring + (unsigned)b * PAGE, a.blob + (size_t)pg * PAGE, PAGE, bars + 8u * b);
  };
  if (lane == 0)
    for (int b = 0; b < NB; ++b)
      if (pg0 + b < pg1) fetch(pg0 + b, b);
  // right-hand sides of 32 consecutive rows, one per lane, a block ahead
  int qb = q0;
  double rr = qb + lane < q1 ? __ldg(a.tperm + qb + lane) : 0.0;
  double rn = qb + 32 + lane < q1 ? __ldg(a.tperm + qb + 32 + lane) : 0.0;
  int q = q0;
  for (int pg = pg0, it = 0; pg < pg1 && !abort; ++pg, ++it) {
    const int b = it % NB;
    {
      const unsigned par = (unsigned)(it / NB) & 1u;
      while (!mbar_try_wait(bars + 8u * b, par)) {}
    }
    const unsigned page = ring + (unsigned)b * PAGE;
    const int nrows = (int)lds_u32(page);
    unsigned off = page + kClusterPageHdr;
    for (int r = 0; r < nrows && !abort; ++r, ++q) {
      if (a.trace && lane == 0) a.trace[q] = clock64();
      int cnt, ne, row, slot;
      asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(cnt), "=r"(ne), "=r"(row), "=r"(slot) : "r"(off));
      double dg, rdg;
      asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(dg), "=d"(rdg) : "r"(off + 16u));
      const unsigned cbase = off + kClusterRowHdr, sbase = cbase + 8u * (unsigned)cnt;
      // the publishing addresses, formed now and pinned in registers: nothing but the last input's
      // FMA, the division and the two stores is left between that input's arrival and the publish
      unsigned my_saddr = xbase + 8u * (unsigned)slot;
      double* my_gaddr = a.xnew + row;
      asm volatile("" : "+r"(my_saddr));
      asm volatile("" : "+l"(my_gaddr));
      if (q - qb == 32) {
        qb += 32;
        rr = rn;
        rn = qb + 32 + lane < q1 ? __ldg(a.tperm + qb + 32 + lane) : 0.0;
      }
      const double rhs = __shfl_sync(FULL, rr, q - qb);
      // ---- early entries: one per lane, two chunks of 32 in flight together -----------
      double sum = 0.0;
      unsigned spins = 0;
      for (int base = 0; base < ne; base += 64) {
        double cf[2];
        unsigned long long v[2];
        unsigned ad[2];
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const int idx = base + 32 * c + lane;
          cf[c] = 0.0;
          v[c] = 0ull;
          ad[c] = xbase;
          if (idx < ne) {
            cf[c] = lds_f64(cbase + 8u * (unsigned)idx);
            const unsigned sc = lds_u32(sbase + 4u * (unsigned)idx);
            if (OLD && (sc >> 31)) {
              v[c] = (unsigned long long)__double_as_longlong(__ldg(a.xold + (sc & 0x7fffffffu)));
            } else {
              v[c] = kSentinel;
              if (GRID) {
                ad[c] = sc & 0x3fffffffu;
              } else {  // bit 0 of the address: a slot of this CTA (ld.shared instead of the cluster load)
                const unsigned ct = (sc >> 24) & 15u, la = xbase + 8u * (sc & 0xffffffu);
                ad[c] = ct == cr ? (la | 1u) : map_rank(la, ct);
              }
            }
          }
        }
        for (;;) {
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            if (gs_published(v[c])) continue;
            if (GRID) v[c] = ld_relaxed_u64(a.xnew + ad[c]);
            else if (ad[c] & 1u) v[c] = ld_shared_volatile_u64(ad[c] & ~1u);
            else v[c] = ld_cluster_u64(ad[c]);
          }
          if (!__any_sync(FULL, !gs_published(v[0]) || !gs_published(v[1]))) break;
          if (a.sleep_ns > 0) __nanosleep((unsigned)a.sleep_ns);
          if (__any_sync(FULL, timed_out(spins))) { abort = true; break; }
        }
#pragma unroll
        for (int c = 0; c < 2; ++c) sum = fma(cf[c], __longlong_as_double((long long)v[c]), sum);
      }
      if (a.trace && lane == 0) a.trace[2 * (size_t)a.n + q] = clock64();
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(FULL, sum, o);
      // ---- late entries and the row's completion: lane 0 alone, tight polls ------
      if (lane == 0 && !abort) {
        double s = rhs - sum;
        for (int k = ne; k < cnt; ++k) {
          const double lc = lds_f64(cbase + 8u * (unsigned)k);
          const unsigned sc = lds_u32(sbase + 4u * (unsigned)k);
          unsigned long long v;
          if (OLD && (sc >> 31)) {
            v = (unsigned long long)__double_as_longlong(__ldg(a.xold + (sc & 0x7fffffffu)));
          } else if (GRID ? (sc >> 30) != 0u : ((sc >> 24) & 15u) == cr) {  // the usual case: this CTA's input
            const unsigned ad = xbase + 8u * (sc & 0xffffffu);
            while (!gs_published(v = ld_shared_volatile_u64(ad)))
              if (timed_out(spins)) { abort = true; break; }
          } else if (GRID) {
            const double* ad = a.xnew + (sc & 0x3fffffffu);
            while (!gs_published(v = ld_relaxed_u64(ad)))
              if (timed_out(spins)) { abort = true; break; }
          } else {
            const unsigned ad = map_rank(xbase + 8u * (sc & 0xffffffu), (sc >> 24) & 15u);
            while (!gs_published(v = ld_cluster_u64(ad)))
              if (timed_out(spins)) { abort = true; break; }
          }
          s = fma(-lc, __longlong_as_double((long long)v), s);
        }
        if (!abort) {
          const double xi = div_rn_markstein(s, dg, rdg);
          if (!GRID || slot >= 0) st_shared_f64(my_saddr, xi);  // grid form: only if polled here
          if (GRID) st_relaxed_f64(my_gaddr, xi);  // polled by other CTAs
          else *my_gaddr = xi;
          if (a.trace) a.trace[(size_t)a.n + q] = clock64();
        }
      }
      abort = __any_sync(FULL, abort);
      off += (unsigned)cluster_row_bytes(cnt);
    }
    // the page is consumed: bring the page NB ahead into its buffer
    __syncwarp();
    if (lane == 0 && pg + NB < pg1) fetch(pg + NB, b);
  }
  if (!GRID) cluster_sync();  // no CTA leaves while a peer may still poll its slice
}

}  // namespace mvamg
