// gs_stream.cuh -- exact-order Gauss-Seidel sweep of a coarse level on one SM
// or one thread-block cluster, level packets streamed by TMA.
//
// Reference: gs_forward / gs_backward (pkg/src/mvamg/_kernels.py:15-38).  The
// serial loop's result depends only on its dependency DAG (row i reads the new
// x_j of every row j it couples to that comes earlier in the sweep), so the
// rows can run in level-set order of that DAG: a batch of mutually independent
// rows, a barrier, the next batch.
//
// Coarse multi-vector levels (C3: 250-160k rows, 20-76 entries per row, DAG
// depth 50-190) are latency bound: one dependent step per DAG level.  Here x
// (and, for a single-SM sweep from a nonzero guess, b) live in shared memory
// -- for a cluster of C CTAs, CTA c holds rows [c R, (c+1) R) and reads the
// others' rows over DSMEM -- so a step costs a barrier plus one row's
// shared-memory reads and arithmetic; the matrix is the only thing streamed
// from HBM/L2.  The host packs the batches, in sweep order, into stages of at
// most `slot_bytes` per CTA (every CTA's stage s holds its rows of the same
// batches); one thread per CTA keeps NS stages in flight with cp.async.bulk
// into a shared-memory ring (one mbarrier per slot), so the stream's latency
// hides behind NS - 1 stages of computation.
//
// Stage blob of one CTA (16-B aligned, offsets relative to its start):
//   [0, 16)            u32 nbatch, u32 nrows, u32 nents, u32 0
//   [16, 16 + 8 nb)    per batch: u32 row_begin (stage row index), u32 nrows
//   rows (16-aligned)  GsStreamRow x nrows, batch order
//   coef (16-aligned)  f64 x nents, per row in CSR order
//   src  (16-aligned)  u32 x nents: column j (one CTA) or owner << 24 | local
// Rows hold the entries the sweep still reads, diagonal excluded: a sweep
// from x = 0 keeps only its dependency side (j < i forward, j > i backward);
// a single-SM sweep from x_old keeps every off-diagonal entry, the other side
// reading x_old from shared memory -- exactly the values the serial loop
// reads.  (Cluster plans are zero-guess only; a backward sweep from x_old
// folds its old lower neighbours into b first, gs_prepare_kernel.)
//
// G == 1: one thread per row, CSR-order subtractions, one rounding each
// (bit-exact with the serial sweep).  G > 1 (tolerance parity): G lanes per
// row, strided FMA partial sums and an xor-shuffle tree; the DAG order is the
// same, only the rounding of each row's sum changes (as gs_level_kernel).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace mvamg {

struct GsStreamRow {  // 32 bytes
  unsigned row, cnt, ebeg, pad;  // row: local index in the owning CTA's slice
  double diag, rdiag;
};

constexpr int kStreamThreads = 256;

struct GsStreamArgs {
  int n;
  int with_old;                  // 1: x starts at x_old, b kept separately; 0: x starts at b (x = 0 guess)
  int nstages, nslots, slot_bytes;
  int rows_per_cta;              // slice of x held by each CTA (n for one CTA)
  const unsigned char* blob;     // stages, 16-B aligned
  const long long* stage_off;    // nstages * ncta + 1 byte offsets, stage-major
  const double* b;
  const double* xold;
  double* xnew;
  long long* trace;              // diagnostics (nullptr: off): CTA 0's clock64 per stage wait / batch
  int trace_cap;
};

__device__ __forceinline__ void gss_mbar_init(unsigned bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void gss_expect_tx(unsigned bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void gss_bulk_g2s(unsigned dst, const void* src, unsigned bytes, unsigned bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}
__device__ __forceinline__ void gss_wait(unsigned bar, unsigned parity) {
  unsigned ok = 0;
  while (!ok) {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                 : "=r"(ok) : "r"(bar), "r"(parity) : "memory");
  }
}
__device__ __forceinline__ unsigned gss_crank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned gss_cn() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void gss_csync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ unsigned gss_mapa(unsigned saddr, unsigned rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ double gss_ld_dsmem(unsigned caddr) {
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(caddr) : "memory");
  return v;
}

template <int G, bool CLU>
__global__ void __launch_bounds__(kStreamThreads, 1) gs_stream_kernel(GsStreamArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ __align__(8) unsigned long long bars[8];
  constexpr int T = kStreamThreads, NG = T / G;
  const int tid = threadIdx.x;
  const unsigned me = CLU ? gss_crank() : 0u, ncta = CLU ? gss_cn() : 1u;
  const int base = (int)me * a.rows_per_cta;
  const int nloc = max(0, min(a.rows_per_cta, a.n - base));
  double* x = reinterpret_cast<double*>(smem);
  const int xw = (a.rows_per_cta + 1) & ~1;
  double* bs = a.with_old ? x + xw : x;          // right-hand side (x itself when starting from zero)
  unsigned char* ring = smem + 8 * xw * (a.with_old ? 2 : 1);
  const unsigned x_s = (unsigned)__cvta_generic_to_shared(x);
  const unsigned ring_s = (unsigned)__cvta_generic_to_shared(ring);
  const unsigned bar_s = (unsigned)__cvta_generic_to_shared(bars);
  const long long* soff = a.stage_off + me;    // stage s of this CTA: soff[s * ncta]
  auto issue = [&](int s, int slot) {           // thread 0: stage s into `slot`
    if (s < a.nstages) {
      const long long off = soff[(size_t)s * ncta];
      const unsigned bytes = (unsigned)(a.stage_off[(size_t)s * ncta + me + 1] - off);
      gss_expect_tx(bar_s + 8u * slot, bytes);
      gss_bulk_g2s(ring_s + (unsigned)slot * (unsigned)a.slot_bytes, a.blob + off, bytes, bar_s + 8u * slot);
    }
  };
  if (tid == 0) {
    for (int q = 0; q < a.nslots; ++q) gss_mbar_init(bar_s + 8u * q, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int s = 0; s < a.nslots; ++s) issue(s, s);
  }
  if (a.with_old) {
    for (int i = tid; i < nloc; i += T) {
      x[i] = __ldg(a.xold + base + i);
      bs[i] = __ldg(a.b + base + i);
    }
  } else {
    for (int i = tid; i < nloc; i += T) x[i] = __ldg(a.b + base + i);
  }
  if (CLU) gss_csync();  // every slice is initialised before anyone reads it
  else __syncthreads();
  // x_j: a local slice entry, or (cluster) owner << 24 | local over DSMEM
  auto xval = [&](unsigned j) -> double {
    if constexpr (CLU) {
      const unsigned own = j >> 24, loc = j & 0xffffffu;
      if (own == me) return x[loc];
      return gss_ld_dsmem(gss_mapa(x_s + 8u * loc, own));
    } else {
      return x[j];
    }
  };
  const int g = tid / G, li = tid % G;
  const bool tr = a.trace != nullptr && tid == 0 && me == 0;
  int tn = 1;
  auto stamp = [&](long long tag) {
    if (tr && tn + 1 < a.trace_cap) {
      a.trace[tn++] = tag;
      a.trace[tn++] = clock64();
    }
  };
  stamp(-1);
  // ---- batch cursor over the ring: the next batch's metadata (row header,
  // this lane's first KE coefficients and columns) is read from shared memory
  // while the current batch's barrier settles, so a DAG level's critical path
  // is only the x loads, the products, the sum and the division ----
  constexpr int KE = 8;
  struct Item {
    const GsStreamRow* rows;
    const double* coef;
    const unsigned* src;
    int r0, rn;
    bool act;
    GsStreamRow m;
    double c[KE];
    unsigned j[KE];
  };
  auto fetch = [&](const unsigned char* st, int bt, Item& it) {
    const unsigned* hdr = reinterpret_cast<const unsigned*>(st);
    const int nb = (int)hdr[0], nr = (int)hdr[1], ne = (int)hdr[2];
    const int rows_off = (16 + 8 * nb + 15) & ~15;
    const int coef_off = rows_off + 32 * nr;
    const int src_off = (coef_off + 8 * ne + 15) & ~15;
    it.rows = reinterpret_cast<const GsStreamRow*>(st + rows_off);
    it.coef = reinterpret_cast<const double*>(st + coef_off);
    it.src = reinterpret_cast<const unsigned*>(st + src_off);
    it.r0 = (int)hdr[4 + 2 * bt];
    it.rn = (int)hdr[5 + 2 * bt];
    it.act = g < it.rn;
    if (it.act) {
      it.m = it.rows[it.r0 + g];
      const int cnt = (int)it.m.cnt;
#pragma unroll
      for (int u = 0; u < KE; ++u) {
        const int k = (G == 1) ? u : li + u * G;
        it.c[u] = 0.0;
        it.j[u] = 0u;
        if (k < cnt) {
          it.c[u] = it.coef[it.m.ebeg + k];
          it.j[u] = it.src[it.m.ebeg + k];
        }
      }
    }
  };
  // one row (group g, lanes li) of a batch; pre: entries 0..KE-1 of this lane prefetched
  auto do_row = [&](bool act, const GsStreamRow& m, const double* c0, const unsigned* j0, const double* coef,
                    const unsigned* src) {
    const int cnt = act ? (int)m.cnt : 0;
    if constexpr (G == 1) {
      if (!act) return;
      // CSR order, one rounding per multiply and subtract (bit-exact)
      double sacc = bs[m.row];
      double xv[KE];
#pragma unroll
      for (int u = 0; u < KE; ++u) xv[u] = u < cnt ? xval(j0[u]) : 0.0;
#pragma unroll
      for (int u = 0; u < KE; ++u)
        if (u < cnt) sacc = __dsub_rn(sacc, __dmul_rn(c0[u], xv[u]));
      const double* c = coef + m.ebeg;
      const unsigned* sj = src + m.ebeg;
      for (int k0 = KE; k0 < cnt; k0 += 8) {
        double p[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) p[u] = (k0 + u < cnt) ? __dmul_rn(c[k0 + u], xval(sj[k0 + u])) : 0.0;
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (k0 + u < cnt) sacc = __dsub_rn(sacc, p[u]);
      }
      x[m.row] = div_rn_markstein(sacc, m.diag, m.rdiag);
    } else {
      double xv[KE];
#pragma unroll
      for (int u = 0; u < KE; ++u) xv[u] = (li + u * G < cnt) ? xval(j0[u]) : 0.0;
      double q0 = 0.0, q1 = 0.0;  // two accumulation chains (absent entries add +0)
#pragma unroll
      for (int u = 0; u < KE; u += 2) {
        q0 = __fma_rn(c0[u], xv[u], q0);
        q1 = __fma_rn(c0[u + 1], xv[u + 1], q1);
      }
      const double* c = coef + m.ebeg;
      const unsigned* sj = src + m.ebeg;
      for (int k = li + KE * G; k < cnt; k += G) q0 = __fma_rn(c[k], xval(sj[k]), q0);
      double part = __dadd_rn(q0, q1);
#pragma unroll
      for (int off = G / 2; off > 0; off >>= 1)
        part = __dadd_rn(part, __shfl_xor_sync(0xffffffffu, part, off, G));
      if (act && li == 0) x[m.row] = div_rn_markstein(__dsub_rn(bs[m.row], part), m.diag, m.rdiag);
    }
  };
  int s = 0, slot = 0, bt = 0;
  unsigned phase = 0;
  gss_wait(bar_s, 0);
  const unsigned char* st = ring;
  Item cur;
  fetch(st, 0, cur);
  for (;;) {
    // the batch: first pass from the prefetched item, further passes (more
    // rows than groups) read their rows directly
    do_row(cur.act, cur.m, cur.c, cur.j, cur.coef, cur.src);
    for (int p0 = NG; p0 < cur.rn; p0 += NG) {
      const int r = p0 + g;
      const bool act = r < cur.rn;
      GsStreamRow m;
      double c0[KE];
      unsigned j0[KE];
      if (act) m = cur.rows[cur.r0 + r];
      const int cnt = act ? (int)m.cnt : 0;
#pragma unroll
      for (int u = 0; u < KE; ++u) {
        const int k = (G == 1) ? u : li + u * G;
        c0[u] = k < cnt ? cur.coef[m.ebeg + k] : 0.0;
        j0[u] = k < cnt ? cur.src[m.ebeg + k] : 0u;
      }
      do_row(act, m, c0, j0, cur.coef, cur.src);
    }
    stamp(-4);
    if (CLU) asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    // next batch: same stage, or the first batch of the next stage
    const int nb = (int)reinterpret_cast<const unsigned*>(st)[0];
    int nslot = slot, ns = s, nbt = bt + 1;
    unsigned nphase = phase;
    bool next_stage = false, done = false;
    if (nbt >= nb) {
      if (s + 1 >= a.nstages) {
        done = true;
      } else {
        next_stage = true;
        ns = s + 1;
        nbt = 0;
        if (++nslot == a.nslots) {
          nslot = 0;
          nphase ^= 1u;
        }
        gss_wait(bar_s + 8u * nslot, nphase);
      }
    }
    Item nit;
    const unsigned char* nst = ring + nslot * a.slot_bytes;
    if (!done) fetch(nst, nbt, nit);
    stamp(-5);
    if (CLU) asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    else __syncthreads();  // batch published (and, when leaving a stage, its slot consumed)
    stamp(cur.rn);
    if (next_stage && tid == 0) issue(s + a.nslots, slot);
    if (done) break;
    s = ns;
    slot = nslot;
    phase = nphase;
    bt = nbt;
    st = nst;
    cur = nit;
  }
  for (int i = tid; i < nloc; i += T) a.xnew[base + i] = x[i];
  if (tr) a.trace[0] = tn;
  if (CLU) gss_csync();  // no CTA leaves while another may still read its slice
}

}  // namespace mvamg
