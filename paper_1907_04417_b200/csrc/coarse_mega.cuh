// coarse_mega.cuh -- the small coarse levels of a cycle in ONE thread block.
//
// The K-cycle (pkg/src/mvamg/cycles.py:150-179 with krylov.py:75-107 inner
// FCG) visits level k 2^k times; on the small coarse levels each visit is a
// couple of dozen tiny kernels, so a composite application (bootstrap.py:
// 98-113) is dominated by launch latency (C3: ~1e5 launches, ~5 us each).
// This kernel runs everything from level k0 down -- pre-smoothing, residual,
// restriction, the nested FCG or V recursion, coarsest solve, prolongation,
// post-smoothing -- in one 1024-thread block with __syncthreads between
// phases.  The recursion is an explicit frame stack in shared memory; every
// thread follows the same (uniform) control flow.
//
// Arithmetic is the multi-kernel path's: SpMV / residual / restriction /
// prolongation in CSR order with one rounding per operation, GS sweeps on the
// single-CTA level-set schedules (forward from zero; backward folded), the
// coarsest GEMV in gemv_kernel's lane-strided FMA + xor-shuffle order.  A
// V-cycle through this kernel is therefore bit-identical to the multi-kernel
// one; FCG dots use a fixed-order block reduction (tolerance-level, as the
// reference's BLAS dots).
#pragma once

namespace mvamg {

struct MegaLevel {
  int n, nlev0, nlev2, pad;
  const int *ip, *ix;                    // A_k
  const double* v;
  const int *rip, *rix;                  // R_k = P_k^T (n_{k+1} rows)
  const double* rv;
  const int *pip, *pix;                  // P_k (n_k rows)
  const double* pv;
  const int *lp0, *lp2;                  // level-set row offsets (forward / backward from zero)
  const GsLevelRow *rows0, *rows2;
  const GsLevelEntry *ents0, *ents2;
  double *xa, *t, *r, *z, *fr, *fx, *fp0, *fp1, *fap0, *fap1;
};

struct MegaArgs {
  int k0, L, entry_fcg, kcycle, inner, nL;
  const MegaLevel* lv;
  const double* inv;  // coarsest dense inverse (nL x nL, row-major)
  const double* in;   // right-hand side of the entry frame (level k0)
  int* status;
};

constexpr int kMegaThreads = 1024;
constexpr int kMegaMaxDepth = 64;

// ---- block-wide building blocks (all threads call; caller syncs) ---------
__device__ __forceinline__ void mk_spmv(int n, const int* ip, const int* ix, const double* v, const double* x,
                                        const double* b, double* y, int mode) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int k0 = __ldg(ip + i), k1 = __ldg(ip + i + 1);
    double s = 0.0;
    for (int k = k0; k < k1; ++k) s = __dadd_rn(s, __dmul_rn(__ldg(v + k), x[__ldg(ix + k)]));
    if (mode == 0) y[i] = s;
    else if (mode == 1) y[i] = __dsub_rn(b[i], s);
    else y[i] = __dadd_rn(y[i], s);
  }
}

// One level-set sweep on the single-CTA schedule: rows of each DAG level in
// parallel, CSR-order chains (products first, subtractions in order).
__device__ __forceinline__ void mk_gs_levels(int nlev, const int* lp, const GsLevelRow* rows,
                                             const GsLevelEntry* ents, const double* rhs, double* x) {
  for (int l = 0; l < nlev; ++l) {
    const int r0 = __ldg(lp + l), r1 = __ldg(lp + l + 1);
    for (int q = r0 + threadIdx.x; q < r1; q += blockDim.x) {
      const int4 hd = __ldg(reinterpret_cast<const int4*>(rows + q));       // row, estart, cnt, pad
      const double2 dd = __ldg(reinterpret_cast<const double2*>(rows + q) + 1);  // diag, RN(1/diag)
      const int row = hd.x, cnt = hd.z;
      double s = rhs[row];
      const GsLevelEntry* e = ents + hd.y;
      for (int k0 = 0; k0 < cnt; k0 += 4) {
        double p[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          p[u] = 0.0;
          if (k0 + u < cnt) {
            const double2 en = __ldg(reinterpret_cast<const double2*>(e + k0 + u));  // coef, src
            p[u] = __dmul_rn(en.x, x[__double2loint(en.y)]);
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (k0 + u < cnt) s = __dsub_rn(s, p[u]);
      }
      x[row] = div_rn_markstein(s, dd.x, dd.y);
    }
    __syncthreads();
  }
}

// Deterministic block sums of x.y and x2.y2 (fixed per-thread order, fixed tree).
__device__ __forceinline__ void mk_dot2(int n, const double* x, const double* y, const double* x2,
                                        const double* y2, double* sh, double& d1, double& d2) {
  double a = 0.0, b = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    a = __dadd_rn(a, __dmul_rn(x[i], y[i]));
    if (x2) b = __dadd_rn(b, __dmul_rn(x2[i], y2[i]));
  }
  a = warp_sum(a);
  b = warp_sum(b);
  const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) {
    sh[w] = a;
    sh[32 + w] = b;
  }
  __syncthreads();
  double ta = 0.0, tb = 0.0;
  for (int k = 0; k < nw; ++k) {
    ta += sh[k];
    tb += sh[32 + k];
  }
  d1 = ta;
  d2 = tb;
  __syncthreads();
}

struct MegaFrame {
  int type, k, phase, it, cur;  // type 0 = descend, 1 = fcg
  const double* in;
};

constexpr int kMegaMaxLevels = 32;

__global__ void __launch_bounds__(kMegaThreads, 1) coarse_mega_kernel(MegaArgs a) {
  __shared__ MegaFrame st[kMegaMaxDepth];
  __shared__ MegaLevel slv[kMegaMaxLevels];  // level descriptors, read on every phase
  __shared__ double sh[64];
  __shared__ double s_beta, s_alpha, s_pap_prev[kMegaMaxDepth];
  int depth = 0;
  {
    const int nw = (int)(sizeof(MegaLevel) / 8);
    const unsigned long long* src = reinterpret_cast<const unsigned long long*>(a.lv);
    unsigned long long* dst = reinterpret_cast<unsigned long long*>(slv);
    for (int i = threadIdx.x; i < (a.L - a.k0) * nw; i += blockDim.x) dst[a.k0 * nw + i] = src[a.k0 * nw + i];
  }
  if (threadIdx.x == 0) {
    st[0].type = a.entry_fcg;
    st[0].k = a.k0;
    st[0].phase = 0;
    st[0].it = 0;
    st[0].cur = 0;
    st[0].in = a.in;
  }
  __syncthreads();
  auto out_of = [&](int type, int k) -> double* {  // where a frame leaves its result
    if (type == 1) return slv[k].fx;
    return k == a.L - 1 ? slv[k].z : slv[k].xa;
  };
  auto fcg_level = [&](int k) { return a.kcycle && a.inner >= 1 && k >= 1 && k < a.L - 1; };
  while (depth >= 0) {
    const MegaFrame f = st[depth];
    __syncthreads();
    const MegaLevel& l = slv[f.k];
    if (f.type == 0) {
      if (f.k == a.L - 1) {  // coarsest: z = Inv r (gemv_kernel's order)
        const int lane = threadIdx.x & 31, n = a.nL;
        for (int row = threadIdx.x >> 5; row < n; row += blockDim.x >> 5) {
          const double* m = a.inv + (size_t)row * n;
          double s = 0.0;
          for (int j = lane; j < n; j += 32) s = fma(__ldg(m + j), f.in[j], s);
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
          if (lane == 0) l.z[row] = s;
        }
        __syncthreads();
        --depth;
        continue;
      }
      const MegaLevel& c = slv[f.k + 1];
      if (f.phase == 0) {
        // pre-smoothing: GS forward from x = 0
        mk_gs_levels(l.nlev0, l.lp0, l.rows0, l.ents0, f.in, l.xa);
        mk_spmv(l.n, l.ip, l.ix, l.v, l.xa, f.in, l.t, 1);  // t = r - A x
        __syncthreads();
        mk_spmv(c.n, l.rip, l.rix, l.rv, l.t, nullptr, c.r, 0);  // rc = R t
        __syncthreads();
        if (threadIdx.x == 0) {
          st[depth].phase = 1;
          MegaFrame& ch = st[depth + 1];
          ch.type = fcg_level(f.k + 1) ? 1 : 0;
          ch.k = f.k + 1;
          ch.phase = 0;
          ch.it = 0;
          ch.cur = 0;
          ch.in = c.r;
        }
        ++depth;
        __syncthreads();
        continue;
      }
      // phase 1: x += P xc, then GS backward (old lower neighbours folded)
      const double* xc = out_of(fcg_level(f.k + 1) ? 1 : 0, f.k + 1);
      mk_spmv(l.n, l.pip, l.pix, l.pv, xc, nullptr, l.xa, 2);
      __syncthreads();
      for (int i = threadIdx.x; i < l.n; i += blockDim.x) {
        double s = f.in[i];
        const int k1 = __ldg(l.ip + i + 1);
        for (int k = __ldg(l.ip + i); k < k1; ++k) {
          const int j = __ldg(l.ix + k);
          if (j >= i) break;
          s = __dsub_rn(s, __dmul_rn(__ldg(l.v + k), l.xa[j]));
        }
        l.t[i] = s;
      }
      __syncthreads();
      mk_gs_levels(l.nlev2, l.lp2, l.rows2, l.ents2, l.t, l.xa);
      --depth;
      continue;
    }
    // ---- FCG with a fixed step count, x0 = 0 (krylov.py:75-107) ----------
    const int n = l.n;
    if (f.phase == 0) {
      for (int i = threadIdx.x; i < n; i += blockDim.x) l.fr[i] = f.in[i];
      __syncthreads();
      if (threadIdx.x == 0) {
        st[depth].phase = 1;
        MegaFrame& ch = st[depth + 1];
        ch.type = 0;
        ch.k = f.k;
        ch.phase = 0;
        ch.it = 0;
        ch.cur = 0;
        ch.in = l.fr;
      }
      ++depth;
      __syncthreads();
      continue;
    }
    // a descend(k, r) just returned z in l.xa: one FCG step
    const int cur = f.cur, it = f.it;
    double* p = cur ? l.fp1 : l.fp0;
    double* ap = cur ? l.fap1 : l.fap0;
    const double* pprev = cur ? l.fp0 : l.fp1;
    const double* apprev = cur ? l.fap0 : l.fap1;
    const double* z = l.xa;
    if (it > 0) {
      double d1, d2;
      mk_dot2(n, z, apprev, nullptr, nullptr, sh, d1, d2);
      if (threadIdx.x == 0) s_beta = d1 / s_pap_prev[depth];
      __syncthreads();
    }
    const double beta = it > 0 ? s_beta : 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) p[i] = it == 0 ? z[i] : __dsub_rn(z[i], __dmul_rn(beta, pprev[i]));
    __syncthreads();
    mk_spmv(n, l.ip, l.ix, l.v, p, nullptr, ap, 0);
    __syncthreads();
    double d1, d2;
    mk_dot2(n, p, ap, p, l.fr, sh, d1, d2);
    if (threadIdx.x == 0) {
      if (!(d1 > 0.0)) {
        atomicOr(a.status, ST_FCG);
        s_alpha = 0.0;
      } else {
        s_alpha = d2 / d1;
      }
      s_pap_prev[depth] = d1;
    }
    __syncthreads();
    const double alpha = s_alpha;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const double xi = it == 0 ? 0.0 : l.fx[i];
      l.fx[i] = __dadd_rn(xi, __dmul_rn(alpha, p[i]));
      l.fr[i] = __dsub_rn(l.fr[i], __dmul_rn(alpha, ap[i]));
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      st[depth].it = it + 1;
      st[depth].cur = cur ^ 1;
    }
    __syncthreads();
    if (it + 1 < a.inner) {
      if (threadIdx.x == 0) {
        MegaFrame& ch = st[depth + 1];
        ch.type = 0;
        ch.k = f.k;
        ch.phase = 0;
        ch.it = 0;
        ch.cur = 0;
        ch.in = l.fr;
      }
      ++depth;
      __syncthreads();
      continue;
    }
    --depth;
  }
}

}  // namespace mvamg
