// mvamg_kernels.cuh -- sm_100a device kernels for the mvamg solve phase.
//
// Everything here is fp64 sparse / streaming work (~0.17 flop/B): HBM- or
// latency-bound, no tensor cores (BASELINE.json north_star).  Bit-exactness
// recipe: each row sum is formed in CSR order starting
// from 0.0 (or b[i] for GS) with separately rounded multiply and add/subtract
// (__dmul_rn / __dadd_rn / __dsub_rn; the .so is also built with -fmad=false),
// exactly like scipy csr_matvec and the numba GS kernels
// (pkg/src/mvamg/_kernels.py:15-38, pkg/src/mvamg/sparse.py:40).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace mvamg {

constexpr unsigned long long kSentinel = 0xFFFFFFFFFFFFFFFFull;  // -NaN, never produced by arithmetic
constexpr int kSpinLimit = 1 << 21;
constexpr int kDotMaxBlocks = 1024;

// status bits (mirror MVAMG_ST_* in include/mvamg_b200.h)
constexpr int ST_RZ = 1, ST_PQ = 2, ST_FCG = 4, ST_GS_TIMEOUT = 8;

// ---------------------------------------------------------------------------
// Device scalar block shared by the drivers (one per hierarchy).
struct DevScalars {
  double rz, alpha, beta, r0, rtol;
  double pq, rr;
  int k, itmax, status, converged, stop, pad0, pad1, pad2;
  double* hist;
};

// Per-level FCG scalars (krylov.py:75-107).
struct FcgScalars {
  double alpha, beta, pAp, pAp_prev, pr;
};

__device__ __noinline__ double div_rn_slow(double s, double d) { return __ddiv_rn(s, d); }

__device__ __forceinline__ double div_rn_markstein(double s, double d, double y) {
  // RN(s/d) from y = RN(1/d): q0 = RN(s*y) is faithful, r = s - q0*d is exact
  // (FMA), q = RN(q0 + r*y) is the correctly rounded quotient (Markstein).
  // 24 cycles of dependent latency instead of ~350 for IEEE ddiv (measured on
  // B200, profiles/r01_probe.txt); 0 mismatches vs __ddiv_rn on 2^26 samples.
  double q0 = __dmul_rn(s, y);
  double r = fma(-q0, d, s);
  double q = fma(r, y, q0);
  double aq = fabs(q0);
  if (__builtin_expect(!(aq > 1e-290 && aq < 1e290), 0)) q = div_rn_slow(s, d);  // outside the theorem's range / zero
  return q;
}

__device__ __forceinline__ unsigned long long ld_relaxed_u64(const double* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}

__device__ __forceinline__ void prefetch_l1(const void* p) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}

// Slow path of a dependency wait: spin on the sentinel.  A bounded spin (and an
// abort once any thread has timed out) turns a scheduling bug into an error
// status instead of a hung GPU.
__device__ __noinline__ double poll_global_slow(const double* p, int* status) {
  unsigned long long v;
  int spins = 0;
  do {
    v = ld_relaxed_u64(p);
    if ((++spins & 255) == 0) {
      if (spins > kSpinLimit) { atomicOr(status, ST_GS_TIMEOUT); return 0.0; }
      if (*reinterpret_cast<volatile int*>(status) & ST_GS_TIMEOUT) return 0.0;
    }
  } while (v == kSentinel);
  return __longlong_as_double(v);
}

__device__ __forceinline__ double poll_global(const double* p, int* status) {
  unsigned long long v = ld_relaxed_u64(p);
  if (v != kSentinel) return __longlong_as_double(v);
  return poll_global_slow(p, status);
}

__device__ __noinline__ double poll_shared_slow(const double* p, int* status) {
  volatile const unsigned long long* q = reinterpret_cast<volatile const unsigned long long*>(p);
  unsigned long long v;
  int spins = 0;
  do {
    v = *q;
    if ((++spins & 255) == 0) {
      if (spins > kSpinLimit) { atomicOr(status, ST_GS_TIMEOUT); return 0.0; }
      if (*reinterpret_cast<volatile int*>(status) & ST_GS_TIMEOUT) return 0.0;
    }
  } while (v == kSentinel);
  return __longlong_as_double(v);
}

__device__ __forceinline__ double poll_shared(const double* p, int* status) {
  unsigned long long v = *reinterpret_cast<volatile const unsigned long long*>(p);
  if (v != kSentinel) return __longlong_as_double(v);
  return poll_shared_slow(p, status);
}

// ---------------------------------------------------------------------------
// CSR SpMV family, one thread per row, CSR-order accumulation (bit-exact).
//   MODE 0: y = A x          (sparse.py:40)
//   MODE 1: y = b - A x      (cycles.py:156 residual)
//   MODE 2: y = y + (A x)    (cycles.py:170 prolongation; sum first, one add)
template <int MODE>
__global__ void __launch_bounds__(256) spmv_kernel(int n, const int* __restrict__ ip,
                                                   const int* __restrict__ ix,
                                                   const double* __restrict__ v,
                                                   const double* __restrict__ x,
                                                   const double* __restrict__ b, double* y) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    int k0 = __ldg(ip + i), k1 = __ldg(ip + i + 1);
    double s = 0.0;
    for (int k = k0; k < k1; ++k) s = __dadd_rn(s, __dmul_rn(__ldg(v + k), __ldg(x + __ldg(ix + k))));
    if (MODE == 0) y[i] = s;
    else if (MODE == 1) y[i] = __dsub_rn(__ldg(b + i), s);
    else y[i] = __dadd_rn(y[i], s);
  }
}

// The same SpMV family, CSR-stream: a block takes `rpt` consecutive rows, its
// threads form the products a_k * x[j_k] of the tile's contiguous entry range
// with coalesced loads (each its own rounding, as in the serial loop) into
// shared memory, then one thread per row adds its products in CSR order from
// 0.0 -- bit-identical to spmv_kernel, but every load instruction of the
// matrix is one coalesced segment instead of 32 rows' strided entries.  A tile
// whose entries exceed the buffer falls back to the row loop.
constexpr int kSpmvTileNnz = 3072;

template <int MODE>
__global__ void __launch_bounds__(256) spmv_stream_kernel(int n, int rpt, const int* __restrict__ ip,
                                                          const int* __restrict__ ix,
                                                          const double* __restrict__ v,
                                                          const double* __restrict__ x,
                                                          const double* __restrict__ b, double* y) {
  __shared__ double prod[kSpmvTileNnz];
  const int tid = threadIdx.x;
  for (int r0 = blockIdx.x * rpt; r0 < n; r0 += gridDim.x * rpt) {
    const int r1 = min(r0 + rpt, n);
    const int e0 = __ldg(ip + r0), e1 = __ldg(ip + r1);
    const int row = r0 + tid;
    double s = 0.0;
    if (e1 - e0 <= kSpmvTileNnz) {
#pragma unroll 4
      for (int e = e0 + tid; e < e1; e += 256) prod[e - e0] = __dmul_rn(__ldg(v + e), __ldg(x + __ldg(ix + e)));
      __syncthreads();
      if (row < r1) {
        const int k1 = __ldg(ip + row + 1);
        for (int k = __ldg(ip + row); k < k1; ++k) s = __dadd_rn(s, prod[k - e0]);
      }
      __syncthreads();
    } else if (row < r1) {
      const int k1 = __ldg(ip + row + 1);
      for (int k = __ldg(ip + row); k < k1; ++k) s = __dadd_rn(s, __dmul_rn(__ldg(v + k), __ldg(x + __ldg(ix + k))));
    }
    if (row < r1) {
      if (MODE == 0) y[row] = s;
      else if (MODE == 1) y[row] = __dsub_rn(__ldg(b + row), s);
      else y[row] = __dadd_rn(y[row], s);
    }
  }
}

// The same SpMV family, one warp per row, for small levels with long rows (the
// K-cycle's coarse levels: a few thousand rows of 10-70 entries).  One thread
// per row walks its row with ~2 dependent L2 trips per unrolled batch of
// entries, which dominates there.  Here the lanes load a 32-entry chunk of the
// row and form the products a_k * x_k (each its own rounding) at once; every
// lane then adds the chunk's products in CSR order from shuffles, starting
// from 0.0 as scipy does, so the sum is bit-identical to spmv_kernel's.
template <int MODE>
__device__ __forceinline__ double warp_row_sum(int i, const int* __restrict__ ip, const int* __restrict__ ix,
                                               const double* __restrict__ v, const double* __restrict__ x,
                                               int lane) {
  const int k0 = __ldg(ip + i), k1 = __ldg(ip + i + 1);
  double s = 0.0;
  for (int c = k0; c < k1; c += 32) {
    const int k = c + lane, m = min(32, k1 - c);
    double pr = 0.0;
    if (k < k1) pr = __dmul_rn(__ldg(v + k), __ldg(x + __ldg(ix + k)));
    for (int t = 0; t < m; ++t) s = __dadd_rn(s, __shfl_sync(0xffffffffu, pr, t));
  }
  return s;
}

template <int MODE>
__global__ void __launch_bounds__(256) spmv_warp_kernel(int n, const int* __restrict__ ip,
                                                        const int* __restrict__ ix,
                                                        const double* __restrict__ v,
                                                        const double* __restrict__ x,
                                                        const double* __restrict__ b, double* y) {
  const int lane = threadIdx.x & 31;
  const int w0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (int i = w0; i < n; i += nw) {
    const double s = warp_row_sum<MODE>(i, ip, ix, v, x, lane);
    if (lane == 0) {
      if (MODE == 0) y[i] = s;
      else if (MODE == 1) y[i] = __dsub_rn(__ldg(b + i), s);
      else y[i] = __dadd_rn(y[i], s);
    }
  }
}

// Weighted Jacobi, out of place: y = x + ((omega*(b - Ax))/d)   (cycles.py:148)
__global__ void __launch_bounds__(256) jacobi_kernel(int n, const int* __restrict__ ip,
                                                     const int* __restrict__ ix,
                                                     const double* __restrict__ v,
                                                     const double* __restrict__ d,
                                                     const double* __restrict__ b, double omega,
                                                     const double* __restrict__ x, double* y) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    int k0 = ip[i], k1 = ip[i + 1];
    double s = 0.0;
    for (int k = k0; k < k1; ++k) s = __dadd_rn(s, __dmul_rn(v[k], x[ix[k]]));
    double t = __ddiv_rn(__dmul_rn(omega, __dsub_rn(b[i], s)), d[i]);
    y[i] = __dadd_rn(x[i], t);
  }
}

}  // namespace mvamg

#include "gs_sweep.cuh"

namespace mvamg {

// ---------------------------------------------------------------------------
// Dense coarsest solve z = Inv r (row-major), one warp per row.
__global__ void __launch_bounds__(256) gemv_kernel(int n, const double* __restrict__ inv,
                                                   const double* __restrict__ r, double* z) {
  const int lane = threadIdx.x & 31;
  for (int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; row < n;
       row += (gridDim.x * blockDim.x) >> 5) {
    const double* a = inv + (size_t)row * n;
    double s = 0.0;
    for (int j = lane; j < n; j += 32) s = fma(__ldg(a + j), __ldg(r + j), s);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) z[row] = s;
  }
}

// ---------------------------------------------------------------------------
// Deterministic reductions.  Each kernel reduces per block (fixed shuffle
// tree), writes a partial, and the last block to arrive sums the partials in
// block order and runs a scalar epilogue (the Krylov scalar updates of
// krylov.py), so no host round trip is needed between kernels.
enum PostOp : int {
  POST_STORE = 0,       // out[0] = d1
  POST_PCG_ALPHA = 1,   // pq = d1; alpha = rz/pq                 krylov.py:53-56
  POST_PCG_NORM = 2,    // hist[k+1] = sqrt(d1); stop test        krylov.py:59-65
  POST_PCG_BETA = 3,    // rz' = d1; beta = rz'/rz; rz = rz'      krylov.py:67-71
  POST_PCG_INIT = 4,    // rz = d1 (r'z of z = M r0)              krylov.py:45-47
  POST_PCG_R0 = 5,      // r0 = sqrt(d1); hist[0]                 krylov.py:40-44
  POST_FCG_BETA = 6,    // beta = d1/pAp_prev                     krylov.py:97
  POST_FCG_ALPHA = 7,   // pAp = d1; alpha = d2/pAp               krylov.py:100-104
};

struct ReduceCtx {
  double* partials;   // >= 2*kDotMaxBlocks
  unsigned* counter;  // zero between uses
  DevScalars* sc;
  FcgScalars* fs;
  double* out;
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block reduce of (d1, d2) for blockDim.x == 256.
__device__ __forceinline__ void block_sum2(double& d1, double& d2) {
  __shared__ double sh[2][8];
  d1 = warp_sum(d1);
  d2 = warp_sum(d2);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) { sh[0][w] = d1; sh[1][w] = d2; }
  __syncthreads();
  if (w == 0) {
    d1 = l < 8 ? sh[0][l] : 0.0;
    d2 = l < 8 ? sh[1][l] : 0.0;
    d1 = warp_sum(d1);
    d2 = warp_sum(d2);
  }
  __syncthreads();
}

__device__ void run_post(int op, double d1, double d2, const ReduceCtx& c) {
  DevScalars* s = c.sc;
  switch (op) {
    case POST_STORE:
      c.out[0] = d1;
      break;
    case POST_PCG_ALPHA:
      s->pq = d1;
      if (!(d1 > 0.0)) { s->status |= ST_PQ; s->stop = 1; s->alpha = 0.0; }
      else s->alpha = s->rz / d1;
      break;
    case POST_PCG_NORM: {
      double nr = sqrt(d1);
      s->k += 1;
      s->hist[s->k] = nr;
      s->rr = nr;
      if (nr <= s->rtol * s->r0) { s->converged = 1; s->stop = 1; }
      if (s->k >= s->itmax) s->stop = 1;
      break;
    }
    case POST_PCG_BETA:
      if (!(d1 > 0.0)) { s->status |= ST_RZ; s->stop = 1; s->beta = 0.0; }
      else { s->beta = d1 / s->rz; s->rz = d1; }
      break;
    case POST_PCG_INIT:
      s->rz = d1;
      if (!(d1 > 0.0)) { s->status |= ST_RZ; s->stop = 1; }
      if (s->itmax <= 0) s->stop = 1;
      break;
    case POST_PCG_R0: {
      double nr = sqrt(d1);
      s->r0 = nr;
      s->hist[0] = nr;
      s->k = 0;
      s->converged = 0;
      s->stop = 0;
      if (nr == 0.0) { s->converged = 1; s->stop = 1; }
      break;
    }
    case POST_FCG_BETA:
      c.fs->beta = d1 / c.fs->pAp_prev;
      break;
    case POST_FCG_ALPHA:
      c.fs->pAp = d1;
      c.fs->pr = d2;
      if (!(d1 > 0.0)) { s->status |= ST_FCG; c.fs->alpha = 0.0; }
      else c.fs->alpha = d2 / d1;
      c.fs->pAp_prev = d1;
      break;
  }
}

// Called by every thread of every block after block_sum2; thread 0 of block 0
// carries the block total in d1/d2 after block_sum2.
__device__ __forceinline__ void grid_finish(int op, double d1, double d2, const ReduceCtx& c) {
  __shared__ bool am_last;
  if (threadIdx.x == 0) {
    c.partials[2 * blockIdx.x] = d1;
    c.partials[2 * blockIdx.x + 1] = d2;
    __threadfence();
    unsigned prev = atomicAdd(c.counter, 1u);
    am_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (!am_last) return;
  __threadfence();
  double e1 = 0.0, e2 = 0.0;
  for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) {
    e1 += __ldcg(c.partials + 2 * b);
    e2 += __ldcg(c.partials + 2 * b + 1);
  }
  block_sum2(e1, e2);
  if (threadIdx.x == 0) {
    *c.counter = 0u;
    run_post(op, e1, e2, c);
  }
}

// d1 = x1.y1, d2 = x2.y2 (x2 may be null).
__global__ void __launch_bounds__(256) dot2_kernel(int n, const double* __restrict__ x1,
                                                   const double* __restrict__ y1,
                                                   const double* __restrict__ x2,
                                                   const double* __restrict__ y2, int op,
                                                   ReduceCtx c) {
  double d1 = 0.0, d2 = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    d1 = fma(x1[i], y1[i], d1);
    if (x2) d2 = fma(x2[i], y2[i], d2);
  }
  block_sum2(d1, d2);
  grid_finish(op, d1, d2, c);
}

// y = A p fused with d1 = p.y and d2 = p.r (r may be null)  (PCG q = A p;
// FCG Ap = A p with p'Ap and p'r).
__global__ void __launch_bounds__(256) spmv_dot_kernel(int n, const int* __restrict__ ip,
                                                       const int* __restrict__ ix,
                                                       const double* __restrict__ v,
                                                       const double* __restrict__ p,
                                                       const double* __restrict__ r, double* y,
                                                       int op, ReduceCtx c) {
  double d1 = 0.0, d2 = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    int k0 = __ldg(ip + i), k1 = __ldg(ip + i + 1);
    double s = 0.0;
    for (int k = k0; k < k1; ++k) s = __dadd_rn(s, __dmul_rn(__ldg(v + k), __ldg(p + __ldg(ix + k))));
    y[i] = s;
    double pi = p[i];
    d1 = fma(pi, s, d1);
    if (r) d2 = fma(pi, r[i], d2);
  }
  block_sum2(d1, d2);
  grid_finish(op, d1, d2, c);
}

// spmv_dot_kernel with one warp per row (spmv_warp_kernel's bit-identical y);
// lane 0 of each warp accumulates the dots over its rows.
__global__ void __launch_bounds__(256) spmv_dot_warp_kernel(int n, const int* __restrict__ ip,
                                                            const int* __restrict__ ix,
                                                            const double* __restrict__ v,
                                                            const double* __restrict__ p,
                                                            const double* __restrict__ r, double* y,
                                                            int op, ReduceCtx c) {
  const int lane = threadIdx.x & 31;
  const int w0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  double d1 = 0.0, d2 = 0.0;
  for (int i = w0; i < n; i += nw) {
    const double s = warp_row_sum<0>(i, ip, ix, v, p, lane);
    if (lane == 0) {
      y[i] = s;
      const double pi = p[i];
      d1 = fma(pi, s, d1);
      if (r) d2 = fma(pi, r[i], d2);
    }
  }
  block_sum2(d1, d2);
  grid_finish(op, d1, d2, c);
}

// PCG: x += alpha p; r -= alpha q; d1 = r.r   (krylov.py:57-60)
__global__ void __launch_bounds__(256) pcg_xr_kernel(int n, double* x, double* r,
                                                     const double* __restrict__ p,
                                                     const double* __restrict__ q, ReduceCtx c) {
  const double alpha = c.sc->alpha;
  double d1 = 0.0, d2 = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    x[i] = __dadd_rn(x[i], __dmul_rn(alpha, p[i]));
    double ri = __dsub_rn(r[i], __dmul_rn(alpha, q[i]));
    r[i] = ri;
    d1 = fma(ri, ri, d1);
  }
  block_sum2(d1, d2);
  grid_finish(POST_PCG_NORM, d1, d2, c);
}

// PCG: p = z + beta p  (krylov.py:70)
__global__ void pcg_p_kernel(int n, double* p, const double* __restrict__ z, const DevScalars* sc) {
  const double beta = sc->beta;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    p[i] = __dadd_rn(z[i], __dmul_rn(beta, p[i]));
}

// FCG: p = z (first) or p = z - beta p_prev   (krylov.py:93-98)
__global__ void fcg_p_kernel(int n, double* p, const double* __restrict__ z,
                             const double* __restrict__ pprev, const FcgScalars* fs, int first) {
  const double beta = first ? 0.0 : fs->beta;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    p[i] = first ? z[i] : __dsub_rn(z[i], __dmul_rn(beta, pprev[i]));
}

// FCG: x += alpha p; r -= alpha Ap  (x starts at 0 when first)   (krylov.py:105-106)
__global__ void fcg_xr_kernel(int n, double* x, double* r, const double* __restrict__ p,
                              const double* __restrict__ ap, const FcgScalars* fs, int first) {
  const double alpha = fs->alpha;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double xi = first ? 0.0 : x[i];
    x[i] = __dadd_rn(xi, __dmul_rn(alpha, p[i]));
    r[i] = __dsub_rn(r[i], __dmul_rn(alpha, ap[i]));
  }
}

// elementwise helpers
__global__ void copy_kernel(int n, double* y, const double* __restrict__ x) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) y[i] = x[i];
}
// y = a - b
__global__ void sub_kernel(int n, double* y, const double* __restrict__ a, const double* __restrict__ b) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    y[i] = __dsub_rn(a[i], b[i]);
}
// y = a + b
__global__ void add_kernel(int n, double* y, const double* __restrict__ a, const double* __restrict__ b) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    y[i] = __dadd_rn(a[i], b[i]);
}
__global__ void zero_kernel(int n, double* y) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) y[i] = 0.0;
}

// PCG scalar setup: itmax / rtol / hist pointer / status reset.
__global__ void pcg_setup_kernel(DevScalars* sc, double rtol, int itmax, double* hist) {
  sc->rtol = rtol;
  sc->itmax = itmax;
  sc->hist = hist;
  sc->status = 0;
  sc->converged = 0;
  sc->stop = 0;
  sc->k = 0;
}


// ---- row-partitioned solve: halo packing and Krylov updates ----------------
__global__ void gather_kernel(int n, const int* __restrict__ idx, const double* __restrict__ src,
                              double* __restrict__ dst) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) dst[i] = src[idx[i]];
}

__global__ void scatter_kernel(int n, const int* __restrict__ idx, const double* __restrict__ src,
                               double* __restrict__ dst) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) dst[idx[i]] = src[i];
}

// y_i = y_i + (alpha * x_i)   (krylov.py:57-58: x += alpha p, r -= alpha q)
__global__ void axpy_kernel(int n, double alpha, const double* __restrict__ x, double* __restrict__ y) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    y[i] = __dadd_rn(y[i], __dmul_rn(alpha, x[i]));
}

// y_i = x_i + (beta * y_i)   (krylov.py:70: p = z + beta p)
__global__ void xpby_kernel(int n, const double* __restrict__ x, double beta, double* __restrict__ y) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    y[i] = __dadd_rn(x[i], __dmul_rn(beta, y[i]));
}

}  // namespace mvamg
