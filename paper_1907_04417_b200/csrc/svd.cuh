// svd.cuh -- the multi-vector setup's batched local SVD on the GPU
// (pkg/src/mvamg/svd.py:17-55, _kernels.py:64-121, multivector.py:181-212;
// SURVEY.md 8(f) #2).
//
// One thread per aggregate.  The reference's one-sided Jacobi is sequential
// inside an aggregate: every column sum runs over the rows in order and each
// rotation depends on the previous one, so the parallelism is across
// aggregates (C2's fine level: ~10^5 of them, m <= 64 rows, k = nsv columns).
// Each thread copies its block into U and rotates it there (the block is
// contiguous, m*k*8 <= 2.5 KB at the defaults, and stays in L1); the
// rotation accumulator V of the host code is not needed for U or sigma and is
// not formed.  Every operation is one IEEE rounding (__d*_rn, no contraction),
// in the host restatement's order, so U and sigma are bit-identical to
// mvamg_jacobi_svd_batch.
#pragma once

#include <cuda_runtime.h>

namespace mvamg {
namespace svd {

constexpr int kMaxCols = 16;

// status[0] = smallest non-converged block, status[1] = smallest empty block (both INT_MAX if none)
__global__ void jacobi_svd_kernel(int nblk, const int* __restrict__ row_ptr, int k, const double* __restrict__ A,
                                  int max_sweeps, double tol, double* __restrict__ U, double* __restrict__ sigma,
                                  int* __restrict__ status) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nblk) return;
  const int r0 = row_ptr[b], m = row_ptr[b + 1] - r0;
  if (m < 1) {
    atomicMin(status + 1, b);
    return;
  }
  double* B = U + (size_t)r0 * k;
  const double* Ab = A + (size_t)r0 * k;
  for (int e = 0; e < m * k; ++e) B[e] = Ab[e];
  // jacobi_orthogonalize (mvamg_b200.cu), _kernels.py:64-121
  if (k >= 2) {
    const double rel_tol = fmax(tol, __dmul_rn(__dmul_rn(2.0, (double)m), 2.220446049250313e-16));
    bool converged = false;
    for (int sweep = 0; sweep < max_sweeps && !converged; ++sweep) {
      double total = 0.0;
      for (int p = 0; p < k; ++p)
        for (int r = 0; r < m; ++r) total = __dadd_rn(total, __dmul_rn(B[r * k + p], B[r * k + p]));
      const double floor_ = __dmul_rn(tol, total);
      int rotated = 0;
      for (int p = 0; p < k - 1; ++p) {
        for (int q = p + 1; q < k; ++q) {
          double alpha = 0.0, beta = 0.0, gamma = 0.0;
          for (int r = 0; r < m; ++r) {
            const double bp = B[r * k + p], bq = B[r * k + q];
            alpha = __dadd_rn(alpha, __dmul_rn(bp, bp));
            beta = __dadd_rn(beta, __dmul_rn(bq, bq));
            gamma = __dadd_rn(gamma, __dmul_rn(bp, bq));
          }
          if (gamma == 0.0) continue;
          const double ag = fabs(gamma);
          if (ag <= __dmul_rn(rel_tol, __dsqrt_rn(__dmul_rn(alpha, beta))) || ag <= floor_) continue;
          ++rotated;
          const double zeta = __ddiv_rn(__dsub_rn(beta, alpha), __dmul_rn(2.0, gamma));
          const double t = __ddiv_rn(copysign(1.0, zeta),
                                     __dadd_rn(fabs(zeta), __dsqrt_rn(__dadd_rn(1.0, __dmul_rn(zeta, zeta)))));
          const double c = __ddiv_rn(1.0, __dsqrt_rn(__dadd_rn(1.0, __dmul_rn(t, t))));
          const double s = __dmul_rn(c, t);
          for (int r = 0; r < m; ++r) {
            const double bp = B[r * k + p], bq = B[r * k + q];
            B[r * k + p] = __dsub_rn(__dmul_rn(c, bp), __dmul_rn(s, bq));
            B[r * k + q] = __dadd_rn(__dmul_rn(s, bp), __dmul_rn(c, bq));
          }
        }
      }
      converged = rotated == 0;
    }
    if (!converged) {
      atomicMin(status, b);
      return;
    }
  }
  // column norms, stable descending order, U = B / sigma (svd.py:40-55)
  double s[kMaxCols];
  int order[kMaxCols];
  for (int p = 0; p < k; ++p) {
    double acc = 0.0;
    for (int r = 0; r < m; ++r) acc = __dadd_rn(acc, __dmul_rn(B[r * k + p], B[r * k + p]));
    s[p] = __dsqrt_rn(acc);
  }
  for (int p = 0; p < k; ++p) {  // stable insertion sort on -s, as std::stable_sort does
    const int v = p;
    int j = p;
    while (j > 0 && -s[v] < -s[order[j - 1]]) {
      order[j] = order[j - 1];
      --j;
    }
    order[j] = v;
  }
  for (int p = 0; p < k; ++p) sigma[(size_t)b * k + p] = s[order[p]];
  double row[kMaxCols];
  for (int r = 0; r < m; ++r) {
    for (int p = 0; p < k; ++p) row[p] = B[r * k + p];
    for (int p = 0; p < k; ++p) {
      const int src = order[p];
      B[r * k + p] = s[src] > 0.0 ? __ddiv_rn(row[src], s[src]) : 0.0;
    }
  }
}

}  // namespace svd
}  // namespace mvamg
