// matching.cuh -- the setup's greedy max-product matching on the GPU
// (pkg/src/mvamg/matching.py:78-122, _kernels.py:41-61).
//
// The reference visits the edges by descending weight c, ties by (i, j), and
// accepts an edge when both ends are free.  Under that strict total order the
// greedy result equals the locally dominant matching: repeatedly, every free
// vertex picks its best edge to a free neighbour, and mutual picks are
// matched.  The globally best remaining edge is always mutual, so every round
// matches at least one pair, and an edge is matched by one algorithm exactly
// when it is matched by the other.  Edge weights are formed exactly as numpy
// does (edge_weights, setup.py): den = d_i (w_i w_i) + d_j (w_j w_j), c =
// 1 - (((2 a) w_i) w_j) / den with i < j, one rounding per operation.
// Non-positive (<= floor), NaN and zero-denominator edges never take part.
#pragma once

#include <cuda_runtime.h>

namespace mvamg {
namespace matching {

__device__ __forceinline__ bool edge_better(double c1, int i1, int j1, double c2, int i2, int j2) {
  return c1 > c2 || (c1 == c2 && (i1 < i2 || (i1 == i2 && j1 < j2)));
}

__device__ __forceinline__ double edge_weight(double a, int i0, int j0, const double* __restrict__ d,
                                              const double* __restrict__ w, bool* ok) {
  const double wi = w[i0], wj = w[j0];
  const double den = __dadd_rn(__dmul_rn(d[i0], __dmul_rn(wi, wi)), __dmul_rn(d[j0], __dmul_rn(wj, wj)));
  *ok = den != 0.0;
  return __dsub_rn(1.0, __ddiv_rn(__dmul_rn(__dmul_rn(__dmul_rn(2.0, a), wi), wj), den));
}

// best[u] = the free neighbour of free vertex u on u's best eligible edge, or -1
__global__ void match_best_kernel(int n, const int* __restrict__ ip, const int* __restrict__ ix,
                                  const double* __restrict__ v, const double* __restrict__ d,
                                  const double* __restrict__ w, double floor_, const int* __restrict__ partner,
                                  int* __restrict__ best) {
  for (int u = blockIdx.x * blockDim.x + threadIdx.x; u < n; u += gridDim.x * blockDim.x) {
    if (partner[u] >= 0) {
      best[u] = -1;
      continue;
    }
    int bj_v = -1, bi = 0, bj = 0;
    double bc = 0.0;
    for (int k = ip[u]; k < ip[u + 1]; ++k) {
      const int j = ix[k];
      if (j == u || partner[j] >= 0) continue;
      const int i0 = u < j ? u : j, j0 = u < j ? j : u;
      // the reference weighs an edge by its upper-triangle entry A[i0, j0]
      double a = v[k];
      if (u > j) {
        int lo = ip[j], hi = ip[j + 1] - 1;
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (ix[mid] < u) lo = mid + 1;
          else hi = mid;
        }
        if (lo > hi || ix[lo] != u) continue;  // pattern not symmetric: the edge exists only below
        a = v[lo];
      }
      bool ok;
      const double c = edge_weight(a, i0, j0, d, w, &ok);
      if (!ok || !(c > floor_)) continue;
      if (bj_v < 0 || edge_better(c, i0, j0, bc, bi, bj)) {
        bj_v = j;
        bc = c;
        bi = i0;
        bj = j0;
      }
    }
    best[u] = bj_v;
  }
}

// mutual picks become pairs (the pair is written by its smaller vertex)
__global__ void match_pair_kernel(int n, const int* __restrict__ best, int* __restrict__ partner,
                                  int* __restrict__ changed) {
  for (int u = blockIdx.x * blockDim.x + threadIdx.x; u < n; u += gridDim.x * blockDim.x) {
    const int b = best[u];
    if (b > u && best[b] == u) {
      partner[u] = b;
      partner[b] = u;
      *changed = 1;
    }
  }
}

__global__ void fill_int_kernel(int n, int* __restrict__ p, int value) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) p[i] = value;
}

}  // namespace matching
}  // namespace mvamg
