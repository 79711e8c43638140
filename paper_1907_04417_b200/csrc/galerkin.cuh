// galerkin.cuh -- the aggregation Galerkin product A_c = (G + G^T) * 0.5,
// G = P^T (A P), on the GPU, bit for bit equal to the reference's scipy recipe
// (pkg/src/mvamg/sparse.py:50-66; SURVEY.md 8(a) A14, Appendix A "Galerkin").
//
// scipy's csr_matmat forms row i of X @ Y as sums[c] += x_ij * y_jc with sums
// starting at 0.0, visiting X's row in CSR order and then Y's row j, and drops
// exact-zero sums.  Every column c of the output row therefore sums its
// products in generation order.  Here one warp owns one output row and walks
// X's row serially; the entries of Y's row j are spread over the lanes.  Within
// one Y row the columns are distinct, so each lane owns a different
// accumulator slot and every slot still receives its products in generation
// order -- the scipy rounding sequence, with no sort of the products at all.
// Accumulators live in a per-warp open-addressing table in shared memory; a
// row whose distinct columns overflow it is redone with a larger table in
// global memory.  Output rows come out sorted (rank counting inside the warp).
//
// P^T (A P) runs csr_matmat on the transposed operands (csc inputs), so
// G[I,J] = 0.0 + sum over k ascending of AP[k,J] * P[k,I]: the same kernel with
// X = P^T (rows ascending in k, a stable transpose) and Y = AP.
// (G + G^T) is csr_plus_csr: a matching pair is added once (commutative), a
// lone entry is kept as is, exact zeros are dropped; then every value * 0.5.
#pragma once

#include <cuda_runtime.h>

namespace mvamg {
namespace galerkin {

constexpr int kWarps = 8;           // warps per CTA of the row kernels
constexpr int kTable = 256;         // shared-memory accumulator slots per warp
constexpr int kTableFill = 192;     // distinct columns before a row overflows to global memory
// dynamic shared memory of spgemm_smem_kernel per warp: table (key, value),
// the list of occupied slots, and the compacted (key, value) output list
constexpr int kSmemBytes = kWarps * (kTable * 12 + kTableFill * 16);

__device__ __forceinline__ unsigned slot_hash(int c) { return (unsigned)c * 2654435761u; }

// Accumulate X row `row` times Y into a (keys, vals) table of H slots
// (H a power of two, keys -1 = empty, vals 0.0); every newly occupied slot is
// appended to `slots`.  Returns the number of distinct columns, or -1 (all
// lanes) once more than `fill` appear -- the slots listed so far are then
// still dirty (clear_slots()).
__device__ __forceinline__ int accumulate_row(int row, const int* __restrict__ xp, const int* __restrict__ xi,
                                              const double* __restrict__ xv, const int* __restrict__ yp,
                                              const int* __restrict__ yi, const double* __restrict__ yv,
                                              int* keys, double* vals, int* slots, int H, int fill) {
  const int lane = threadIdx.x & 31;
  const int j0 = xp[row], j1 = xp[row + 1];
  int distinct = 0;
  for (int jj = j0; jj < j1; ++jj) {
    const int j = xi[jj];
    const double a = xv[jj];
    const int k0 = yp[j], k1 = yp[j + 1];
    for (int base = k0; base < k1; base += 32) {
      const int kk = base + lane;
      bool added = false;
      unsigned h = 0;
      if (kk < k1) {
        const int c = yi[kk];
        const double prod = __dmul_rn(a, yv[kk]);
        h = slot_hash(c) & (H - 1);
        for (int probe = 0; probe < H; ++probe) {
          int key = *(volatile int*)&keys[h];
          if (key == -1) {
            key = atomicCAS(&keys[h], -1, c);
            if (key == -1) {
              added = true;
              key = c;
            }
          }
          if (key == c) {  // this lane owns the slot for this Y row: ordered update
            vals[h] = __dadd_rn(vals[h], prod);
            break;
          }
          h = (h + 1) & (H - 1);
        }
      }
      const unsigned m = __ballot_sync(0xffffffffu, added);
      const int at = distinct + __popc(m & ((1u << lane) - 1u));
      if (added && at < fill) slots[at] = (int)h;
      distinct += __popc(m);
      __syncwarp();
      if (distinct > fill) return -1;
    }
  }
  return distinct;
}

__device__ __forceinline__ void clear_table(int* keys, double* vals, int H) {
  for (int s = threadIdx.x & 31; s < H; s += 32) {
    keys[s] = -1;
    vals[s] = 0.0;
  }
  __syncwarp();
}

// After an overflow: the listed slots plus any slot claimed in the last chunk
// may be dirty, so clear the whole table.
__device__ __forceinline__ void clear_slots(int* keys, double* vals, int H) { clear_table(keys, vals, H); }

// Compact the nonzero listed slots into (lk, lv) while clearing them, then
// (FILL) write them sorted by column at ci/cv + ofs.  Exact-zero sums are
// dropped as csr_matmat does.  Returns the row's nnz.
template <bool FILL>
__device__ __forceinline__ int emit_row(int distinct, const int* slots, int* keys, double* vals, int* lk,
                                        double* lv, int* __restrict__ ci, double* __restrict__ cv, long long ofs) {
  const int lane = threadIdx.x & 31;
  int count = 0;
  for (int e0 = 0; e0 < distinct; e0 += 32) {
    const int e = e0 + lane;
    bool live = false;
    int key = 0;
    double val = 0.0;
    if (e < distinct) {
      const int s = slots[e];
      key = keys[s];
      val = vals[s];
      live = val != 0.0;
      keys[s] = -1;
      vals[s] = 0.0;
    }
    const unsigned m = __ballot_sync(0xffffffffu, live);
    if (FILL && live) {
      const int at = count + __popc(m & ((1u << lane) - 1u));
      lk[at] = key;
      lv[at] = val;
    }
    count += __popc(m);
  }
  __syncwarp();
  if (FILL) {
    for (int e = lane; e < count; e += 32) {
      const int key = lk[e];
      int rank = 0;
      for (int f = 0; f < count; ++f) rank += lk[f] < key;
      ci[ofs + rank] = key;
      cv[ofs + rank] = lv[e];
    }
    __syncwarp();
  }
  return count;
}

// One warp per row, shared-memory tables.  FILL = false: cnt[row] = nnz of the
// row, or overflow -> flagged and appended to ovf_rows (counted by the global
// pass).  FILL = true: rows not flagged are written at cp[row].
template <bool FILL>
__global__ void __launch_bounds__(kWarps * 32) spgemm_smem_kernel(
    int nrows, const int* __restrict__ xp, const int* __restrict__ xi, const double* __restrict__ xv,
    const int* __restrict__ yp, const int* __restrict__ yi, const double* __restrict__ yv,
    int* __restrict__ cnt, unsigned char* __restrict__ ovf_flag, int* __restrict__ ovf_rows, int* __restrict__ n_ovf,
    int* __restrict__ max_ovf_ub, const long long* __restrict__ cp, int* __restrict__ ci, double* __restrict__ cv) {
  extern __shared__ __align__(16) unsigned char g_smem[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* vals = reinterpret_cast<double*>(g_smem) + w * kTable;
  double* lv = reinterpret_cast<double*>(g_smem) + kWarps * kTable + w * kTableFill;
  int* ibase = reinterpret_cast<int*>(g_smem + kWarps * (kTable + kTableFill) * 8);
  int* keys = ibase + w * kTable;
  int* slots = ibase + kWarps * kTable + w * kTableFill;
  int* lk = ibase + kWarps * (kTable + kTableFill) + w * kTableFill;
  clear_table(keys, vals, kTable);
  const int warps = gridDim.x * kWarps;
  for (int row = blockIdx.x * kWarps + w; row < nrows; row += warps) {
    if (FILL && ovf_flag[row]) continue;
    const int distinct = accumulate_row(row, xp, xi, xv, yp, yi, yv, keys, vals, slots, kTable, kTableFill);
    if (distinct < 0) {
      clear_slots(keys, vals, kTable);
      if (!FILL && lane == 0) {
        ovf_flag[row] = 1;
        ovf_rows[atomicAdd(n_ovf, 1)] = row;
        long long ub = 0;  // upper bound on the row's distinct columns: its product count
        for (int jj = xp[row]; jj < xp[row + 1]; ++jj) ub += yp[xi[jj] + 1] - yp[xi[jj]];
        atomicMax(max_ovf_ub, (int)(ub < 0x3fffffff ? ub : 0x3fffffff));
      }
      continue;
    }
    const int c = emit_row<FILL>(distinct, slots, keys, vals, lk, lv, ci, cv, FILL ? cp[row] : 0);
    if (!FILL && lane == 0) {
      cnt[row] = c;
      ovf_flag[row] = 0;
    }
  }
}

// Overflow rows: one warp per listed row with a private table (and list) of H
// slots in global memory -- a pool of gridDim.x * kWarps tables.
template <bool FILL>
__global__ void __launch_bounds__(kWarps * 32) spgemm_global_kernel(
    int nlist, const int* __restrict__ rows, const int* __restrict__ xp, const int* __restrict__ xi,
    const double* __restrict__ xv, const int* __restrict__ yp, const int* __restrict__ yi,
    const double* __restrict__ yv, int H, int* __restrict__ pool_keys, double* __restrict__ pool_vals,
    int* __restrict__ cnt, const long long* __restrict__ cp, int* __restrict__ ci, double* __restrict__ cv) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long gw = (long long)blockIdx.x * kWarps + w;
  int* keys = pool_keys + gw * 3 * (long long)H;
  int* slots = keys + H;
  int* lk = keys + 2 * H;
  double* vals = pool_vals + gw * 2 * (long long)H;
  double* lv = vals + H;
  clear_table(keys, vals, H);
  const int warps = gridDim.x * kWarps;
  for (int t = (int)gw; t < nlist; t += warps) {
    const int row = rows[t];
    const int distinct = accumulate_row(row, xp, xi, xv, yp, yi, yv, keys, vals, slots, H, H);
    const int c = emit_row<FILL>(distinct, slots, keys, vals, lk, lv, ci, cv, FILL ? cp[row] : 0);
    if (!FILL && lane == 0) cnt[row] = c;
  }
}

// ---- stable transpose (rows of the result list source rows ascending) -------
__global__ void col_count_kernel(long long nnz, const int* __restrict__ ix, int* __restrict__ cnt) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < nnz; k += (long long)gridDim.x * blockDim.x)
    atomicAdd(&cnt[ix[k]], 1);
}

// Scatter entry (i, c, v) to column c's segment in arrival order (unordered).
__global__ void transpose_scatter_kernel(int n, const int* __restrict__ ip, const int* __restrict__ ix,
                                         const double* __restrict__ v, const long long* __restrict__ tp,
                                         int* __restrict__ cursor, int* __restrict__ tix, double* __restrict__ tv) {
  const int warps = gridDim.x * (blockDim.x >> 5);
  const int lane = threadIdx.x & 31;
  for (int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < n; i += warps) {
    for (int k = ip[i] + lane; k < ip[i + 1]; k += 32) {
      const int c = ix[k];
      const long long p = tp[c] + atomicAdd(&cursor[c], 1);
      tix[p] = i;
      tv[p] = v[k];
    }
  }
}

// Order each row of the scattered transpose by source row (keys are distinct
// within a row): rank counting, one warp per row, out of place.
__global__ void segment_rank_sort_kernel(int nrows, const long long* __restrict__ tp, const int* __restrict__ in_ix,
                                         const double* __restrict__ in_v, int* __restrict__ out_ix,
                                         double* __restrict__ out_v) {
  const int warps = gridDim.x * (blockDim.x >> 5);
  const int lane = threadIdx.x & 31;
  for (int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < nrows; r += warps) {
    const long long a = tp[r], b = tp[r + 1];
    for (long long e = a + lane; e < b; e += 32) {
      const int key = in_ix[e];
      int rank = 0;
      for (long long f = a; f < b; ++f) rank += in_ix[f] < key;
      out_ix[a + rank] = key;
      out_v[a + rank] = in_v[e];
    }
  }
}

// ---- (G + G^T) * 0.5 -----------------------------------------------------
// Row i merges G's row i with G^T's row i (both sorted).  csr_plus_csr: a
// matching pair is added once, a lone entry is added to 0.0, exact-zero sums
// are dropped; the stored value is then scaled by 0.5.
template <bool FILL>
__global__ void symmetrize_kernel(int n, const long long* __restrict__ gp, const int* __restrict__ gi,
                                  const double* __restrict__ gv, const long long* __restrict__ tp,
                                  const int* __restrict__ ti, const double* __restrict__ tv, int* __restrict__ cnt,
                                  const long long* __restrict__ sp, int* __restrict__ si, double* __restrict__ sv) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    long long a = gp[i], b = tp[i];
    const long long ae = gp[i + 1], be = tp[i + 1];
    long long o = FILL ? sp[i] : 0;
    int c = 0;
    while (a < ae || b < be) {
      int col;
      double s;
      if (b >= be || (a < ae && gi[a] < ti[b])) {
        col = gi[a];
        s = __dadd_rn(gv[a], 0.0);
        ++a;
      } else if (a >= ae || ti[b] < gi[a]) {
        col = ti[b];
        s = __dadd_rn(0.0, tv[b]);
        ++b;
      } else {
        col = gi[a];
        s = __dadd_rn(gv[a], tv[b]);
        ++a;
        ++b;
      }
      if (s != 0.0) {
        if (FILL) {
          si[o] = col;
          sv[o] = __dmul_rn(s, 0.5);
          ++o;
        }
        ++c;
      }
    }
    if (!FILL) cnt[i] = c;
  }
}

// ---- exclusive scan of int counts into int64 offsets ------------------------
constexpr int kScanThreads = 1024;
constexpr int kScanItems = 4;  // per thread

__device__ __forceinline__ long long block_excl_scan(long long v, long long* s_warp, long long* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  long long x = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const long long y = __shfl_up_sync(0xffffffffu, x, d);
    if (lane >= d) x += y;
  }
  if (lane == 31) s_warp[w] = x;
  __syncthreads();
  if (w == 0) {
    long long t = lane < (blockDim.x >> 5) ? s_warp[lane] : 0;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const long long y = __shfl_up_sync(0xffffffffu, t, d);
      if (lane >= d) t += y;
    }
    s_warp[lane] = t;  // inclusive over warps
  }
  __syncthreads();
  const long long before = (w ? s_warp[w - 1] : 0) + x - v;
  *total = s_warp[(blockDim.x >> 5) - 1];
  __syncthreads();
  return before;
}

// out[i] = sum of in[0..i) for i in [0, n]; block sums to bsum.
__global__ void __launch_bounds__(kScanThreads) scan_blocks_kernel(int n, const int* __restrict__ in,
                                                                   long long* __restrict__ out,
                                                                   long long* __restrict__ bsum) {
  __shared__ long long s_warp[32];
  const long long base = (long long)blockIdx.x * kScanThreads * kScanItems;
  long long loc[kScanItems];
  long long acc = 0;
#pragma unroll
  for (int t = 0; t < kScanItems; ++t) {
    const long long i = base + (long long)threadIdx.x * kScanItems + t;
    loc[t] = acc;
    acc += i < n ? in[i] : 0;
  }
  long long total;
  const long long before = block_excl_scan(acc, s_warp, &total);
#pragma unroll
  for (int t = 0; t < kScanItems; ++t) {
    const long long i = base + (long long)threadIdx.x * kScanItems + t;
    if (i <= n) out[i] = before + loc[t];
  }
  if (threadIdx.x == 0) bsum[blockIdx.x] = total;
}

// Serial-in-chunks scan of the block sums by one CTA, then added back.
__global__ void __launch_bounds__(kScanThreads) scan_sums_kernel(int nb, long long* __restrict__ bsum) {
  __shared__ long long s_warp[32];
  long long carry = 0;
  for (int c0 = 0; c0 < nb; c0 += kScanThreads) {
    const int i = c0 + threadIdx.x;
    const long long v = i < nb ? bsum[i] : 0;
    long long total;
    const long long before = block_excl_scan(v, s_warp, &total);
    if (i < nb) bsum[i] = carry + before;
    carry += total;
  }
}

__global__ void scan_add_kernel(int n, long long* __restrict__ out, const long long* __restrict__ bsum) {
  const long long per = (long long)kScanThreads * kScanItems;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i <= n; i += (long long)gridDim.x * blockDim.x)
    out[i] += bsum[i / per];
}

__global__ void narrow_offsets_kernel(int n, const long long* __restrict__ in, int* __restrict__ out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i <= n; i += gridDim.x * blockDim.x) out[i] = (int)in[i];
}

__global__ void widen_offsets_kernel(int n, const int* __restrict__ in, long long* __restrict__ out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i <= n; i += gridDim.x * blockDim.x) out[i] = in[i];
}

}  // namespace galerkin
}  // namespace mvamg
