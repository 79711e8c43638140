// mvamg_b200.cu -- native runtime + C ABI of libmvamg_b200.so (sm_100a).
//
// The drivers below restate, as device launch sequences on one CUDA stream, the
// reference solve path of arXiv 1907.04417's `mvamg`:
//   descend / cycle  : pkg/src/mvamg/cycles.py:150-179 (V and K cycles)
//   fcg              : pkg/src/mvamg/krylov.py:75-107  (K-cycle inner solve)
//   pcg              : pkg/src/mvamg/krylov.py:28-72
//   composite        : pkg/src/mvamg/bootstrap.py:98-113
// All scalars stay on the device (reductions finish in their last block and
// update the Krylov scalars in place); repeated launch sequences (one cycle, one
// PCG half-iteration) are captured once into CUDA graphs and replayed.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "../../include/mvamg_b200.h"
#include "mvamg_kernels.cuh"
#include "galerkin.cuh"
#include "gs_stream.cuh"
#include "gs_cluster.cuh"
#include "matching.cuh"
#include "svd.cuh"

using namespace mvamg;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CUDA_TRY(expr)                                                                 \
  do {                                                                                 \
    cudaError_t e_ = (expr);                                                           \
    if (e_ != cudaSuccess)                                                             \
      return fail(MVAMG_E_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_));   \
  } while (0)

int g_num_sms = 0;
long long g_kernel_launches = 0;
long long* g_gs_trace = nullptr;  // diagnostics: per-warp GS round/cycle counters (device)
int g_gs_debug = [] {
  const char* e = getenv("MVAMG_GS_DEBUG");
  return e ? atoi(e) : 0;
}();  // kernels launched by this library (graph nodes counted per replay)
int g_row_sleep = [] {
  const char* e = getenv("MVAMG_ROW_SLEEP");
  return e ? atoi(e) : 0;
}();
int g_cluster_cap10 = [] {  // diagnostics: a CTA's share of a DAG level (x10) the plan lets it exceed ...
  const char* e = getenv("MVAMG_CLUSTER_CAP10");
  return e ? atoi(e) : 15;
}();
int g_cluster_tot10 = [] {  // ... and of all rows so far (x10), when a row follows its latest input's CTA
  const char* e = getenv("MVAMG_CLUSTER_TOT10");
  return e ? atoi(e) : 11;
}();
int g_cluster_local = [] {  // diagnostics: 0 = the cluster plan ignores where a row's latest input lives
  const char* e = getenv("MVAMG_CLUSTER_LOCAL");
  return e ? atoi(e) : 1;
}();
int g_cluster_sleep = [] {  // diagnostics: overrides a cluster schedule's poll back-off (ns)
  const char* e = getenv("MVAMG_CLUSTER_SLEEP");
  return e ? atoi(e) : -1;
}();

int num_sms() {
  if (g_num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  return g_num_sms;
}

inline int grid_for(int n, int threads = 256, int per_sm = 8) {
  long long g = ((long long)n + threads - 1) / threads;
  long long cap = (long long)num_sms() * per_sm;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

inline int dot_grid(int n) { return std::min(grid_for(n, 256, 8), kDotMaxBlocks); }
constexpr int kWarpRowMaxRows = 65536;  // levels up to this size with >= kWarpRowMinAvg entries per row
constexpr int kWarpRowMinAvg = 8;       //   run their SpMVs one warp per row

bool g_attr_done = false;
int g_max_dyn_smem = 48 * 1024;
void set_kernel_attrs() {
  if (g_attr_done) return;
  g_attr_done = true;
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  int maxsm = optin - 1024;  // leave room for the kernel's static shared memory
  if (maxsm < 48 * 1024) maxsm = 48 * 1024;
  bool ok = true;
#define MVAMG_GS_ATTR(F, R, D) \
  ok &= cudaFuncSetAttribute(gs_sweep_kernel<F, R, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm) == cudaSuccess;
#define MVAMG_GS_ATTR_D(F, R) MVAMG_GS_ATTR(F, R, 2) MVAMG_GS_ATTR(F, R, 4) MVAMG_GS_ATTR(F, R, 8)
  MVAMG_GS_ATTR_D(true, 1) MVAMG_GS_ATTR_D(true, 2) MVAMG_GS_ATTR_D(true, 4) MVAMG_GS_ATTR_D(true, 8)
  MVAMG_GS_ATTR_D(false, 1) MVAMG_GS_ATTR_D(false, 2) MVAMG_GS_ATTR_D(false, 4) MVAMG_GS_ATTR_D(false, 8)
#undef MVAMG_GS_ATTR_D
#undef MVAMG_GS_ATTR
#define MVAMG_LEAN_ATTR(F, CC, RR, DD)                                                                   \
  ok &= cudaFuncSetAttribute(gs_lean_kernel<F, CC, RR, DD>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm) == \
        cudaSuccess;                                                                                     \
  ok &= cudaFuncSetAttribute(gs_lean_kernel<F, CC, RR, DD, 1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                             maxsm) == cudaSuccess;
#define MVAMG_LEAN_ATTR_C(F, RR, DD) MVAMG_LEAN_ATTR(F, 2, RR, DD) MVAMG_LEAN_ATTR(F, 4, RR, DD) MVAMG_LEAN_ATTR(F, 8, RR, DD)
  MVAMG_LEAN_ATTR_C(true, 8, 3) MVAMG_LEAN_ATTR_C(true, 8, 2) MVAMG_LEAN_ATTR_C(true, 4, 4) MVAMG_LEAN_ATTR_C(true, 4, 2) MVAMG_LEAN_ATTR_C(true, 2, 2) MVAMG_LEAN_ATTR_C(true, 2, 8) MVAMG_LEAN_ATTR_C(true, 1, 8)
  MVAMG_LEAN_ATTR_C(false, 8, 3) MVAMG_LEAN_ATTR_C(false, 8, 2) MVAMG_LEAN_ATTR_C(false, 4, 4) MVAMG_LEAN_ATTR_C(false, 4, 2) MVAMG_LEAN_ATTR_C(false, 2, 2) MVAMG_LEAN_ATTR_C(false, 2, 8) MVAMG_LEAN_ATTR_C(false, 1, 8)
#define MVAMG_LEANK_ATTR(F, CC, RR, DD, KK) \
  ok &= cudaFuncSetAttribute(gs_lean_kernel<F, CC, RR, DD, KK>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm) == cudaSuccess;
#define MVAMG_LEANK_ATTR_F(F)                                                               \
  MVAMG_LEANK_ATTR(F, 2, 2, 3, 4) MVAMG_LEANK_ATTR(F, 4, 2, 3, 4) MVAMG_LEANK_ATTR(F, 2, 2, 2, 4) \
  MVAMG_LEANK_ATTR(F, 4, 2, 2, 4) MVAMG_LEANK_ATTR(F, 2, 4, 2, 2) MVAMG_LEANK_ATTR(F, 4, 4, 2, 2)
  MVAMG_LEANK_ATTR_F(true) MVAMG_LEANK_ATTR_F(false)
#undef MVAMG_LEANK_ATTR_F
#undef MVAMG_LEANK_ATTR
#undef MVAMG_LEAN_ATTR_C
#undef MVAMG_LEAN_ATTR
  g_max_dyn_smem = ok ? maxsm : 48 * 1024;
  cudaGetLastError();
}

struct Csr {
  int n = 0, m = 0, nnz = 0;
  const int* ip = nullptr;
  const int* ix = nullptr;
  const double* v = nullptr;
};

struct GsPlan {
  int ntiles = 0, threads = 32, window = 0;
  const int* chain_ptr = nullptr;
  const int* tile_ptr = nullptr;     // tiles: ranges of the chain order
  const int* chain_order = nullptr;  // processing order of the chains (nullptr: natural)
  int wmask = -1;                    // window positions mod (wmask + 1); -1: whole chains
};

// Static round schedule of one sweep mode (0 forward from x = 0, 1 forward,
// 2 backward): round-major records, per-round offsets, per-warp round bases,
// per-tile warp bases, the row -> (round, lane) permutation and its rhs buffer.
struct GsList {
  int lean_C = 0;  // > 0: uniform records of 3 + 2C words, lean kernel
  const unsigned long long* rec = nullptr;
  const int* round_off = nullptr;
  const int* tbase = nullptr;
  const int* tile_wbase = nullptr;
  const int* perm = nullptr;
  double* tperm = nullptr;
  int R = 1, D = 2, slot_words = 0, rec_words_max = 0;
};

// Level-set schedule of one sweep mode for the single-CTA small-level kernel
// (0 forward from x = 0, 1 forward, 2 backward from x = 0, 3 backward).
struct GsLevels {
  int ncta = 1, rows_per_cta = 0;
  const int* lev_ptr = nullptr;
  const int* lev_eptr = nullptr;
  const GsLevelRow* rows = nullptr;
  const GsLevelEntry* ents = nullptr;
  const int* perm = nullptr;
  double* tperm = nullptr;
  int nlev = 0, max_rows = 0, max_ents = 0, threads = 256;
  int group = 1;  // lanes per row: 1 = bit-exact CSR order, 2..16 = tolerance parity
  int reg = 0;    // single CTA, group > 1: register-prefetch kernel (x only in shared memory)
};

// Streamed level-set schedule (gs_stream.cuh) of one sweep mode: one SM, x (and
// b) in shared memory, level packets through a TMA ring.
struct GsStream {
  int nstages = 0, nslots = 0, slot_bytes = 0, group = 1, ncta = 1;
  const unsigned char* blob = nullptr;
  const long long* stage_off = nullptr;
  double* tfold = nullptr;  // n doubles: folded right-hand side (mode-2 plan used from x_old)
};

// Dataflow row schedule (gs_row_kernel) of one sweep mode.
struct GsRows {
  int mode = 0, threads = 128, ctas = 0, max_tile_slots = 0;
  const int* rowid = nullptr;
  const int* cnt = nullptr;
  const int* crit = nullptr;
  const int* wofs = nullptr;
  const double* coef = nullptr;
  const int* src = nullptr;
  const double* dg = nullptr;
  const double* rdg = nullptr;
  const int* perm = nullptr;
  double* tperm = nullptr;
};

// Cluster dataflow schedule (gs_cluster_kernel) of one sweep mode
// (mvamg_gs_cluster_plan).
struct GsCluster {
  int mode = 0, ncta = 0, wpc = 0, slots = 0, page_bytes = 0, sleep_ns = 0, grid = 0;
  const int* wptr = nullptr;
  const int* wpage = nullptr;
  const unsigned char* blob = nullptr;
  const int* perm = nullptr;
  double* tperm = nullptr;
};

struct Smoother {
  int kind, sweeps;
  double omega;
};

// ---- raw launches ----------------------------------------------------------
// small levels with long rows: one warp per row (bit-identical, see spmv_warp_kernel)
inline bool warp_rows(const Csr& A) {
  return A.n > 0 && A.n <= kWarpRowMaxRows && (long long)A.nnz >= (long long)kWarpRowMinAvg * A.n;
}

// GS preparation (gs_prepare_kernel); the backward fold of a small long-row
// level runs one warp per row (bit-identical)
void launch_prepare(const Csr& A, const double* b, const double* xold, const int* perm, double* tperm,
                    double* xnew, int* ticket, int fold, cudaStream_t s) {
  const int n = A.n;
  // (one warp per row at any size was measured level with the thread-per-row fold on C5's
  // 2.86M- and 900k-row levels -- its CSR-order shuffle chain costs what the coalescing saves)
  if (fold && warp_rows(A)) {
    const int gw = std::max(1, std::min((n + 7) / 8, num_sms() * 8));
    gs_prepare_fold_warp_kernel<<<gw, 256, 0, s>>>(n, A.ip, A.ix, A.v, b, xold, perm, tperm, xnew, ticket);
  } else {
    gs_prepare_kernel<<<grid_for(n), 256, 0, s>>>(n, A.ip, A.ix, A.v, b, xold, perm, tperm, xnew, ticket, fold);
  }
}

bool g_spmv_stream = true;  // CSR-stream SpMV for the thread-per-row cases (mvamg_set_spmv_stream)

int launch_spmv(int mode, const Csr& A, const double* x, const double* b, double* y, cudaStream_t s) {
  if (A.n == 0) return 0;
  if (warp_rows(A)) {
    const int gw = std::max(1, std::min((A.n + 7) / 8, num_sms() * 8));
    if (mode == 0) spmv_warp_kernel<0><<<gw, 256, 0, s>>>(A.n, A.ip, A.ix, A.v, x, b, y);
    else if (mode == 1) spmv_warp_kernel<1><<<gw, 256, 0, s>>>(A.n, A.ip, A.ix, A.v, x, b, y);
    else spmv_warp_kernel<2><<<gw, 256, 0, s>>>(A.n, A.ip, A.ix, A.v, x, b, y);
    CUDA_TRY(cudaGetLastError());
    return 0;
  }
  if (g_spmv_stream) {
    // CSR-stream tiles of rpt rows sized so a tile's entries usually fit the buffer
    const double avg = A.nnz > 0 ? (double)A.nnz / A.n : 8.0;
    const int rpt = avg <= 11.0 ? 256 : (avg <= 23.0 ? 128 : (avg <= 47.0 ? 64 : 32));
    const long long tiles = ((long long)A.n + rpt - 1) / rpt;
    const int g = (int)std::max(1LL, std::min(tiles, (long long)num_sms() * 8));
    if (mode == 0) spmv_stream_kernel<0><<<g, 256, 0, s>>>(A.n, rpt, A.ip, A.ix, A.v, x, b, y);
    else if (mode == 1) spmv_stream_kernel<1><<<g, 256, 0, s>>>(A.n, rpt, A.ip, A.ix, A.v, x, b, y);
    else spmv_stream_kernel<2><<<g, 256, 0, s>>>(A.n, rpt, A.ip, A.ix, A.v, x, b, y);
    CUDA_TRY(cudaGetLastError());
    return 0;
  }
  int g = grid_for(A.n);
  if (mode == 0) spmv_kernel<0><<<g, 256, 0, s>>>(A.n, A.ip, A.ix, A.v, x, b, y);
  else if (mode == 1) spmv_kernel<1><<<g, 256, 0, s>>>(A.n, A.ip, A.ix, A.v, x, b, y);
  else spmv_kernel<2><<<g, 256, 0, s>>>(A.n, A.ip, A.ix, A.v, x, b, y);
  CUDA_TRY(cudaGetLastError());
  return 0;
}

size_t gs_smem_bytes(const GsPlan& p, const GsList& ls) {
  const int warps = p.threads / 32;
  size_t words = (size_t)((p.window + 1) & ~1) + (size_t)warps * ls.D * ls.slot_words;
  return words * 8 + (size_t)warps * ls.D * 8;  // + one mbarrier per slot
}

int gs_blocks(const GsPlan& p, const GsList& ls) {
  static std::map<std::pair<int, size_t>, int> occ_cache;
  size_t smem = gs_smem_bytes(p, ls);
  auto key = std::make_pair(p.threads, smem);
  auto it = occ_cache.find(key);
  int per_sm;
  if (it != occ_cache.end()) {
    per_sm = it->second;
  } else {
    per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gs_sweep_kernel<true, 4, 2>, p.threads, smem);
    if (per_sm < 1) per_sm = 1;
    occ_cache[key] = per_sm;
  }
  return std::max(1, std::min(p.ntiles, per_sm * num_sms()));
}

// Lean-kernel launch, optionally as thread-block clusters of `cluster` CTAs.
template <class Kern>
void launch_lean_k(Kern k, int g, int threads, size_t smem, cudaStream_t s, const GsArgs& a, int cluster) {
  if (cluster <= 1) {
    k<<<g, threads, smem, s>>>(a);
    return;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(std::max(cluster, (g / cluster) * cluster));
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k, a);
}

// One sweep: gs_prepare_kernel writes the right-hand side in (round, lane)
// order (folding the backward sweep's old upper neighbours), fills x_new with
// the sentinel and resets the ticket; gs_sweep_kernel then runs the schedule.
int launch_gs(bool fwd, const Csr& A, const GsList& ls, const GsPlan& p, const double* b,
              const double* xold, double* xnew, int* ticket, int* status, cudaStream_t s) {
  const int n = A.n;
  if (n == 0) return 0;
  if (!ls.rec) return fail(MVAMG_E_STATE, "gs: schedule for this sweep mode was not set");
  set_kernel_attrs();
  const size_t smem = gs_smem_bytes(p, ls);
  if (smem > (size_t)g_max_dyn_smem)
    return fail(MVAMG_E_ARG, "gs: shared memory plan of " + std::to_string(smem) + " bytes exceeds the limit");
  const int fold = (!fwd && xold != nullptr) ? 1 : 0;
  launch_prepare(A, b, xold, ls.perm, ls.tperm, xnew, ticket, fold, s);
  GsArgs a;
  a.n = n;
  a.ntiles = p.ntiles;
  a.window = p.window;
  a.slot_words = ls.slot_words;
  a.rec_words_max = ls.rec_words_max;
  a.rec = ls.rec;
  a.round_off = ls.round_off;
  a.tbase = ls.tbase;
  a.tile_wbase = ls.tile_wbase;
  a.chain_ptr = p.chain_ptr;
  a.tile_ptr = p.tile_ptr;
  a.chain_order = p.chain_order;
  a.wmask = p.wmask;
  a.tperm = ls.tperm;
  a.xold = xold;
  a.xnew = xnew;
  a.ticket = ticket;
  a.status = status;
  a.trace = g_gs_trace;
  a.debug = g_gs_debug;
  const int g = gs_blocks(p, ls);
  if (ls.lean_C > 0) {
    const int lc = ls.lean_C & 0xff, lk = (ls.lean_C >> 8) & 0xff, lcl = (ls.lean_C >> 16) & 0xff;
    if (lk > 1) {  // K rows per lane per round (C <= 4; (R, D, K) in {(2,2,4), (2,3,4), (4,2,2)})
#define MVAMG_LEANK(F, RR, DD, KK)                                                \
  do {                                                                            \
    if (lc <= 2) launch_lean_k(gs_lean_kernel<F, 2, RR, DD, KK>, g, p.threads, smem, s, a, 0); \
    else launch_lean_k(gs_lean_kernel<F, 4, RR, DD, KK>, g, p.threads, smem, s, a, 0);         \
  } while (0)
#define MVAMG_LEANK_F(F)                                                          \
  do {                                                                            \
    if (lk == 4 && ls.D >= 3) MVAMG_LEANK(F, 2, 3, 4);                            \
    else if (lk == 4) MVAMG_LEANK(F, 2, 2, 4);                                    \
    else MVAMG_LEANK(F, 4, 2, 2);                                                 \
  } while (0)
      if (fwd) MVAMG_LEANK_F(true); else MVAMG_LEANK_F(false);
#undef MVAMG_LEANK_F
#undef MVAMG_LEANK
      CUDA_TRY(cudaGetLastError());
      return 0;
    }
#define MVAMG_LEAN(F, CC, RR, DD)                                                                   \
  do {                                                                                             \
    if (lcl > 1) launch_lean_k(gs_lean_kernel<F, CC, RR, DD, 1, true>, g, p.threads, smem, s, a, lcl); \
    else launch_lean_k(gs_lean_kernel<F, CC, RR, DD, 1, false>, g, p.threads, smem, s, a, 0);         \
  } while (0)
#define MVAMG_LEAN_C(F, RR, DD)                                                   \
  do {                                                                            \
    if (lc <= 2) MVAMG_LEAN(F, 2, RR, DD);                                        \
    else if (lc <= 4) MVAMG_LEAN(F, 4, RR, DD);                                   \
    else MVAMG_LEAN(F, 8, RR, DD);                                                \
  } while (0)
#define MVAMG_LEAN_R(F)                                                           \
  do {                                                                            \
    if (ls.R >= 8 && ls.D >= 3) MVAMG_LEAN_C(F, 8, 3);                            \
    else if (ls.R >= 8) MVAMG_LEAN_C(F, 8, 2);                                    \
    else if (ls.R >= 4 && ls.D >= 4) MVAMG_LEAN_C(F, 4, 4);                       \
    else if (ls.R >= 4) MVAMG_LEAN_C(F, 4, 2);                                    \
    else if (ls.R >= 2 && ls.D >= 8) MVAMG_LEAN_C(F, 2, 8);                       \
    else if (ls.R >= 2) MVAMG_LEAN_C(F, 2, 2);                                    \
    else MVAMG_LEAN_C(F, 1, 8);                                                   \
  } while (0)
    if (fwd) MVAMG_LEAN_R(true); else MVAMG_LEAN_R(false);
#undef MVAMG_LEAN_R
#undef MVAMG_LEAN_C
#undef MVAMG_LEAN
    CUDA_TRY(cudaGetLastError());
    return 0;
  }
#define MVAMG_GS_LAUNCH(F, RR, DD) gs_sweep_kernel<F, RR, DD><<<g, p.threads, smem, s>>>(a)
#define MVAMG_GS_LAUNCH_D(F, RR)                                     \
  do {                                                               \
    if (ls.D >= 8) MVAMG_GS_LAUNCH(F, RR, 8);                        \
    else if (ls.D >= 4) MVAMG_GS_LAUNCH(F, RR, 4);                   \
    else MVAMG_GS_LAUNCH(F, RR, 2);                                  \
  } while (0)
  if (fwd) {
    if (ls.R >= 8) MVAMG_GS_LAUNCH_D(true, 8); else if (ls.R >= 4) MVAMG_GS_LAUNCH_D(true, 4);
    else if (ls.R >= 2) MVAMG_GS_LAUNCH_D(true, 2); else MVAMG_GS_LAUNCH_D(true, 1);
  } else {
    if (ls.R >= 8) MVAMG_GS_LAUNCH_D(false, 8); else if (ls.R >= 4) MVAMG_GS_LAUNCH_D(false, 4);
    else if (ls.R >= 2) MVAMG_GS_LAUNCH_D(false, 2); else MVAMG_GS_LAUNCH_D(false, 1);
  }
#undef MVAMG_GS_LAUNCH_D
#undef MVAMG_GS_LAUNCH
  CUDA_TRY(cudaGetLastError());
  return 0;
}

size_t gs_level_smem(const GsLevels& g) {
  const size_t xw = (size_t)((g.rows_per_cta + 1) & ~1);
  const size_t buf = (size_t)g.max_rows * 32 + (size_t)g.max_ents * 16 + (((size_t)(g.max_rows + 2) * 8 + 15) & ~(size_t)15);
  return xw * 8 + 3 * buf;
}

// gs_stream_kernel on one SM.  with_old: x starts at x_old and b is kept in
// shared memory too (every off-diagonal entry is in the plan); otherwise x
// starts at b (a sweep from x = 0).
long long* g_stream_trace = nullptr;  // diagnostics: mvamg_gs_stream_set_trace
int g_stream_trace_cap = 0;

size_t gs_stream_smem(int n, int with_old, const GsStream& g) {
  const int R = g.ncta > 1 ? (n + g.ncta - 1) / g.ncta : n;
  const size_t xw = (size_t)((R + 1) & ~1);
  return xw * 8 * (with_old ? 2 : 1) + (size_t)g.nslots * (size_t)g.slot_bytes;
}

int launch_gs_stream(int n, const GsStream& g, int with_old, const double* b, const double* xold, double* xnew,
                     cudaStream_t s) {
  if (n == 0) return 0;
  static bool attr = false;
  if (!attr) {
    attr = true;
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
#define MVAMG_STREAM_ATTR(GG)                                                                                 \
  cudaFuncSetAttribute(gs_stream_kernel<GG, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - 1024); \
  cudaFuncSetAttribute(gs_stream_kernel<GG, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - 1024);  \
  cudaFuncSetAttribute(gs_stream_kernel<GG, true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    MVAMG_STREAM_ATTR(1) MVAMG_STREAM_ATTR(2) MVAMG_STREAM_ATTR(4) MVAMG_STREAM_ATTR(8) MVAMG_STREAM_ATTR(16)
#undef MVAMG_STREAM_ATTR
    cudaGetLastError();
  }
  if (g.nslots < 1 || g.nslots > 8 || g.slot_bytes < 64 || (g.slot_bytes & 127))
    return fail(MVAMG_E_ARG, "gs stream: 1..8 slots of a multiple of 128 bytes");
  if (g.ncta < 1 || g.ncta > 16 || (g.ncta > 1 && with_old))
    return fail(MVAMG_E_ARG, "gs stream: clusters of 1..16 CTAs, zero-guess plans only");
  if (with_old && !xold) return fail(MVAMG_E_ARG, "gs stream: sweep from x_old without x_old");
  const size_t smem = gs_stream_smem(n, with_old, g);
  if (smem > (size_t)g_max_dyn_smem) return fail(MVAMG_E_ARG, "gs stream: x, b and the ring exceed shared memory");
  GsStreamArgs a;
  a.n = n;
  a.with_old = with_old;
  a.nstages = g.nstages;
  a.nslots = g.nslots;
  a.slot_bytes = g.slot_bytes;
  a.blob = g.blob;
  a.stage_off = g.stage_off;
  a.b = b;
  a.xold = xold;
  a.xnew = xnew;
  a.rows_per_cta = g.ncta > 1 ? (n + g.ncta - 1) / g.ncta : n;
  a.trace = g_stream_trace;
  a.trace_cap = g_stream_trace_cap;
  void (*kern)(GsStreamArgs) = nullptr;
  const bool clu = g.ncta > 1;
  switch (g.group) {
    case 1: kern = clu ? gs_stream_kernel<1, true> : gs_stream_kernel<1, false>; break;
    case 2: kern = clu ? gs_stream_kernel<2, true> : gs_stream_kernel<2, false>; break;
    case 4: kern = clu ? gs_stream_kernel<4, true> : gs_stream_kernel<4, false>; break;
    case 8: kern = clu ? gs_stream_kernel<8, true> : gs_stream_kernel<8, false>; break;
    case 16: kern = clu ? gs_stream_kernel<16, true> : gs_stream_kernel<16, false>; break;
    default: return fail(MVAMG_E_ARG, "gs stream: lanes per row must be 1, 2, 4, 8 or 16");
  }
  if (!clu) {
    kern<<<1, kStreamThreads, smem, s>>>(a);
  } else {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)g.ncta);
    cfg.blockDim = dim3(kStreamThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)g.ncta;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, a));
  }
  CUDA_TRY(cudaGetLastError());
  return 0;
}

bool g_level_attr = false;
int launch_gs_levels(const Csr& A, const GsLevels& g, bool zero, const double* b, const double* xold,
                     double* xnew, int* ticket, cudaStream_t s, bool fold = false) {
  const int n = A.n;
  if (n == 0) return 0;
  if (!g_level_attr) {
    g_level_attr = true;
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
#define MVAMG_LEVEL_ATTR(GG)                                                                              \
  cudaFuncSetAttribute(gs_level_kernel<false, GG>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - 1024); \
  cudaFuncSetAttribute(gs_level_kernel<true, GG>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - 1024);  \
  cudaFuncSetAttribute(gs_level_kernel<true, GG>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    MVAMG_LEVEL_ATTR(1) MVAMG_LEVEL_ATTR(2) MVAMG_LEVEL_ATTR(4) MVAMG_LEVEL_ATTR(8) MVAMG_LEVEL_ATTR(16)
#undef MVAMG_LEVEL_ATTR
    cudaGetLastError();
  }
  const size_t smem = gs_level_smem(g);
  const bool reg_path = g.ncta == 1 && g.group > 1 && g.reg;
  if (reg_path ? (size_t)(n + 2 + g.max_ents + g.nlev) * 8 > (size_t)g_max_dyn_smem + 1024
               : smem > (size_t)g_max_dyn_smem)
    return fail(MVAMG_E_ARG, "gs levels: shared memory plan too large");
  if (g.ncta < 1 || g.ncta > 16) return fail(MVAMG_E_ARG, "gs levels: cluster of 1..16 CTAs");
  // right-hand side in the schedule's row layout; a backward sweep from a
  // nonzero guess folds its old upper neighbours here and then runs the
  // zero-guess schedule (only new values are read during the sweep)
  launch_prepare(A, b, xold, g.perm, g.tperm, xnew, ticket, fold ? 1 : 0, s);
  GsLevelArgs a;
  a.n = n;
  a.nlev = g.nlev;
  a.zero_init = (zero || fold) ? 1 : 0;
  a.max_rows = g.max_rows;
  a.max_ents = g.max_ents;
  a.rows_per_cta = g.rows_per_cta;
  a.lev_ptr = g.lev_ptr;
  a.lev_eptr = g.lev_eptr;
  a.rows = g.rows;
  a.ents = g.ents;
  a.tperm = g.tperm;
  a.xold = xold;
  a.xnew = xnew;
  if (g.group != 1 && g.group != 2 && g.group != 4 && g.group != 8 && g.group != 16)
    return fail(MVAMG_E_ARG, "gs levels: lanes per row must be 1, 2, 4, 8 or 16");
  if (g.ncta == 1 && g.group > 1 && g.reg) {
    // tolerance parity, x in shared memory, entries prefetched into registers
    static bool reg_attr = false;
    if (!reg_attr) {
      reg_attr = true;
      int dev = 0, optin = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
      cudaFuncSetAttribute(gs_level_reg_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
      cudaFuncSetAttribute(gs_level_reg_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
      cudaFuncSetAttribute(gs_level_reg_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
      cudaFuncSetAttribute(gs_level_reg_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
      cudaGetLastError();
    }
    const int T = kRegThreads;
    if ((long long)g.max_ents > (long long)T * kRegEnts)
      return fail(MVAMG_E_ARG, "gs levels (register path): a level exceeds 512 * 8 entries");
    const size_t xs = ((size_t)(n + 1) & ~(size_t)1) * 8 + (size_t)g.max_ents * 8 + (size_t)(g.nlev + 1) * 8;
    switch (g.group) {
      case 2: gs_level_reg_kernel<2><<<1, T, xs, s>>>(a); break;
      case 4: gs_level_reg_kernel<4><<<1, T, xs, s>>>(a); break;
      case 8: gs_level_reg_kernel<8><<<1, T, xs, s>>>(a); break;
      default: gs_level_reg_kernel<16><<<1, T, xs, s>>>(a); break;
    }
    CUDA_TRY(cudaGetLastError());
    return 0;
  }
  if (g.ncta == 1) {
    switch (g.group) {
      case 1: gs_level_kernel<false, 1><<<1, g.threads, smem, s>>>(a); break;
      case 2: gs_level_kernel<false, 2><<<1, g.threads, smem, s>>>(a); break;
      case 4: gs_level_kernel<false, 4><<<1, g.threads, smem, s>>>(a); break;
      case 8: gs_level_kernel<false, 8><<<1, g.threads, smem, s>>>(a); break;
      default: gs_level_kernel<false, 16><<<1, g.threads, smem, s>>>(a); break;
    }
    CUDA_TRY(cudaGetLastError());
    return 0;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(g.ncta);
  cfg.blockDim = dim3(g.threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = g.ncta;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  switch (g.group) {
    case 1: CUDA_TRY(cudaLaunchKernelEx(&cfg, gs_level_kernel<true, 1>, a)); break;
    case 2: CUDA_TRY(cudaLaunchKernelEx(&cfg, gs_level_kernel<true, 2>, a)); break;
    case 4: CUDA_TRY(cudaLaunchKernelEx(&cfg, gs_level_kernel<true, 4>, a)); break;
    case 8: CUDA_TRY(cudaLaunchKernelEx(&cfg, gs_level_kernel<true, 8>, a)); break;
    default: CUDA_TRY(cudaLaunchKernelEx(&cfg, gs_level_kernel<true, 16>, a)); break;
  }
  return 0;
}

bool g_row_attr = false;
// Dataflow row sweep: prepare (rhs in position order, fold, sentinel fill,
// ticket reset), then gs_row_kernel on `ctas` resident CTAs (0 = one per SM).
int launch_gs_rows(const Csr& A, const GsRows& g, const double* b, const double* xold, double* xnew,
                   int* ticket, int* status, cudaStream_t s) {
  const int n = A.n;
  if (n == 0) return 0;
  if (!g.rowid) return fail(MVAMG_E_STATE, "gs rows: schedule for this sweep mode was not set");
  set_kernel_attrs();
  if (g.threads < 32 || g.threads > 128 || g.threads % 32) return fail(MVAMG_E_ARG, "gs rows: threads must be 32..128");
  bool fold = false;
  if (xold) {
    if (g.mode == 2) fold = true;
    else if (g.mode == 0) return fail(MVAMG_E_ARG, "gs rows: zero-guess forward schedule with x_old");
  } else if (g.mode == 1 || g.mode == 3) {
    return fail(MVAMG_E_ARG, "gs rows: schedule needs x_old");
  }
  if (!g_row_attr) {
    g_row_attr = true;
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncSetAttribute(gs_row_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - 1024);
    cudaFuncSetAttribute(gs_row_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - 1024);
    cudaGetLastError();
  }
  const size_t smem = (size_t)g.max_tile_slots * 384;
  if (smem > (size_t)g_max_dyn_smem) return fail(MVAMG_E_ARG, "gs rows: tile slices exceed shared memory");
  launch_prepare(A, b, xold, g.perm, g.tperm, xnew, ticket, fold ? 1 : 0, s);
  GsRowArgs a;
  a.n = n;
  a.ntiles = (n + g.threads - 1) / g.threads;
  a.rowid = g.rowid;
  a.cnt = g.cnt;
  a.crit = g.crit;
  a.wofs = g.wofs;
  a.coef = g.coef;
  a.src = g.src;
  a.dg = g.dg;
  a.rdg = g.rdg;
  a.tperm = g.tperm;
  a.xold = xold;
  a.xnew = xnew;
  a.ticket = ticket;
  a.status = status;
  a.trace = g_gs_trace;
  a.debug = g_row_sleep;
  a.mirror_ptr = nullptr;
  a.mirror_dst = nullptr;
  a.peers = nullptr;
  a.sys = 0;
  const int grid = std::max(1, std::min(a.ntiles, g.ctas > 0 ? g.ctas : num_sms()));
  if (g.mode == 1 || g.mode == 3) gs_row_kernel<true><<<grid, g.threads, smem, s>>>(a);
  else gs_row_kernel<false><<<grid, g.threads, smem, s>>>(a);
  CUDA_TRY(cudaGetLastError());
  return 0;
}


bool g_cluster_attr = false;
// Cluster dataflow sweep: prepare (rhs in position order, fold), then ONE
// thread-block cluster of g.ncta CTAs x g.wpc worker warps with x in its
// distributed shared memory.
int launch_gs_cluster(const Csr& A, const GsCluster& g, const double* b, const double* xold, double* xnew,
                      int* ticket, int* status, cudaStream_t s) {
  const int n = A.n;
  if (n == 0) return 0;
  if (!g.blob) return fail(MVAMG_E_STATE, "gs cluster: plan for this sweep mode was not set");
  set_kernel_attrs();
  if (g.grid ? (g.ncta < 1 || g.ncta > num_sms()) : (g.ncta < 1 || g.ncta > 16 || (g.ncta & (g.ncta - 1))))
    return fail(MVAMG_E_ARG, "gs cluster: 1, 2, 4, 8 or 16 CTAs (grid form: 1 .. the number of SMs)");
  if (g.wpc < 1 || g.wpc > 32) return fail(MVAMG_E_ARG, "gs cluster: 1..32 worker warps per CTA");
  bool fold = false;
  if (xold) {
    if (g.mode == 2) fold = true;
    else if (g.mode == 0) return fail(MVAMG_E_ARG, "gs cluster: zero-guess forward schedule with x_old");
  } else if (g.mode == 1 || g.mode == 3) {
    return fail(MVAMG_E_ARG, "gs cluster: schedule needs x_old");
  }
  if (!g_cluster_attr) {
    g_cluster_attr = true;
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncSetAttribute(gs_cluster_kernel<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - 1024);
    cudaFuncSetAttribute(gs_cluster_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - 1024);
    cudaFuncSetAttribute(gs_cluster_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - 1024);
    cudaFuncSetAttribute(gs_cluster_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - 1024);
    cudaFuncSetAttribute(gs_cluster_kernel<false, false>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(gs_cluster_kernel<true, false>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaGetLastError();
  }
  if (g.page_bytes < 128 || g.page_bytes % 128) return fail(MVAMG_E_ARG, "gs cluster: pages of a multiple of 128 bytes");
  // x slice | wpc rings of kClusterRing pages | their mbarriers
  const size_t smem = (((size_t)g.slots * 8 + 127) & ~(size_t)127) +
                      (size_t)g.wpc * kClusterRing * ((size_t)g.page_bytes + 8);
  if (smem > (size_t)g_max_dyn_smem) return fail(MVAMG_E_ARG, "gs cluster: x slice and page rings exceed shared memory");
  launch_prepare(A, b, xold, g.perm, g.tperm, xnew, ticket, fold ? 1 : 0, s);
  GsClusterArgs a;
  a.n = n;
  a.wpc = g.wpc;
  a.slots = g.slots;
  a.page_bytes = g.page_bytes;
  a.wptr = g.wptr;
  a.wpage = g.wpage;
  a.blob = g.blob;
  a.tperm = g.tperm;
  a.xold = xold;
  a.xnew = xnew;
  a.status = status;
  a.trace = g_gs_trace;
  a.sleep_ns = g_cluster_sleep >= 0 ? g_cluster_sleep : g.sleep_ns;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(g.ncta);
  cfg.blockDim = dim3(g.wpc * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = g.ncta;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (g.grid) {  // ordinary CTAs, all resident; x_new (sentinel-filled by the prepare kernel) carries the early inputs
    if (g.mode == 1 || g.mode == 3) gs_cluster_kernel<true, true><<<g.ncta, g.wpc * 32, smem, s>>>(a);
    else gs_cluster_kernel<false, true><<<g.ncta, g.wpc * 32, smem, s>>>(a);
    CUDA_TRY(cudaGetLastError());
    return 0;
  }
  if (g.mode == 1 || g.mode == 3) CUDA_TRY(cudaLaunchKernelEx(&cfg, gs_cluster_kernel<true, false>, a));
  else CUDA_TRY(cudaLaunchKernelEx(&cfg, gs_cluster_kernel<false, false>, a));
  return 0;
}

}  // namespace

// ============================================================================
// Hierarchy
// ============================================================================
struct Level {
  Csr A;
  const double* diag = nullptr;
  const double* rdiag = nullptr;
  GsPlan plan;
  GsList gl[3];
  GsStream gss[4];  // streamed single-SM schedules (used first when set)
  GsLevels glv[4];  // small-level single-CTA schedules (used when set)
  GsRows grw[4];    // dataflow row schedules (used when set and glv is not)
  GsCluster gcl[4]; // cluster dataflow schedules (used first when set)
  Csr P, R;  // valid for k < L-1
  double *xa = nullptr, *xb = nullptr, *t = nullptr, *r = nullptr, *z = nullptr;
  double *fr = nullptr, *fx = nullptr, *fp[2] = {nullptr, nullptr}, *fap[2] = {nullptr, nullptr};
  FcgScalars* fs = nullptr;
};

struct mvamg_hierarchy {
  int L = 0, kind = 0, inner = 2;
  Smoother pre{MVAMG_GS_FORWARD, 1, 1.0}, post{MVAMG_GS_BACKWARD, 1, 1.0};
  std::vector<Level> lv;
  const double* inv = nullptr;
  bool bound = false, use_graphs = true;
  // workspace carve-outs
  double* partials = nullptr;
  unsigned* counter = nullptr;
  int* ticket = nullptr;
  DevScalars* sc = nullptr;
  double *px = nullptr, *pr = nullptr, *pp = nullptr, *pq = nullptr, *pt = nullptr, *pu = nullptr,
         *pz = nullptr, *in = nullptr;
  DevScalars* host_sc = nullptr;  // pinned mirror
  std::map<std::string, cudaGraphExec_t> graphs;
  std::map<std::string, int> graph_kernels;

  ReduceCtx ctx(FcgScalars* fs = nullptr, double* out = nullptr) const {
    ReduceCtx c;
    c.partials = partials;
    c.counter = counter;
    c.sc = sc;
    c.fs = fs;
    c.out = out;
    return c;
  }
  int* status_ptr() const { return reinterpret_cast<int*>(reinterpret_cast<char*>(sc) + offsetof(DevScalars, status)); }
  bool fcg_level(int k) const { return kind == MVAMG_CYCLE_K && inner >= 1 && k >= 1 && k < L - 1; }

  ~mvamg_hierarchy() {
    for (auto& kv : graphs) cudaGraphExecDestroy(kv.second);
    if (host_sc) cudaFreeHost(host_sc);
  }

  // ---- smoothing (cycles.py:139-148) ----------------------------------------
  // x_cur holds the current iterate (nullptr == zero).  Returns the buffer with
  // the smoothed iterate (one of xa / xb).
  int smooth(const Smoother& sp, int k, const double* b, double*& x_cur, cudaStream_t s) {
    Level& l = lv[k];
    int st;
    if (sp.sweeps == 0 && x_cur == nullptr) {
      zero_kernel<<<grid_for(l.A.n), 256, 0, s>>>(l.A.n, l.xa);
      x_cur = l.xa;
      return 0;
    }
    for (int it = 0; it < sp.sweeps; ++it) {
      double* out = (x_cur == l.xa) ? l.xb : l.xa;
      if (sp.kind == MVAMG_WEIGHTED_JACOBI) {
        if (x_cur == nullptr) {
          zero_kernel<<<grid_for(l.A.n), 256, 0, s>>>(l.A.n, l.xb);
          x_cur = l.xb;
          out = l.xa;
        }
        jacobi_kernel<<<grid_for(l.A.n), 256, 0, s>>>(l.A.n, l.A.ip, l.A.ix, l.A.v, l.diag, b,
                                                       sp.omega, x_cur, out);
      } else {
        bool fwd = sp.kind == MVAMG_GS_FORWARD;
        int lmode = (fwd ? 0 : 2) + (x_cur == nullptr ? 0 : 1);
        if (l.gcl[lmode].blob) {
          st = launch_gs_cluster(l.A, l.gcl[lmode], b, x_cur, out, ticket, status_ptr(), s);
        } else if (!fwd && x_cur != nullptr && l.gcl[2].blob) {  // folded backward sweep from x_old
          st = launch_gs_cluster(l.A, l.gcl[2], b, x_cur, out, ticket, status_ptr(), s);
        } else if (l.gss[lmode].nstages) {
          st = launch_gs_stream(l.A.n, l.gss[lmode], x_cur != nullptr, b, x_cur, out, s);
        } else if (!fwd && x_cur != nullptr && l.gss[2].nstages && l.gss[2].tfold) {
          // backward from x_old with the zero-guess plan: fold the old lower
          // neighbours into the right-hand side first (same roundings, CSR order)
          launch_prepare(l.A, b, x_cur, nullptr, l.gss[2].tfold, out, ticket, 1, s);
          st = launch_gs_stream(l.A.n, l.gss[2], 0, l.gss[2].tfold, nullptr, out, s);
        } else if (!fwd && x_cur != nullptr && l.glv[2].rows) {
          st = launch_gs_levels(l.A, l.glv[2], false, b, x_cur, out, ticket, s, /*fold=*/true);
        } else if (l.glv[lmode].rows) {
          st = launch_gs_levels(l.A, l.glv[lmode], x_cur == nullptr, b, x_cur, out, ticket, s);
        } else if (!fwd && x_cur != nullptr && l.grw[2].rowid) {
          st = launch_gs_rows(l.A, l.grw[2], b, x_cur, out, ticket, status_ptr(), s);
        } else if (l.grw[lmode].rowid) {
          st = launch_gs_rows(l.A, l.grw[lmode], b, x_cur, out, ticket, status_ptr(), s);
        } else {
          int mode = fwd ? (x_cur == nullptr ? 0 : 1) : 2;
          st = launch_gs(fwd, l.A, l.gl[mode], l.plan, b, x_cur, out, ticket, status_ptr(), s);
        }
        if (st) return st;
      }
      x_cur = out;
    }
    return 0;
  }

  // ---- coarsest solve --------------------------------------------------------
  int coarse(const double* r, const double*& out, cudaStream_t s) {
    Level& l = lv[L - 1];
    int n = l.A.n;
    int g = std::max(1, std::min((n * 32 + 255) / 256, num_sms() * 8));
    gemv_kernel<<<g, 256, 0, s>>>(n, inv, r, l.z);
    out = l.z;
    return 0;
  }

  // ---- recursive cycle (cycles.py:150-172) ------------------------------------
  int descend(int k, const double* r, const double*& out, cudaStream_t s) {
    if (k == L - 1) return coarse(r, out, s);
    Level& l = lv[k];
    Level& c = lv[k + 1];
    double* x = nullptr;
    int st = smooth(pre, k, r, x, s);
    if (st) return st;
    if ((st = launch_spmv(1, l.A, x, r, l.t, s))) return st;     // t = r - A x
    if ((st = launch_spmv(0, l.R, l.t, nullptr, c.r, s))) return st;  // rc = R t
    const double* xc = nullptr;
    if (fcg_level(k + 1)) st = fcg(k + 1, c.r, xc, s);
    else st = descend(k + 1, c.r, xc, s);
    if (st) return st;
    if ((st = launch_spmv(2, l.P, xc, nullptr, x, s))) return st;  // x += P xc
    st = smooth(post, k, r, x, s);
    out = x;
    return st;
  }

  // ---- FCG with a fixed step count, x0 = 0 (krylov.py:75-107) -----------------
  int fcg(int k, const double* b, const double*& out, cudaStream_t s) {
    Level& l = lv[k];
    int n = l.A.n, g = grid_for(n), st;
    copy_kernel<<<g, 256, 0, s>>>(n, l.fr, b);
    int cur = 0;
    for (int it = 0; it < inner; ++it) {
      const double* z = nullptr;
      if ((st = descend(k, l.fr, z, s))) return st;
      double* p = l.fp[cur];
      double* ap = l.fap[cur];
      if (it > 0) {
        dot2_kernel<<<dot_grid(n), 256, 0, s>>>(n, z, l.fap[cur ^ 1], nullptr, nullptr,
                                                POST_FCG_BETA, ctx(l.fs));
      }
      fcg_p_kernel<<<g, 256, 0, s>>>(n, p, z, l.fp[cur ^ 1], l.fs, it == 0);
      if (warp_rows(l.A))
        spmv_dot_warp_kernel<<<std::min((n + 7) / 8, kDotMaxBlocks), 256, 0, s>>>(
            n, l.A.ip, l.A.ix, l.A.v, p, l.fr, ap, POST_FCG_ALPHA, ctx(l.fs));
      else
        spmv_dot_kernel<<<dot_grid(n), 256, 0, s>>>(n, l.A.ip, l.A.ix, l.A.v, p, l.fr, ap,
                                                    POST_FCG_ALPHA, ctx(l.fs));
      fcg_xr_kernel<<<g, 256, 0, s>>>(n, l.fx, l.fr, p, ap, l.fs, it == 0);
      cur ^= 1;
    }
    CUDA_TRY(cudaGetLastError());
    out = l.fx;
    return 0;
  }

  // z = B r for the level-0 cycle.  `r` must stay valid while the sequence runs.
  int cycle(const double* r, const double*& out, cudaStream_t s) {
    if (L == 1) return coarse(r, out, s);
    return descend(0, r, out, s);
  }

  // ---- graph helper ----------------------------------------------------------
  template <class F>
  int run_graph(const std::string& key, cudaStream_t s, F&& body) {
    if (!use_graphs) return body(s);
    auto it = graphs.find(key);
    if (it == graphs.end()) {
      cudaStream_t cs;
      CUDA_TRY(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
      CUDA_TRY(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
      int st = body(cs);
      cudaGraph_t graph;
      cudaError_t e = cudaStreamEndCapture(cs, &graph);
      cudaStreamDestroy(cs);
      if (st) return st;
      if (e != cudaSuccess) return fail(MVAMG_E_CUDA, std::string("graph capture: ") + cudaGetErrorString(e));
      size_t nn = 0;
      cudaGraphGetNodes(graph, nullptr, &nn);
      std::vector<cudaGraphNode_t> nodes(nn);
      if (nn) cudaGraphGetNodes(graph, nodes.data(), &nn);
      int nk = 0;
      for (auto nd : nodes) {
        cudaGraphNodeType ty;
        if (cudaGraphNodeGetType(nd, &ty) == cudaSuccess && ty == cudaGraphNodeTypeKernel) ++nk;
      }
      cudaGraphExec_t exec;
      e = cudaGraphInstantiate(&exec, graph, 0);
      cudaGraphDestroy(graph);
      if (e != cudaSuccess) return fail(MVAMG_E_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(e));
      it = graphs.emplace(key, exec).first;
      graph_kernels[key] = nk;
    }
    CUDA_TRY(cudaGraphLaunch(it->second, s));
    g_kernel_launches += graph_kernels[key];
    return 0;
  }
};

// Graphs that replay a composite are cached on its first component's
// hierarchy, which usually outlives the composite (the bootstrap builds a new
// composite per stage over the same components).  They are keyed by a serial
// number, never by the composite's address: a new composite allocated at a
// freed one's address must not replay the old graph (stale component list and
// freed buffers -- an intermittent wrong result or illegal address).
unsigned long long g_composite_serial = 0;

struct mvamg_composite {
  std::vector<mvamg_hierarchy*> ops;
  double *t = nullptr, *acc = nullptr;
  int n = 0;
  unsigned long long serial = 0;
  std::map<std::string, cudaGraphExec_t> graphs;
  ~mvamg_composite() {
    for (auto& kv : graphs) cudaGraphExecDestroy(kv.second);
    if (t) cudaFree(t);
    if (acc) cudaFree(acc);
  }

  // x <- E_1..E_r E_r..E_1 x, E_i x = x - B_i (A x)   (bootstrap.py:98-113)
  int symmetrized(double* x, cudaStream_t s) {
    int r = (int)ops.size(), st;
    const Csr& A = ops[0]->lv[0].A;
    for (int pass = 0; pass < 2 * r; ++pass) {
      mvamg_hierarchy* h = ops[pass < r ? pass : 2 * r - 1 - pass];
      if ((st = launch_spmv(0, A, x, nullptr, t, s))) return st;
      const double* z = nullptr;
      if ((st = h->cycle(t, z, s))) return st;
      sub_kernel<<<grid_for(n), 256, 0, s>>>(n, x, x, z);
    }
    CUDA_TRY(cudaGetLastError());
    return 0;
  }

  // acc = Bsym r: acc = 0; for i in 1..r, r..1: acc += B_i (r - A acc)
  int precond(const double* r, const double*& out, cudaStream_t s) {
    int nops = (int)ops.size(), st;
    const Csr& A = ops[0]->lv[0].A;
    for (int pass = 0; pass < 2 * nops; ++pass) {
      mvamg_hierarchy* h = ops[pass < nops ? pass : 2 * nops - 1 - pass];
      const double* u = nullptr;
      if (pass == 0) {
        if ((st = h->cycle(r, u, s))) return st;
        copy_kernel<<<grid_for(n), 256, 0, s>>>(n, acc, u);
      } else {
        if ((st = launch_spmv(1, A, acc, r, t, s))) return st;  // t = r - A acc
        if ((st = h->cycle(t, u, s))) return st;
        add_kernel<<<grid_for(n), 256, 0, s>>>(n, acc, acc, u);
      }
    }
    CUDA_TRY(cudaGetLastError());
    out = acc;
    return 0;
  }
};

// ---- PCG (krylov.py:28-72) --------------------------------------------------
namespace {

int precond_apply(mvamg_hierarchy* h, int pc, mvamg_composite* comp, const double* r,
                  const double*& z, cudaStream_t s) {
  if (pc == MVAMG_PC_CYCLE) return h->cycle(r, z, s);
  if (pc == MVAMG_PC_COMPOSITE) return comp->precond(r, z, s);
  z = r;
  return 0;
}

int pcg_device(mvamg_hierarchy* h, int pc, mvamg_composite* comp, const double* b, double rtol,
               int itmax, double* hist, int* nit, int* converged, int* status, cudaStream_t s) {
  if (!h->bound) return fail(MVAMG_E_STATE, "workspace not bound");
  if (pc == MVAMG_PC_COMPOSITE && comp == nullptr) return fail(MVAMG_E_ARG, "composite preconditioner missing");
  const Level& l0 = h->lv[0];
  const Csr& A = l0.A;
  const int n = A.n, g = grid_for(n), gd = dot_grid(n);
  int st;
  pcg_setup_kernel<<<1, 1, 0, s>>>(h->sc, rtol, itmax, hist);
  copy_kernel<<<g, 256, 0, s>>>(n, h->pr, b);
  zero_kernel<<<g, 256, 0, s>>>(n, h->px);
  dot2_kernel<<<gd, 256, 0, s>>>(n, h->pr, h->pr, nullptr, nullptr, POST_PCG_R0, h->ctx());
  CUDA_TRY(cudaGetLastError());
  g_kernel_launches += 4;
  auto sync_flags = [&]() -> int {
    CUDA_TRY(cudaMemcpyAsync(h->host_sc, h->sc, sizeof(DevScalars), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    return 0;
  };
  if ((st = sync_flags())) return st;
  if (!h->host_sc->stop) {
    // z = M r ; rz = r'z ; p = z
    const std::string cid = comp ? std::to_string(comp->serial) : std::string("-");
    std::string key0 = "pcg0/" + std::to_string(pc) + "/" + cid;
    st = h->run_graph(key0, s, [&](cudaStream_t cs) -> int {
      const double* z = nullptr;
      int e = precond_apply(h, pc, comp, h->pr, z, cs);
      if (e) return e;
      dot2_kernel<<<gd, 256, 0, cs>>>(n, h->pr, z, nullptr, nullptr, POST_PCG_INIT, h->ctx());
      copy_kernel<<<g, 256, 0, cs>>>(n, h->pp, z);
      return 0;
    });
    if (st) return st;
    if ((st = sync_flags())) return st;
    std::string keyA = "pcgA", keyB = "pcgB/" + std::to_string(pc) + "/" + cid;
    while (!h->host_sc->stop) {
      // q = A p ; alpha = rz/p'q ; x += alpha p ; r -= alpha q ; hist ; stop test
      st = h->run_graph(keyA, s, [&](cudaStream_t cs) -> int {
        spmv_dot_kernel<<<gd, 256, 0, cs>>>(n, A.ip, A.ix, A.v, h->pp, nullptr, h->pq,
                                            POST_PCG_ALPHA, h->ctx());
        pcg_xr_kernel<<<gd, 256, 0, cs>>>(n, h->px, h->pr, h->pp, h->pq, h->ctx());
        return 0;
      });
      if (st) return st;
      if ((st = sync_flags())) return st;
      if (h->host_sc->stop) break;
      // z = M r ; beta = r'z/rz ; p = z + beta p
      st = h->run_graph(keyB, s, [&](cudaStream_t cs) -> int {
        const double* z = nullptr;
        int e = precond_apply(h, pc, comp, h->pr, z, cs);
        if (e) return e;
        dot2_kernel<<<gd, 256, 0, cs>>>(n, h->pr, z, nullptr, nullptr, POST_PCG_BETA, h->ctx());
        pcg_p_kernel<<<g, 256, 0, cs>>>(n, h->pp, z, h->sc);
        return 0;
      });
      if (st) return st;
    }
  }
  *nit = h->host_sc->k;
  *converged = h->host_sc->converged;
  *status = h->host_sc->status;
  return 0;
}


// ---------------------------------------------------------------------------
// Galerkin product on the device (galerkin.cuh)
// ---------------------------------------------------------------------------
// Device CSR owned by the library (intermediates and the returned A_c).
// Intermediates are stream-ordered allocations (cudaMallocAsync / cudaFreeAsync
// on the working stream), so freeing them never synchronises the device.
struct DevCsr {
  int n = 0, m = 0;
  long long nnz = 0;
  int* ip = nullptr;
  int* ix = nullptr;
  double* v = nullptr;
  cudaStream_t s = nullptr;
  void release() {
    for (void* p : {(void*)ip, (void*)ix, (void*)v})
      if (p) cudaFreeAsync(p, s);
    ip = ix = nullptr;
    v = nullptr;
  }
};

struct DevTmp {  // scoped stream-ordered allocation
  void* p = nullptr;
  cudaStream_t s = nullptr;
  explicit DevTmp(cudaStream_t st = nullptr) : s(st) {}
  cudaError_t alloc(size_t bytes) { return cudaMallocAsync(&p, bytes, s); }
  ~DevTmp() {
    if (p) cudaFreeAsync(p, s);
  }
  template <class T>
  T* get() const {
    return static_cast<T*>(p);
  }
};

#define GK_LAUNCH_CHECK()                                                         \
  do {                                                                            \
    ++g_kernel_launches;                                                          \
    cudaError_t e_ = cudaGetLastError();                                          \
    if (e_ != cudaSuccess) return fail(MVAMG_E_CUDA, std::string("galerkin: ") + cudaGetErrorString(e_)); \
  } while (0)

// offsets[0..n] = exclusive scan of cnt[0..n); *total = offsets[n].
int scan_counts(int n, const int* cnt, long long* offsets, long long* total, cudaStream_t s) {
  using namespace galerkin;
  const long long per = (long long)kScanThreads * kScanItems;
  const int nb = (int)(((long long)n + 1 + per - 1) / per);
  DevTmp bsum(s);
  CUDA_TRY(bsum.alloc((size_t)nb * 8));
  scan_blocks_kernel<<<nb, kScanThreads, 0, s>>>(n, cnt, offsets, bsum.get<long long>());
  GK_LAUNCH_CHECK();
  scan_sums_kernel<<<1, kScanThreads, 0, s>>>(nb, bsum.get<long long>());
  GK_LAUNCH_CHECK();
  scan_add_kernel<<<grid_for(n + 1), 256, 0, s>>>(n, offsets, bsum.get<long long>());
  GK_LAUNCH_CHECK();
  CUDA_TRY(cudaMemcpyAsync(total, offsets + n, 8, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  return 0;
}

int alloc_csr(DevCsr& C, int n, int m, long long nnz, const long long* offsets64, cudaStream_t s) {
  if (nnz >= 0x7fffffffLL) return fail(MVAMG_E_ARG, "galerkin: more than 2^31 - 1 nonzeros");
  C.n = n;
  C.m = m;
  C.nnz = nnz;
  C.s = s;
  CUDA_TRY(cudaMallocAsync((void**)&C.ip, (size_t)(n + 1) * 4, s));
  CUDA_TRY(cudaMallocAsync((void**)&C.ix, (size_t)std::max(nnz, 1LL) * 4, s));
  CUDA_TRY(cudaMallocAsync((void**)&C.v, (size_t)std::max(nnz, 1LL) * 8, s));
  galerkin::narrow_offsets_kernel<<<grid_for(n + 1), 256, 0, s>>>(n, offsets64, C.ip);
  GK_LAUNCH_CHECK();
  return 0;
}

// Stable transpose of an n x m CSR (rows of the result list source rows ascending).
int csr_transpose(int n, int m, const int* ip, const int* ix, const double* v, long long nnz, DevCsr& T,
                  cudaStream_t s) {
  using namespace galerkin;
  DevTmp cnt(s), off(s), cur(s), tix(s), tv(s);
  CUDA_TRY(cnt.alloc((size_t)(m + 1) * 4));
  CUDA_TRY(off.alloc((size_t)(m + 1) * 8));
  CUDA_TRY(cur.alloc((size_t)(m + 1) * 4));
  CUDA_TRY(tix.alloc((size_t)std::max(nnz, 1LL) * 4));
  CUDA_TRY(tv.alloc((size_t)std::max(nnz, 1LL) * 8));
  CUDA_TRY(cudaMemsetAsync(cnt.p, 0, (size_t)(m + 1) * 4, s));
  CUDA_TRY(cudaMemsetAsync(cur.p, 0, (size_t)(m + 1) * 4, s));
  if (nnz > 0) {
    col_count_kernel<<<grid_for((int)std::min(nnz, 1LL << 30)), 256, 0, s>>>(nnz, ix, cnt.get<int>());
    GK_LAUNCH_CHECK();
  }
  long long total = 0;
  if (int e = scan_counts(m, cnt.get<int>(), off.get<long long>(), &total, s)) return e;
  if (total != nnz) return fail(MVAMG_E_ARG, "galerkin: column index out of range");
  if (int e = alloc_csr(T, m, n, nnz, off.get<long long>(), s)) return e;
  if (nnz > 0) {
    transpose_scatter_kernel<<<grid_for(n * 32), 256, 0, s>>>(n, ip, ix, v, off.get<long long>(), cur.get<int>(),
                                                               tix.get<int>(), tv.get<double>());
    GK_LAUNCH_CHECK();
    segment_rank_sort_kernel<<<grid_for(m * 32), 256, 0, s>>>(m, off.get<long long>(), tix.get<int>(),
                                                               tv.get<double>(), T.ix, T.v);
    GK_LAUNCH_CHECK();
  }
  return 0;
}

// C = X @ Y in csr_matmat's summation order (galerkin.cuh), sorted, zeros dropped.
int spgemm_ordered(int nrows, int ncols, const int* xp, const int* xi, const double* xv, const int* yp,
                   const int* yi, const double* yv, DevCsr& C, cudaStream_t s) {
  using namespace galerkin;
  static bool attr = false;
  if (!attr) {
    CUDA_TRY(cudaFuncSetAttribute(spgemm_smem_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes));
    CUDA_TRY(cudaFuncSetAttribute(spgemm_smem_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes));
    attr = true;
  }
  DevTmp cnt(s), flag(s), rows(s), ctr(s), off(s);
  CUDA_TRY(cnt.alloc((size_t)(nrows + 1) * 4));
  CUDA_TRY(flag.alloc((size_t)nrows + 1));
  CUDA_TRY(rows.alloc((size_t)(nrows + 1) * 4));
  CUDA_TRY(ctr.alloc(16));
  CUDA_TRY(off.alloc((size_t)(nrows + 1) * 8));
  CUDA_TRY(cudaMemsetAsync(ctr.p, 0, 16, s));
  CUDA_TRY(cudaMemsetAsync(cnt.p, 0, (size_t)(nrows + 1) * 4, s));
  int* n_ovf = ctr.get<int>();
  int* max_ub = n_ovf + 1;
  const int grid = std::max(1, std::min((nrows + kWarps - 1) / kWarps, num_sms() * 4));
  if (nrows > 0) {
    spgemm_smem_kernel<false><<<grid, kWarps * 32, kSmemBytes, s>>>(nrows, xp, xi, xv, yp, yi, yv, cnt.get<int>(),
                                                                    flag.get<unsigned char>(), rows.get<int>(), n_ovf,
                                                                    max_ub, nullptr, nullptr, nullptr);
    GK_LAUNCH_CHECK();
  }
  int hctr[2] = {0, 0};
  CUDA_TRY(cudaMemcpyAsync(hctr, ctr.p, 8, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  const int novf = hctr[0];
  int H = 0, ggrid = 0;
  DevTmp pk(s), pv(s);
  if (novf > 0) {
    const long long need = std::min<long long>(std::max(hctr[1], 1), std::max(ncols, 1));
    H = 64;
    while (H < 2 * need) H <<= 1;
    long long nw = std::min<long long>(novf, (long long)num_sms() * 2 * kWarps);
    const long long cap = (1LL << 30) / ((long long)H * 28 * kWarps);  // pool <= 1 GiB
    nw = std::max<long long>(kWarps, std::min(nw, cap * kWarps));
    ggrid = (int)((nw + kWarps - 1) / kWarps);
    CUDA_TRY(pk.alloc((size_t)ggrid * kWarps * 3 * H * 4));
    CUDA_TRY(pv.alloc((size_t)ggrid * kWarps * 2 * H * 8));
    spgemm_global_kernel<false><<<ggrid, kWarps * 32, 0, s>>>(novf, rows.get<int>(), xp, xi, xv, yp, yi, yv, H,
                                                              pk.get<int>(), pv.get<double>(), cnt.get<int>(), nullptr,
                                                              nullptr, nullptr);
    GK_LAUNCH_CHECK();
  }
  long long total = 0;
  if (int e = scan_counts(nrows, cnt.get<int>(), off.get<long long>(), &total, s)) return e;
  if (int e = alloc_csr(C, nrows, ncols, total, off.get<long long>(), s)) return e;
  if (nrows > 0 && total > 0) {
    spgemm_smem_kernel<true><<<grid, kWarps * 32, kSmemBytes, s>>>(nrows, xp, xi, xv, yp, yi, yv, nullptr,
                                                                   flag.get<unsigned char>(), nullptr, nullptr, nullptr,
                                                                   off.get<long long>(), C.ix, C.v);
    GK_LAUNCH_CHECK();
    if (novf > 0) {
      spgemm_global_kernel<true><<<ggrid, kWarps * 32, 0, s>>>(novf, rows.get<int>(), xp, xi, xv, yp, yi, yv, H,
                                                               pk.get<int>(), pv.get<double>(), nullptr,
                                                               off.get<long long>(), C.ix, C.v);
      GK_LAUNCH_CHECK();
    }
  }
  return 0;
}

int galerkin_device(int n, int nc, Csr A, Csr P, DevCsr& S, cudaStream_t s, float* phase_ms) {
  using namespace galerkin;
  cudaEvent_t ev[5];
  for (auto& e : ev) CUDA_TRY(cudaEventCreate(&e));
  struct EvGuard {
    cudaEvent_t* e;
    ~EvGuard() {
      for (int i = 0; i < 5; ++i) cudaEventDestroy(e[i]);
    }
  } guard{ev};
  DevCsr R, AP, G, GT;
  struct CsrGuard {
    DevCsr* m[4];
    ~CsrGuard() {
      for (auto* x : m) x->release();
    }
  } cg{{&R, &AP, &G, &GT}};
  CUDA_TRY(cudaEventRecord(ev[0], s));
  if (int e = csr_transpose(n, nc, P.ip, P.ix, P.v, P.nnz, R, s)) return e;           // R = P^T
  CUDA_TRY(cudaEventRecord(ev[1], s));
  if (int e = spgemm_ordered(n, nc, A.ip, A.ix, A.v, P.ip, P.ix, P.v, AP, s)) return e;  // A P
  CUDA_TRY(cudaEventRecord(ev[2], s));
  if (int e = spgemm_ordered(nc, nc, R.ip, R.ix, R.v, AP.ip, AP.ix, AP.v, G, s)) return e;  // P^T (A P)
  CUDA_TRY(cudaEventRecord(ev[3], s));
  if (int e = csr_transpose(nc, nc, G.ip, G.ix, G.v, G.nnz, GT, s)) return e;
  DevTmp cnt(s), off(s);
  CUDA_TRY(cnt.alloc((size_t)(nc + 1) * 4));
  CUDA_TRY(off.alloc((size_t)(nc + 1) * 8));
  DevTmp gp(s), tp(s);  // int64 row offsets for the merge
  CUDA_TRY(gp.alloc((size_t)(nc + 1) * 8));
  CUDA_TRY(tp.alloc((size_t)(nc + 1) * 8));
  widen_offsets_kernel<<<grid_for(nc + 1), 256, 0, s>>>(nc, G.ip, gp.get<long long>());
  GK_LAUNCH_CHECK();
  widen_offsets_kernel<<<grid_for(nc + 1), 256, 0, s>>>(nc, GT.ip, tp.get<long long>());
  GK_LAUNCH_CHECK();
  symmetrize_kernel<false><<<grid_for(nc), 256, 0, s>>>(nc, gp.get<long long>(), G.ix, G.v, tp.get<long long>(),
                                                        GT.ix, GT.v, cnt.get<int>(), nullptr, nullptr, nullptr);
  GK_LAUNCH_CHECK();
  long long total = 0;
  if (int e = scan_counts(nc, cnt.get<int>(), off.get<long long>(), &total, s)) return e;
  if (int e = alloc_csr(S, nc, nc, total, off.get<long long>(), s)) return e;
  symmetrize_kernel<true><<<grid_for(nc), 256, 0, s>>>(nc, gp.get<long long>(), G.ix, G.v, tp.get<long long>(),
                                                       GT.ix, GT.v, nullptr, off.get<long long>(), S.ix, S.v);
  GK_LAUNCH_CHECK();
  CUDA_TRY(cudaEventRecord(ev[4], s));
  CUDA_TRY(cudaEventSynchronize(ev[4]));
  if (phase_ms)
    for (int i = 0; i < 4; ++i) CUDA_TRY(cudaEventElapsedTime(&phase_ms[i], ev[i], ev[i + 1]));
  return 0;
}
#undef GK_LAUNCH_CHECK
}  // namespace

// ============================================================================
// C ABI
// ============================================================================
extern "C" {

int mvamg_version(void) { return 1; }

int mvamg_gs_set_trace(long long* trace_dev) {
  g_gs_trace = trace_dev;
  return 0;
}

int mvamg_kernel_launches(long long* count, int reset) {
  if (count) *count = g_kernel_launches;
  if (reset) g_kernel_launches = 0;
  return 0;
}
const char* mvamg_last_error(void) { return g_err.c_str(); }

int mvamg_gs_analyse(int n, const int* indptr, const int* indices, int max_chain, int max_threads,
                     int max_window, int* nchains, int* ntiles, int* chain_ptr, int* tile_ptr,
                     int* threads_out, int* window_out, int* depth_out, const int* chain_order) {
  if (n < 0 || !indptr || (n > 0 && !indices) || !nchains || !ntiles)
    return fail(MVAMG_E_ARG, "gs_analyse: bad arguments");
  if (max_chain < 1) max_chain = 1;
  if (max_threads < 1) max_threads = 1;
  if (max_window < 1) max_window = 1;
  // chains: consecutive rows with a stored (i, i-1) entry (pattern is symmetric)
  std::vector<int> cp;
  cp.reserve(n / 4 + 2);
  int len = 0;
  for (int i = 0; i < n; ++i) {
    bool dep = false;
    if (i > 0 && len < max_chain) {
      const int* b = indices + indptr[i];
      const int* e = indices + indptr[i + 1];
      dep = std::binary_search(b, e, i - 1);
    }
    if (!dep) {
      cp.push_back(i);
      len = 0;
    }
    ++len;
  }
  cp.push_back(n);
  int nc = (int)cp.size() - 1;
  // tiles: consecutive chains, <= max_threads chains, and a position-major
  // shared window of roundup32(chains) x (longest chain) slots <= max_window
  if (max_threads > 256) max_threads = 256;
  auto r32 = [](int v) { return ((v + 31) / 32) * 32; };
  std::vector<int> tp;
  tp.push_back(0);
  int cnt = 0, maxlen = 0, maxcnt = 1, maxslots = 1;
  for (int c = 0; c < nc; ++c) {
    const int oc = chain_order ? chain_order[c] : c;  // tiles are ranges of the chain order
    if (oc < 0 || oc >= nc) return fail(MVAMG_E_ARG, "gs_analyse: chain order out of range");
    int cl = cp[oc + 1] - cp[oc];
    if (cnt > 0 && (cnt + 1 > max_threads || (long long)r32(cnt + 1) * std::max(maxlen, cl) > max_window)) {
      tp.push_back(c);
      maxcnt = std::max(maxcnt, cnt);
      maxslots = std::max(maxslots, r32(cnt) * maxlen);
      cnt = 0;
      maxlen = 0;
    }
    ++cnt;
    maxlen = std::max(maxlen, cl);
  }
  if (nc > 0) {
    tp.push_back(nc);
    maxcnt = std::max(maxcnt, cnt);
    maxslots = std::max(maxslots, r32(cnt) * maxlen);
  }
  int nt = (int)tp.size() - 1;
  *nchains = nc;
  *ntiles = nt;
  if (chain_ptr) std::copy(cp.begin(), cp.end(), chain_ptr);
  if (tile_ptr) std::copy(tp.begin(), tp.end(), tile_ptr);
  if (threads_out) *threads_out = r32(maxcnt);
  if (window_out) *window_out = maxslots;
  if (depth_out) {
    // level-set depth of the forward sweep DAG (diagnostic: the critical path)
    std::vector<int> lvl(n, 0);
    int depth = 0;
    for (int i = 0; i < n; ++i) {
      int m = 0;
      for (int k = indptr[i]; k < indptr[i + 1]; ++k) {
        int j = indices[k];
        if (j < i) m = std::max(m, lvl[j]);
      }
      lvl[i] = m + 1;
      depth = std::max(depth, m + 1);
    }
    *depth_out = depth;
  }
  return 0;
}

int mvamg_csr_spmv_f64(int n, const int* indptr, const int* indices, const double* data,
                       const double* x, double* y, void* stream) {
  Csr A;
  A.n = n; A.ip = indptr; A.ix = indices; A.v = data;
  return launch_spmv(0, A, x, nullptr, y, (cudaStream_t)stream);
}

int mvamg_csr_spmv_mode_f64(int mode, int n, int nnz, const int* indptr, const int* indices, const double* data,
                            const double* x, const double* b, double* y, void* stream) {
  if (mode < 0 || mode > 2 || n < 0 || nnz < 0) return fail(MVAMG_E_ARG, "csr_spmv_mode: bad arguments");
  Csr A;
  A.n = n; A.m = n; A.nnz = nnz; A.ip = indptr; A.ix = indices; A.v = data;
  return launch_spmv(mode, A, x, b, y, (cudaStream_t)stream);
}

int mvamg_csr_residual_f64(int n, const int* indptr, const int* indices, const double* data,
                           const double* b, const double* x, double* r, void* stream) {
  Csr A;
  A.n = n; A.ip = indptr; A.ix = indices; A.v = data;
  return launch_spmv(1, A, x, b, r, (cudaStream_t)stream);
}

int mvamg_csr_spmv_add_f64(int n, const int* indptr, const int* indices, const double* data,
                           const double* x, double* y, void* stream) {
  Csr A;
  A.n = n; A.ip = indptr; A.ix = indices; A.v = data;
  return launch_spmv(2, A, x, nullptr, y, (cudaStream_t)stream);
}

int mvamg_gs_schedule(int n, const int* indptr, const int* indices, const double* data, int ntiles,
                      const int* chain_ptr, const int* tile_ptr, int window, int mode, int R,
                      int uniform_S, int rows_per_round, long long* nwords, int* nrounds, int* nwarps,
                      int* max_S, unsigned long long* rec, int* round_off, int* tbase, int* tile_wbase,
                      int* perm, const int* chain_order, int wpos) {
  if (n < 0 || !indptr || !chain_ptr || !tile_ptr || !nwords || !nrounds || !nwarps || mode < 0 ||
      mode > 2 || R < 1 || R > 31)
    return fail(MVAMG_E_ARG, "gs_schedule: bad arguments");
  if (n >= (1 << 29)) return fail(MVAMG_E_ARG, "gs_schedule: n >= 2^29 not encodable");
  // rows_per_round: K | (cluster << 8); cluster > 1 marks sources in the previous
  // tile of the same thread-block cluster (processing order) for DSMEM reads
  const int cluster = (rows_per_round >> 8) & 0xff;
  rows_per_round &= 0xff;
  const int K = rows_per_round < 1 ? 1 : rows_per_round;
  if (K > 8 || (K > 1 && uniform_S <= 0))
    return fail(MVAMG_E_ARG, "gs_schedule: rows_per_round 1..8, > 1 only with uniform (lean) records");
  const bool fwd = mode < 2, with_old = mode == 1;
  auto dbits = [](double d) {
    unsigned long long u;
    std::memcpy(&u, &d, 8);
    return u;
  };
  auto keep = [&](int i, int j) {  // entries a row's record holds, in CSR order
    if (j == i) return false;
    if (fwd) return j < i || with_old;
    return j > i;
  };
  auto lower = [&](int i, int j) { return fwd ? (j < i) : (j > i); };
  const int nch = tile_ptr[ntiles];
  // wpos > 0: a tile's shared window keeps chain positions modulo wpos (one-warp
  // tiles only: every window read is then a same-warp value of an earlier
  // round, and each read is checked below to precede the slot's next write)
  if (wpos < 0 || (wpos & (wpos - 1))) return fail(MVAMG_E_ARG, "gs_schedule: wpos must be 0 or a power of two");
  if (wpos > 0)
    for (int t = 0; t < ntiles; ++t)
      if (tile_ptr[t + 1] - tile_ptr[t] > 32) return fail(MVAMG_E_ARG, "gs_schedule: wpos needs one-warp tiles");
  if (chain_order && cluster > 1) return fail(MVAMG_E_ARG, "gs_schedule: chain order and cluster tiles exclude each other");
  // chains are ranges of rows; warps / tiles are ranges of the chain order
  // (position cl holds chain ord(cl)); `pos_of` inverts it
  auto ord = [&](int cl) { return chain_order ? chain_order[cl] : cl; };
  std::vector<int> chain_of(n > 0 ? n : 1), pos_of(nch > 0 ? nch : 1), lidx(n > 0 ? n : 1, 0);
  for (int c = 0; c < nch; ++c)
    for (int i = chain_ptr[c]; i < chain_ptr[c + 1]; ++i) chain_of[i] = c;
  for (int cl = 0; cl < nch; ++cl) {
    const int c = ord(cl);
    if (c < 0 || c >= nch) return fail(MVAMG_E_ARG, "gs_schedule: chain order out of range");
    pos_of[c] = cl;
  }
  std::vector<int> tile_of_chain(nch > 0 ? nch : 1), warp_of_chain(nch > 0 ? nch : 1);
  for (int t = 0; t < ntiles; ++t)
    for (int cl = tile_ptr[t]; cl < tile_ptr[t + 1]; ++cl) tile_of_chain[ord(cl)] = t;
  {
    int w = 0;
    for (int t = 0; t < ntiles; ++t)
      for (int cA = tile_ptr[t]; cA < tile_ptr[t + 1]; cA += 32, ++w)
        for (int cl = cA; cl < std::min(cA + 32, tile_ptr[t + 1]); ++cl) warp_of_chain[ord(cl)] = w;
  }
  // an inter-warp input must come from a warp earlier in processing order, or
  // warps could wait on each other (the natural order of grid lines has it)
  for (int i = 0; i < n; ++i)
    for (int k = indptr[i]; k < indptr[i + 1]; ++k) {
      const int j = indices[k];
      if (j == i || !lower(i, j)) continue;
      const int wi = warp_of_chain[chain_of[i]], wj = warp_of_chain[chain_of[j]];
      if (wi != wj && (fwd ? wj > wi : wj < wi))
        return fail(MVAMG_E_ARG, "gs_schedule: the chain order puts an input in a later warp");
    }
  std::vector<int> wrows;
  auto ptk = [&](int t) { return fwd ? t : ntiles - 1 - t; };  // processing order of tile t
  long long w = 0;
  int gr = 0, gw = 0, smax = 1;
  std::vector<int> rnd, slot_of, rows_of_round, cnt_of;
  for (int t = 0; t < ntiles; ++t) {
    const int c0 = tile_ptr[t], c1 = tile_ptr[t + 1];
    const int TS = ((c1 - c0 + 31) / 32) * 32;
    if (tile_wbase) tile_wbase[t] = gw;
    for (int cA = c0; cA < c1; cA += 32, ++gw) {
      const int cB = std::min(cA + 32, c1);
      // the warp's rows in sweep order (its chains need not be consecutive)
      wrows.clear();
      for (int cl = cA; cl < cB; ++cl)
        for (int i = chain_ptr[ord(cl)]; i < chain_ptr[ord(cl) + 1]; ++i) wrows.push_back(i);
      std::sort(wrows.begin(), wrows.end());
      if (!fwd) std::reverse(wrows.begin(), wrows.end());
      const int nwr = (int)wrows.size();
      for (int q = 0; q < nwr; ++q) lidx[wrows[q]] = q;
      rnd.assign(nwr, 0);
      slot_of.assign(nwr, 0);
      int last[32], used[32];
      for (int L = 0; L < 32; ++L) last[L] = -1, used[L] = 0;
      int nr = 0;
      for (int q = 0; q < nwr; ++q) {
        const int i = wrows[q];
        const int L = pos_of[chain_of[i]] - cA;
        const int c = chain_of[i], pred = fwd ? i - 1 : i + 1;
        const bool has_pred = fwd ? (i - 1 >= chain_ptr[c]) : (i + 1 < chain_ptr[c + 1]);
        // every intra-warp input other than the chain predecessor must come
        // from an earlier round (its value is read from the window at the
        // round's start); the predecessor may share the round (register)
        int rmin = 0;
        for (int k = indptr[i]; k < indptr[i + 1]; ++k) {
          const int j = indices[k];
          if (j != i && lower(i, j) && warp_of_chain[chain_of[j]] == gw && !(has_pred && j == pred))
            rmin = std::max(rmin, rnd[lidx[j]] + 1);
        }
        int r;
        if (last[L] >= 0 && used[L] < K && rmin <= last[L]) {
          r = last[L];
          ++used[L];
        } else {
          r = std::max(last[L] + 1, rmin);
          used[L] = 1;
        }
        rnd[q] = r;
        slot_of[q] = used[L] - 1;
        last[L] = r;
        nr = std::max(nr, r + 1);
      }
      nr = ((nr + R - 1) / R) * R;
      if (nr == 0) nr = R;
      if (tbase) tbase[gw] = gr;
      // rows of each round: K slots per lane
      rows_of_round.assign((size_t)nr * K * 32, -1);
      for (int q = 0; q < nwr; ++q)
        rows_of_round[((size_t)rnd[q] * K + slot_of[q]) * 32 + (pos_of[chain_of[wrows[q]]] - cA)] = wrows[q];
      for (int r = 0; r < nr; ++r, ++gr) {
        int maxcnt = -1;
        for (int L = 0; L < 32 * K; ++L) {
          const int i = rows_of_round[(size_t)r * K * 32 + L];
          if (i < 0) continue;
          int cnt = 0;
          for (int k = indptr[i]; k < indptr[i + 1]; ++k) cnt += keep(i, indices[k]);
          maxcnt = std::max(maxcnt, cnt);
        }
        int S = maxcnt < 0 ? 1 : 3 + 2 * maxcnt;
        if (uniform_S > 0) {
          if (S > uniform_S) return fail(MVAMG_E_ARG, "gs_schedule: row longer than the uniform record");
          S = uniform_S;
        }
        smax = std::max(smax, S);
        if (round_off) round_off[gr] = (int)w;
        if (rec) for (int sl = 0; sl < K; ++sl) {
          unsigned long long* blk = rec + w + (size_t)sl * 32 * S;
          std::memset(blk, 0, sizeof(unsigned long long) * 32 * S);
          // lean records: absent entries carry source code 3 ("none") and the
          // header word's bits 16-31 hold the 2-bit source type of every entry
          const int nent = uniform_S > 0 ? (S - 3) / 2 : 0;
          if (uniform_S > 0 && nent > 8) return fail(MVAMG_E_ARG, "gs_schedule: lean records hold <= 8 entries");
          for (int L = 0; L < 32; ++L)
            for (int u = 0; u < nent; ++u) blk[(size_t)32 * (4 + 2 * u) + L] = 3ull;
          for (int L = 0; L < 32; ++L) {
            const int i = rows_of_round[((size_t)r * K + sl) * 32 + L];
            if (i < 0) {
              blk[L] = kGsNoRow | (uniform_S > 0 ? 0xffff0000ull : 0ull);
              continue;
            }
            const int c = chain_of[i], cs = chain_ptr[c], ce = chain_ptr[c + 1];
            int cnt = 0;
            bool fast = true;
            double dg = 0.0;
            for (int k = indptr[i]; k < indptr[i + 1]; ++k) {
              const int j = indices[k];
              if (j == i) dg = data[k];
              if (!keep(i, j)) continue;
              int code;
              if (!lower(i, j)) {
                code = (j << 2) | 3;
              } else if ((fwd && j == i - 1 && j >= cs) || (!fwd && j == i + 1 && j < ce)) {
                code = 0;
              } else if (tile_of_chain[chain_of[j]] == t) {
                const int cj = chain_of[j];
                const int pos = fwd ? j - chain_ptr[cj] : chain_ptr[cj + 1] - 1 - j;
                long long slot = (long long)pos * TS + (pos_of[cj] - c0);
                if (wpos > 0) {
                  slot = (long long)(pos & (wpos - 1)) * TS + (pos_of[cj] - c0);
                  // the slot's next write: chain cj's row wpos positions later
                  const int pn = pos + wpos, len = chain_ptr[cj + 1] - chain_ptr[cj];
                  if (pn < len) {
                    const int jn = fwd ? chain_ptr[cj] + pn : chain_ptr[cj + 1] - 1 - pn;
                    if (rnd[lidx[jn]] <= r)
                      return fail(MVAMG_E_ARG, "gs_schedule: window of " + std::to_string(wpos) +
                                                   " positions too short for this schedule");
                  }
                }
                if (slot >= window) return fail(MVAMG_E_ARG, "gs_schedule: window slot out of range");
                code = (int)(slot << 2) | 1;
              } else {
                const int cj = chain_of[j], st = tile_of_chain[cj];
                if (cluster > 1 && ptk(st) == ptk(t) - 1 && ptk(t) % cluster != 0) {
                  // previous tile of the same cluster: its window slot, read over DSMEM
                  const int sc0 = tile_ptr[st], sTS = ((tile_ptr[st + 1] - sc0 + 31) / 32) * 32;
                  const int pos = fwd ? j - chain_ptr[cj] : chain_ptr[cj + 1] - 1 - j;
                  const long long slot = (long long)pos * sTS + (cj - sc0);
                  if (slot >= window || slot >= (long long)kGsRemote)
                    return fail(MVAMG_E_ARG, "gs_schedule: remote window slot out of range");
                  code = (int)((((unsigned)slot | kGsRemote) << 2) | 2u);
                } else {
                  code = (j << 2) | 2;
                }
              }
              blk[(size_t)32 * (3 + 2 * cnt) + L] = dbits(data[k]);
              blk[(size_t)32 * (4 + 2 * cnt) + L] = (unsigned long long)(unsigned)code;
              fast = fast && ((code & 3) == 0 || (code & 3) == 1);
              ++cnt;
            }
            if (cnt >= (int)kGsNoRow) return fail(MVAMG_E_ARG, "gs_schedule: row with too many entries");
            if (uniform_S > 0) {
              unsigned tb = 0xffffu;  // types of entries >= cnt stay 3
              for (int u = 0; u < cnt; ++u) {
                const unsigned t = (unsigned)blk[(size_t)32 * (4 + 2 * u) + L] & 3u;
                tb = (tb & ~(3u << (2 * u))) | (t << (2 * u));
              }
              blk[L] = (unsigned long long)(unsigned)cnt | ((unsigned long long)tb << 16);
            } else {
              blk[L] = (unsigned long long)(unsigned)cnt | (fast ? 0x10000ull : 0ull);
            }
            blk[32 + L] = dbits(dg);
            blk[64 + L] = dbits(1.0 / dg);
            if (perm) perm[i] = (gr * K + sl) * 32 + L;
          }
        }
        w += (long long)32 * K * S;
        if (w >= (1LL << 31)) return fail(MVAMG_E_ARG, "gs_schedule: record stream exceeds 2^31 words");
        if ((long long)gr * 32 * K >= (1LL << 31)) return fail(MVAMG_E_ARG, "gs_schedule: too many rounds");
      }
    }
  }
  if (round_off) round_off[gr] = (int)w;
  if (tbase) tbase[gw] = gr;
  if (tile_wbase) tile_wbase[ntiles] = gw;
  *nwords = w;
  *nrounds = gr;
  *nwarps = gw;
  if (max_S) *max_S = smax;
  return 0;
}

int mvamg_gs_sweep_f64(int direction, int n, const int* indptr, const int* indices, const double* data,
                       const unsigned long long* rec, const int* round_off, const int* tbase,
                       const int* tile_wbase, const int* perm, double* tperm, int R, int D,
                       int lean_C, int slot_words, int rec_words_max, int ntiles,
                       const int* chain_ptr, const int* tile_ptr, const int* chain_order, int threads,
                       int window, int wpos, const double* b, const double* x_old, double* x_new, int* ws,
                       void* stream) {
  if (threads < 32 || threads > 256 || threads % 32) return fail(MVAMG_E_ARG, "gs: threads must be 32..256, multiple of 32");
  if (R != 1 && R != 2 && R != 4 && R != 8) return fail(MVAMG_E_ARG, "gs: R must be 1, 2, 4 or 8");
  if (D != 2 && D != 3 && D != 4 && D != 8) return fail(MVAMG_E_ARG, "gs: D must be 2, 3, 4 or 8");
  if (x_old != nullptr && x_old == x_new) return fail(MVAMG_E_ARG, "gs: x_new must not alias x_old");
  Csr A;
  A.n = n; A.ip = indptr; A.ix = indices; A.v = data;
  GsList ls;
  ls.rec = rec; ls.round_off = round_off; ls.tbase = tbase; ls.tile_wbase = tile_wbase; ls.perm = perm;
  ls.tperm = tperm; ls.R = R; ls.D = D; ls.slot_words = slot_words; ls.rec_words_max = rec_words_max;
  ls.lean_C = lean_C;
  const int lean_K = (lean_C >> 8) & 0xff;
  if (lean_C > 0 && lean_K <= 1 && ((R == 8 && D != 2 && D != 3) || (R == 4 && D != 4 && D != 2) || (R == 2 && D != 8 && D != 2) ||
                                    (R == 1 && D != 8)))
    return fail(MVAMG_E_ARG, "gs: lean kernel ring must be (R, D) in {(8,3), (8,2), (4,4), (4,2), (2,8), (2,2), (1,8)}");
  if (lean_K > 1 && ((lean_C & 0xff) > 4 ||
                     !((lean_K == 4 && R == 2 && (D == 2 || D == 3)) || (lean_K == 2 && R == 4 && D == 2))))
    return fail(MVAMG_E_ARG, "gs: lean kernel with K rows per round needs C <= 4 and (R, D, K) in "
                             "{(2,2,4), (2,3,4), (4,2,2)}");
  GsPlan p;
  p.ntiles = ntiles; p.threads = threads; p.window = window; p.chain_ptr = chain_ptr; p.tile_ptr = tile_ptr;
  p.chain_order = chain_order;
  if (wpos < 0 || (wpos & (wpos - 1))) return fail(MVAMG_E_ARG, "gs: wpos must be 0 or a power of two");
  p.wmask = wpos > 0 ? wpos - 1 : -1;
  return launch_gs(direction == 0, A, ls, p, b, x_old, x_new, ws, ws + 1, (cudaStream_t)stream);
}

int mvamg_gs_levels(int n, const int* indptr, const int* indices, const double* data, int mode, int ncta,
                    int row_cap, int ent_cap, int* nlev, long long* nents, int* max_rows, int* max_ents,
                    int* rows_per_cta, int* lev_ptr, int* lev_eptr, void* rows_out, void* ents_out,
                    int* perm) {
  if (n < 0 || !indptr || !nlev || !nents || !max_rows || !max_ents || !rows_per_cta || mode < 0 ||
      mode > 3 || ncta < 1 || ncta > 16)
    return fail(MVAMG_E_ARG, "gs_levels: bad arguments");
  const bool fwd = mode < 2, zero = (mode % 2) == 0;
  auto keep = [&](int i, int j) {
    if (j == i) return false;
    if (!zero) return true;
    return fwd ? j < i : j > i;
  };
  if (row_cap <= 0) row_cap = 1 << 30;
  if (ent_cap <= 0) ent_cap = 1 << 30;
  const int rpc = (n + ncta - 1) / ncta;
  if (rpc >= (1 << 26)) return fail(MVAMG_E_ARG, "gs_levels: too many rows per CTA");
  // level sets of the sweep's dependency DAG
  std::vector<int> lvl(n > 0 ? n : 1, 0), rowcnt(n > 0 ? n : 1, 0);
  int nl = 0;
  for (int q = 0; q < n; ++q) {
    const int i = fwd ? q : n - 1 - q;
    int m = 0;
    for (int k = indptr[i]; k < indptr[i + 1]; ++k) {
      const int j = indices[k];
      if (fwd ? j < i : j > i) m = std::max(m, lvl[j] + 1);
    }
    lvl[i] = m;
    nl = std::max(nl, m + 1);
  }
  if (n == 0) nl = 0;
  for (int i = 0; i < n; ++i) {
    int c = 0;
    for (int k = indptr[i]; k < indptr[i + 1]; ++k) c += keep(i, indices[k]);
    rowcnt[i] = c;
  }
  // rows of every (cta, level) bucket, ascending
  std::vector<std::vector<int>> bucket((size_t)ncta * nl);
  for (int i = 0; i < n; ++i) bucket[(size_t)(i / rpc) * nl + lvl[i]].push_back(i);
  // split each level into cluster-uniform sub-levels whose (cta) buckets fit the caps
  std::vector<int> sub(nl > 0 ? nl : 1, 1);
  std::vector<std::vector<int>> cut((size_t)ncta * nl);  // greedy group boundaries per bucket
  for (int l = 0; l < nl; ++l) {
    int need = 1;
    for (int c = 0; c < ncta; ++c) {
      auto& bk = bucket[(size_t)c * nl + l];
      auto& ct = cut[(size_t)c * nl + l];
      ct.assign(1, 0);
      long long ents = 0;
      int rows = 0;
      for (int p = 0; p < (int)bk.size(); ++p) {
        const int rc = rowcnt[bk[p]];
        if (rows > 0 && (rows + 1 > row_cap || ents + rc > ent_cap)) {
          ct.push_back(p);
          ents = 0;
          rows = 0;
        }
        ents += rc;
        ++rows;
      }
      ct.push_back((int)bk.size());
      need = std::max(need, (int)ct.size() - 1);
    }
    sub[l] = need;
  }
  int nsub = 0;
  for (int l = 0; l < nl; ++l) nsub += sub[l];
  const size_t L1 = (size_t)nsub + 1;
  // offsets over (cta, sub-level), CTA-major
  std::vector<long long> rstart((size_t)ncta * L1), estart((size_t)ncta * L1);
  long long rofs = 0, eofs = 0, mr = 0, me = 0;
  for (int c = 0; c < ncta; ++c) {
    int s = 0;
    for (int l = 0; l < nl; ++l) {
      auto& bk = bucket[(size_t)c * nl + l];
      auto& ct = cut[(size_t)c * nl + l];
      for (int g = 0; g < sub[l]; ++g, ++s) {
        rstart[(size_t)c * L1 + s] = rofs;
        estart[(size_t)c * L1 + s] = eofs;
        const int p0 = g + 1 < (int)ct.size() ? ct[g] : (int)bk.size();
        const int p1 = g + 1 < (int)ct.size() ? ct[g + 1] : (int)bk.size();
        long long e = 0;
        for (int p = p0; p < p1; ++p) e += rowcnt[bk[p]];
        rofs += p1 - p0;
        eofs += e;
        mr = std::max(mr, (long long)(p1 - p0));
        me = std::max(me, e);
      }
    }
    rstart[(size_t)c * L1 + nsub] = rofs;
    estart[(size_t)c * L1 + nsub] = eofs;
  }
  if (eofs >= (1LL << 31)) return fail(MVAMG_E_ARG, "gs_levels: more than 2^31 entries");
  *nlev = nsub;
  *nents = eofs;
  *max_rows = (int)mr;
  *max_ents = (int)me;
  *rows_per_cta = rpc;
  if (!rows_out) return 0;
  for (size_t k = 0; k < rstart.size(); ++k) {
    lev_ptr[k] = (int)rstart[k];
    lev_eptr[k] = (int)estart[k];
  }
  GsLevelRow* R = static_cast<GsLevelRow*>(rows_out);
  GsLevelEntry* E = static_cast<GsLevelEntry*>(ents_out);
  for (int c = 0; c < ncta; ++c) {
    int s = 0;
    for (int l = 0; l < nl; ++l) {
      auto& bk = bucket[(size_t)c * nl + l];
      auto& ct = cut[(size_t)c * nl + l];
      for (int g = 0; g < sub[l]; ++g, ++s) {
        long long pos = rstart[(size_t)c * L1 + s], epos = estart[(size_t)c * L1 + s];
        const int p0 = g + 1 < (int)ct.size() ? ct[g] : (int)bk.size();
        const int p1 = g + 1 < (int)ct.size() ? ct[g + 1] : (int)bk.size();
        for (int p = p0; p < p1; ++p, ++pos) {
          const int i = bk[p];
          GsLevelRow& r = R[pos];
          r.row = i;
          r.estart = (int)epos;
          r.cnt = rowcnt[i];
          r.pad = 0;
          double dg = 0.0;
          for (int k = indptr[i]; k < indptr[i + 1]; ++k) {
            const int j = indices[k];
            if (j == i) dg = data[k];
            if (!keep(i, j)) continue;
            GsLevelEntry& e = E[epos++];
            e.coef = data[k];
            e.src = ((j / rpc) << 26) | (j % rpc);
            e.pad = 0;
          }
          r.diag = dg;
          r.rdiag = 1.0 / dg;
          if (perm) perm[i] = (int)pos;
        }
      }
    }
  }
  return 0;
}

int mvamg_gs_level_sweep_f64(int direction, int n, const int* indptr, const int* indices,
                             const double* data, int ncta, int rows_per_cta, int nlev, int max_rows,
                             int max_ents, int threads, int group, const int* lev_ptr, const int* lev_eptr,
                             const void* rows, const void* ents, const int* perm, double* tperm,
                             const double* b, const double* x_old, double* x_new, int* ws, void* stream) {
  if (threads < 32 || threads > 1024 || threads % 32) return fail(MVAMG_E_ARG, "gs levels: bad thread count");
  Csr A;
  A.n = n; A.ip = indptr; A.ix = indices; A.v = data;
  GsLevels g;
  g.lev_ptr = lev_ptr; g.lev_eptr = lev_eptr; g.rows = static_cast<const GsLevelRow*>(rows);
  g.ents = static_cast<const GsLevelEntry*>(ents); g.perm = perm; g.tperm = tperm;
  g.nlev = nlev; g.max_rows = max_rows; g.max_ents = max_ents; g.threads = threads;
  g.ncta = ncta; g.rows_per_cta = rows_per_cta; g.group = group & 0xff; g.reg = (group >> 8) & 1;
  (void)direction;  // encoded in the schedule
  set_kernel_attrs();
  return launch_gs_levels(A, g, x_old == nullptr, b, x_old, x_new, ws, (cudaStream_t)stream);
}

int mvamg_gs_level_sweep_folded_f64(int n, const int* indptr, const int* indices, const double* data,
                                    int ncta, int rows_per_cta, int nlev, int max_rows, int max_ents,
                                    int threads, int group, const int* lev_ptr, const int* lev_eptr,
                                    const void* rows, const void* ents, const int* perm,
                                    double* tperm, const double* b, const double* x_old,
                                    double* x_new, int* ws, void* stream) {
  if (!x_old) return fail(MVAMG_E_ARG, "gs levels folded: needs x_old");
  Csr A;
  A.n = n; A.ip = indptr; A.ix = indices; A.v = data;
  GsLevels g;
  g.lev_ptr = lev_ptr; g.lev_eptr = lev_eptr; g.rows = static_cast<const GsLevelRow*>(rows);
  g.ents = static_cast<const GsLevelEntry*>(ents); g.perm = perm; g.tperm = tperm;
  g.nlev = nlev; g.max_rows = max_rows; g.max_ents = max_ents; g.threads = threads;
  g.ncta = ncta; g.rows_per_cta = rows_per_cta; g.group = group & 0xff; g.reg = (group >> 8) & 1;
  set_kernel_attrs();
  return launch_gs_levels(A, g, false, b, x_old, x_new, ws, (cudaStream_t)stream, true);
}

int mvamg_hierarchy_set_gs_levels(mvamg_hierarchy* h, int k, int mode, int ncta, int rows_per_cta,
                                  int nlev, int max_rows, int max_ents, int threads, int group,
                                  const int* lev_ptr, const int* lev_eptr, const void* rows, const void* ents,
                                  const int* perm, double* tperm) {
  if (!h || k < 0 || k >= h->L || mode < 0 || mode > 3) return fail(MVAMG_E_ARG, "set_gs_levels: bad index");
  GsLevels& g = h->lv[k].glv[mode];
  g.lev_ptr = lev_ptr; g.lev_eptr = lev_eptr; g.rows = static_cast<const GsLevelRow*>(rows);
  g.ents = static_cast<const GsLevelEntry*>(ents); g.perm = perm; g.tperm = tperm;
  g.nlev = nlev; g.max_rows = max_rows; g.max_ents = max_ents; g.threads = threads;
  g.ncta = ncta; g.rows_per_cta = rows_per_cta; g.group = group & 0xff; g.reg = (group >> 8) & 1;
  return 0;
}

// Streamed level-set plan (gs_stream.cuh).  Call with blob == nullptr to size
// it (*blob_bytes, *nstages), then with buffers of those sizes.  Rows go into
// batches by their level in the sweep's dependency DAG -- for a sweep from
// x_old also after every row whose old value they read on the other side
// (anti-dependence through the transposed pattern) -- in sweep order within a
// level.  With ncta > 1 CTA c owns rows [c R, (c+1) R), R = ceil(n / ncta),
// and its blob of stage s holds its rows of that stage's batches; a level
// whose part on some CTA exceeds a slot is split into several batches on all.
int mvamg_gs_stream_plan(int n, const int* indptr, const int* indices, const double* data, int mode,
                         int slot_bytes, int ncta, long long* blob_bytes, int* nstages, int* nlevels,
                         unsigned char* blob, long long* stage_off) {
  if (n < 0 || !indptr || (n > 0 && (!indices || !data)) || mode < 0 || mode > 3 || slot_bytes < 256 ||
      !blob_bytes || !nstages || ncta < 1 || ncta > 16 || (ncta > 1 && (mode & 1)))
    return fail(MVAMG_E_ARG, "gs_stream_plan: bad arguments (clusters: zero-guess modes only)");
  const bool fwd = mode < 2, old = (mode & 1) != 0;
  const int R = ncta > 1 ? (n + ncta - 1) / ncta : std::max(n, 1);
  if (ncta > 1 && R >= (1 << 24)) return fail(MVAMG_E_ARG, "gs_stream_plan: slice too large to encode");
  auto dep = [&](int i, int j) { return fwd ? j < i : j > i; };
  auto keep = [&](int i, int j) { return j != i && (old || dep(i, j)); };
  std::vector<int> lvl(n > 0 ? n : 1, 0), cnt(n > 0 ? n : 1, 0);
  std::vector<double> dg(n > 0 ? n : 1, 0.0);
  // transposed pattern (anti-dependences of a sweep from x_old)
  std::vector<int> tp, tix;
  if (old) {
    tp.assign(n + 1, 0);
    for (int i = 0; i < n; ++i)
      for (int k = indptr[i]; k < indptr[i + 1]; ++k) tp[indices[k] + 1]++;
    for (int i = 0; i < n; ++i) tp[i + 1] += tp[i];
    tix.resize(tp[n] > 0 ? tp[n] : 1);
    std::vector<int> cur(tp.begin(), tp.end() - 1);
    for (int i = 0; i < n; ++i)
      for (int k = indptr[i]; k < indptr[i + 1]; ++k) tix[cur[indices[k]]++] = i;
  }
  int nl = 0;
  for (int q = 0; q < n; ++q) {
    const int i = fwd ? q : n - 1 - q;
    int m = 0;
    for (int k = indptr[i]; k < indptr[i + 1]; ++k) {
      const int j = indices[k];
      if (j == i) dg[i] = data[k];
      if (keep(i, j)) ++cnt[i];
      if (j != i && dep(i, j)) m = std::max(m, lvl[j] + 1);
    }
    if (old)  // row r read x_old[i] on its other side: i must run after r
      for (int k = tp[i]; k < tp[i + 1]; ++k) {
        const int r = tix[k];
        if (r != i && dep(i, r)) m = std::max(m, lvl[r] + 1);
      }
    lvl[i] = m;
    nl = std::max(nl, m + 1);
  }
  if (n > 0 && *std::min_element(dg.begin(), dg.begin() + n) == 0.0)
    return fail(MVAMG_E_NOT_SPD, "gs_stream_plan: zero diagonal");
  // rows by (level, CTA), sweep order within
  const int NC = ncta;
  std::vector<int> lp((size_t)nl * NC + 1, 0), order(n > 0 ? n : 1);
  for (int i = 0; i < n; ++i) lp[(size_t)lvl[i] * NC + i / R + 1]++;
  for (size_t t = 0; t + 1 < lp.size(); ++t) lp[t + 1] += lp[t];
  {
    std::vector<int> cur(lp.begin(), lp.end() - 1);
    for (int q = 0; q < n; ++q) {
      const int i = fwd ? q : n - 1 - q;
      order[cur[(size_t)lvl[i] * NC + i / R]++] = i;
    }
  }
  auto a16 = [](long long v) { return (v + 15) & ~15LL; };
  auto stage_size = [&](long long nb, long long nr, long long ne) {
    return a16(a16(a16(16 + 8 * nb) + 32 * nr + 8 * ne) + 4 * ne);
  };
  // batches: per CTA a (first position, rows) range of `order`; a level split
  // where one CTA's part does not fit a slot (same split count on every CTA)
  struct Part { int p, r; long long e; };
  std::vector<std::vector<Part>> batches;  // batch -> NC parts
  for (int l = 0; l < nl; ++l) {
    int parts = 1;
    std::vector<std::vector<Part>> chunks(NC);
    for (int c = 0; c < NC; ++c) {
      const int b0 = lp[(size_t)l * NC + c], b1 = lp[(size_t)l * NC + c + 1];
      int p = b0;
      while (p < b1) {
        int q = p;
        long long ne = 0;
        while (q < b1 && stage_size(1, q - p + 1, ne + cnt[order[q]]) <= slot_bytes) ne += cnt[order[q++]];
        if (q == p) return fail(MVAMG_E_ARG, "gs_stream_plan: a row does not fit one slot");
        chunks[c].push_back({p, q - p, ne});
        p = q;
      }
      parts = std::max(parts, (int)chunks[c].size());
    }
    for (int k = 0; k < parts; ++k) {
      std::vector<Part> bt(NC);
      for (int c = 0; c < NC; ++c) bt[c] = k < (int)chunks[c].size() ? chunks[c][k] : Part{0, 0, 0};
      batches.push_back(bt);
    }
  }
  // stages: consecutive batches while every CTA's part of the stage fits a slot
  std::vector<std::pair<int, int>> stages;  // (first batch, batches)
  {
    size_t bi = 0;
    while (bi < batches.size()) {
      size_t bj = bi;
      std::vector<long long> nr(NC, 0), ne(NC, 0);
      while (bj < batches.size()) {
        bool fits = true;
        for (int c = 0; c < NC && fits; ++c)
          fits = stage_size((long long)(bj - bi + 1), nr[c] + batches[bj][c].r, ne[c] + batches[bj][c].e) <=
                 slot_bytes;
        if (!fits) break;
        for (int c = 0; c < NC; ++c) {
          nr[c] += batches[bj][c].r;
          ne[c] += batches[bj][c].e;
        }
        ++bj;
      }
      stages.push_back({(int)bi, (int)(bj - bi)});
      bi = bj;
    }
  }
  const size_t NS = stages.size();
  std::vector<long long> off(NS * NC + 1, 0);
  long long total = 0;
  for (size_t s = 0; s < NS; ++s)
    for (int c = 0; c < NC; ++c) {
      long long nr = 0, ne = 0;
      for (int b = stages[s].first; b < stages[s].first + stages[s].second; ++b) {
        nr += batches[b][c].r;
        ne += batches[b][c].e;
      }
      total += stage_size(stages[s].second, nr, ne);
      off[s * NC + c + 1] = total;
    }
  *blob_bytes = total;
  *nstages = (int)NS;
  if (nlevels) *nlevels = nl;
  if (!blob) return 0;
  if (!stage_off) return fail(MVAMG_E_ARG, "gs_stream_plan: stage offsets buffer missing");
  std::memset(blob, 0, (size_t)total);
  for (size_t s = 0; s < NS; ++s)
    for (int c = 0; c < NC; ++c) {
      unsigned char* st = blob + off[s * NC + c];
      const int b0 = stages[s].first, nb = stages[s].second;
      unsigned nr = 0, ne = 0;
      for (int b = b0; b < b0 + nb; ++b) {
        nr += (unsigned)batches[b][c].r;
        ne += (unsigned)batches[b][c].e;
      }
      unsigned* hdr = reinterpret_cast<unsigned*>(st);
      hdr[0] = (unsigned)nb;
      hdr[1] = nr;
      hdr[2] = ne;
      const long long rows_off = a16(16 + 8LL * nb), coef_off = rows_off + 32LL * nr;
      const long long src_off = a16(coef_off + 8LL * ne);
      GsStreamRow* rows = reinterpret_cast<GsStreamRow*>(st + rows_off);
      double* coef = reinterpret_cast<double*>(st + coef_off);
      unsigned* src = reinterpret_cast<unsigned*>(st + src_off);
      unsigned r = 0, e = 0;
      for (int b = b0; b < b0 + nb; ++b) {
        hdr[4 + 2 * (b - b0)] = r;
        hdr[5 + 2 * (b - b0)] = (unsigned)batches[b][c].r;
        for (int t = 0; t < batches[b][c].r; ++t, ++r) {
          const int i = order[batches[b][c].p + t];
          GsStreamRow& m = rows[r];
          m.row = (unsigned)(i - c * (NC > 1 ? R : 0));
          m.cnt = (unsigned)cnt[i];
          m.ebeg = e;
          m.pad = 0;
          m.diag = dg[i];
          m.rdiag = 1.0 / dg[i];
          for (int k = indptr[i]; k < indptr[i + 1]; ++k) {
            const int j = indices[k];
            if (!keep(i, j)) continue;
            coef[e] = data[k];
            src[e] = NC > 1 ? ((unsigned)(j / R) << 24) | (unsigned)(j % R) : (unsigned)j;
            ++e;
          }
        }
      }
    }
  std::copy(off.begin(), off.end(), stage_off);
  return 0;
}

int mvamg_gs_stream_sweep_f64(int n, int mode, int nstages, int nslots, int slot_bytes, int group, int ncta,
                              const void* blob, const long long* stage_off, const double* b, const double* x_old,
                              double* x_new, void* stream) {
  if (n < 0 || mode < 0 || mode > 3 || (n > 0 && (!blob || !stage_off || !b || !x_new)))
    return fail(MVAMG_E_ARG, "gs_stream_sweep: bad arguments");
  GsStream g;
  g.nstages = nstages; g.nslots = nslots; g.slot_bytes = slot_bytes; g.group = group; g.ncta = ncta;
  g.blob = static_cast<const unsigned char*>(blob);
  g.stage_off = stage_off;
  return launch_gs_stream(n, g, mode & 1, b, x_old, x_new, (cudaStream_t)stream);
}

int mvamg_gs_stream_sweep_folded_f64(int n, const int* indptr, const int* indices, const double* data, int nstages,
                                     int nslots, int slot_bytes, int group, int ncta, const void* blob,
                                     const long long* stage_off, double* tfold, const double* b,
                                     const double* x_old, double* x_new, int* ws, void* stream) {
  if (n < 0 || (n > 0 && (!indptr || !indices || !data || !blob || !stage_off || !tfold || !b || !x_old || !x_new ||
                          !ws)))
    return fail(MVAMG_E_ARG, "gs_stream_sweep_folded: bad arguments");
  Csr A;
  A.n = n; A.m = n; A.ip = indptr; A.ix = indices; A.v = data;
  A.nnz = 0;
  cudaStream_t s = (cudaStream_t)stream;
  GsStream g;
  g.nstages = nstages; g.nslots = nslots; g.slot_bytes = slot_bytes; g.group = group; g.ncta = ncta;
  g.blob = static_cast<const unsigned char*>(blob);
  g.stage_off = stage_off;
  launch_prepare(A, b, x_old, nullptr, tfold, x_new, ws, 1, s);
  return launch_gs_stream(n, g, 0, tfold, nullptr, x_new, s);
}

// ---- NCCL (row-partitioned solve) ---------------------
// libnccl.so.2 is opened at run time, not linked: in a process where PyTorch
// already loaded its NCCL, dlopen returns that same library (one NCCL per
// process, as SURVEY 5 asks); MVAMG_NCCL overrides the path.
namespace ncclabi {
typedef struct { char internal[128]; } UniqueId;
typedef void* Comm;
typedef int (*GetUniqueId_t)(UniqueId*);
typedef int (*CommInitRank_t)(Comm*, int, UniqueId, int);
typedef int (*CommDestroy_t)(Comm);
typedef int (*Group_t)();
typedef int (*Send_t)(const void*, size_t, int, int, Comm, cudaStream_t);
typedef int (*Recv_t)(void*, size_t, int, int, Comm, cudaStream_t);
typedef int (*AllReduce_t)(const void*, void*, size_t, int, int, Comm, cudaStream_t);
typedef const char* (*ErrStr_t)(int);
constexpr int kFloat64 = 8, kSum = 0;
struct Api {
  bool ok = false;
  GetUniqueId_t get_id = nullptr;
  CommInitRank_t init = nullptr;
  CommDestroy_t destroy = nullptr;
  Group_t gstart = nullptr, gend = nullptr;
  Send_t send = nullptr;
  Recv_t recv = nullptr;
  AllReduce_t allreduce = nullptr;
  ErrStr_t errstr = nullptr;
};
Api& api() {
  static Api a;
  static bool tried = false;
  if (tried) return a;
  tried = true;
  const char* path = std::getenv("MVAMG_NCCL");
  void* h = dlopen(path ? path : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return a;
  a.get_id = (GetUniqueId_t)dlsym(h, "ncclGetUniqueId");
  a.init = (CommInitRank_t)dlsym(h, "ncclCommInitRank");
  a.destroy = (CommDestroy_t)dlsym(h, "ncclCommDestroy");
  a.gstart = (Group_t)dlsym(h, "ncclGroupStart");
  a.gend = (Group_t)dlsym(h, "ncclGroupEnd");
  a.send = (Send_t)dlsym(h, "ncclSend");
  a.recv = (Recv_t)dlsym(h, "ncclRecv");
  a.allreduce = (AllReduce_t)dlsym(h, "ncclAllReduce");
  a.errstr = (ErrStr_t)dlsym(h, "ncclGetErrorString");
  a.ok = a.get_id && a.init && a.destroy && a.gstart && a.gend && a.send && a.recv && a.allreduce;
  return a;
}
}  // namespace ncclabi

struct mvamg_comm {
  ncclabi::Comm c = nullptr;
  int rank = 0, nranks = 1;
};

#define NCCL_TRY(x)                                                                        \
  do {                                                                                     \
    int r_ = (x);                                                                          \
    if (r_ != 0)                                                                           \
      return fail(MVAMG_E_CUDA, std::string("nccl: ") +                                    \
                                    (ncclabi::api().errstr ? ncclabi::api().errstr(r_) : "error")); \
  } while (0)

int mvamg_comm_unique_id(void* id128) {
  if (!id128) return fail(MVAMG_E_ARG, "comm_unique_id: null");
  if (!ncclabi::api().ok) return fail(MVAMG_E_STATE, "comm_unique_id: libnccl.so.2 not available");
  ncclabi::UniqueId id;
  NCCL_TRY(ncclabi::api().get_id(&id));
  std::memcpy(id128, &id, sizeof(id));
  return 0;
}

int mvamg_comm_init(mvamg_comm** comm, int rank, int nranks, const void* id128) {
  if (!comm || !id128 || nranks < 1 || rank < 0 || rank >= nranks) return fail(MVAMG_E_ARG, "comm_init: bad arguments");
  if (!ncclabi::api().ok) return fail(MVAMG_E_STATE, "comm_init: libnccl.so.2 not available");
  ncclabi::UniqueId id;
  std::memcpy(&id, id128, sizeof(id));
  mvamg_comm* c = new mvamg_comm();
  c->rank = rank;
  c->nranks = nranks;
  int r = ncclabi::api().init(&c->c, nranks, id, rank);
  if (r != 0) {
    delete c;
    NCCL_TRY(r);
  }
  *comm = c;
  return 0;
}

int mvamg_comm_destroy(mvamg_comm* comm) {
  if (!comm) return 0;
  if (comm->c && ncclabi::api().ok) ncclabi::api().destroy(comm->c);
  delete comm;
  return 0;
}

int mvamg_halo_exchange(mvamg_comm* comm, int nsend, const int* send_peer, const double* const* send_buf,
                        const long long* send_count, int nrecv, const int* recv_peer, double* const* recv_buf,
                        const long long* recv_count, void* stream) {
  if (!comm || nsend < 0 || nrecv < 0 || (nsend && (!send_peer || !send_buf || !send_count)) ||
      (nrecv && (!recv_peer || !recv_buf || !recv_count)))
    return fail(MVAMG_E_ARG, "halo_exchange: bad arguments");
  auto& a = ncclabi::api();
  cudaStream_t s = (cudaStream_t)stream;
  NCCL_TRY(a.gstart());
  for (int q = 0; q < nsend; ++q)
    if (send_count[q] > 0) NCCL_TRY(a.send(send_buf[q], (size_t)send_count[q], ncclabi::kFloat64, send_peer[q], comm->c, s));
  for (int q = 0; q < nrecv; ++q)
    if (recv_count[q] > 0) NCCL_TRY(a.recv(recv_buf[q], (size_t)recv_count[q], ncclabi::kFloat64, recv_peer[q], comm->c, s));
  NCCL_TRY(a.gend());
  return 0;
}

int mvamg_allreduce_sum_f64(mvamg_comm* comm, double* buf, long long count, void* stream) {
  if (!comm || !buf || count < 0) return fail(MVAMG_E_ARG, "allreduce: bad arguments");
  NCCL_TRY(ncclabi::api().allreduce(buf, buf, (size_t)count, ncclabi::kFloat64, ncclabi::kSum, comm->c,
                                    (cudaStream_t)stream));
  return 0;
}

int mvamg_set_spmv_stream(int enable) {
  g_spmv_stream = enable != 0;
  return 0;
}

int mvamg_gs_stream_set_trace(long long* trace_dev, int cap) {
  g_stream_trace = trace_dev;
  g_stream_trace_cap = trace_dev ? cap : 0;
  return 0;
}

int mvamg_hierarchy_set_gs_stream(mvamg_hierarchy* h, int k, int mode, int nstages, int nslots, int slot_bytes,
                                  int group, int ncta, const void* blob, const long long* stage_off, double* tfold) {
  if (!h || k < 0 || k >= h->L || mode < 0 || mode > 3) return fail(MVAMG_E_ARG, "set_gs_stream: bad index");
  GsStream& g = h->lv[k].gss[mode];
  g.nstages = nstages; g.nslots = nslots; g.slot_bytes = slot_bytes; g.group = group; g.ncta = ncta;
  g.blob = static_cast<const unsigned char*>(blob);
  g.stage_off = stage_off;
  g.tfold = tfold;
  return 0;
}

int mvamg_gs_rows(int n_all, const int* indptr, const int* indices, const double* data, int mode, int entry_order,
                  long long* nslots, int* nlev, int* rowid, int* cnt, int* crit, double* dg, double* rdg,
                  int* perm, int* wofs, double* coef, int* src, int row_lo, int row_hi) {
  if (n_all < 0 || !indptr || !nslots || !nlev || mode < 0 || mode > 3) return fail(MVAMG_E_ARG, "gs_rows: bad arguments");
  // rows [row_lo, row_hi) are swept (positions); the others are external inputs
  // (ghosts of a row-partitioned level, final before or published during the sweep)
  if (row_lo < 0 && row_hi < 0) { row_lo = 0; row_hi = n_all; }
  if (row_lo < 0 || row_hi < row_lo || row_hi > n_all) return fail(MVAMG_E_ARG, "gs_rows: bad row range");
  const int n = row_hi - row_lo;
  const bool fwd = mode < 2, zero = (mode % 2) == 0;
  auto swept = [&](int j) { return j >= row_lo && j < row_hi; };
  // level sets of the sweep's dependency DAG (external inputs: level -1)
  std::vector<int> lvl(n_all > 0 ? n_all : 1, -1), c(n_all > 0 ? n_all : 1, 0);
  int nl = 0;
  for (int q = 0; q < n; ++q) {
    const int i = fwd ? row_lo + q : row_hi - 1 - q;
    int m = 0;
    for (int k = indptr[i]; k < indptr[i + 1]; ++k) {
      const int j = indices[k];
      if (fwd ? j < i : j > i) m = std::max(m, lvl[j] + 1);
    }
    lvl[i] = m;
    nl = std::max(nl, m + 1);
  }
  for (int i = row_lo; i < row_hi; ++i) {
    int m = 0;
    for (int k = indptr[i]; k < indptr[i + 1]; ++k) {
      const int j = indices[k];
      if (j == i) continue;
      if (zero && (fwd ? j > i : j < i)) continue;
      ++m;
    }
    c[i] = m;
  }
  // topological positions: by level, then longest row first (uniform warps)
  std::vector<int> order(n > 0 ? n : 1);
  for (int q = 0; q < n; ++q) order[q] = row_lo + q;
  std::stable_sort(order.begin(), order.begin() + n, [&](int x, int y) {
    if (lvl[x] != lvl[y]) return lvl[x] < lvl[y];
    return c[x] > c[y];
  });
  const int nw = (n + 31) / 32;
  long long tot = 0;
  for (int w = 0; w < nw; ++w) {
    int m = 0;
    for (int l = 0; l < 32 && w * 32 + l < n; ++l) m = std::max(m, c[order[w * 32 + l]]);
    tot += m;
  }
  if (tot * 32 >= (1LL << 31)) return fail(MVAMG_E_ARG, "gs_rows: too many entries");
  *nslots = tot;
  *nlev = n > 0 ? nl : 0;
  if (!rowid) return 0;
  if (entry_order != 0 && entry_order != 1)
    return fail(MVAMG_E_ARG, "gs_rows: entry order must be 0 (CSR) or 1 (by input level)");
  std::vector<int> ents;
  long long off = 0;
  for (int w = 0; w < nw; ++w) {
    int m = 0;
    for (int l = 0; l < 32 && w * 32 + l < n; ++l) m = std::max(m, c[order[w * 32 + l]]);
    wofs[w] = (int)off;
    for (int l = 0; l < 32; ++l) {
      const int p = w * 32 + l;
      int u = 0;
      if (p < n) {
        const int i = order[p];
        rowid[p] = i;
        cnt[p] = c[i];
        perm[i] = p;
        double dgv = 0.0;
        int lmax = -1, e1 = -1;
        // the row's entries in consumption order: CSR order (entry_order = 0, the
        // reference's rounding), or by the level at which each input becomes
        // final, old values first, CSR order within a level (entry_order = 1:
        // tolerance parity -- the chain is consumed as the inputs land, so
        // only one subtraction is left when the last one arrives)
        ents.clear();
        for (int k = indptr[i]; k < indptr[i + 1]; ++k) {
          const int j = indices[k];
          if (j == i) { dgv = data[k]; continue; }
          const bool isnew = fwd ? j < i : j > i;
          if (zero && !isnew) continue;
          ents.push_back(k);
        }
        auto avail = [&](int k) {
          const int j = indices[k];
          return (fwd ? j < i : j > i) ? lvl[j] : -1;
        };
        if (entry_order == 1)
          std::stable_sort(ents.begin(), ents.end(), [&](int x, int y) { return avail(x) < avail(y); });
        for (int k : ents) {
          const int j = indices[k];
          const bool isnew = fwd ? j < i : j > i;
          const size_t e = (size_t)(off + u) * 32 + l;
          coef[e] = data[k];
          src[e] = isnew ? j : (int)(0x80000000u | (unsigned)j);
          if (isnew && lvl[j] >= lmax && swept(j)) { lmax = lvl[j]; e1 = u; }
          ++u;
        }
        // wait hints: e1 = the entry of the latest input; e2 = the latest one
        // at least two levels earlier (the pre-scan trigger)
        int e2 = -1, l2 = -1;
        for (int uu = 0; uu < (int)ents.size(); ++uu) {
          const int j = indices[ents[uu]];
          const bool isnew = fwd ? j < i : j > i;
          if (isnew && lvl[j] <= lmax - 2 && lvl[j] > l2) { l2 = lvl[j]; e2 = uu; }
        }
        if (u >= 0xffff) e1 = e2 = -1;
        crit[p] = (e1 < 0 ? 0xffff : e1) | ((e2 < 0 ? 0xffff : e2) << 16);
        dg[p] = dgv;
        rdg[p] = 1.0 / dgv;
      }
      for (; u < m; ++u) {  // padding
        const size_t e = (size_t)(off + u) * 32 + l;
        coef[e] = 0.0;
        src[e] = 0;
      }
    }
    off += m;
  }
  wofs[nw] = (int)off;
  return 0;
}

int mvamg_gs_row_sweep_f64(int mode, int n, const int* indptr, const int* indices, const double* data,
                           const int* rowid, const int* cnt, const int* crit, const double* dg, const double* rdg,
                           const int* perm, const int* wofs, const double* coef, const int* src,
                           int threads, int ctas, int max_tile_slots, double* tperm, const double* b,
                           const double* x_old, double* x_new, int* ws, void* stream) {
  if (mode < 0 || mode > 3) return fail(MVAMG_E_ARG, "gs rows: bad mode");
  set_kernel_attrs();
  if (x_old != nullptr && x_old == x_new) return fail(MVAMG_E_ARG, "gs rows: x_new must not alias x_old");
  Csr A;
  A.n = n; A.ip = indptr; A.ix = indices; A.v = data;
  GsRows g;
  g.mode = mode; g.threads = threads; g.ctas = ctas; g.max_tile_slots = max_tile_slots;
  g.rowid = rowid; g.cnt = cnt; g.crit = crit; g.wofs = wofs;
  g.coef = coef; g.src = src; g.dg = dg; g.rdg = rdg; g.perm = perm; g.tperm = tperm;
  return launch_gs_rows(A, g, b, x_old, x_new, ws, ws + 1, (cudaStream_t)stream);
}

// Pipelined sweep of one rank's rows of a row-partitioned level over its
// extended layout [lower ghosts | own rows | upper ghosts] (distributed.py):
// positions are the own rows (mvamg_gs_rows with row range [row_lo, row_hi)),
// ghost inputs are polled in x_ext -- their owners' kernels store them there
// over NVLink as they finish them (mirror tables) -- and every own row's value
// goes to x_ext and to the peers that read it.  x_ext's own and ghost slots
// must hold the sentinel (all-ones) when the ranks start (the caller resets
// them, then synchronises the ranks); for a backward sweep from x_old the old
// lower neighbours (own and ghost, x_old_ext) are folded into the right-hand
// side first, in CSR order.
__global__ void __launch_bounds__(256) gs_prepare_ext_kernel(int npos, const int* __restrict__ rowid, int row_lo,
                                                             const int* __restrict__ ip, const int* __restrict__ ix,
                                                             const double* __restrict__ v,
                                                             const double* __restrict__ b_own,
                                                             const double* __restrict__ xold_ext, double* tperm,
                                                             int* ticket, int fold) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < npos; p += gridDim.x * blockDim.x) {
    const int i = __ldg(rowid + p);
    double s = __ldg(b_own + (i - row_lo));
    if (fold) {
      const int k1 = __ldg(ip + i + 1);
      for (int k = __ldg(ip + i); k < k1; ++k) {
        const int j = __ldg(ix + k);
        if (j >= i) break;
        s = __dsub_rn(s, __dmul_rn(__ldg(v + k), __ldg(xold_ext + j)));
      }
    }
    tperm[p] = s;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *ticket = 0;
}

int mvamg_gs_row_sweep_ext_f64(int mode, int n_ext, int row_lo, int row_hi, const int* indptr, const int* indices,
                               const double* data, const int* rowid, const int* cnt, const int* crit,
                               const double* dg, const double* rdg, const int* wofs, const double* coef,
                               const int* src, int threads, int ctas, int max_tile_slots, double* tperm,
                               const double* b_own, const double* x_old_ext, double* x_ext,
                               const int* mirror_ptr, const unsigned* mirror_dst, double* const* peers,
                               int* ws, void* stream) {
  if (mode != 0 && mode != 2) return fail(MVAMG_E_ARG, "gs rows ext: zero-guess schedules (0, 2) only");
  if (row_lo < 0 || row_hi < row_lo || row_hi > n_ext) return fail(MVAMG_E_ARG, "gs rows ext: bad row range");
  if (threads < 32 || threads > 128 || threads % 32) return fail(MVAMG_E_ARG, "gs rows ext: threads must be 32..128");
  if (x_old_ext && mode != 2) return fail(MVAMG_E_ARG, "gs rows ext: x_old only with the backward schedule");
  const int npos = row_hi - row_lo;
  if (npos == 0) return 0;
  set_kernel_attrs();
  if (!g_row_attr) {
    g_row_attr = true;
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncSetAttribute(gs_row_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - 1024);
    cudaFuncSetAttribute(gs_row_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - 1024);
    cudaGetLastError();
  }
  const size_t smem = (size_t)max_tile_slots * 384;
  if (smem > (size_t)g_max_dyn_smem) return fail(MVAMG_E_ARG, "gs rows ext: tile slices exceed shared memory");
  cudaStream_t s = (cudaStream_t)stream;
  gs_prepare_ext_kernel<<<grid_for(npos), 256, 0, s>>>(npos, rowid, row_lo, indptr, indices, data, b_own,
                                                         x_old_ext, tperm, ws, x_old_ext ? 1 : 0);
  GsRowArgs a;
  a.n = npos;
  a.ntiles = (npos + threads - 1) / threads;
  a.rowid = rowid; a.cnt = cnt; a.crit = crit; a.wofs = wofs; a.coef = coef; a.src = src;
  a.dg = dg; a.rdg = rdg; a.tperm = tperm;
  a.xold = nullptr;
  a.xnew = x_ext;
  a.ticket = ws;
  a.status = ws + 1;
  a.trace = nullptr;
  a.debug = 0;
  a.mirror_ptr = mirror_ptr;
  a.mirror_dst = mirror_dst;
  a.peers = peers;
  a.sys = 1;
  const int grid = std::max(1, std::min(a.ntiles, ctas > 0 ? ctas : num_sms()));
  gs_row_kernel<false><<<grid, threads, smem, s>>>(a);
  CUDA_TRY(cudaGetLastError());
  return 0;
}

// CUDA IPC of a device buffer (the extended x of a rank, for its peers' mirror
// stores): 64-byte handle out / open / close.
int mvamg_ipc_handle(const void* dptr, void* handle64) {
  if (!dptr || !handle64) return fail(MVAMG_E_ARG, "ipc_handle: null");
  cudaIpcMemHandle_t h;
  CUDA_TRY(cudaIpcGetMemHandle(&h, const_cast<void*>(dptr)));
  std::memcpy(handle64, &h, sizeof(h));
  return 0;
}

int mvamg_ipc_open(const void* handle64, void** dptr) {
  if (!handle64 || !dptr) return fail(MVAMG_E_ARG, "ipc_open: null");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle64, sizeof(h));
  CUDA_TRY(cudaIpcOpenMemHandle(dptr, h, cudaIpcMemLazyEnablePeerAccess));
  return 0;
}

int mvamg_ipc_close(void* dptr) {
  if (dptr) CUDA_TRY(cudaIpcCloseMemHandle(dptr));
  return 0;
}

int mvamg_hierarchy_set_gs_rows(mvamg_hierarchy* h, int k, int mode, const int* rowid, const int* cnt,
                                const int* crit, const double* dg, const double* rdg, const int* perm, const int* wofs,
                                const double* coef, const int* src, int threads, int ctas,
                                int max_tile_slots, double* tperm) {
  if (!h || k < 0 || k >= h->L || mode < 0 || mode > 3) return fail(MVAMG_E_ARG, "set_gs_rows: bad index");
  GsRows& g = h->lv[k].grw[mode];
  g.mode = mode; g.threads = threads; g.ctas = ctas; g.max_tile_slots = max_tile_slots;
  g.rowid = rowid; g.cnt = cnt; g.crit = crit; g.wofs = wofs;
  g.coef = coef; g.src = src; g.dg = dg; g.rdg = rdg; g.perm = perm; g.tperm = tperm;
  return 0;
}

int mvamg_gs_cluster_plan(int n, const int* indptr, const int* indices, const double* data, int mode, int grid,
                          int ncta, int wpc, int page_bytes, long long* npages, int* nlev, int* slots_per_cta,
                          int* local_late, int* wptr, int* wpage, int* rowid, int* perm, void* blob) {
  if (n < 0 || !indptr || !npages || !nlev || !slots_per_cta || mode < 0 || mode > 3)
    return fail(MVAMG_E_ARG, "gs_cluster_plan: bad arguments");
  if (wpc < 1 || wpc > 32 || ncta < 1 || (grid ? ncta > 1024 : (ncta > 16 || (ncta & (ncta - 1)))))
    return fail(MVAMG_E_ARG, "gs_cluster_plan: ncta in {1,2,4,8,16} (grid form: 1..1024), wpc in 1..32");
  if (grid && n >= (1 << 30)) return fail(MVAMG_E_ARG, "gs_cluster_plan: too many rows");
  if (page_bytes < 128 || page_bytes % 128) return fail(MVAMG_E_ARG, "gs_cluster_plan: pages of a multiple of 128 bytes");
  const bool fwd = mode < 2, zero = (mode % 2) == 0;
  const int G = ncta * wpc;
  // level sets of the sweep's dependency DAG; crit[i] = an input of the last level
  std::vector<int> lvl(n > 0 ? n : 1, 0), crit(n > 0 ? n : 1, -1), cn(n > 0 ? n : 1, 0);
  int nl = 0;
  for (int q = 0; q < n; ++q) {
    const int i = fwd ? q : n - 1 - q;
    int m = 0, cj = -1, cc = 0;
    for (int k = indptr[i]; k < indptr[i + 1]; ++k) {
      const int j = indices[k];
      if (j == i) continue;
      const bool isnew = fwd ? j < i : j > i;
      if (isnew && lvl[j] + 1 >= m) { m = lvl[j] + 1; cj = j; }
      if (isnew || !zero) ++cc;
    }
    lvl[i] = m;
    crit[i] = cj;
    cn[i] = cc;
    if (kClusterPageHdr + cluster_row_bytes(cc) > page_bytes)
      return fail(MVAMG_E_ARG, "gs_cluster_plan: a row record exceeds the page");
    nl = std::max(nl, m + 1);
  }
  *nlev = n > 0 ? nl : 0;
  // topological positions: by level, original order within a level (stable)
  std::vector<int> order(n > 0 ? n : 1);
  for (int q = 0; q < n; ++q) order[q] = q;
  std::stable_sort(order.begin(), order.begin() + n, [&](int x, int y) { return lvl[x] < lvl[y]; });
  // CTA of every row: its critical input's, while that CTA holds no more than 1.5x
  // its share of the row's DAG level and 1.1x its share of all rows so far; else the
  // CTA with the fewest rows of the level (then the fewest overall)
  std::vector<int> cta(n > 0 ? n : 1, 0), nin(ncta, 0), load(ncta, 0);
  int hits = 0;
  for (int p0 = 0; p0 < n;) {
    int p1 = p0;
    while (p1 < n && lvl[order[p1]] == lvl[order[p0]]) ++p1;
    const int w = p1 - p0;
    const int cap = (g_cluster_cap10 * w + 10 * ncta - 1) / (10 * ncta);
    std::fill(load.begin(), load.end(), 0);
    for (int p = p0; p < p1; ++p) {
      const int i = order[p];
      int c = (g_cluster_local && crit[i] >= 0) ? cta[crit[i]] : -1;
      if (c >= 0 && load[c] < cap && 10LL * nin[c] <= (long long)g_cluster_tot10 * (p / ncta) + 10LL * wpc) {
        ++hits;
      } else {
        c = 0;
        for (int t = 1; t < ncta; ++t)
          if (load[t] < load[c] || (load[t] == load[c] && nin[t] < nin[c])) c = t;
      }
      cta[i] = c;
      ++load[c];
      ++nin[c];
    }
    p0 = p1;
  }
  // a row's entries in consumption order and its late tail: by the level at which each input
  // becomes final (old values first), CSR order within one -- but the critical input (whose CTA
  // the row mostly shares) last of all; late = the inputs of the last level, at most kClusterLate
  auto row_entries = [&](int i, std::vector<int>& ents) -> int {
    ents.clear();
    for (int k = indptr[i]; k < indptr[i + 1]; ++k) {
      const int j = indices[k];
      if (j == i) continue;
      const bool isnew = fwd ? j < i : j > i;
      if (zero && !isnew) continue;
      ents.push_back(k);
    }
    auto avail = [&](int k) {
      const int j = indices[k];
      if (!(fwd ? j < i : j > i)) return -1;
      return 2 * lvl[j] + (j == crit[i] ? 1 : 0);
    };
    std::stable_sort(ents.begin(), ents.end(), [&](int x, int y) { return avail(x) < avail(y); });
    const int cnt = (int)ents.size();
    int late = 0;
    while (late < kClusterLate && late < cnt && avail(ents[cnt - 1 - late]) >= 0 &&
           avail(ents[cnt - 1 - late]) / 2 == avail(ents[cnt - 1]) / 2)
      ++late;
    return late;
  };
  // x slots: every row in the cluster form (peers read them over DSMEM); in the grid form only
  // the rows some row of the same CTA polls as a late input -- shared memory holds nothing else
  std::vector<int> ents;
  std::vector<char> need(n > 0 ? n : 1, grid ? 0 : 1);
  if (grid) {
    for (int i = 0; i < n; ++i) {
      const int late = row_entries(i, ents), cnt = (int)ents.size();
      for (int u = cnt - late; u < cnt; ++u) {
        const int j = indices[ents[u]];
        if (cta[j] == cta[i]) need[j] = 1;
      }
    }
  }
  // a CTA's rows go round-robin to its warps in position order; worker g = warp * ncta + cta
  std::vector<int> seen(ncta, 0), nslot(ncta, 0), wcount(G + 1, 0), wk(n > 0 ? n : 1, 0), sl(n > 0 ? n : 1, -1);
  for (int p = 0; p < n; ++p) {
    const int i = order[p], c = cta[i];
    if (need[i]) sl[i] = nslot[c]++;
    wk[i] = (seen[c] % wpc) * ncta + c;
    ++seen[c];
    ++wcount[wk[i] + 1];
  }
  int slots = 2;
  for (int c = 0; c < ncta; ++c) slots = std::max(slots, nslot[c]);
  if (slots >= (1 << 24)) return fail(MVAMG_E_ARG, "gs_cluster_plan: too many slots per CTA");
  *slots_per_cta = slots;
  if (local_late) *local_late = hits;
  for (int g = 0; g < G; ++g) wcount[g + 1] += wcount[g];
  std::vector<int> fill(wcount.begin(), wcount.end() - 1), qrow(n > 0 ? n : 1, 0);
  for (int p = 0; p < n; ++p) {
    const int i = order[p];
    qrow[fill[wk[i]]++] = i;
  }
  // pages: each worker's records back to back, no record across a page boundary
  std::vector<int> pg_first(G + 1, 0);
  long long pages = 0;
  for (int g = 0; g < G; ++g) {
    pg_first[g] = (int)pages;
    int used = page_bytes;  // forces a first page when the worker has rows
    for (int q = wcount[g]; q < wcount[g + 1]; ++q) {
      const int rb = cluster_row_bytes(cn[qrow[q]]);
      if (used + rb > page_bytes) { ++pages; used = kClusterPageHdr; }
      used += rb;
    }
  }
  pg_first[G] = (int)pages;
  if (pages * (long long)page_bytes >= (1LL << 40)) return fail(MVAMG_E_ARG, "gs_cluster_plan: too many pages");
  *npages = pages;
  if (!blob) return 0;
  if (!wptr || !wpage || !rowid || !perm) return fail(MVAMG_E_ARG, "gs_cluster_plan: missing outputs");
  for (int g = 0; g <= G; ++g) { wptr[g] = wcount[g]; wpage[g] = pg_first[g]; }
  unsigned char* out = static_cast<unsigned char*>(blob);
  std::memset(out, 0, (size_t)pages * page_bytes);
  for (int g = 0; g < G; ++g) {
    long long pg = pg_first[g] - 1;
    int used = page_bytes, rows_in_page = 0;
    for (int q = wcount[g]; q < wcount[g + 1]; ++q) {
      const int i = qrow[q];
      rowid[q] = i;
      perm[i] = q;
      const int cnt = cn[i], rb = cluster_row_bytes(cnt);
      if (used + rb > page_bytes) {
        if (pg >= pg_first[g]) std::memcpy(out + (size_t)pg * page_bytes, &rows_in_page, 4);
        ++pg;
        used = kClusterPageHdr;
        rows_in_page = 0;
      }
      unsigned char* rec = out + (size_t)pg * page_bytes + used;
      double dgv = 0.0;
      for (int k = indptr[i]; k < indptr[i + 1]; ++k)
        if (indices[k] == i) dgv = data[k];
      const int late = row_entries(i, ents);
      const int hdr[4] = {cnt, cnt - late, i, sl[i]};
      const double dd[2] = {dgv, 1.0 / dgv};
      std::memcpy(rec, hdr, 16);
      std::memcpy(rec + 16, dd, 16);
      double* cf = reinterpret_cast<double*>(rec + kClusterRowHdr);
      unsigned* sc = reinterpret_cast<unsigned*>(rec + kClusterRowHdr + 8 * (size_t)cnt);
      for (int u = 0; u < cnt; ++u) {
        const int k = ents[u], j = indices[k];
        const bool isnew = fwd ? j < i : j > i;
        cf[u] = data[k];
        if (!isnew) sc[u] = 0x80000000u | (unsigned)j;
        else if (!grid) sc[u] = ((unsigned)cta[j] << 24) | (unsigned)sl[j];
        else sc[u] = (u >= cnt - late && cta[j] == cta[i]) ? (0x40000000u | (unsigned)sl[j]) : (unsigned)j;
      }
      used += rb;
      ++rows_in_page;
    }
    if (pg >= pg_first[g]) std::memcpy(out + (size_t)pg * page_bytes, &rows_in_page, 4);
  }
  return 0;
}

int mvamg_gs_cluster_sweep_f64(int mode, int n, const int* indptr, const int* indices, const double* data,
                               const int* wptr, const int* wpage, const void* blob, const int* perm, int grid,
                               int ncta, int wpc, int slots, int page_bytes, int sleep_ns, double* tperm,
                               const double* b, const double* x_old, double* x_new, int* ws, void* stream) {
  if (mode < 0 || mode > 3) return fail(MVAMG_E_ARG, "gs cluster: bad mode");
  if (x_old != nullptr && x_old == x_new) return fail(MVAMG_E_ARG, "gs cluster: x_new must not alias x_old");
  Csr A;
  A.n = n; A.ip = indptr; A.ix = indices; A.v = data;
  GsCluster g;
  g.mode = mode; g.ncta = ncta; g.wpc = wpc; g.slots = slots; g.page_bytes = page_bytes; g.sleep_ns = sleep_ns;
  g.grid = grid;
  g.wptr = wptr; g.wpage = wpage; g.blob = static_cast<const unsigned char*>(blob); g.perm = perm; g.tperm = tperm;
  return launch_gs_cluster(A, g, b, x_old, x_new, ws, ws + 1, (cudaStream_t)stream);
}

int mvamg_hierarchy_set_gs_cluster(mvamg_hierarchy* h, int k, int mode, const int* wptr, const int* wpage,
                                   const void* blob, const int* perm, int grid, int ncta, int wpc, int slots,
                                   int page_bytes, int sleep_ns, double* tperm) {
  if (!h || k < 0 || k >= h->L || mode < 0 || mode > 3) return fail(MVAMG_E_ARG, "set_gs_cluster: bad index");
  GsCluster& g = h->lv[k].gcl[mode];
  g.mode = mode; g.ncta = ncta; g.wpc = wpc; g.slots = slots; g.page_bytes = page_bytes; g.sleep_ns = sleep_ns;
  g.grid = grid;
  g.wptr = wptr; g.wpage = wpage; g.blob = static_cast<const unsigned char*>(blob); g.perm = perm; g.tperm = tperm;
  return 0;
}

// ---- setup helpers (host) ---------------------------------------------------
int mvamg_greedy_match(long long ne, const long long* ei, const long long* ej, int n, long long* partner,
                       long long* pair_i, long long* pair_j, long long* npairs) {
  // Accept vertex-disjoint edges in the given (sorted) order -- the greedy
  // 1/2-approximate maximum-product matching (pkg/src/mvamg/_kernels.py:41-61).
  if (n < 0 || ne < 0 || !partner || !npairs) return fail(MVAMG_E_ARG, "greedy_match: bad arguments");
  for (int v = 0; v < n; ++v) partner[v] = -1;
  long long np_ = 0;
  for (long long k = 0; k < ne; ++k) {
    const long long i = ei[k], j = ej[k];
    if (i < 0 || j < 0 || i >= n || j >= n) return fail(MVAMG_E_ARG, "greedy_match: vertex out of range");
    if (partner[i] < 0 && partner[j] < 0) {
      partner[i] = j;
      partner[j] = i;
      if (pair_i) pair_i[np_] = i;
      if (pair_j) pair_j[np_] = j;
      ++np_;
    }
  }
  *npairs = np_;
  return 0;
}

namespace {
// One-sided Jacobi column orthogonalisation of B (m x k, row-major) with V
// (k x k) accumulating the rotations -- the same sweep, pair order, skip rules
// and roundings as pkg/src/mvamg/_kernels.py:64-121.
int jacobi_orthogonalize(double* B, double* V, int m, int k, int max_sweeps, double tol) {
  if (k < 2) return 1;
  const double rel_tol = std::max(tol, 2.0 * m * 2.220446049250313e-16);
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    double total = 0.0;
    for (int p = 0; p < k; ++p)
      for (int r = 0; r < m; ++r) total += B[r * k + p] * B[r * k + p];
    const double floor_ = tol * total;
    int rotated = 0;
    for (int p = 0; p < k - 1; ++p) {
      for (int q = p + 1; q < k; ++q) {
        double alpha = 0.0, beta = 0.0, gamma = 0.0;
        for (int r = 0; r < m; ++r) {
          alpha += B[r * k + p] * B[r * k + p];
          beta += B[r * k + q] * B[r * k + q];
          gamma += B[r * k + p] * B[r * k + q];
        }
        if (gamma == 0.0) continue;
        if (std::fabs(gamma) <= rel_tol * std::sqrt(alpha * beta) || std::fabs(gamma) <= floor_) continue;
        ++rotated;
        const double zeta = (beta - alpha) / (2.0 * gamma);
        const double t = std::copysign(1.0, zeta) / (std::fabs(zeta) + std::sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / std::sqrt(1.0 + t * t);
        const double s = c * t;
        for (int r = 0; r < m; ++r) {
          const double bp = B[r * k + p], bq = B[r * k + q];
          B[r * k + p] = c * bp - s * bq;
          B[r * k + q] = s * bp + c * bq;
        }
        for (int r = 0; r < k; ++r) {
          const double vp = V[r * k + p], vq = V[r * k + q];
          V[r * k + p] = c * vp - s * vq;
          V[r * k + q] = s * vp + c * vq;
        }
      }
    }
    if (rotated == 0) return 1;
  }
  return 0;
}
}  // namespace

int mvamg_jacobi_svd_batch(int nblk, const int* row_ptr, int k, const double* A, int max_sweeps,
                           double tol, double* U, double* sigma, int* failed_block) {
  // Batched thin SVD of stacked blocks (rows row_ptr[b]..row_ptr[b+1], k
  // columns, row-major): pkg/src/mvamg/svd.py:17-55 -- Jacobi, column norms,
  // stable descending sort, U = B / sigma for nonzero sigma.
  if (nblk < 0 || k < 1 || !row_ptr || !A || !U || !sigma) return fail(MVAMG_E_ARG, "jacobi_svd_batch: bad arguments");
  if (failed_block) *failed_block = -1;
  std::vector<double> B, V, s(k);
  std::vector<int> order(k);
  for (int b = 0; b < nblk; ++b) {
    const int r0 = row_ptr[b], m = row_ptr[b + 1] - r0;
    if (m < 1) return fail(MVAMG_E_ARG, "jacobi_svd_batch: empty block");
    B.assign(A + (size_t)r0 * k, A + (size_t)(r0 + m) * k);
    V.assign((size_t)k * k, 0.0);
    for (int i = 0; i < k; ++i) V[(size_t)i * k + i] = 1.0;
    if (!jacobi_orthogonalize(B.data(), V.data(), m, k, max_sweeps, tol)) {
      if (failed_block) *failed_block = b;
      return fail(MVAMG_E_NOT_SPD, "Jacobi SVD did not converge");
    }
    for (int p = 0; p < k; ++p) {
      double acc = 0.0;
      for (int r = 0; r < m; ++r) acc += B[(size_t)r * k + p] * B[(size_t)r * k + p];
      s[p] = std::sqrt(acc);
    }
    for (int p = 0; p < k; ++p) order[p] = p;
    std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return -s[x] < -s[y]; });
    for (int p = 0; p < k; ++p) {
      const int src = order[p];
      sigma[(size_t)b * k + p] = s[src];
      for (int r = 0; r < m; ++r)
        U[(size_t)(r0 + r) * k + p] = s[src] > 0.0 ? B[(size_t)r * k + src] / s[src] : 0.0;
    }
  }
  return 0;
}

int mvamg_dense_gemv_f64(int n, const double* inv, const double* r, double* z, void* stream) {
  int g = std::max(1, std::min((n * 32 + 255) / 256, num_sms() * 8));
  gemv_kernel<<<g, 256, 0, (cudaStream_t)stream>>>(n, inv, r, z);
  CUDA_TRY(cudaGetLastError());
  return 0;
}

int mvamg_dot_ws_bytes(void) { return (2 * kDotMaxBlocks + 1) * 8 + 64; }

int mvamg_dot_f64(int n, const double* x, const double* y, double* result, void* ws, void* stream) {
  ReduceCtx c;
  c.partials = (double*)ws;
  c.counter = (unsigned*)((char*)ws + 2 * kDotMaxBlocks * 8);
  c.sc = nullptr;
  c.fs = nullptr;
  c.out = result;
  dot2_kernel<<<dot_grid(n), 256, 0, (cudaStream_t)stream>>>(n, x, y, nullptr, nullptr, POST_STORE, c);
  CUDA_TRY(cudaGetLastError());
  return 0;
}

int mvamg_hierarchy_create(mvamg_hierarchy** h, int nlevels, int cycle_kind, int inner_fcg_iters,
                           int pre_kind, int pre_sweeps, double pre_omega, int post_kind,
                           int post_sweeps, double post_omega) {
  if (!h || nlevels < 1) return fail(MVAMG_E_ARG, "hierarchy_create: need >= 1 level");
  if (cycle_kind != MVAMG_CYCLE_V && cycle_kind != MVAMG_CYCLE_K) return fail(MVAMG_E_ARG, "unknown cycle kind");
  if (pre_sweeps < 0 || post_sweeps < 0 || inner_fcg_iters < 0) return fail(MVAMG_E_ARG, "negative sweeps/iters");
  auto* H = new mvamg_hierarchy();
  H->L = nlevels;
  H->kind = cycle_kind;
  H->inner = inner_fcg_iters;
  H->pre = Smoother{pre_kind, pre_sweeps, pre_omega};
  H->post = Smoother{post_kind, post_sweeps, post_omega};
  H->lv.resize(nlevels);
  *h = H;
  return 0;
}

int mvamg_hierarchy_destroy(mvamg_hierarchy* h) {
  delete h;
  return 0;
}

int mvamg_hierarchy_set_level(mvamg_hierarchy* h, int k, int n, int nnz, const int* indptr,
                              const int* indices, const double* data, const double* diag,
                              const double* rdiag, int ntiles, const int* chain_ptr,
                              const int* tile_ptr, const int* chain_order, int gs_threads, int gs_window,
                              int gs_wpos) {
  if (!h || k < 0 || k >= h->L) return fail(MVAMG_E_ARG, "set_level: bad level index");
  Level& l = h->lv[k];
  l.A.n = n; l.A.m = n; l.A.nnz = nnz; l.A.ip = indptr; l.A.ix = indices; l.A.v = data;
  l.diag = diag;
  l.rdiag = rdiag;
  l.plan.ntiles = ntiles;
  l.plan.chain_ptr = chain_ptr;
  l.plan.tile_ptr = tile_ptr;
  l.plan.chain_order = chain_order;
  if (gs_wpos < 0 || (gs_wpos & (gs_wpos - 1))) return fail(MVAMG_E_ARG, "set_level: wpos must be 0 or a power of two");
  l.plan.wmask = gs_wpos > 0 ? gs_wpos - 1 : -1;
  l.plan.threads = gs_threads;
  l.plan.window = gs_window;
  return 0;
}

int mvamg_hierarchy_set_gs_schedule(mvamg_hierarchy* h, int k, int mode, const unsigned long long* rec,
                                    const int* round_off, const int* tbase, const int* tile_wbase,
                                    const int* perm, double* tperm, int R, int D, int lean_C,
                                    int slot_words, int rec_words_max) {
  if (!h || k < 0 || k >= h->L || mode < 0 || mode > 2) return fail(MVAMG_E_ARG, "set_gs_schedule: bad index");
  GsList& g = h->lv[k].gl[mode];
  g.lean_C = lean_C;
  g.rec = rec; g.round_off = round_off; g.tbase = tbase; g.tile_wbase = tile_wbase; g.perm = perm;
  g.tperm = tperm; g.R = R; g.D = D; g.slot_words = slot_words; g.rec_words_max = rec_words_max;
  return 0;
}

int mvamg_hierarchy_set_transfer(mvamg_hierarchy* h, int k, const int* p_indptr, const int* p_indices,
                                 const double* p_data, const int* r_indptr, const int* r_indices,
                                 const double* r_data) {
  if (!h || k < 0 || k >= h->L - 1) return fail(MVAMG_E_ARG, "set_transfer: bad level index");
  if (!p_indptr || !p_indices || !p_data || !r_indptr || !r_indices || !r_data)
    return fail(MVAMG_E_ARG, "set_transfer: null operand");
  // P's and R's shapes come from the levels on both sides: both must be set first
  if (!h->lv[k].A.ip || !h->lv[k + 1].A.ip)
    return fail(MVAMG_E_STATE, "set_transfer: levels " + std::to_string(k) + " and " + std::to_string(k + 1) +
                                   " must be set (mvamg_hierarchy_set_level) before transfer " + std::to_string(k));
  Level& l = h->lv[k];
  l.P.n = l.A.n; l.P.m = h->lv[k + 1].A.n; l.P.ip = p_indptr; l.P.ix = p_indices; l.P.v = p_data;
  l.R.n = h->lv[k + 1].A.n; l.R.m = l.A.n; l.R.ip = r_indptr; l.R.ix = r_indices; l.R.v = r_data;
  // entry counts (one small read each, at setup): they pick the warp-per-row SpMV on small levels.
  // The caller's uploads may still be in flight on any stream: wait for the device first.
  CUDA_TRY(cudaDeviceSynchronize());
  CUDA_TRY(cudaMemcpy(&l.P.nnz, p_indptr + l.P.n, sizeof(int), cudaMemcpyDeviceToHost));
  CUDA_TRY(cudaMemcpy(&l.R.nnz, r_indptr + l.R.n, sizeof(int), cudaMemcpyDeviceToHost));
  return 0;
}

int mvamg_hierarchy_set_coarse(mvamg_hierarchy* h, const double* inv) {
  if (!h) return fail(MVAMG_E_ARG, "set_coarse: null");
  h->inv = inv;
  return 0;
}

static size_t al(size_t b) { return (b + 255) & ~(size_t)255; }

static size_t workspace_layout(mvamg_hierarchy* h, char* base) {
  size_t off = 0;
  auto take = [&](size_t bytes) -> char* {
    char* p = base ? base + off : nullptr;
    off += al(bytes);
    return p;
  };
  h->partials = (double*)take(2 * kDotMaxBlocks * 8);
  h->counter = (unsigned*)take(64);
  h->ticket = (int*)take(64);
  h->sc = (DevScalars*)take(sizeof(DevScalars));
  int n0 = h->lv[0].A.n;
  for (double** p : {&h->px, &h->pr, &h->pp, &h->pq, &h->pt, &h->pu, &h->pz, &h->in})
    *p = (double*)take((size_t)n0 * 8);
  for (int k = 0; k < h->L; ++k) {
    Level& l = h->lv[k];
    size_t n = (size_t)l.A.n * 8;
    l.r = (double*)take(n);
    if (k < h->L - 1) {
      l.xa = (double*)take(n);
      l.xb = (double*)take(n);
      l.t = (double*)take(n);
    } else {
      l.z = (double*)take(n);
    }
    if (h->fcg_level(k)) {
      l.fr = (double*)take(n);
      l.fx = (double*)take(n);
      for (int q = 0; q < 2; ++q) {
        l.fp[q] = (double*)take(n);
        l.fap[q] = (double*)take(n);
      }
      l.fs = (FcgScalars*)take(sizeof(FcgScalars));
    }
  }
  return off;
}

int mvamg_hierarchy_workspace_bytes(mvamg_hierarchy* h, long long* bytes) {
  if (!h || !bytes) return fail(MVAMG_E_ARG, "workspace_bytes: null");
  *bytes = (long long)workspace_layout(h, nullptr);
  return 0;
}

int mvamg_hierarchy_bind_workspace(mvamg_hierarchy* h, void* ws, void* stream) {
  if (!h || !ws) return fail(MVAMG_E_ARG, "bind_workspace: null");
  for (int k = 0; k < h->L; ++k)
    if (!h->lv[k].A.ip) return fail(MVAMG_E_STATE, "bind_workspace: level " + std::to_string(k) + " not set");
  if (!h->inv) return fail(MVAMG_E_STATE, "bind_workspace: coarse inverse not set");
  for (int k = 0; k < h->L - 1; ++k) {
    const Level& l = h->lv[k];
    if (!l.P.ip || !l.R.ip) return fail(MVAMG_E_STATE, "bind_workspace: transfer " + std::to_string(k) + " not set");
    if (l.P.n != l.A.n || l.P.m != h->lv[k + 1].A.n || l.R.n != h->lv[k + 1].A.n || l.R.m != l.A.n)
      return fail(MVAMG_E_STATE, "bind_workspace: transfer " + std::to_string(k) +
                                     " was set before a level it connects changed size");
  }
  workspace_layout(h, (char*)ws);
  set_kernel_attrs();
  for (int k = 0; k < h->L - 1; ++k)
    for (int m = 0; m < 3; ++m)
      if (h->lv[k].plan.ntiles > 0 && h->lv[k].gl[m].rec) gs_blocks(h->lv[k].plan, h->lv[k].gl[m]);
  cudaStream_t s = (cudaStream_t)stream;
  CUDA_TRY(cudaMemsetAsync(h->counter, 0, 64, s));
  CUDA_TRY(cudaMemsetAsync(h->ticket, 0, 64, s));
  CUDA_TRY(cudaMemsetAsync(h->sc, 0, sizeof(DevScalars), s));
  if (!h->host_sc) CUDA_TRY(cudaMallocHost(&h->host_sc, sizeof(DevScalars)));
  for (auto& kv : h->graphs) cudaGraphExecDestroy(kv.second);
  h->graphs.clear();
  h->bound = true;
  return 0;
}

int mvamg_hierarchy_set_graphs(mvamg_hierarchy* h, int enable) {
  if (!h) return fail(MVAMG_E_ARG, "null");
  h->use_graphs = enable != 0;
  return 0;
}

int mvamg_cycle_apply(mvamg_hierarchy* h, const double* r, double* z, void* stream) {
  if (!h || !h->bound) return fail(MVAMG_E_STATE, "cycle_apply: workspace not bound");
  cudaStream_t s = (cudaStream_t)stream;
  int n = h->lv[0].A.n;
  CUDA_TRY(cudaMemcpyAsync(h->in, r, (size_t)n * 8, cudaMemcpyDeviceToDevice, s));
  const double* out = nullptr;
  int st = h->run_graph("apply", s, [&](cudaStream_t cs) -> int {
    int e = h->cycle(h->in, out, cs);
    if (e) return e;
    copy_kernel<<<grid_for(n), 256, 0, cs>>>(n, h->pz, out);
    return 0;
  });
  if (st) return st;
  CUDA_TRY(cudaMemcpyAsync(z, h->pz, (size_t)n * 8, cudaMemcpyDeviceToDevice, s));
  return 0;
}

int mvamg_error_propagation(mvamg_hierarchy* h, const double* x, double* e, void* stream) {
  if (!h || !h->bound) return fail(MVAMG_E_STATE, "error_propagation: workspace not bound");
  cudaStream_t s = (cudaStream_t)stream;
  int n = h->lv[0].A.n;
  CUDA_TRY(cudaMemcpyAsync(h->pu, x, (size_t)n * 8, cudaMemcpyDeviceToDevice, s));
  int st = h->run_graph("errprop", s, [&](cudaStream_t cs) -> int {
    int q = launch_spmv(0, h->lv[0].A, h->pu, nullptr, h->in, cs);
    if (q) return q;
    const double* out = nullptr;
    if ((q = h->cycle(h->in, out, cs))) return q;
    sub_kernel<<<grid_for(n), 256, 0, cs>>>(n, h->pz, h->pu, out);
    return 0;
  });
  if (st) return st;
  CUDA_TRY(cudaMemcpyAsync(e, h->pz, (size_t)n * 8, cudaMemcpyDeviceToDevice, s));
  return 0;
}

int mvamg_hierarchy_status(mvamg_hierarchy* h, int* status, int reset) {
  if (!h || !h->bound) return fail(MVAMG_E_STATE, "status: workspace not bound");
  int v = 0;
  CUDA_TRY(cudaMemcpy(&v, h->status_ptr(), sizeof(int), cudaMemcpyDeviceToHost));
  *status = v;
  if (reset) CUDA_TRY(cudaMemset(h->status_ptr(), 0, sizeof(int)));
  return 0;
}

int mvamg_pcg_solve(mvamg_hierarchy* h, int pc_kind, mvamg_composite* comp, const double* b,
                    double* x, double rtol, int itmax, double* hist, int* nit, int* converged,
                    int* status, void* stream) {
  if (!h) return fail(MVAMG_E_ARG, "pcg: null hierarchy");
  cudaStream_t s = (cudaStream_t)stream;
  int st = pcg_device(h, pc_kind, comp, b, rtol, itmax, hist, nit, converged, status, s);
  if (st) return st;
  CUDA_TRY(cudaMemcpyAsync(x, h->px, (size_t)h->lv[0].A.n * 8, cudaMemcpyDeviceToDevice, s));
  return 0;
}

int mvamg_pcg_solve_host(mvamg_hierarchy* h, int pc_kind, mvamg_composite* comp, const double* b_host,
                         double* x_host, double rtol, int itmax, double* hist_host, int* nit,
                         int* converged, int* status, void* stream) {
  if (!h || !h->bound) return fail(MVAMG_E_STATE, "pcg_host: workspace not bound");
  cudaStream_t s = (cudaStream_t)stream;
  size_t nb = (size_t)h->lv[0].A.n * 8;
  // stage b in the PCG input buffer, solve, read back x and the history
  CUDA_TRY(cudaMemcpyAsync(h->in, b_host, nb, cudaMemcpyHostToDevice, s));
  double* hist_dev = h->pt;  // n0 doubles; itmax+1 must fit
  if ((size_t)itmax + 1 > (size_t)h->lv[0].A.n) {
    // history longer than one level-0 vector: use a temporary allocation
    CUDA_TRY(cudaMallocAsync((void**)&hist_dev, ((size_t)itmax + 1) * 8, s));
  }
  int st = pcg_device(h, pc_kind, comp, h->in, rtol, itmax, hist_dev, nit, converged, status, s);
  if (st) {
    if (hist_dev != h->pt) cudaFreeAsync(hist_dev, s);
    return st;
  }
  CUDA_TRY(cudaMemcpyAsync(x_host, h->px, nb, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaMemcpyAsync(hist_host, hist_dev, ((size_t)*nit + 1) * 8, cudaMemcpyDeviceToHost, s));
  if (hist_dev != h->pt) CUDA_TRY(cudaFreeAsync(hist_dev, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  return 0;
}

int mvamg_composite_create(mvamg_composite** c, int ncomp, mvamg_hierarchy* const* comps) {
  if (!c || ncomp < 1 || !comps) return fail(MVAMG_E_ARG, "composite has no components");
  int n = comps[0]->lv[0].A.n;
  for (int i = 0; i < ncomp; ++i) {
    if (!comps[i] || !comps[i]->bound) return fail(MVAMG_E_STATE, "composite: component not bound");
    if (comps[i]->lv[0].A.n != n) return fail(MVAMG_E_ARG, "composite: component sizes differ");
  }
  auto* C = new mvamg_composite();
  C->ops.assign(comps, comps + ncomp);
  C->n = n;
  C->serial = ++g_composite_serial;
  if (cudaMalloc(&C->t, (size_t)n * 8) != cudaSuccess || cudaMalloc(&C->acc, (size_t)n * 8) != cudaSuccess) {
    delete C;
    return fail(MVAMG_E_CUDA, "composite: cudaMalloc failed");
  }
  *c = C;
  return 0;
}

int mvamg_composite_destroy(mvamg_composite* c) {
  delete c;
  return 0;
}

int mvamg_composite_apply_symmetrized(mvamg_composite* c, double* x, void* stream) {
  if (!c) return fail(MVAMG_E_ARG, "composite: null");
  cudaStream_t s = (cudaStream_t)stream;
  mvamg_hierarchy* h0 = c->ops[0];
  CUDA_TRY(cudaMemcpyAsync(c->acc, x, (size_t)c->n * 8, cudaMemcpyDeviceToDevice, s));
  int st = h0->run_graph("composite/" + std::to_string(c->serial), s,
                         [&](cudaStream_t cs) -> int { return c->symmetrized(c->acc, cs); });
  if (st) return st;
  CUDA_TRY(cudaMemcpyAsync(x, c->acc, (size_t)c->n * 8, cudaMemcpyDeviceToDevice, s));
  return 0;
}

int mvamg_composite_precond(mvamg_composite* c, const double* r, double* z, void* stream) {
  if (!c) return fail(MVAMG_E_ARG, "composite: null");
  cudaStream_t s = (cudaStream_t)stream;
  mvamg_hierarchy* h0 = c->ops[0];
  CUDA_TRY(cudaMemcpyAsync(h0->in, r, (size_t)c->n * 8, cudaMemcpyDeviceToDevice, s));
  const double* out = nullptr;
  int st = h0->run_graph("compprec/" + std::to_string(c->serial), s, [&](cudaStream_t cs) -> int {
    int e = c->precond(h0->in, out, cs);
    if (e) return e;
    copy_kernel<<<grid_for(c->n), 256, 0, cs>>>(c->n, h0->pz, out);
    return 0;
  });
  if (st) return st;
  CUDA_TRY(cudaMemcpyAsync(z, h0->pz, (size_t)c->n * 8, cudaMemcpyDeviceToDevice, s));
  return 0;
}


struct mvamg_spmat {
  DevCsr m;
};

int mvamg_galerkin_f64(int n, int nc, const int* a_indptr, const int* a_indices, const double* a_data,
                       const int* p_indptr, const int* p_indices, const double* p_data, mvamg_spmat** out,
                       long long* nnz_out, float* phase_ms, void* stream) {
  if (!out || n < 0 || nc < 0 || !a_indptr || !p_indptr) return fail(MVAMG_E_ARG, "galerkin: bad arguments");
  *out = nullptr;
  cudaStream_t s = (cudaStream_t)stream;
  int nnz_a = 0, nnz_p = 0;
  CUDA_TRY(cudaMemcpyAsync(&nnz_a, a_indptr + n, 4, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaMemcpyAsync(&nnz_p, p_indptr + n, 4, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  Csr A, P;
  A.n = A.m = n;
  A.nnz = nnz_a;
  A.ip = a_indptr;
  A.ix = a_indices;
  A.v = a_data;
  P.n = n;
  P.m = nc;
  P.nnz = nnz_p;
  P.ip = p_indptr;
  P.ix = p_indices;
  P.v = p_data;
  auto* h = new mvamg_spmat();
  int e = galerkin_device(n, nc, A, P, h->m, s, phase_ms);
  if (e) {
    h->m.release();
    delete h;
    return e;
  }
  *out = h;
  if (nnz_out) *nnz_out = h->m.nnz;
  return 0;
}

int mvamg_spmat_copy(const mvamg_spmat* m, int* indptr, int* indices, double* data, void* stream) {
  if (!m || !indptr) return fail(MVAMG_E_ARG, "spmat_copy: bad arguments");
  cudaStream_t s = (cudaStream_t)stream;
  CUDA_TRY(cudaMemcpyAsync(indptr, m->m.ip, (size_t)(m->m.n + 1) * 4, cudaMemcpyDeviceToDevice, s));
  if (m->m.nnz > 0) {
    CUDA_TRY(cudaMemcpyAsync(indices, m->m.ix, (size_t)m->m.nnz * 4, cudaMemcpyDeviceToDevice, s));
    CUDA_TRY(cudaMemcpyAsync(data, m->m.v, (size_t)m->m.nnz * 8, cudaMemcpyDeviceToDevice, s));
  }
  return 0;
}

int mvamg_spmat_destroy(mvamg_spmat* m) {
  if (m) {
    for (void* p : {(void*)m->m.ip, (void*)m->m.ix, (void*)m->m.v})
      if (p) cudaFree(p);  // synchronous: the creating stream may be gone
    delete m;
  }
  return 0;
}


int mvamg_gather_f64(int n, const int* idx, const double* src, double* dst, void* stream) {
  if (n < 0) return fail(MVAMG_E_ARG, "gather: n < 0");
  if (n == 0) return 0;
  gather_kernel<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(n, idx, src, dst);
  ++g_kernel_launches;
  CUDA_TRY(cudaGetLastError());
  return 0;
}

int mvamg_scatter_f64(int n, const int* idx, const double* src, double* dst, void* stream) {
  if (n < 0) return fail(MVAMG_E_ARG, "scatter: n < 0");
  if (n == 0) return 0;
  scatter_kernel<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(n, idx, src, dst);
  ++g_kernel_launches;
  CUDA_TRY(cudaGetLastError());
  return 0;
}

int mvamg_axpy_f64(int n, double alpha, const double* x, double* y, void* stream) {
  if (n < 0) return fail(MVAMG_E_ARG, "axpy: n < 0");
  if (n == 0) return 0;
  axpy_kernel<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(n, alpha, x, y);
  ++g_kernel_launches;
  CUDA_TRY(cudaGetLastError());
  return 0;
}

int mvamg_xpby_f64(int n, const double* x, double beta, double* y, void* stream) {
  if (n < 0) return fail(MVAMG_E_ARG, "xpby: n < 0");
  if (n == 0) return 0;
  xpby_kernel<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(n, x, beta, y);
  ++g_kernel_launches;
  CUDA_TRY(cudaGetLastError());
  return 0;
}


int mvamg_greedy_match_device(int n, const int* indptr, const int* indices, const double* data,
                              const double* diag, const double* w, double weight_floor, int* partner,
                              int* rounds_out, void* stream) {
  using namespace matching;
  if (n < 0 || (n > 0 && (!indptr || !indices || !data || !diag || !w || !partner)))
    return fail(MVAMG_E_ARG, "greedy_match_device: bad arguments");
  if (rounds_out) *rounds_out = 0;
  if (n == 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  DevTmp best(s), flag(s);
  CUDA_TRY(best.alloc((size_t)n * 4));
  CUDA_TRY(flag.alloc(16));
  fill_int_kernel<<<grid_for(n), 256, 0, s>>>(n, partner, -1);
  ++g_kernel_launches;
  int rounds = 0;
  for (;;) {
    CUDA_TRY(cudaMemsetAsync(flag.p, 0, 4, s));
    match_best_kernel<<<grid_for(n), 256, 0, s>>>(n, indptr, indices, data, diag, w, weight_floor, partner,
                                                  best.get<int>());
    match_pair_kernel<<<grid_for(n), 256, 0, s>>>(n, best.get<int>(), partner, flag.get<int>());
    g_kernel_launches += 2;
    CUDA_TRY(cudaGetLastError());
    int changed = 0;
    CUDA_TRY(cudaMemcpyAsync(&changed, flag.p, 4, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    ++rounds;
    if (!changed) break;
    if (rounds > n + 1) return fail(MVAMG_E_STATE, "greedy_match_device: no progress");
  }
  if (rounds_out) *rounds_out = rounds;
  return 0;
}

int mvamg_jacobi_svd_batch_device(int nblk, const int* row_ptr, int k, const double* A, int max_sweeps,
                                  double tol, double* U, double* sigma, int* failed_block, void* stream) {
  // mvamg_jacobi_svd_batch on the GPU (svd.cuh): device pointers, bit-identical U and sigma.
  if (nblk < 0 || k < 1 || k > svd::kMaxCols || (nblk > 0 && (!row_ptr || !A || !U || !sigma)))
    return fail(MVAMG_E_ARG, "jacobi_svd_batch_device: bad arguments (k must be 1..16)");
  if (failed_block) *failed_block = -1;
  if (nblk == 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  DevTmp status(s);
  CUDA_TRY(status.alloc(8));
  matching::fill_int_kernel<<<1, 32, 0, s>>>(2, status.get<int>(), 0x7fffffff);
  svd::jacobi_svd_kernel<<<(nblk + 63) / 64, 64, 0, s>>>(nblk, row_ptr, k, A, max_sweeps, tol, U, sigma,
                                                         status.get<int>());
  g_kernel_launches += 2;
  CUDA_TRY(cudaGetLastError());
  int st[2];
  CUDA_TRY(cudaMemcpyAsync(st, status.p, 8, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  if (st[1] != 0x7fffffff && st[1] < st[0]) return fail(MVAMG_E_ARG, "jacobi_svd_batch_device: empty block");
  if (st[0] != 0x7fffffff) {
    if (failed_block) *failed_block = st[0];
    return fail(MVAMG_E_NOT_SPD, "Jacobi SVD did not converge");
  }
  return 0;
}

}  // extern "C"
