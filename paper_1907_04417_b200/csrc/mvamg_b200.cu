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

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "../../include/mvamg_b200.h"
#include "mvamg_kernels.cuh"

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
  bool ok = cudaFuncSetAttribute(gs_sweep_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm) == cudaSuccess;
  ok &= cudaFuncSetAttribute(gs_sweep_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm) == cudaSuccess;
  ok &= cudaFuncSetAttribute(gs_sweep_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm) == cudaSuccess;
  ok &= cudaFuncSetAttribute(gs_sweep_kernel<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm) == cudaSuccess;
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
  const int* tile_ptr = nullptr;
};

struct Smoother {
  int kind, sweeps;
  double omega;
};

// ---- raw launches ----------------------------------------------------------
int launch_spmv(int mode, const Csr& A, const double* x, const double* b, double* y, cudaStream_t s) {
  if (A.n == 0) return 0;
  int g = grid_for(A.n);
  if (mode == 0) spmv_kernel<0><<<g, 256, 0, s>>>(A.n, A.ip, A.ix, A.v, x, b, y);
  else if (mode == 1) spmv_kernel<1><<<g, 256, 0, s>>>(A.n, A.ip, A.ix, A.v, x, b, y);
  else spmv_kernel<2><<<g, 256, 0, s>>>(A.n, A.ip, A.ix, A.v, x, b, y);
  CUDA_TRY(cudaGetLastError());
  return 0;
}

int gs_blocks(const GsPlan& p) {
  static std::map<std::pair<int, int>, int> occ_cache;
  size_t smem = (size_t)p.window * sizeof(double);
  auto key = std::make_pair(p.threads, p.window);
  auto it = occ_cache.find(key);
  int per_sm;
  if (it != occ_cache.end()) {
    per_sm = it->second;
  } else {
    per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gs_sweep_kernel<true, true>, p.threads, smem);
    if (per_sm < 1) per_sm = 1;
    occ_cache[key] = per_sm;
  }
  return std::max(1, std::min(p.ntiles, per_sm * num_sms()));
}

int launch_gs(bool fwd, bool zero, const Csr& A, const double* diag, const double* rdiag,
              const GsPlan& p, const double* b, const double* xold, double* xnew, int* ticket,
              int* status, cudaStream_t s) {
  if (A.n == 0) return 0;
  set_kernel_attrs();
  if ((size_t)p.window * sizeof(double) > (size_t)g_max_dyn_smem)
    return fail(MVAMG_E_ARG, "gs: window of " + std::to_string(p.window) + " rows exceeds shared memory");
  gs_prep_kernel<<<grid_for(A.n), 256, 0, s>>>(A.n, xnew, ticket);
  GsArgs a;
  a.n = A.n;
  a.ntiles = p.ntiles;
  a.window = p.window;
  a.ip = A.ip;
  a.ix = A.ix;
  a.v = A.v;
  a.diag = diag;
  a.rdiag = rdiag;
  a.chain_ptr = p.chain_ptr;
  a.tile_ptr = p.tile_ptr;
  a.b = b;
  a.xold = xold;
  a.xnew = xnew;
  a.ticket = ticket;
  a.status = status;
  int g = gs_blocks(p);
  size_t smem = (size_t)p.window * sizeof(double);
  if (fwd && zero) gs_sweep_kernel<true, true><<<g, p.threads, smem, s>>>(a);
  else if (fwd) gs_sweep_kernel<true, false><<<g, p.threads, smem, s>>>(a);
  else if (zero) gs_sweep_kernel<false, true><<<g, p.threads, smem, s>>>(a);
  else gs_sweep_kernel<false, false><<<g, p.threads, smem, s>>>(a);
  CUDA_TRY(cudaGetLastError());
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
        st = launch_gs(fwd, x_cur == nullptr, l.A, l.diag, l.rdiag, l.plan, b, x_cur, out, ticket,
                       status_ptr(), s);
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
      cudaGraphExec_t exec;
      e = cudaGraphInstantiate(&exec, graph, 0);
      cudaGraphDestroy(graph);
      if (e != cudaSuccess) return fail(MVAMG_E_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(e));
      it = graphs.emplace(key, exec).first;
    }
    CUDA_TRY(cudaGraphLaunch(it->second, s));
    return 0;
  }
};

struct mvamg_composite {
  std::vector<mvamg_hierarchy*> ops;
  double *t = nullptr, *acc = nullptr;
  int n = 0;
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
  auto sync_flags = [&]() -> int {
    CUDA_TRY(cudaMemcpyAsync(h->host_sc, h->sc, sizeof(DevScalars), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    return 0;
  };
  if ((st = sync_flags())) return st;
  if (!h->host_sc->stop) {
    // z = M r ; rz = r'z ; p = z
    std::string key0 = "pcg0/" + std::to_string(pc) + "/" + std::to_string((size_t)comp);
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
    std::string keyA = "pcgA", keyB = "pcgB/" + std::to_string(pc) + "/" + std::to_string((size_t)comp);
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

}  // namespace

// ============================================================================
// C ABI
// ============================================================================
extern "C" {

int mvamg_version(void) { return 1; }
const char* mvamg_last_error(void) { return g_err.c_str(); }

int mvamg_gs_analyse(int n, const int* indptr, const int* indices, int max_chain, int max_threads,
                     int max_window, int* nchains, int* ntiles, int* chain_ptr, int* tile_ptr,
                     int* threads_out, int* window_out, int* depth_out) {
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
  // tiles: consecutive chains, <= max_threads chains, rows <= max_window
  std::vector<int> tp;
  tp.push_back(0);
  int cnt = 0, rows = 0, maxcnt = 1, maxrows = 0;
  for (int c = 0; c < nc; ++c) {
    int cl = cp[c + 1] - cp[c];
    if (cnt > 0 && (cnt + 1 > max_threads || rows + cl > max_window)) {
      tp.push_back(c);
      maxcnt = std::max(maxcnt, cnt);
      maxrows = std::max(maxrows, rows);
      cnt = 0;
      rows = 0;
    }
    ++cnt;
    rows += cl;
  }
  if (nc > 0) {
    tp.push_back(nc);
    maxcnt = std::max(maxcnt, cnt);
    maxrows = std::max(maxrows, rows);
  }
  int nt = (int)tp.size() - 1;
  *nchains = nc;
  *ntiles = nt;
  if (chain_ptr) std::copy(cp.begin(), cp.end(), chain_ptr);
  if (tile_ptr) std::copy(tp.begin(), tp.end(), tile_ptr);
  if (threads_out) *threads_out = std::min(256, ((maxcnt + 31) / 32) * 32);
  if (window_out) *window_out = std::min(maxrows, max_window);
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
  if (max_threads > 256) return fail(MVAMG_E_ARG, "gs_analyse: max_threads > 256");
  return 0;
}

int mvamg_csr_spmv_f64(int n, const int* indptr, const int* indices, const double* data,
                       const double* x, double* y, void* stream) {
  Csr A;
  A.n = n; A.ip = indptr; A.ix = indices; A.v = data;
  return launch_spmv(0, A, x, nullptr, y, (cudaStream_t)stream);
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

int mvamg_gs_sweep_f64(int direction, int zero_init, int n, const int* indptr, const int* indices,
                       const double* data, const double* diag, const double* rdiag, int ntiles,
                       const int* chain_ptr, const int* tile_ptr, int threads, int window,
                       const double* b, const double* x_old, double* x_new, int* ws, void* stream) {
  if (threads < 32 || threads > 256 || threads % 32) return fail(MVAMG_E_ARG, "gs: threads must be 32..256, multiple of 32");
  if (!zero_init && x_old == x_new) return fail(MVAMG_E_ARG, "gs: x_new must not alias x_old");
  Csr A;
  A.n = n; A.ip = indptr; A.ix = indices; A.v = data;
  GsPlan p;
  p.ntiles = ntiles; p.threads = threads; p.window = window; p.chain_ptr = chain_ptr; p.tile_ptr = tile_ptr;
  return launch_gs(direction == 0, zero_init != 0, A, diag, rdiag, p, b, x_old, x_new, ws, ws + 1,
                   (cudaStream_t)stream);
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
                              const int* tile_ptr, int gs_threads, int gs_window) {
  if (!h || k < 0 || k >= h->L) return fail(MVAMG_E_ARG, "set_level: bad level index");
  Level& l = h->lv[k];
  l.A.n = n; l.A.m = n; l.A.nnz = nnz; l.A.ip = indptr; l.A.ix = indices; l.A.v = data;
  l.diag = diag;
  l.rdiag = rdiag;
  l.plan.ntiles = ntiles;
  l.plan.chain_ptr = chain_ptr;
  l.plan.tile_ptr = tile_ptr;
  l.plan.threads = gs_threads;
  l.plan.window = gs_window;
  return 0;
}

int mvamg_hierarchy_set_transfer(mvamg_hierarchy* h, int k, const int* p_indptr, const int* p_indices,
                                 const double* p_data, const int* r_indptr, const int* r_indices,
                                 const double* r_data) {
  if (!h || k < 0 || k >= h->L - 1) return fail(MVAMG_E_ARG, "set_transfer: bad level index");
  Level& l = h->lv[k];
  l.P.n = l.A.n; l.P.m = h->lv[k + 1].A.n; l.P.ip = p_indptr; l.P.ix = p_indices; l.P.v = p_data;
  l.R.n = h->lv[k + 1].A.n; l.R.m = l.A.n; l.R.ip = r_indptr; l.R.ix = r_indices; l.R.v = r_data;
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
  workspace_layout(h, (char*)ws);
  set_kernel_attrs();
  for (int k = 0; k < h->L - 1; ++k)
    if (h->lv[k].plan.ntiles > 0) gs_blocks(h->lv[k].plan);
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
  if (st) return st;
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
  int st = h0->run_graph("composite/" + std::to_string((size_t)c), s,
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
  int st = h0->run_graph("compprec/" + std::to_string((size_t)c), s, [&](cudaStream_t cs) -> int {
    int e = c->precond(h0->in, out, cs);
    if (e) return e;
    copy_kernel<<<grid_for(c->n), 256, 0, cs>>>(c->n, h0->pz, out);
    return 0;
  });
  if (st) return st;
  CUDA_TRY(cudaMemcpyAsync(z, h0->pz, (size_t)c->n * 8, cudaMemcpyDeviceToDevice, s));
  return 0;
}

}  // extern "C"
