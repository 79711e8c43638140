// gs_scan.cuh -- chain-scan Gauss-Seidel sweep for fine levels with chain
// structure (tolerance parity: GpuConfig.exact_gs = False).
//
// The reference sweep (pkg/src/mvamg/_kernels.py:15-38) updates rows in order.
// On a grid, consecutive rows form chains (grid lines).  Within a chain, row i
// depends on row i-1; every other new-value source lies in an earlier chain.
// For one chain the update is the affine recurrence
//     x_i = o_i + s_i * x_{i-1},   s_i = -a_{i,i-1} / a_ii,
//     o_i = (b_i - sum_old a_ij x_j - sum_{j in earlier chains} a_ij x_j) / a_ii.
// A warp takes 32 rows of a chain at a time (a segment).  It forms their o_i
// from the earlier chains, composes the 32 affine maps with a 5-step shuffle
// scan, and applies the carry from the previous segment.  The in-line
// dependency chain of 32 rows becomes log2(32) steps.  The DAG is the
// reference's: every row still uses the new values of all earlier rows and
// the old values of all later rows.  Only the rounding differs (sums
// reassociated, o_i scaled by RN(1/a_ii)).
//
// Depth: a segment waits for the source segments of its rows, e.g. on a
// 2-D grid line L segment s waits for line L-1 segment s+1.  The wavefront is
// therefore 2 x (lines) + (segments per line) steps: 2,080 on C2's fine level,
// against 3,070 row levels for the exact sweep.  Each step is one warp scan,
// not one row.
//
// One CTA runs the whole sweep.  Chains go round-robin to its warps.  The x
// values of the last S chains live in a shared-memory ring (slot = chain mod
// S).  Progress counters in shared memory order the warps; nothing crosses
// L2 on the dependency path.  The old-value terms and b are folded into o_i by
// a fully parallel pre-pass (gs_scan_prepass_kernel) before the sweep.
#pragma once

#include <cuda_runtime.h>

namespace mvamg {
namespace gsscan {

constexpr int kMaxDeps = 4;  // distinct source-chain distances

constexpr int kStages = 3;     // segments of records in flight per warp (TMA bulk copies)

// Per-segment header (32 B, one bulk copy with the records): the two waits
// ((delta << 20) | segments needed), the deferred source of the last row
// (same encoding) and its position, then its coefficient.
struct __align__(16) SegInfo {
  int wait0, wait1, defer, defpos;
  double defcoef, pad;
};

struct ScanArgs {
  int nchains, S, ring_len;     // ring: S slots of ring_len doubles
  int window;                   // > 0: slots hold positions mod window (single distance 1), producers
                                // wait for their reader before overwriting; 0: whole chains
  int ndelta, delta[kMaxDeps];  // distinct source-chain distances (slot-reuse guard)
  int n, fwd, stage_bytes;
  int spin_polls, sleep_ns;     // busy polls before backing off with __nanosleep(sleep_ns)
  const int* seg_ptr;           // chain -> first segment (nchains + 1)
  const int* chain_start;       // chain -> first row, sweep order
  const int* chain_len;         // chain -> rows
  const double2* recv;          // [(segment * NV + v) * 32 + lane]: (slope, c0), (c1, c2), ...
  const uint4* addr;            // [segment * 32 + lane]: (delta << 20) | position, per source
  const SegInfo* seginfo;       // [segment]
  const double* o0;             // pre-pass output, record layout
  double* xnew;                 // original row order
  int* status;
  long long* trace;             // diagnostics (null): per segment, %globaltimer at 4 points of its step
};

__device__ __forceinline__ long long scan_clock() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ unsigned long long scan_enc(int chain, int S, unsigned done) {
  return ((unsigned long long)(unsigned)(chain + S + 1) << 32) | done;
}

__device__ __forceinline__ unsigned long long ld_volatile_shared_u64(const unsigned long long* p) {
  return *reinterpret_cast<const volatile unsigned long long*>(p);
}

__device__ __forceinline__ unsigned addr_k(const uint4& a, int k) {
  return k == 0 ? a.x : k == 1 ? a.y : k == 2 ? a.z : a.w;
}

// Every lane of the warp runs the same waits on the same shared-memory words
// (uniform control flow, no divergent spinning); a failed poll backs off with
// __nanosleep so waiting warps leave the issue slots to the working ones.
// Progress of a chain = its number of complete segments.  A segment whose
// last row has a deferred source is completed (that row fixed, then
// published) when the warp starts the next segment, or at the chain's end.
// Each warp streams its segments' records into kStages shared-memory stages
// with TMA bulk copies (one elected lane, an mbarrier per stage), so no
// global load sits on the dependency path.
template <int K>
__global__ void __launch_bounds__(1024, 1) gs_scan_kernel(ScanArgs a) {
  constexpr int NV = (K + 2) / 2;
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const unsigned FULL = 0xffffffffu;
  const int S = a.S, RL = a.ring_len, WIN = a.window;
  unsigned long long* prog = reinterpret_cast<unsigned long long*>(smem);
  double* ring = reinterpret_cast<double*>(smem + 8 * ((S + 1) & ~1));
  unsigned char* stages = smem + ((8 * ((S + 1) & ~1) + 8 * (size_t)S * RL + 127) & ~(size_t)127);
  unsigned char* my_stages = stages + (size_t)warp * kStages * a.stage_bytes;
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(stages + (size_t)nw * kStages * a.stage_bytes);
  const unsigned bar0 = (unsigned)__cvta_generic_to_shared(bars + warp * kStages);
  const unsigned st0 = (unsigned)__cvta_generic_to_shared(my_stages);
  for (int i = threadIdx.x; i < S; i += blockDim.x) prog[i] = scan_enc(i - S, S, 0x7fffffffu);
  for (int i = threadIdx.x; i < S * RL; i += blockDim.x) ring[i] = 0.0;
  if (lane == 0) {
    for (int k = 0; k < kStages; ++k) mbar_init(bar0 + 8u * k, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // stage layout: o0 (32 doubles) | recv (NV x 32 double2) | addr (32 uint4) | SegInfo
  constexpr int OFF_RV = 256, OFF_AD = 256 + NV * 512, OFF_SI = 256 + NV * 512 + 512;
  unsigned phase = 0;  // parity bit per stage
  bool dead = false;
  auto issue = [&](int g, int k) {
    if (lane == 0) {
      const unsigned dst = st0 + (unsigned)(k * a.stage_bytes), bar = bar0 + 8u * k;
      mbar_expect_tx(bar, (unsigned)(OFF_SI + 32));
      bulk_g2s(dst, a.o0 + (size_t)g * 32, 256u, bar);
      bulk_g2s(dst + OFF_RV, a.recv + (size_t)g * NV * 32, (unsigned)(NV * 512), bar);
      bulk_g2s(dst + OFF_AD, a.addr + (size_t)g * 32, 512u, bar);
      bulk_g2s(dst + OFF_SI, a.seginfo + g, 32u, bar);
    }
  };
  auto wait_stage = [&](int k) {
    while (!mbar_try_wait(bar0 + 8u * k, (phase >> k) & 1u)) {}
    phase ^= 1u << k;
  };
  // wait until chain c (ring slot cslot) has `need` complete segments
  auto wait_for = [&](int c, int cslot, unsigned need) {
    const unsigned long long want = scan_enc(c, S, need);
    const unsigned long long* p = prog + cslot;
    if (ld_volatile_shared_u64(p) >= want) return;
    long long spins = 0;
    while (ld_volatile_shared_u64(p) < want) {
      if (++spins > a.spin_polls) __nanosleep(a.sleep_ns);
      if (spins > (1LL << 24)) {  // a broken schedule must not hang the GPU
        if (lane == 0) atomicOr(a.status, 8);
        dead = true;
        return;
      }
    }
  };
  auto wait_word = [&](int L, int slot, int w) {
    if (w == 0) return;
    const int dl = w >> 20;
    int cs_ = slot - dl;
    if (cs_ < 0) cs_ += S;
    wait_for(L - dl, cs_, (unsigned)(w & 0xfffff));
  };
  auto publish = [&](int L, int slot, unsigned done) {
    __threadfence_block();
    __syncwarp();
    if (lane == 0) *reinterpret_cast<volatile unsigned long long*>(prog + slot) = scan_enc(L, S, done);
  };
  auto ring_at = [&](int src_slot, int pos) -> double* {
    return ring + (size_t)src_slot * RL + (WIN ? (pos & (WIN - 1)) : pos);
  };
  int slot = warp % S;
  for (int L = warp; L < a.nchains && !dead; L += nw) {
    const int g0 = a.seg_ptr[L], nseg = a.seg_ptr[L + 1] - g0;
    for (int k = 0; k < kStages && k < nseg; ++k) issue(g0 + k, k);
    // the slot's previous occupant (chain L - S) has no readers left
    for (int d = 0; d < a.ndelta; ++d) {
      const int c = L - S + a.delta[d];
      if (c >= 0) {
        int cs_ = slot + a.delta[d];
        if (cs_ >= S) cs_ -= S;
        wait_for(c, cs_, (unsigned)(a.seg_ptr[c + 1] - a.seg_ptr[c]));
      }
    }
    __threadfence_block();
    const int cs = a.chain_start[L], len = a.chain_len[L];
    int rslot = slot + 1;  // window mode: the reader of this chain is chain L + 1
    if (rslot >= S) rslot -= S;
    double carry = 0.0;
    int pend_z = 0, pend_w = 0;  // deferred source of the previous segment's last row
    double pend_c = 0.0;
    auto store_ring = [&](int q, double x) { *ring_at(slot, q) = x; };
    auto store_global = [&](int q, double x) { a.xnew[a.fwd ? cs + q : a.n - 1 - (cs + q)] = x; };
    auto fix_pending = [&](int s) {  // complete segment s - 1: its last row's deferred term
      wait_word(L, slot, pend_z);
      __threadfence_block();
      const int dl = pend_z >> 20;
      int ss = slot - dl;
      if (ss < 0) ss += S;
      const double xv = *reinterpret_cast<volatile double*>(ring_at(ss, pend_w));
      carry = __fma_rn(-pend_c, xv, carry);
      if (lane == 31) store_ring(s * 32 - 1, carry);
      publish(L, slot, (unsigned)s);
      if (lane == 31) store_global(s * 32 - 1, carry);
      pend_z = 0;
    };
    for (int s = 0; s < nseg; ++s) {
      const int k = s % kStages;
      wait_stage(k);
      const unsigned char* st = my_stages + (size_t)k * a.stage_bytes;
      const double o0 = reinterpret_cast<const double*>(st)[lane];
      double2 rv[NV];
#pragma unroll
      for (int v = 0; v < NV; ++v) rv[v] = reinterpret_cast<const double2*>(st + OFF_RV)[v * 32 + lane];
      const uint4 ad = reinterpret_cast<const uint4*>(st + OFF_AD)[lane];
      const SegInfo si = *reinterpret_cast<const SegInfo*>(st + OFF_SI);
      __syncwarp();
      if (s + kStages < nseg) issue(g0 + s + kStages, k);  // the stage is free again
      if (pend_z) fix_pending(s);
      // window mode: segment s overwrites segment s - WIN/32 of this slot;
      // its reader must be done with it
      if (WIN && s >= WIN / 32 && L + 1 < a.nchains) wait_for(L + 1, rslot, (unsigned)(s - WIN / 32 + 2));
      wait_word(L, slot, si.wait0);
      wait_word(L, slot, si.wait1);
      __threadfence_block();
      double o = o0;
#pragma unroll
      for (int kk = 0; kk < K; ++kk) {
        const unsigned w = addr_k(ad, kk);
        const int d = (int)(w >> 20), pos = (int)(w & 0xfffffu);
        int ss = slot - d;
        if (ss < 0) ss += S;
        const double c = (kk + 1) % 2 == 0 ? rv[(kk + 1) / 2].x : rv[(kk + 1) / 2].y;
        const double xv = *reinterpret_cast<volatile double*>(ring_at(ss, pos));
        o = __fma_rn(-c, xv, o);
      }
      // inclusive scan of x -> o + slope * x over the 32 lanes
      double A = o, B = rv[0].x;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const double Ap = __shfl_up_sync(FULL, A, d), Bp = __shfl_up_sync(FULL, B, d);
        if (lane >= d) {
          A = __fma_rn(B, Ap, A);
          B = __dmul_rn(B, Bp);
        }
      }
      const double x = __fma_rn(B, carry, A);
      carry = __shfl_sync(FULL, x, 31);
      const int q = s * 32 + lane;
      const bool deferred = si.defer != 0;
      const bool mine = q < len && !(deferred && lane == 31);
      if (mine) store_ring(q, x);
      if (deferred) {
        pend_z = si.defer;
        pend_w = si.defpos;
        pend_c = si.defcoef;
      } else {
        publish(L, slot, (unsigned)(s + 1));
      }
      if (mine) store_global(q, x);
    }
    if (pend_z) fix_pending(nseg);
    slot += nw % S;
    if (slot >= S) slot -= S;
  }
}

// ---------------------------------------------------------------------------
// Cluster version (window mode: every source lies in the previous chain).
// Chain L runs on CTA L mod C of a thread-block cluster, so consecutive lines
// -- the wavefront -- are spread over C SMs.  Its x values and progress word
// live in the shared memory of its reader's CTA ((L + 1) mod C): the producer
// stores them there (st.shared::cluster, then a release store of the progress
// word) and the reader waits on its own shared memory.  Only the producer's
// occasional checks (slot reuse, the reader's progress before overwriting a
// window position) read another CTA's shared memory.
__device__ __forceinline__ void st_cluster_f64(unsigned caddr, double v) {
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(caddr), "d"(v) : "memory");
}
__device__ __forceinline__ void st_release_cluster_u64(unsigned caddr, unsigned long long v) {
  asm volatile("st.release.cluster.shared::cluster.u64 [%0], %1;" ::"r"(caddr), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_cluster_u64(unsigned caddr) {
  unsigned long long v;
  asm volatile("ld.acquire.cluster.shared::cluster.u64 %0, [%1];" : "=l"(v) : "r"(caddr) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_acquire_local_u64(unsigned saddr) {
  // the word is released by a thread of another CTA: acquire at cluster scope
  unsigned long long v;
  asm volatile("ld.acquire.cluster.shared::cta.u64 %0, [%1];" : "=l"(v) : "r"(saddr) : "memory");
  return v;
}

__device__ __forceinline__ void bulk_s2g(void* gdst, unsigned ssrc, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(ssrc), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}

template <int K>
__global__ void __launch_bounds__(256, 1) gs_scan_cluster_kernel(ScanArgs a) {
  constexpr int NV = (K + 2) / 2;
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const unsigned FULL = 0xffffffffu;
  const int C = (int)cluster_nctas(), me = (int)cluster_rank();
  const int S = a.S, WIN = a.window;  // S slots of WIN doubles per CTA
  const long long BIAS = (long long)C * S + 1;
  auto enc = [&](int chain, unsigned done) -> unsigned long long {
    return ((unsigned long long)(chain + BIAS) << 32) | done;
  };
  unsigned long long* prog = reinterpret_cast<unsigned long long*>(smem);
  double* ring = reinterpret_cast<double*>(smem + 8 * ((S + 1) & ~1));
  unsigned char* stages = smem + ((8 * ((S + 1) & ~1) + 8 * (size_t)S * WIN + 127) & ~(size_t)127);
  unsigned char* my_stages = stages + (size_t)warp * kStages * a.stage_bytes;
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(stages + (size_t)nw * kStages * a.stage_bytes);
  const unsigned bar0 = (unsigned)__cvta_generic_to_shared(bars + warp * kStages);
  const unsigned st0 = (unsigned)__cvta_generic_to_shared(my_stages);
  // x_new leaves through TMA bulk stores from two 32-value staging buffers per
  // warp: asynchronous-proxy stores, so a segment's release store of its
  // progress word never waits for global memory
  double* xout = reinterpret_cast<double*>(
      (reinterpret_cast<size_t>(bars + (size_t)nw * kStages) + 15) & ~(size_t)15) + warp * 64;
  const unsigned xout_s = (unsigned)__cvta_generic_to_shared(xout);
  const unsigned prog_s = (unsigned)__cvta_generic_to_shared(prog);
  const unsigned ring_s = (unsigned)__cvta_generic_to_shared(ring);
  // slot k of this CTA first serves chain k*C + (me - 1 mod C): mark its
  // fictitious predecessor (C*S chains earlier) complete
  const int first_owner = (me + C - 1) % C;
  for (int i = threadIdx.x; i < S; i += blockDim.x) prog[i] = enc(i * C + first_owner - C * S, 0x7fffffffu);
  for (int i = threadIdx.x; i < S * WIN; i += blockDim.x) ring[i] = 0.0;
  if (lane == 0) {
    for (int k = 0; k < kStages; ++k) mbar_init(bar0 + 8u * k, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  cluster_sync();  // every CTA's rings and progress words exist before remote stores
  constexpr int OFF_RV = 256, OFF_AD = 256 + NV * 512, OFF_SI = 256 + NV * 512 + 512;
  unsigned phase = 0;
  bool dead = false;
  auto issue = [&](int g, int k) {
    if (lane == 0) {
      const unsigned dst = st0 + (unsigned)(k * a.stage_bytes), bar = bar0 + 8u * k;
      mbar_expect_tx(bar, (unsigned)(OFF_SI + 32));
      bulk_g2s(dst, a.o0 + (size_t)g * 32, 256u, bar);
      bulk_g2s(dst + OFF_RV, a.recv + (size_t)g * NV * 32, (unsigned)(NV * 512), bar);
      bulk_g2s(dst + OFF_AD, a.addr + (size_t)g * 32, 512u, bar);
      bulk_g2s(dst + OFF_SI, a.seginfo + g, 32u, bar);
    }
  };
  auto wait_stage = [&](int k) {
    while (!mbar_try_wait(bar0 + 8u * k, (phase >> k) & 1u)) {}
    phase ^= 1u << k;
  };
  // a chain's progress word: in the shared memory of CTA (c + 1) mod C, slot (c / C) mod S
  auto prog_addr = [&](int c) -> unsigned {
    return map_rank(prog_s + 8u * (unsigned)((c / C) % S), (unsigned)((c + 1) % C));
  };
  auto wait_remote = [&](int c, unsigned need) {
    if (c < 0) return;
    const unsigned long long want = enc(c, need);
    const unsigned ad = prog_addr(c);
    long long spins = 0;
    while (ld_acquire_cluster_u64(ad) < want) {
      if (++spins > (1LL << 24)) {
        if (lane == 0) atomicOr(a.status, 8);
        dead = true;
        return;
      }
      __nanosleep(32);
    }
  };
  auto wait_local = [&](int c, unsigned need) {  // c's word lives here: (c + 1) mod C == me
    if (c < 0) return;
    const unsigned long long want = enc(c, need);
    const unsigned ad = prog_s + 8u * (unsigned)((c / C) % S);
    long long spins = 0;
    while (ld_acquire_local_u64(ad) < want) {
      if (++spins > (1LL << 26)) {
        if (lane == 0) atomicOr(a.status, 8);
        dead = true;
        return;
      }
    }
  };
  for (int j = warp; !dead; j += nw) {
    const int L = j * C + me;
    if (L >= a.nchains) break;
    const int g0 = a.seg_ptr[L], nseg = a.seg_ptr[L + 1] - g0;
    for (int k = 0; k < kStages && k < nseg; ++k) issue(g0 + k, k);
    const int rcta = (L + 1) % C, wslot = (L / C) % S;
    const unsigned my_ring = map_rank(ring_s + 8u * (unsigned)(wslot * WIN), (unsigned)rcta);
    const unsigned my_prog = map_rank(prog_s + 8u * (unsigned)wslot, (unsigned)rcta);
    // the slot's previous occupant (chain L - C*S) has no reader left
    if (L - C * S >= 0) {
      const int c = L - C * S + 1;
      wait_remote(c, (unsigned)(a.seg_ptr[c + 1] - a.seg_ptr[c]));
    }
    // source chain L - 1: its ring is in this CTA
    const int src = L - 1;
    const double* src_ring = ring + (size_t)(src >= 0 ? (src / C) % S : 0) * WIN;
    const int cs = a.chain_start[L], len = a.chain_len[L];
    double carry = 0.0;
    int pend_z = 0, pend_w = 0;
    double pend_c = 0.0;
    // x goes to the reader's ring before the release store of the progress
    // word, and to x_new (global) after it, so the release never waits on
    // global-memory stores
    auto store_ring = [&](int q, double x) { st_cluster_f64(my_ring + 8u * (unsigned)(q & (WIN - 1)), x); };
    auto store_global = [&](int q, double x) { a.xnew[a.fwd ? cs + q : a.n - 1 - (cs + q)] = x; };
    // whole 32-row segments go out by bulk copy when the chain's x_new span is 16-byte aligned
    const bool bulk = ((a.fwd ? cs : a.n - cs) & 1) == 0;
    auto stage_out = [&](int seg, int ln, double x) { xout[(seg & 1) * 32 + (a.fwd ? ln : 31 - ln)] = x; };
    auto flush_out = [&](int seg) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        const size_t start = a.fwd ? (size_t)cs + 32 * seg : (size_t)a.n - 1 - ((size_t)cs + 32 * seg + 31);
        bulk_s2g(a.xnew + start, xout_s + 256u * (unsigned)(seg & 1), 256u);
        bulk_commit();
      }
    };
    auto publish = [&](unsigned done) {
      __syncwarp();
      if (lane == 0) st_release_cluster_u64(my_prog, enc(L, done));
    };
    auto fix_pending = [&](int s) {
      wait_local(src, (unsigned)(pend_z & 0xfffff));
      const double xv = *reinterpret_cast<const volatile double*>(src_ring + (pend_w & (WIN - 1)));
      carry = __fma_rn(-pend_c, xv, carry);
      if (lane == 31) store_ring(s * 32 - 1, carry);
      publish((unsigned)s);
      const bool full = (s - 1) * 32 + 32 <= len;
      if (bulk && full) {
        if (lane == 31) stage_out(s - 1, 31, carry);
        flush_out(s - 1);
      } else if (lane == 31) {
        store_global(s * 32 - 1, carry);
      }
      pend_z = 0;
    };
    unsigned long long reader_seen = 0;  // last observed progress word of chain L + 1 (remote reads are rare)
    for (int s = 0; s < nseg; ++s) {
      const int k = s % kStages;
      long long* tr = a.trace ? a.trace + 4 * (size_t)(g0 + s) : nullptr;
      if (tr && lane == 0) tr[0] = scan_clock();
      wait_stage(k);
      const unsigned char* st = my_stages + (size_t)k * a.stage_bytes;
      const double o0 = reinterpret_cast<const double*>(st)[lane];
      double2 rv[NV];
#pragma unroll
      for (int v = 0; v < NV; ++v) rv[v] = reinterpret_cast<const double2*>(st + OFF_RV)[v * 32 + lane];
      const uint4 ad = reinterpret_cast<const uint4*>(st + OFF_AD)[lane];
      const SegInfo si = *reinterpret_cast<const SegInfo*>(st + OFF_SI);
      __syncwarp();
      if (tr && lane == 0) tr[1] = scan_clock();
      if (s + kStages < nseg) issue(g0 + s + kStages, k);
      if (pend_z) fix_pending(s);
      // window: segment s overwrites segment s - WIN/32; the reader (chain L + 1) must be past it
      if (s >= WIN / 32 && L + 1 < a.nchains) {
        const unsigned long long want = enc(L + 1, (unsigned)(s - WIN / 32 + 2));
        if (reader_seen < want) {
          const unsigned pa = prog_addr(L + 1);
          reader_seen = ld_acquire_cluster_u64(pa);
          if (reader_seen < want) {
            wait_remote(L + 1, (unsigned)(s - WIN / 32 + 2));
            reader_seen = ld_acquire_cluster_u64(pa);
          }
        }
      }
      if (si.wait0) wait_local(src, (unsigned)(si.wait0 & 0xfffff));
      if (tr && lane == 0) tr[2] = scan_clock();
      double o = o0;
#pragma unroll
      for (int kk = 0; kk < K; ++kk) {
        const unsigned w = addr_k(ad, kk);
        const int pos = (int)(w & 0xfffffu);
        const double c = (kk + 1) % 2 == 0 ? rv[(kk + 1) / 2].x : rv[(kk + 1) / 2].y;
        const double xv = (w >> 20) ? *reinterpret_cast<const volatile double*>(src_ring + (pos & (WIN - 1))) : 0.0;
        o = __fma_rn(-c, xv, o);
      }
      double A = o, B = rv[0].x;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const double Ap = __shfl_up_sync(FULL, A, d), Bp = __shfl_up_sync(FULL, B, d);
        if (lane >= d) {
          A = __fma_rn(B, Ap, A);
          B = __dmul_rn(B, Bp);
        }
      }
      const double x = __fma_rn(B, carry, A);
      carry = __shfl_sync(FULL, x, 31);
      const int q = s * 32 + lane;
      const bool deferred = si.defer != 0;
      const bool mine = q < len && !(deferred && lane == 31);
      const bool full = s * 32 + 32 <= len;
      if (mine) store_ring(q, x);
      if (bulk && full) {
        // the staging buffer of segment s last held segment s - 2: its bulk read must be done
        if (lane == 0) bulk_wait_read<1>();
        __syncwarp();
        if (mine) stage_out(s, lane, x);
      }
      if (deferred) {
        pend_z = si.defer;
        pend_w = si.defpos;
        pend_c = si.defcoef;
      } else {
        publish((unsigned)(s + 1));
        if (bulk && full) flush_out(s);
      }
      if (mine && !(bulk && full)) store_global(q, x);
      if (tr && lane == 0) tr[3] = scan_clock();
    }
    if (pend_z) fix_pending(nseg);
  }
  if (lane == 0) bulk_wait<0>();  // x_new complete before the kernel ends
  cluster_sync();  // nobody leaves while others may still store into its shared memory
}

// o0[rec(i)] = (b_i - sum over the row's old-value entries a_ij xold_j) * rdiag_i,
// in the sweep's record layout.  old: 0 none (sweep from zero), 1 entries j > i
// (forward from x_old), 2 entries j < i (backward from x_old).
__global__ void gs_scan_prepass_kernel(int n, const int* __restrict__ ip, const int* __restrict__ ix,
                                       const double* __restrict__ v, const double* __restrict__ rdiag,
                                       const int* __restrict__ rec, const double* __restrict__ b,
                                       const double* __restrict__ xold, int old, double* __restrict__ o0) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double s = b[i];
    if (old) {
      for (int k = ip[i]; k < ip[i + 1]; ++k) {
        const int j = ix[k];
        if (old == 1 ? j > i : j < i) s = __fma_rn(-v[k], xold[j], s);
      }
    }
    o0[rec[i]] = __dmul_rn(s, rdiag[i]);
  }
}

}  // namespace gsscan
}  // namespace mvamg
