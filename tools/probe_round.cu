// Microbenchmark of the GS round body's pieces (one warp, synthetic data).
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("ERR %s line %d\n", cudaGetErrorString(e), __LINE__); return 1;}}while(0)

__device__ __forceinline__ unsigned long long lds(unsigned a) { unsigned long long v; asm volatile("ld.shared.b64 %0, [%1];" : "=l"(v) : "r"(a)); return v; }
__device__ __forceinline__ unsigned long long ldsv(unsigned a) { unsigned long long v; asm volatile("ld.volatile.shared.b64 %0, [%1];" : "=l"(v) : "r"(a)); return v; }
__device__ __noinline__ double slowdiv(double s, double d) { return __ddiv_rn(s, d); }
__device__ __forceinline__ double mdiv(double s, double d, double y) {
  double q0 = __dmul_rn(s, y); double r = fma(-q0, d, s); double q = fma(r, y, q0);
  double aq = fabs(q0); if (__builtin_expect(!(aq > 1e-290 && aq < 1e290), 0)) q = slowdiv(s, d); return q;
}

template <int V>
__global__ void rounds(int nr, double* out, long long* cyc, double* gx) {
  extern __shared__ unsigned long long sm[];
  const unsigned base = (unsigned)__cvta_generic_to_shared(sm);
  const int lane = threadIdx.x;
  for (int i = lane; i < 8192; i += 32) sm[i] = __double_as_longlong(1.0 + 1e-3 * i);
  for (int i = 0; i < 32; ++i) sm[4096 + i * 32 + lane] = (unsigned long long)((lane * 8) << 2 | 1);
  __syncwarp();
  double xprev = 1.0, acc = 0.0;
  long long t0 = clock64();
  for (int r = 0; r < nr; ++r) {
    if (V >= 1) {
      const unsigned rec = base + 8u * (unsigned)(((r & 7) * 160) + lane);
      double s = __longlong_as_double(lds(rec + 256u * 40));
      double a0 = __longlong_as_double(lds(rec + 256u * 3)), a1 = __longlong_as_double(lds(rec + 256u * 5));
      unsigned c0 = (unsigned)lds(base + 8u * (4096 + (r & 31) * 32 + lane));
      double x0 = xprev;
      if (V >= 2) { unsigned long long v = ldsv(base + 8u * (c0 >> 2)); if ((unsigned)(v >> 32) == 0xffffffffu) acc += 1; x0 = __longlong_as_double(v); }
      s = __dsub_rn(s, __dmul_rn(a0, x0));
      s = __dsub_rn(s, __dmul_rn(a1, xprev));
      double d = __longlong_as_double(lds(rec + 256u)), y = 1.0 / 4.0;
      double x = (V >= 3) ? mdiv(s, d, y) : s * y;
      if (V >= 4) asm volatile("st.volatile.shared.f64 [%0], %1;" :: "r"(base + 8u * (unsigned)(6000 + (r & 63) * 32 + lane)), "d"(x));
      if (V >= 5) gx[(size_t)r * 32 + lane] = x;
      xprev = x * 1e-9 + 1.0;
    }
    if (V >= 6) { bool ok = __all_sync(0xffffffffu, xprev > 0); if (!ok) acc += 1; }
    __syncwarp();
  }
  long long t1 = clock64();
  out[lane] = xprev + acc;
  if (lane == 0) cyc[0] = t1 - t0;
}

int main() {
  double* out; long long* cyc; double* gx;
  CK(cudaMalloc(&out, 256)); CK(cudaMalloc(&cyc, 8)); CK(cudaMalloc(&gx, 4096 * 32 * 8));
  const int nr = 4096; const size_t smem = 100 * 1024;
  auto run = [&](auto kern, const char* name) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<1, 32, smem>>>(nr, out, cyc, gx); cudaDeviceSynchronize();
    kern<<<1, 32, smem>>>(nr, out, cyc, gx); cudaError_t e = cudaDeviceSynchronize();
    long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-40s %7.1f cycles/round %s\n", name, (double)c / nr, cudaGetErrorString(e));
  };
  run(rounds<0>, "V0 empty (syncwarp)");
  run(rounds<1>, "V1 + LDS record + 2 fmul/fsub + mul");
  run(rounds<2>, "V2 + window LDS.volatile + check");
  run(rounds<3>, "V3 + markstein division");
  run(rounds<4>, "V4 + STS.volatile publish");
  run(rounds<5>, "V5 + STG xnew");
  run(rounds<6>, "V6 + all_sync vote");
  return 0;
}
