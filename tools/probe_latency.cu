// Microprobes: fp64 dependent latency, Markstein division exactness, cross-CTA flag hop latency.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("ERR %s line %d\n", cudaGetErrorString(e), __LINE__); exit(1);}}while(0)

__global__ void lat_chain(double* out, double a, double b, int iters, long long* cyc, int mode) {
  double s = a;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (mode == 0) { s = __dsub_rn(s, __dmul_rn(b, s)); }          // mul+sub
    else if (mode == 1) { s = __ddiv_rn(s, b); }                      // div
    else { double q = __dmul_rn(s, a); double r = fma(-q, b, s); s = fma(r, a, q); } // markstein
  }
  long long t1 = clock64();
  out[0] = s; cyc[0] = t1 - t0;
}

__global__ void div_check(const double* s, const double* d, long n, unsigned long long* bad) {
  long i = blockIdx.x * (long)blockDim.x + threadIdx.x;
  for (; i < n; i += (long)gridDim.x * blockDim.x) {
    double y = __drcp_rn(d[i]);
    double q0 = __dmul_rn(s[i], y);
    double r = fma(-q0, d[i], s[i]);
    double q = fma(r, y, q0);
    double t = __ddiv_rn(s[i], d[i]);
    if (__double_as_longlong(q) != __double_as_longlong(t)) atomicAdd(bad, 1ULL);
  }
}

// ping-pong between two CTAs through a global word
__global__ void pingpong(volatile long long* flag, int rounds, long long* cyc) {
  int me = blockIdx.x;
  if (threadIdx.x != 0) return;
  long long t0 = clock64();
  for (int r = 0; r < rounds; ++r) {
    long long want = 2 * r + me;
    while (flag[0] != want) {}
    flag[0] = want + 1;
  }
  long long t1 = clock64();
  if (me == 0) cyc[0] = t1 - t0;
}

int main() {
  double* out; long long* cyc; CK(cudaMalloc(&out, 8)); CK(cudaMalloc(&cyc, 8));
  const char* nm[3] = {"mul+sub", "ddiv", "markstein3"};
  for (int m = 0; m < 3; ++m) {
    lat_chain<<<1,1>>>(out, 0.999, 0.5, 10000, cyc, m); CK(cudaDeviceSynchronize());
    long long c; CK(cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost));
    printf("latency %s: %.2f cycles/iter\n", nm[m], c / 10000.0);
  }
  long n = 1L << 26;
  double *hs = (double*)malloc(n * 8), *hd = (double*)malloc(n * 8);
  srand(1);
  for (long i = 0; i < n; ++i) {
    double u = (rand() / (double)RAND_MAX) * 2 - 1; double v = (rand() / (double)RAND_MAX);
    int e1 = rand() % 80 - 40, e2 = rand() % 20 - 10;
    hs[i] = ldexp(u + (rand() / (double)RAND_MAX) * 1e-9, e1); hd[i] = ldexp(0.5 + v, e2);
    if (i % 7 == 0) hd[i] = ldexp(1.0 - ldexp(1.0, -52) * (rand() % 5), e2);  // near power of two
    if (i % 11 == 0) hs[i] = ldexp(1.0 - ldexp(1.0, -52) * (rand() % 5), e1);
  }
  double *ds, *dd; unsigned long long* bad; CK(cudaMalloc(&ds, n * 8)); CK(cudaMalloc(&dd, n * 8)); CK(cudaMalloc(&bad, 8));
  CK(cudaMemcpy(ds, hs, n * 8, cudaMemcpyHostToDevice)); CK(cudaMemcpy(dd, hd, n * 8, cudaMemcpyHostToDevice));
  CK(cudaMemset(bad, 0, 8));
  div_check<<<1184, 256>>>(ds, dd, n, bad); CK(cudaDeviceSynchronize());
  unsigned long long hb; CK(cudaMemcpy(&hb, bad, 8, cudaMemcpyDeviceToHost));
  printf("markstein mismatches: %llu of %ld\n", hb, n);
  long long* flag; CK(cudaMalloc(&flag, 8)); CK(cudaMemset(flag, 0, 8));
  pingpong<<<2, 32>>>((volatile long long*)flag, 10000, cyc); CK(cudaDeviceSynchronize());
  long long c; CK(cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost));
  printf("cross-CTA pingpong: %.1f cycles per one-way hop\n", c / 20000.0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0); printf("clock kHz %d\n", clk);
  return 0;
}
