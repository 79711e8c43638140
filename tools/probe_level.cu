// Microprobe: the floor of one DAG-level step of a single-CTA level-set sweep
// on B200 -- a block barrier plus one row's shared-memory chain.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/probe_level tools/probe_level.cu
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("ERR %s line %d\n", cudaGetErrorString(e), __LINE__); return 1;}}while(0)

// mode 0: barrier only; 1: thread 0 x[i] = fma(x[i-1], a, b) + barrier;
// 2: 8 lanes read 8 x values, FMA, 3-step shuffle tree, Markstein, store + barrier;
// 3: as 2 but the 8 column indices come from shared memory too (dependent load)
__global__ void level_probe(int mode, int iters, double a, double b, long long* cyc, double* out) {
  extern __shared__ double sm[];
  int* idx = reinterpret_cast<int*>(sm + 4096);
  const int tid = threadIdx.x;
  for (int i = tid; i < 4096; i += blockDim.x) { sm[i] = 1.0 + i * 1e-3; idx[i] = (i * 37) & 4095; }
  __syncthreads();
  long long t0 = clock64();
  for (int i = 1; i < iters; ++i) {
    if (mode == 1) {
      if (tid == 0) sm[i & 4095] = fma(sm[(i - 1) & 4095], a, b);
    } else if (mode >= 2) {
      if (tid < 8) {
        int j = mode == 3 ? idx[(i * 8 + tid) & 4095] : ((i * 8 + tid * 13) & 4095);
        double v = sm[j];
        double p = fma(v, a, b);
        p += __shfl_xor_sync(0xffu, p, 4, 8);
        p += __shfl_xor_sync(0xffu, p, 2, 8);
        p += __shfl_xor_sync(0xffu, p, 1, 8);
        double q0 = p * b, r = fma(-q0, a, p), q = fma(r, b, q0);
        if (tid == 0) sm[(i * 101) & 4095] = q;
      }
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (tid == 0) { cyc[0] = t1 - t0; out[0] = sm[7]; }
}

int main() {
  long long* cyc; double* out;
  CK(cudaMalloc(&cyc, 8)); CK(cudaMalloc(&out, 8));
  CK(cudaFuncSetAttribute(level_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  const int iters = 20000;
  for (int threads : {32, 256, 512, 1024})
    for (int smem : {48 * 1024, 200 * 1024})
      for (int mode = 0; mode < 4; ++mode) {
        level_probe<<<1, threads, smem>>>(mode, iters, 0.999, 0.5, cyc, out);
        CK(cudaDeviceSynchronize());
        long long c; CK(cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost));
        printf("threads %4d smem %3d KB mode %d: %.1f cycles per level\n", threads, smem / 1024, mode, c / (double)(iters - 1));
      }
  return 0;
}
