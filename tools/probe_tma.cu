// Cost of per-warp TMA bulk-copy streaming (elected lane issues, all lanes wait).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count)); }
__device__ __forceinline__ void mbar_expect_tx(unsigned bar, unsigned bytes) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory"); }
__device__ __forceinline__ void bulk_g2s(unsigned dst, const void* src, unsigned bytes, unsigned bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory"); }
__device__ __forceinline__ bool mbar_try_wait(unsigned bar, unsigned parity) {
  unsigned ok; asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}" : "=r"(ok) : "r"(bar), "r"(parity) : "memory"); return ok != 0; }
__device__ __forceinline__ unsigned long long lds(unsigned a) { unsigned long long v; asm volatile("ld.shared.b64 %0, [%1];" : "=l"(v) : "r"(a)); return v; }

template <int R, int D>
__global__ void stream(const unsigned long long* src, int nchunk, int chunk_bytes, long long* cyc, double* out, int work) {
  extern __shared__ __align__(16) unsigned long long sm[];
  const unsigned base = (unsigned)__cvta_generic_to_shared(sm);
  const unsigned bars = base + (unsigned)(D * chunk_bytes);
  const int lane = threadIdx.x;
  if (lane == 0) { for (int d = 0; d < D; ++d) mbar_init(bars + 8 * d, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  __syncwarp();
  auto issue = [&](int k) { int d = k % D; mbar_expect_tx(bars + 8 * d, chunk_bytes);
    bulk_g2s(base + d * chunk_bytes, (const char*)src + (size_t)k * chunk_bytes, chunk_bytes, bars + 8 * d); };
  if (lane == 0) for (int k = 0; k < D && k < nchunk; ++k) issue(k);
  unsigned parity = 0; double acc = 0;
  long long t0 = clock64();
  for (int k = 0; k < nchunk; ++k) {
    int d = k % D;
    while (!mbar_try_wait(bars + 8 * d, (parity >> d) & 1u)) {}
    parity ^= 1u << d;
    for (int r = 0; r < R; ++r) {
      unsigned long long v = lds(base + d * chunk_bytes + 8 * ((r * 64 + lane) % (chunk_bytes / 8)));
      double x = __longlong_as_double(v);
      for (int w = 0; w < work; ++w) x = x * 0.999 + 1e-3;   // ~ dependent fp work per round
      acc += x;
      __syncwarp();
    }
    __syncwarp();
    if (lane == 0 && k + D < nchunk) issue(k + D);
  }
  long long t1 = clock64();
  out[lane] = acc;
  if (lane == 0) cyc[0] = t1 - t0;
}

int main() {
  const int nchunk = 2048, chunk_bytes = 8192;
  unsigned long long* src; long long* cyc; double* out;
  cudaMalloc(&src, (size_t)nchunk * chunk_bytes); cudaMemset(src, 0, (size_t)nchunk * chunk_bytes);
  cudaMalloc(&cyc, 8); cudaMalloc(&out, 256);
  auto run = [&](auto kern, int R, int D, int work) {
    size_t smem = (size_t)D * chunk_bytes + 8 * D;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<1, 32, smem>>>(src, nchunk, chunk_bytes, cyc, out, work); cudaDeviceSynchronize();
    kern<<<1, 32, smem>>>(src, nchunk, chunk_bytes, cyc, out, work); cudaError_t e = cudaDeviceSynchronize();
    long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("R=%d D=%d work=%3d: %8.1f cycles/chunk %7.1f cycles/round  %s\n", R, D, work, (double)c / nchunk, (double)c / nchunk / R, cudaGetErrorString(e));
  };
  for (int work : {0, 20}) {
    run(stream<1, 2>, 1, 2, work); run(stream<1, 8>, 1, 8, work); run(stream<4, 2>, 4, 2, work);
    run(stream<8, 2>, 8, 2, work); run(stream<4, 8>, 4, 8, work); run(stream<8, 4>, 8, 4, work);
  }
  return 0;
}
