// probe_hop.cu -- raw latency of a publish -> poll -> publish hop through L2 on
// B200 (diagnostics for the dataflow GS row sweep).  Row r waits for x[r-1]
// (sentinel-filled) and publishes x[r]; rows are handed to CTAs by ticket.
//   A: one thread per row, every lane spins on its own predecessor (intra-warp
//      dependencies inside a warp, cross-warp between warps)
//   B: like A but the warp polls in lockstep (all lanes loop until all done)
//   C: one row per warp (lane 0), rows of consecutive warps depend on each other
//   D: one row per CTA (cross-CTA hops only)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o probe_hop probe_hop.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long ldr(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ void str(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
constexpr unsigned long long S = ~0ull;

template <int MODE>
__global__ void hop(unsigned long long* x, int n, int* ticket, int rows_per_cta) {
  __shared__ int t;
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) t = atomicAdd(ticket, 1);
    __syncthreads();
    const int tk = t;
    if (tk * rows_per_cta >= n) return;
    int r = -1;
    if (MODE == 0 || MODE == 1) r = tk * rows_per_cta + threadIdx.x;
    if (MODE == 2) r = (threadIdx.x & 31) == 0 ? tk * rows_per_cta + (threadIdx.x >> 5) : -1;
    if (MODE == 3) r = threadIdx.x == 0 ? tk : -1;
    const bool have = r >= 0 && r < n;
    if (MODE == 1) {
      bool done = !have;
      while (!__all_sync(0xffffffffu, done)) {
        if (!done) {
          unsigned long long v = r == 0 ? 0ull : ldr(x + r - 1);
          if (v != S) { str(x + r, v + 1); done = true; }
        }
      }
    } else if (have) {
      unsigned long long v = 0;
      if (r > 0) do { v = ldr(x + r - 1); } while (v == S);
      str(x + r, v + 1);
    }
  }
}

int main() {
  const int n = 8192;
  unsigned long long* x;
  int* ticket;
  cudaMalloc(&x, n * 8);
  cudaMalloc(&ticket, 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  struct Cfg { const char* name; int mode, threads, rpc, grid; };
  Cfg cfgs[] = {{"A lanes own spin T=128 grid=8", 0, 128, 128, 8}, {"A T=32 grid=16", 0, 32, 32, 16},
                {"B warp lockstep T=128 grid=8", 1, 128, 128, 8}, {"B T=32 grid=16", 1, 32, 32, 16},
                {"C row per warp T=128 (4 rows/CTA) grid=16", 2, 128, 4, 16},
                {"D row per CTA grid=64", 3, 32, 1, 64}, {"D row per CTA grid=148", 3, 32, 1, 148}};
  for (auto& c : cfgs) {
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaMemset(x, 0xff, n * 8);
      cudaMemset(ticket, 0, 4);
      cudaEventRecord(e0);
      if (c.mode == 0) hop<0><<<c.grid, c.threads>>>(x, n, ticket, c.rpc);
      if (c.mode == 1) hop<1><<<c.grid, c.threads>>>(x, n, ticket, c.rpc);
      if (c.mode == 2) hop<2><<<c.grid, c.threads>>>(x, n, ticket, c.rpc);
      if (c.mode == 3) hop<3><<<c.grid, c.threads>>>(x, n, ticket, c.rpc);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    unsigned long long last;
    cudaMemcpy(&last, x + n - 1, 8, cudaMemcpyDeviceToHost);
    printf("%-44s %8.1f ns/hop  (check %llu == %d) %s\n", c.name, best * 1e6 / n, last, n - 1,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
