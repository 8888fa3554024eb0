#include <cuda_runtime.h>
#include <cstdio>
#include "sm100_prims.cuh"
using namespace lcb;
__device__ __forceinline__ unsigned long long clk() { unsigned long long t; asm volatile("mov.u64 %0, %%clock64;" : "=l"(t)); return t; }
__device__ __forceinline__ bool test_wait(uint32_t bar, uint32_t parity) {
  uint32_t done;
  asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(done) : "r"(bar), "r"(parity) : "memory");
  return done;
}
__global__ void k(int iters, unsigned long long* out) {
  __shared__ uint64_t bar[2];
  if (threadIdx.x == 0) { mbar_init(smem_u32(&bar[0]), 1); mbar_init(smem_u32(&bar[1]), 1); fence_mbar_init(); }
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_arrive(smem_u32(&bar[0]));  // phase 0 complete
    unsigned long long t0 = clk();
    for (int i = 0; i < iters; ++i) mbar_wait(smem_u32(&bar[0]), 0);
    unsigned long long t1 = clk();
    for (int i = 0; i < iters; ++i) while (!test_wait(smem_u32(&bar[0]), 0)) {}
    unsigned long long t2 = clk();
    uint32_t ph = 0;
    for (int i = 0; i < iters; ++i) { mbar_arrive(smem_u32(&bar[1])); mbar_wait(smem_u32(&bar[1]), ph); ph ^= 1; }
    unsigned long long t3 = clk();
    ph = 0;
    for (int i = 0; i < iters; ++i) { mbar_arrive(smem_u32(&bar[1])); while (!test_wait(smem_u32(&bar[1]), ph)) {} ph ^= 1; }
    unsigned long long t4 = clk();
    out[0] = t1 - t0; out[1] = t2 - t1; out[2] = t3 - t2; out[3] = t4 - t3;
  }
}
int main() {
  unsigned long long* d; cudaMalloc(&d, 64);
  const int it = 10000;
  k<<<1, 32>>>(it, d); cudaDeviceSynchronize();
  unsigned long long h[4]; cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
  printf("try_wait(complete) %.1f cyc, test_wait(complete) %.1f cyc, arrive+try_wait %.1f, arrive+test_wait %.1f  (%s)\n",
         double(h[0]) / it, double(h[1]) / it, double(h[2]) / it, double(h[3]) / it, cudaGetErrorString(cudaGetLastError()));
}
