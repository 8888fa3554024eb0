// Micro-benchmark: tcgen05.mma issue/execute rate (kind::f16, M=128, K=16,
// SW128 K-major operands in shared memory) for N = 64 / 128 / 256, issued
// back to back by one elected lane of a whole warp; reports cycles per MMA
// and MAC/clk/SM. Operand values are irrelevant (zeros).
// Build: nvcc -std=c++17 -O2 -gencode arch=compute_100a,code=sm_100a
//        -I paper_2101_07344_b200/csrc/kernels tests/cuda/mma_rate.cu -o mma_rate
#include <cuda_runtime.h>

#include <cstdio>

#include "sm100_prims.cuh"

using namespace lcb;

__device__ __forceinline__ unsigned long long clk() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));
  return t;
}

template <int N>
__global__ void mma_kernel(int iters, int per_commit, int row_shift, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t holder;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < (16384 + 1024 + N * 128) / 16; i += blockDim.x) reinterpret_cast<uint4*>(sm)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bar), 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(smem_u32(&holder), 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = holder;
  unsigned long long t0 = 0, t1 = 0;
  if (warp == 0) {
    constexpr uint32_t idesc = umma_idesc_bf16(128, N);
    const uint64_t da = umma_desc_sw128(smem_u32(sm) + 128 * row_shift), db = umma_desc_sw128(smem_u32(sm + 16384 + 1024));
    uint32_t phase = 0;
    t0 = clk();
    for (int it = 0; it < iters; ++it) {
      for (int k = 0; k < per_commit; ++k) umma_bf16_warp(tmem, da + 2 * (k & 3), db + 2 * (k & 3), idesc, k > 0);
      umma_commit_warp(smem_u32(&bar));
      mbar_wait(smem_u32(&bar), phase);
      phase ^= 1;
    }
    t1 = clk();
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  if (warp == 0) tmem_dealloc(tmem, 512);
}

template <int N>
void run(int per_commit, int row_shift = 0) {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  const int iters = 2000;
  const int smem = 16384 + 1024 + N * 128 + 1024;
  cudaFuncSetAttribute(mma_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  mma_kernel<N><<<148, 128, smem>>>(iters, per_commit, row_shift, d);
  cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, d, 148 * 8, cudaMemcpyDeviceToHost);
  const double cyc = double(h[0]) / (double(iters) * per_commit);
  printf("N=%3d MMAs/commit=%3d A row shift %d: %.1f cycles/MMA, %.0f MAC/clk/SM (err %s)\n", N, per_commit, row_shift, cyc,
         128.0 * N * 16 / cyc, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  for (int pc : {12, 48}) {
    run<64>(pc);
    run<128>(pc);
    run<256>(pc);
  }
  for (int rs : {1, 3, 8}) {
    run<64>(48, rs);
    run<128>(48, rs);
  }
  return 0;
}
