// Micro-benchmark: the conv kernel's bf16x3 stacked MMA pattern per K-step
// (4 x [N=2*BN stacked hi*[hi;lo]] + 4 x [N=BN lo*hi], same accumulator), with a
// tcgen05.commit per K-step that nobody waits on (as the stage release), vs the
// same MMAs with no per-step commit. Reports cycles per MMA.
// Build: nvcc -std=c++17 -O2 -gencode arch=compute_100a,code=sm_100a
//        -I paper_2101_07344_b200/csrc/kernels tests/cuda/mma_mix.cu -o mma_mix
#include <cuda_runtime.h>

#include <cstdio>

#include "sm100_prims.cuh"

using namespace lcb;

__device__ __forceinline__ unsigned long long clk() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));
  return t;
}

template <int BN>
__global__ void mix_kernel(int steps, int mode, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar[8];
  __shared__ uint32_t holder;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < (2 * 16384 + 2 * BN * 128) / 16; i += blockDim.x) reinterpret_cast<uint4*>(sm)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    for (int i = 0; i < 8; ++i) mbar_init(smem_u32(&bar[i]), 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(smem_u32(&holder), 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = holder;
  unsigned long long t0 = 0, t1 = 0;
  if (warp == 0) {
    constexpr uint32_t idesc = umma_idesc_bf16(128, BN);
    constexpr uint32_t idesc2 = umma_idesc_bf16(128, 2 * BN);
    const uint64_t dah = umma_desc_sw128(smem_u32(sm)), dal = umma_desc_sw128(smem_u32(sm + 16384));
    const uint64_t dbh = umma_desc_sw128(smem_u32(sm + 32768));
    t0 = clk();
    for (int s = 0; s < steps; ++s) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (mode == 2) {  // plain: 3 MMAs of N=BN per K16
          umma_bf16_warp(tmem, dah + 2 * k, dbh + 2 * k, idesc, (s | k) ? 1u : 0u);
          umma_bf16_warp(tmem, dah + 2 * k, dbh + 2 * k, idesc, 1u);
          umma_bf16_warp(tmem, dal + 2 * k, dbh + 2 * k, idesc, 1u);
        } else {
          umma_bf16_warp(tmem, dah + 2 * k, dbh + 2 * k, idesc2, (s | k) ? 1u : 0u);
          umma_bf16_warp(tmem, dal + 2 * k, dbh + 2 * k, idesc, 1u);
        }
      }
      if (mode >= 1) umma_commit_warp(smem_u32(&bar[s & 7]));
    }
    umma_commit_warp(smem_u32(&bar[0]));
    t1 = clk();
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  if (warp == 0) tmem_dealloc(tmem, 512);
}

// M = 64 rates (weights-as-A formulation): N in {64, 128, 256}, 48 MMAs per commit.
template <int N>
__global__ void m64_kernel(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t holder;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < (16384 + N * 128) / 16; i += blockDim.x) reinterpret_cast<uint4*>(sm)[i] = make_uint4(0, 0, 0, 0);
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
    constexpr uint32_t idesc = umma_idesc_bf16(64, N);
    const uint64_t da = umma_desc_sw128(smem_u32(sm)), db = umma_desc_sw128(smem_u32(sm + 16384));
    uint32_t phase = 0;
    t0 = clk();
    for (int it = 0; it < iters; ++it) {
      for (int k = 0; k < 48; ++k) umma_bf16_warp(tmem, da + 2 * (k & 3), db + 2 * (k & 3), idesc, k > 0);
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
void run_m64() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  const int iters = 500;
  const int smem = 16384 + N * 128 + 1024;
  cudaFuncSetAttribute(m64_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  m64_kernel<N><<<148, 128, smem>>>(iters, d);
  cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, d, 148 * 8, cudaMemcpyDeviceToHost);
  const double cyc = double(h[0]) / (iters * 48.0);
  printf("M= 64 N=%3d: %.1f cycles/MMA, %.0f MAC/clk/SM (err %s)\n", N, cyc, 64.0 * N * 16 / cyc,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

template <int BN>
void run(int mode) {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  const int steps = 2000;
  const int smem = 2 * 16384 + 2 * BN * 128 + 1024;
  cudaFuncSetAttribute(mix_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  mix_kernel<BN><<<148, 128, smem>>>(steps, mode, d);
  cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, d, 148 * 8, cudaMemcpyDeviceToHost);
  const int per = mode == 2 ? 12 : 8;
  printf("BN=%3d mode %d (%s): %.1f cycles/K-step, %.1f cycles/MMA (err %s)\n", BN, mode,
         mode == 0 ? "stacked, no per-step commit" : (mode == 1 ? "stacked + commit per K-step" : "3 MMAs/K16 + commit"),
         double(h[0]) / steps, double(h[0]) / (steps * per), cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  for (int m : {0, 1, 2}) {
    run<64>(m);
    run<128>(m);
  }
  run_m64<64>();
  run_m64<128>();
  run_m64<256>();
  return 0;
}
