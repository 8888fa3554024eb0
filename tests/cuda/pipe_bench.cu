// Micro-benchmark of the producer/consumer handshake used by tc_conv: one
// producer thread (warp 0) and one consumer thread (warp 1) pass S stages
// through full/empty mbarriers. Variants: the consumer releases a stage with
// a plain mbarrier.arrive or with tcgen05.commit (as the MMA warp does), with
// and without issuing MMAs; the producer optionally issues a TMA-free
// arrive.expect_tx(0). Reports cycles per step.
//
// Build: nvcc -std=c++17 -O2 -gencode arch=compute_100a,code=sm_100a
//        -I paper_2101_07344_b200/csrc/kernels tests/cuda/pipe_bench.cu -o pipe_bench
#include <cuda_runtime.h>

#include <cstdio>

#include "sm100_prims.cuh"

using namespace lcb;

__device__ __forceinline__ unsigned long long clk() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));
  return t;
}

template <int S>
__global__ void pipe_kernel(int steps, int mode, unsigned long long* out) {
  __shared__ uint64_t bars[2 * S + 2];
  __shared__ uint32_t holder;
  __shared__ __align__(1024) uint8_t buf[2 * 16384];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t full0 = smem_u32(bars), empty0 = smem_u32(bars + S);
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(full0 + 8 * i, 1);
      mbar_init(empty0 + 8 * i, 1);
    }
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(smem_u32(&holder), 64);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = holder;
  unsigned long long t0 = clk();
  if (warp == 0 && lane == 0) {
    int stage = 0;
    uint32_t phase = 0;
    for (int s = 0; s < steps; ++s) {
      mbar_wait(empty0 + 8 * stage, phase ^ 1);
      mbar_expect_tx(full0 + 8 * stage, 0);
      if (++stage == S) {
        stage = 0;
        phase ^= 1;
      }
    }
  } else if (warp == 1 && lane == 0) {
    int stage = 0;
    uint32_t phase = 0;
    constexpr uint32_t idesc = umma_idesc_bf16(128, 64);
    for (int s = 0; s < steps; ++s) {
      mbar_wait(full0 + 8 * stage, phase);
      tc_fence_after();
      if (mode & 2) {
        const uint32_t a = smem_u32(buf), b = smem_u32(buf + 16384);
        for (int k = 0; k < 12; ++k)
          umma_bf16(tmem, umma_desc_sw128(a + 32 * (k & 3)), umma_desc_sw128(b + 32 * (k & 3)), idesc, k > 0);
      }
      if (mode & 1)
        umma_commit(empty0 + 8 * stage);
      else
        mbar_arrive(empty0 + 8 * stage);
      if (++stage == S) {
        stage = 0;
        phase ^= 1;
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 32) out[blockIdx.x] = clk() - t0;
  if (warp == 0) tmem_dealloc(tmem, 64);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  const int steps = 4096;
  const char* names[4] = {"arrive", "tcgen05.commit", "12 MMAs + arrive", "12 MMAs + commit"};
  for (int mode = 0; mode < 4; ++mode) {
    for (int grid : {1, 148}) {
      pipe_kernel<4><<<grid, 64>>>(steps, mode, d);
      cudaDeviceSynchronize();
      unsigned long long h[148];
      cudaMemcpy(h, d, grid * 8, cudaMemcpyDeviceToHost);
      printf("S=4 %-18s grid=%3d: %.1f cycles/step\n", names[mode], grid, double(h[0]) / steps);
    }
  }
  for (int mode = 1; mode < 4; mode += 2) {
    pipe_kernel<8><<<148, 64>>>(steps, mode, d);
    cudaDeviceSynchronize();
    unsigned long long h[148];
    cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
    printf("S=8 %-18s grid=148: %.1f cycles/step\n", names[mode], double(h[0]) / steps);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
