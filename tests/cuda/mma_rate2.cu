// Micro-benchmark: tcgen05.mma issue/execute rate of CTA PAIRS (cta_group::2,
// M = 256 over two SMs of a TPC) against single-CTA M = 128, kind::f16,
// K = 16, SW128 K-major operands in shared memory (zeros), for N = 64 / 128
// / 256 and the bf16x3 stacked pattern used by tc_conv for 64-channel convs
// (N = 128 then N = 64 per K16). Reports cycles per K16 step and MAC/clk/SM.
// Question answered: does a CTA pair halve the per-instruction cost of the
// small-N MMAs (tc_conv's 64-channel layers are MMA-issue bound at N = 64)?
// Build: nvcc -std=c++17 -O2 -gencode arch=compute_100a,code=sm_100a
//        -I paper_2101_07344_b200/csrc/kernels tests/cuda/mma_rate2.cu -o mma_rate2
#include <cuda_runtime.h>

#include <cstdio>

#include "sm100_prims.cuh"

using namespace lcb;

__device__ __forceinline__ unsigned long long clk() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
}

// mode 0: one MMA of N per K16; mode 1: stacked bf16x3 (N = 2n then N = n)
template <int N, int MODE>
__global__ void __cluster_dims__(2, 1, 1) mma2_kernel(int iters, int per_commit, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t holder;
  const int warp = threadIdx.x >> 5;
  const unsigned rank = cluster_rank();
  constexpr int kB = (MODE ? 2 * N : N) * 128;
  for (int i = threadIdx.x; i < (16384 + kB) / 16; i += blockDim.x) reinterpret_cast<uint4*>(sm)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bar), 1);
    fence_mbar_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&holder)), "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = holder;
  unsigned long long t0 = 0, t1 = 0;
  if (warp == 0 && rank == 0) {
    // M = 256 (two CTAs x 128 rows); per CTA the B operand holds N/2 rows
    constexpr uint32_t idesc = umma_idesc_bf16(256, N);
    constexpr uint32_t idesc2 = umma_idesc_bf16(256, 2 * N);
    const uint64_t da = umma_desc_sw128(smem_u32(sm)), db = umma_desc_sw128(smem_u32(sm + 16384));
    uint32_t phase = 0;
    t0 = clk();
    for (int it = 0; it < iters; ++it) {
      for (int k = 0; k < per_commit; ++k) {
        const uint32_t acc = k > 0 ? 1u : 0u;
        if (MODE == 0) {
          asm volatile(
              "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
              "l"(da + 2 * (k & 3)), "l"(db + 2 * (k & 3)), "r"(idesc), "r"(acc)
              : "memory");
        } else {
          asm volatile(
              "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %5, 0;\n\t"
              "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t"
              "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %4, 1;\n\t}" ::"r"(tmem),
              "l"(da + 2 * (k & 3)), "l"(db + 2 * (k & 3)), "r"(idesc2), "r"(idesc), "r"(acc)
              : "memory");
        }
      }
      asm volatile(
          "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
          "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::"r"(
              smem_u32(&bar)),
          "h"(static_cast<unsigned short>(3))
          : "memory");
      mbar_wait(smem_u32(&bar), phase);
      phase ^= 1;
    }
    t1 = clk();
  }
  if (warp == 0 && rank == 1) {  // the peer's barrier receives the multicast arrivals: follow them
    uint32_t phase = 0;
    for (int it = 0; it < iters; ++it) {
      mbar_wait(smem_u32(&bar), phase);
      phase ^= 1;
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  if (threadIdx.x == 0 && rank == 0) out[blockIdx.x / 2] = t1 - t0;
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
  }
}

template <int N, int MODE>
void run(int per_commit) {
  unsigned long long* d;
  cudaMalloc(&d, 74 * 8);
  cudaMemset(d, 0, 74 * 8);
  const int iters = 2000;
  constexpr int kB = (MODE ? 2 * N : N) * 128;
  const int smem = 16384 + kB + 1024;
  cudaFuncSetAttribute(mma2_kernel<N, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  mma2_kernel<N, MODE><<<148, 128, smem>>>(iters, per_commit, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[74];
  cudaMemcpy(h, d, 74 * 8, cudaMemcpyDeviceToHost);
  const double cyc = double(h[0]) / (double(iters) * per_commit);
  // MACs per K16 step per SM: 128 rows x (N or 3N/2... ) -> report per-SM MACs of the step
  const double macs_sm = 128.0 * 16 * (MODE ? 3 * N : N);
  printf("pair M=256 N=%3d %s K16-steps/commit=%2d: %6.1f cycles/step, %5.0f MAC/clk/SM%s (err %s)\n", N,
         MODE ? "stacked x3 (2N + N)" : "single            ", per_commit, cyc, macs_sm / cyc,
         MODE ? " (x3 product MACs)" : "", cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  for (int pc : {12, 48}) {
    run<64, 0>(pc);
    run<128, 0>(pc);
    run<256, 0>(pc);
    run<64, 1>(pc);
    run<128, 1>(pc);
  }
  return 0;
}
