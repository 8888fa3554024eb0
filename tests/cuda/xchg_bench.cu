// Micro-benchmark of tc_conv's split-K partial exchange pattern: every CTA
// (one per SM) writes a 64 KB fp32 partial tile with st.global.cg, arrives on
// a grid counter (atom.add.acq_rel), spins until all CTAs arrived, then reads
// 64 KB with ld.global.cg (all loads of a thread in flight) — its own slot,
// the next CTA's slot, or slots written long before (no fresh writes). Reports
// cycles per phase (CTA 0 and the max over CTAs) to locate the cost of the
// reduction's partial loads seen in the deep layers (~6k cycles).
// Build: nvcc -std=c++17 -O2 -gencode arch=compute_100a,code=sm_100a
//        -I paper_2101_07344_b200/csrc/kernels tests/cuda/xchg_bench.cu -o xchg_bench
#include <cuda_runtime.h>

#include <cstdio>

#include "gpu_sync.cuh"

using namespace lcb;

__device__ __forceinline__ unsigned long long clk() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// mode: 0 = read own slot, 1 = read the next CTA's slot, 2 = read the next CTA's slot without writing first
__global__ void __launch_bounds__(256, 1) xchg_kernel(float4* ws, int* ctr, int mode, unsigned long long* out) {
  const int tid = threadIdx.x;
  const int G = gridDim.x;
  constexpr int kF4 = 65536 / 16;  // float4 per slot
  float4* mine = ws + static_cast<size_t>(blockIdx.x) * kF4;
  const unsigned long long t0 = clk();
  if (mode != 2) {
#pragma unroll 4
    for (int i = tid; i < kF4; i += blockDim.x) __stcg(mine + i, make_float4(1.f, 2.f, 3.f, static_cast<float>(i)));
  }
  __syncthreads();
  const unsigned long long t1 = clk();
  if (tid == 0) {
    atom_add_acq_rel_gpu(ctr, 1);
    while (ld_acquire_gpu(ctr) < G) __nanosleep(32);
  }
  __syncthreads();
  const unsigned long long t2 = clk();
  const float4* src = ws + static_cast<size_t>(mode == 0 ? blockIdx.x : (blockIdx.x + 1) % G) * kF4;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  float4 v[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) v[k] = __ldcg(src + tid + k * blockDim.x);  // 16 x 256 x 16 B = 64 KB, all in flight
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    acc.x += v[k].x;
    acc.y += v[k].y;
    acc.z += v[k].z;
    acc.w += v[k].w;
  }
  __syncthreads();
  const unsigned long long t3 = clk();
  if (acc.x == -1.f) out[1000] = 1;  // keep the loads
  if (tid == 0) {
    out[blockIdx.x * 3 + 0] = t1 - t0;
    out[blockIdx.x * 3 + 1] = t2 - t1;
    out[blockIdx.x * 3 + 2] = t3 - t2;
  }
}

int main() {
  const int G = 148;
  float4* ws;
  int* ctr;
  unsigned long long* d;
  cudaMalloc(&ws, static_cast<size_t>(G) * 65536);
  cudaMalloc(&ctr, 4);
  cudaMalloc(&d, 2048 * 8);
  const char* names[3] = {"own slot  ", "next slot ", "next, stale"};
  for (int rep = 0; rep < 2; ++rep)
    for (int mode = 0; mode < 3; ++mode) {
      cudaMemset(ctr, 0, 4);
      xchg_kernel<<<G, 256>>>(ws, ctr, mode, d);
      cudaError_t e = cudaDeviceSynchronize();
      unsigned long long h[3 * 148];
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      unsigned long long mx[3] = {0, 0, 0};
      for (int c = 0; c < G; ++c)
        for (int f = 0; f < 3; ++f) mx[f] = h[c * 3 + f] > mx[f] ? h[c * 3 + f] : mx[f];
      printf("%s: ns write %5llu arrive+wait %5llu read64KB %5llu | max over CTAs %5llu %5llu %5llu (%s)\n", names[mode],
             h[0], h[1], h[2], mx[0], mx[1], mx[2], cudaGetErrorString(e));
    }
  return 0;
}
