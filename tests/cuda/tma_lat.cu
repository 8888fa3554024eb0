// Micro-benchmark: TMA (cp.async.bulk.tensor.2d, SW128, 64 x rows bf16 boxes)
// load latency / throughput from an L2-resident source, one CTA per SM, with
// D loads in flight per CTA. Reports cycles per load and GB/s per SM.
// Build: nvcc -std=c++17 -O2 -gencode arch=compute_100a,code=sm_100a
//        -I paper_2101_07344_b200/csrc/kernels tests/cuda/tma_lat.cu paper_2101_07344_b200/csrc/kernels/tc_conv.cu -lcuda -o tma_lat
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdio>

#include "sm100_prims.cuh"
#include "tc_conv.cuh"

using namespace lcb;

__device__ __forceinline__ unsigned long long clk() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));
  return t;
}

__global__ void tma_kernel(const __grid_constant__ CUtensorMap map, int rows_total, int box_rows, int depth, int iters,
                           unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bars[16];
  if (threadIdx.x == 0) {
    for (int i = 0; i < 16; ++i) mbar_init(smem_u32(&bars[i]), 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const uint32_t bytes = static_cast<uint32_t>(box_rows) * 128;
  uint32_t phase[16] = {};
  int row = (blockIdx.x * 977) % (rows_total - box_rows);
  const unsigned long long t0 = clk();
  for (int it = 0; it < iters; ++it) {
    const int slot = it % depth;
    if (it >= depth) {
      mbar_wait(smem_u32(&bars[slot]), phase[slot]);
      phase[slot] ^= 1;
    }
    mbar_expect_tx(smem_u32(&bars[slot]), bytes);
    tma_load_2d(smem_u32(sm + slot * bytes), &map, smem_u32(&bars[slot]), 0, row);
    row += 4099;
    if (row + box_rows > rows_total) row -= rows_total - box_rows;
  }
  for (int k = 0; k < depth; ++k) {
    const int it = iters + k;
    const int slot = it % depth;
    mbar_wait(smem_u32(&bars[slot]), phase[slot]);
    phase[slot] ^= 1;
  }
  out[blockIdx.x] = clk() - t0;
}

// Activation boxes as tc_conv loads them: 5-D map (C, W, H, N, P), box
// {64, wb, hb, 1, 1}, random tile origins incl. tap offsets (OOB zero fill).
__global__ void tma5_kernel(const __grid_constant__ CUtensorMap map, int W, int H, int N, int wb, int hb, int depth,
                            int iters, int per_stage, int oob, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bars[16];
  if (threadIdx.x == 0) {
    for (int i = 0; i < 16; ++i) mbar_init(smem_u32(&bars[i]), 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const uint32_t bytes = static_cast<uint32_t>(wb * hb) * 128;
  uint32_t phase[16] = {};
  unsigned int seed = blockIdx.x * 2654435761u;
  const unsigned long long t0 = clk();
  for (int it = 0; it < iters; ++it) {
    const int slot = it % depth;
    if (it >= depth) {
      mbar_wait(smem_u32(&bars[slot]), phase[slot]);
      phase[slot] ^= 1;
    }
    mbar_expect_tx(smem_u32(&bars[slot]), bytes * per_stage);
    for (int j = 0; j < per_stage; ++j) {
      seed = seed * 1664525u + 1013904223u;
      const int n = (seed >> 8) % N;
      const int h0 = ((seed >> 4) % (H / hb)) * hb - (oob & 1 ? (seed & 1) : 0);
      const int w0 = oob & 2 ? -static_cast<int>((seed >> 1) & 1) : 0;
      tma_load_5d(smem_u32(sm + (slot * per_stage + j) * bytes), &map, smem_u32(&bars[slot]), 0, w0, h0, n, 0);
    }
  }
  for (int k = 0; k < depth; ++k) {
    const int slot = (iters + k) % depth;
    mbar_wait(smem_u32(&bars[slot]), phase[slot]);
    phase[slot] ^= 1;
  }
  out[blockIdx.x] = clk() - t0;
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__device__ __forceinline__ void tma_load_4d_(uint32_t dst, const void* tmap, uint32_t bar, int c0, int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d_(uint32_t dst, const void* tmap, uint32_t bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
      : "memory");
}

// Issue-parallel variant: the per_stage boxes of a stage are issued by per_stage
// lanes of the warp in one instruction (lane 0 arms the barrier).
__global__ void tma_lanes_kernel(const __grid_constant__ CUtensorMap map, int W, int H, int N, int wb, int hb,
                                 int depth, int iters, int per_stage, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bars[16];
  const int lane = threadIdx.x;
  if (lane == 0) {
    for (int i = 0; i < 16; ++i) mbar_init(smem_u32(&bars[i]), 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (lane >= per_stage) return;
  const uint32_t bytes = static_cast<uint32_t>(wb * hb) * 128;
  uint32_t phase[16] = {};
  unsigned int seed = blockIdx.x * 2654435761u + lane * 977u;
  const unsigned long long t0 = clk();
  for (int it = 0; it < iters; ++it) {
    const int slot = it % depth;
    if (it >= depth) {
      mbar_wait(smem_u32(&bars[slot]), phase[slot]);
      phase[slot] ^= 1;
    }
    if (lane == 0) mbar_expect_tx(smem_u32(&bars[slot]), bytes * per_stage);
    seed = seed * 1664525u + 1013904223u;
    const int n = (seed >> 8) % N, h0 = ((seed >> 4) % (H / hb)) * hb;
    tma_load_5d(smem_u32(sm + (slot * per_stage + lane) * bytes), &map, smem_u32(&bars[slot]), 0, 0, h0, n, 0);
  }
  for (int k = 0; k < depth; ++k) {
    const int slot = (iters + k) % depth;
    mbar_wait(smem_u32(&bars[slot]), phase[slot]);
    phase[slot] ^= 1;
  }
  if (lane == 0) out[blockIdx.x] = clk() - t0;
}

// dims = 3: (C, W, H*N); 4: (C, W, H, N). Same boxes {64, wb, hb(, 1)} as tc_conv's A loads.
__global__ void tmaN_kernel(const __grid_constant__ CUtensorMap map, int dims, int W, int H, int N, int wb, int hb,
                            int depth, int iters, int per_stage, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bars[16];
  if (threadIdx.x == 0) {
    for (int i = 0; i < 16; ++i) mbar_init(smem_u32(&bars[i]), 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const uint32_t bytes = static_cast<uint32_t>(wb * hb) * 128;
  uint32_t phase[16] = {};
  unsigned int seed = blockIdx.x * 2654435761u;
  const unsigned long long t0 = clk();
  for (int it = 0; it < iters; ++it) {
    const int slot = it % depth;
    if (it >= depth) {
      mbar_wait(smem_u32(&bars[slot]), phase[slot]);
      phase[slot] ^= 1;
    }
    mbar_expect_tx(smem_u32(&bars[slot]), bytes * per_stage);
    for (int j = 0; j < per_stage; ++j) {
      seed = seed * 1664525u + 1013904223u;
      const int n = (seed >> 8) % N, h0 = ((seed >> 4) % (H / hb)) * hb;
      const uint32_t dst = smem_u32(sm + (slot * per_stage + j) * bytes);
      if (dims == 3) tma_load_3d_(dst, &map, smem_u32(&bars[slot]), 0, 0, n * H + h0);
      else tma_load_4d_(dst, &map, smem_u32(&bars[slot]), 0, 0, h0, n);
    }
  }
  for (int k = 0; k < depth; ++k) {
    const int slot = (iters + k) % depth;
    mbar_wait(smem_u32(&bars[slot]), phase[slot]);
    phase[slot] ^= 1;
  }
  out[blockIdx.x] = clk() - t0;
}

int main() {
  const int rows_total = 256 * 1024;  // 64 ch x 256K rows bf16 = 32 MB (L2 resident)
  __nv_bfloat16* src;
  cudaMalloc(&src, static_cast<size_t>(rows_total) * 128);
  cudaMemset(src, 0, static_cast<size_t>(rows_total) * 128);
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  for (int box_rows : {64, 128, 256}) {
    CUtensorMap map;
    if (!encode_weight_map(&map, src, 64, rows_total, box_rows)) {
      printf("encode failed\n");
      return 1;
    }
    for (int depth : {1, 2, 4, 8}) {
      const int iters = 2000;
      const int smem = depth * box_rows * 128 + 1024;
      cudaFuncSetAttribute(tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      tma_kernel<<<148, 32, smem>>>(map, rows_total, box_rows, depth, iters, d);
      cudaDeviceSynchronize();
      unsigned long long h[148];
      cudaMemcpy(h, d, 148 * 8, cudaMemcpyDeviceToHost);
      double mx = 0;
      for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
      const double cyc = mx / iters;
      printf("box %3d rows (%5d B) depth %d: %7.1f cycles/load, %6.1f B/clk/SM, chip %.2f TB/s @1.965GHz (%s)\n",
             box_rows, box_rows * 128, depth, cyc, box_rows * 128 / cyc, 148 * box_rows * 128 / cyc * 1.965e9 / 1e12,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  {
    const int C = 64, W = 32, H = 32, N = 256;
    __nv_bfloat16* act;
    cudaMalloc(&act, static_cast<size_t>(N) * H * W * C * 2);
    cudaMemset(act, 0, static_cast<size_t>(N) * H * W * C * 2);
    struct Cfg { int wb, hb, per_stage, depth, oob; };
    for (Cfg c : {Cfg{32, 4, 2, 4, 0}, Cfg{32, 4, 2, 4, 1}, Cfg{32, 4, 2, 4, 2}, Cfg{32, 4, 2, 4, 3}, Cfg{4, 4, 8, 4, 0},
                  Cfg{4, 4, 8, 4, 3}}) {
      CUtensorMap map;
      if (!encode_act_map(&map, act, C, W, H, N, 1, c.wb, c.hb, 1)) {
        printf("encode5 failed\n");
        return 1;
      }
      const int iters = 1000;
      const int smem = c.depth * c.per_stage * c.wb * c.hb * 128 + 1024;
      cudaFuncSetAttribute(tma5_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      tma5_kernel<<<148, 32, smem>>>(map, W, H, N, c.wb, c.hb, c.depth, iters, c.per_stage, c.oob, d);
      cudaDeviceSynchronize();
      unsigned long long h[148];
      cudaMemcpy(h, d, 148 * 8, cudaMemcpyDeviceToHost);
      double mx = 0;
      for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
      const double cyc = mx / iters;
      const double by = double(c.per_stage) * c.wb * c.hb * 128;
      printf("5-D box {64,%d,%d} x%d per stage, depth %d, oob h%d w%d: %7.1f cycles/stage, %6.1f B/clk/SM (%s)\n",
             c.wb, c.hb, c.per_stage, c.depth, c.oob & 1, (c.oob >> 1) & 1, cyc, by / cyc,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  {
    const int C = 64, W = 32, H = 32, N = 256;
    __nv_bfloat16* act;
    cudaMalloc(&act, static_cast<size_t>(N) * H * W * C * 2);
    cudaMemset(act, 0, static_cast<size_t>(N) * H * W * C * 2);
    for (int wbhb : {0, 1}) {
      const int wb = wbhb ? 4 : 32, hb = 4;
      CUtensorMap map;
      if (!encode_act_map(&map, act, C, W, H, N, 1, wb, hb, 1)) return 1;
      for (int ps : {1, 2, 4, 8}) {
        const int iters = 1000, depth = 4;
        const int smem = depth * ps * wb * hb * 128 + 1024;
        cudaFuncSetAttribute(tma_lanes_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        tma_lanes_kernel<<<148, 32, smem>>>(map, W, H, N, wb, hb, depth, iters, ps, d);
        cudaDeviceSynchronize();
        unsigned long long h[148];
        cudaMemcpy(h, d, 148 * 8, cudaMemcpyDeviceToHost);
        double mx = 0;
        for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
        const double cyc = mx / iters;
        printf("lanes: 5-D box {64,%d,%d} x%d per stage from %d lanes, depth 4: %7.1f cycles/stage, %6.1f B/clk/SM (%s)\n",
               wb, hb, ps, ps, cyc, double(ps) * wb * hb * 128 / cyc, cudaGetErrorString(cudaGetLastError()));
      }
    }
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
    EncFn enc = reinterpret_cast<EncFn>(fp);
    for (int dims : {3, 4}) {
      for (int hb : {4, 8}) {
        CUtensorMap map;
        cuuint64_t gd[4], gs[3];
        cuuint32_t box[4], es[4] = {1, 1, 1, 1};
        gd[0] = C; gd[1] = W;
        if (dims == 3) { gd[2] = static_cast<cuuint64_t>(H) * N; } else { gd[2] = H; gd[3] = N; }
        gs[0] = C * 2; gs[1] = gs[0] * W; gs[2] = gs[1] * H;
        box[0] = 64; box[1] = 32; box[2] = hb; box[3] = 1;
        CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, dims, act, gd, gs, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) { printf("enc %d failed\n", dims); return 1; }
        const int iters = 1000, depth = 4, per_stage = 2;
        const int smem = depth * per_stage * 32 * hb * 128 + 1024;
        cudaFuncSetAttribute(tmaN_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        tmaN_kernel<<<148, 32, smem>>>(map, dims, W, H, N, 32, hb, depth, iters, per_stage, d);
        cudaDeviceSynchronize();
        unsigned long long h[148];
        cudaMemcpy(h, d, 148 * 8, cudaMemcpyDeviceToHost);
        double mx = 0;
        for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
        const double cyc = mx / iters;
        printf("%d-D box {64,32,%d} x2 per stage, depth 4: %7.1f cycles/stage, %6.1f B/clk/SM (%s)\n", dims, hb, cyc,
               2.0 * 32 * hb * 128 / cyc, cudaGetErrorString(cudaGetLastError()));
      }
    }
  }
  return 0;
}
