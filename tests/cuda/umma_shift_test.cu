// Micro-test of tcgen05 shared-memory descriptor semantics needed by the
// halo (shifted-window) implicit-GEMM conv: an A operand whose start row is
// shifted by an arbitrary number of 128-byte (SW128) or 16-byte (no-swizzle)
// rows inside a TMA-loaded tile.
//
// Build: nvcc -std=c++17 -O2 -gencode arch=compute_100a,code=sm_100a
//        -I paper_2101_07344_b200/csrc/kernels tests/cuda/umma_shift_test.cu -o umma_shift_test -lcuda
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "sm100_prims.cuh"

using namespace lcb;

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e = (x);                                                             \
    if (e != cudaSuccess) {                                                          \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(2);                                                                       \
    }                                                                                \
  } while (0)

constexpr int kRows = 256, kK = 64, kN = 64;
__constant__ int kShifts[] = {0, 1, 3, 5, 8, 13, 34, 35, 71, 127};
static const int hShifts[] = {0, 1, 3, 5, 8, 13, 34, 35, 71, 127};
constexpr int kNS = 10;

__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr, uint32_t base_off) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr & 0x3FFFFu) >> 4);
  d |= static_cast<uint64_t>(1) << 16;
  d |= static_cast<uint64_t>(1024 >> 4) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(base_off & 7) << 49;
  d |= static_cast<uint64_t>(2) << 61;
  return d;
}
// No swizzle, K-major: core matrix = 8 rows x 16 B; lbo = K-direction core
// matrix stride, sbo = M/N-direction 8-row group stride.
__device__ __forceinline__ uint64_t desc_none(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr & 0x3FFFFu) >> 4);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  return d;
}

struct Maps {
  CUtensorMap a_sw, b_sw, a_ns, b_ns;
};

// out[variant][shift][128][64] fp32; variants: 0 SW128 base_off 0, 1 SW128
// base_off (addr>>7)&7, 2 no-swizzle (lbo=region, sbo=128), 3 no-swizzle swapped.
__global__ void __launch_bounds__(128, 1) shift_kernel(const __grid_constant__ Maps m, float* out, int only_v) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint8_t* a_sw = sm;                       // 256 x 128 B = 32 KB
  uint8_t* b_sw = sm + 32768;               // 64 x 128 B = 8 KB
  uint8_t* a_ns = sm + 40960;               // [8 groups][256 rows][16 B] = 32 KB
  uint8_t* b_ns = sm + 73728;               // [8 groups][64 rows][16 B] = 8 KB
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 81920);
  uint32_t* holder = reinterpret_cast<uint32_t*>(sm + 81920 + 64);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bar[0]), 1);
    mbar_init(smem_u32(&bar[1]), 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(smem_u32(holder), 64);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *holder;
  if (threadIdx.x == 0) {
    mbar_expect_tx(smem_u32(&bar[0]), 32768 + 8192 + 32768 + 8192);
    tma_load_2d(smem_u32(a_sw), &m.a_sw, smem_u32(&bar[0]), 0, 0);
    tma_load_2d(smem_u32(b_sw), &m.b_sw, smem_u32(&bar[0]), 0, 0);
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
            smem_u32(a_ns)),
        "l"(reinterpret_cast<uint64_t>(&m.a_ns)), "r"(0), "r"(0), "r"(0), "r"(smem_u32(&bar[0]))
        : "memory");
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
            smem_u32(b_ns)),
        "l"(reinterpret_cast<uint64_t>(&m.b_ns)), "r"(0), "r"(0), "r"(0), "r"(smem_u32(&bar[0]))
        : "memory");
  }
  mbar_wait(smem_u32(&bar[0]), 0);
  uint32_t phase = 0;
  constexpr uint32_t idesc = umma_idesc_bf16(128, kN);
  for (int v = only_v; v <= only_v; ++v) {
    for (int si = 0; si < kNS; ++si) {
      const int sh = kShifts[si];
      if (threadIdx.x == 0) {
        tc_fence_after();
        for (int k = 0; k < 4; ++k) {
          uint64_t ad, bd;
          if (v < 2) {
            const uint32_t a = smem_u32(a_sw) + sh * 128 + 32 * k;
            ad = desc_sw128(a, v == 1 ? ((a >> 7) & 7) : 0);
            bd = desc_sw128(smem_u32(b_sw) + 32 * k, 0);
          } else {
            // k16 step = 2 core-matrix columns = 2 groups
            const uint32_t a = smem_u32(a_ns) + sh * 16 + k * 2 * (kRows * 16);
            const uint32_t b = smem_u32(b_ns) + k * 2 * (kN * 16);
            ad = v == 2 ? desc_none(a, kRows * 16, 128) : desc_none(a, 128, kRows * 16);
            bd = v == 2 ? desc_none(b, kN * 16, 128) : desc_none(b, 128, kN * 16);
          }
          umma_bf16(tmem, ad, bd, idesc, k > 0 ? 1u : 0u);
        }
        umma_commit(smem_u32(&bar[1]));
      }
      mbar_wait(smem_u32(&bar[1]), phase);
      phase ^= 1;
      tc_fence_after();
      const int row = warp * 32 + lane;
      float* o = out + ((static_cast<size_t>(v) * kNS + si) * 128 + row) * kN;
      for (int c = 0; c < kN; c += 16) {
        float r[16];
        tmem_ld16(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c, r);
        for (int i = 0; i < 16; ++i) o[c + i] = r[i];
      }
      tc_fence_before();
      __syncthreads();
    }
  }
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 64);
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  const int only_v = argc > 1 ? atoi(argv[1]) : 0;
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q));
  EncodeFn enc = reinterpret_cast<EncodeFn>(fp);
  std::vector<__nv_bfloat16> A(kRows * kK), B(kN * kK);
  std::vector<float> Af(kRows * kK), Bf(kN * kK);
  srand(7);
  for (int i = 0; i < kRows * kK; ++i) {
    Af[i] = static_cast<float>(rand() % 9 - 4);
    A[i] = __float2bfloat16(Af[i]);
  }
  for (int i = 0; i < kN * kK; ++i) {
    Bf[i] = static_cast<float>(rand() % 7 - 3);
    B[i] = __float2bfloat16(Bf[i]);
  }
  __nv_bfloat16 *dA, *dB;
  CK(cudaMalloc(&dA, A.size() * 2));
  CK(cudaMalloc(&dB, B.size() * 2));
  CK(cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice));
  Maps m;
  {
    cuuint64_t dims[2] = {kK, kRows}, str[1] = {kK * 2};
    cuuint32_t box[2] = {64, kRows}, es[2] = {1, 1};
    CUresult r = enc(&m.a_sw, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dA, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode a_sw: %d\n", (int)r);
    cuuint64_t dimsb[2] = {kK, kN};
    cuuint32_t boxb[2] = {64, kN};
    r = enc(&m.b_sw, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dB, dimsb, str, boxb, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode b_sw: %d\n", (int)r);
  }
  {
    // (k%8, row, k/8) with strides row = 128 B, group = 16 B (non-monotonic).
    cuuint64_t dims[3] = {8, kRows, 8}, str[2] = {kK * 2, 16};
    cuuint32_t box[3] = {8, kRows, 8}, es[3] = {1, 1, 1};
    CUresult r = enc(&m.a_ns, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, dA, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode a_ns (3-D, group stride 16 B): %d\n", (int)r);
    cuuint64_t dimsb[3] = {8, kN, 8};
    cuuint32_t boxb[3] = {8, kN, 8};
    r = enc(&m.b_ns, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, dB, dimsb, str, boxb, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode b_ns: %d\n", (int)r);
  }
  float* dOut;
  const size_t on = 4ull * kNS * 128 * kN;
  CK(cudaMalloc(&dOut, on * 4));
  CK(cudaMemset(dOut, 0, on * 4));
  CK(cudaFuncSetAttribute(shift_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 90 * 1024));
  shift_kernel<<<1, 128, 90 * 1024>>>(m, dOut, only_v);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  std::vector<float> out(on);
  CK(cudaMemcpy(out.data(), dOut, on * 4, cudaMemcpyDeviceToHost));
  const char* names[4] = {"SW128 base_off=0", "SW128 base_off=(a>>7)&7", "NONE lbo=K sbo=M", "NONE lbo=M sbo=K"};
  for (int v = only_v; v <= only_v; ++v) {
    printf("%-26s", names[v]);
    for (int si = 0; si < kNS; ++si) {
      const int sh = hShifts[si];
      long bad = 0;
      for (int r = 0; r < 128; ++r)
        for (int n = 0; n < kN; ++n) {
          float ref = 0;
          for (int k = 0; k < kK; ++k) ref += Af[(r + sh) * kK + k] * Bf[n * kK + k];
          if (out[((static_cast<size_t>(v) * kNS + si) * 128 + r) * kN + n] != ref) ++bad;
        }
      printf(" sh%-3d:%s", sh, bad ? "BAD" : "ok ");
    }
    printf("\n");
  }
  return 0;
}
