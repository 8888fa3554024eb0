// tcgen05 / TMA / TMEM implicit-GEMM kernel. See tc_conv.cuh for the contract.
//
// Warp roles (192 threads, one CTA per SM, persistent over tiles):
//   warp 0      : TMA producer (lane 0) + TMEM allocator (whole warp)
//   warp 1      : MMA issuer (lane 0)
//   warps 2..5  : epilogue, one TMEM lane quadrant (warp % 4) each
// Pipelines: smem ring full/empty (TMA <-> MMA), TMEM double buffer
// tfull/tempty (MMA <-> epilogue).
#include "sm100_prims.cuh"
#include "tc_conv.cuh"

#include <cstdio>

namespace lcb {

namespace {

constexpr int kBM = 128;
constexpr int kABytes = kBM * 128;  // 128 rows x 64 bf16

template <int BN>
struct TcCfg {
  static constexpr int kBBytes = BN * 128;
  static constexpr int kStages = BN == 256 ? 4 : (BN == 128 ? 6 : 8);
  static constexpr int kSmem = kStages * (kABytes + kBBytes) + 1024 /*bars*/ + 1024 /*align*/;
  static constexpr uint32_t kTmemCols = 2 * BN;
};

struct TileGeom {
  int count, n_groups, tiles_w, tiles_img, tiles_n, total, nk;
};

__device__ __forceinline__ TileGeom tile_geom(const TcConvParams& p, int BN) {
  TileGeom g;
  g.count = p.count ? *p.count : p.count_static;
  if (p.plain) {
    g.n_groups = 1;
    g.tiles_w = (g.count + kBM - 1) / kBM;
  } else {
    g.n_groups = (g.count + p.ipt - 1) / p.ipt;
    g.tiles_w = p.tiles_w;
  }
  g.tiles_img = p.tiles_h * g.tiles_w;
  g.tiles_n = p.Cout / BN;
  g.total = g.n_groups * g.tiles_img * g.tiles_n * p.ksplit;
  g.nk = p.ntaps * (p.C / 64) * p.segs;
  return g;
}

struct Tile {
  int tn, ks, grp, h0, w0, s_begin, s_end;
};

__device__ __forceinline__ Tile decode_tile(int t, const TcConvParams& p, const TileGeom& g) {
  Tile x;
  x.ks = t % p.ksplit;
  t /= p.ksplit;
  x.tn = t % g.tiles_n;
  const int tm = t / g.tiles_n;
  x.grp = tm / g.tiles_img;
  const int r = tm % g.tiles_img;
  x.h0 = (r / g.tiles_w) * p.hb;
  x.w0 = (r % g.tiles_w) * p.wb;
  x.s_begin = static_cast<int>((static_cast<long long>(g.nk) * x.ks) / p.ksplit);
  x.s_end = static_cast<int>((static_cast<long long>(g.nk) * (x.ks + 1)) / p.ksplit);
  return x;
}

__device__ __forceinline__ int image_of(const TcConvParams& p, int idx) { return p.surv ? p.surv[idx] : idx; }

template <int BN>
__global__ void __launch_bounds__(192, 1) tc_conv_kernel(const __grid_constant__ TcConvParams p) {
  using Cfg = TcCfg<BN>;
  constexpr int S = Cfg::kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + S * kABytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sB + S * Cfg::kBBytes);
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 2 * S + 4);
  const uint32_t full0 = smem_u32(bars);
  const uint32_t empty0 = smem_u32(bars + S);
  const uint32_t tfull0 = smem_u32(bars + 2 * S);
  const uint32_t tempty0 = smem_u32(bars + 2 * S + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(full0 + 8 * i, 1);
      mbar_init(empty0 + 8 * i, 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(tfull0 + 8 * i, 1);
      mbar_init(tempty0 + 8 * i, 4);
    }
    fence_mbar_init();
    tma_prefetch_desc(&p.tmA[0]);
    tma_prefetch_desc(&p.tmB[0]);
    if (p.segs > 1) {
      tma_prefetch_desc(&p.tmA[1]);
      tma_prefetch_desc(&p.tmB[1]);
    }
  }
  if (warp == 0) tmem_alloc(smem_u32(tmem_holder), Cfg::kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  const TileGeom g = tile_geom(p, BN);
  const int cchunks = p.C / 64;

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------ TMA producer
      int stage = 0;
      uint32_t phase = 0;
      const int box_bytes = p.hb * p.wb * 128;
      for (int t = blockIdx.x; t < g.total; t += gridDim.x) {
        const Tile x = decode_tile(t, p, g);
        int imgs[8];
        if (p.plain) {
          imgs[0] = 0;
        } else {
          for (int j = 0; j < p.ipt; ++j) {
            int idx = x.grp * p.ipt + j;
            if (idx >= g.count) idx = g.count - 1;  // rows discarded by the epilogue
            imgs[j] = image_of(p, idx);
          }
        }
        const int ipt = p.plain ? 1 : p.ipt;
        for (int s = x.s_begin; s < x.s_end; ++s) {
          mbar_wait(empty0 + 8 * stage, phase ^ 1);
          const uint32_t fb = full0 + 8 * stage;
          mbar_expect_tx(fb, kABytes + Cfg::kBBytes);
          const int seg = s % p.segs;
          const int cc = (s / p.segs) % cchunks;
          const int tap = s / (p.segs * cchunks);
          const CUtensorMap* am = (seg == 2) ? &p.tmA[1] : &p.tmA[0];
          const CUtensorMap* bm = (seg == 1) ? &p.tmB[1] : &p.tmB[0];
          const uint32_t a_dst = smem_u32(sA + stage * kABytes);
          const int dh = p.tap_dh[tap], dw = p.tap_dw[tap], ph = p.tap_phase[tap];
          for (int j = 0; j < ipt; ++j) {
            tma_load_5d(a_dst + j * box_bytes, am, fb, cc * 64, x.w0 + dw, x.h0 + dh, imgs[j], ph);
          }
          tma_load_2d(smem_u32(sB + stage * Cfg::kBBytes), bm, fb, tap * p.C + cc * 64, x.tn * BN);
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ------------------------------------------------ MMA issuer
      constexpr uint32_t idesc = umma_idesc_bf16(kBM, BN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int t = blockIdx.x; t < g.total; t += gridDim.x) {
        const Tile x = decode_tile(t, p, g);
        mbar_wait(tempty0 + 8 * acc, acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int s = x.s_begin; s < x.s_end; ++s) {
          mbar_wait(full0 + 8 * stage, phase);
          tc_fence_after();
          const uint32_t a_base = smem_u32(sA + stage * kABytes);
          const uint32_t b_base = smem_u32(sB + stage * Cfg::kBBytes);
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            umma_bf16(d_tmem, umma_desc_sw128(a_base + 32 * k), umma_desc_sw128(b_base + 32 * k), idesc,
                      (s > x.s_begin || k > 0) ? 1u : 0u);
          }
          umma_commit(empty0 + 8 * stage);
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit(tfull0 + 8 * acc);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else {
    // ------------------------------------------------ epilogue
    const int quad = warp & 3;
    const int row = quad * 32 + lane;
    int acc = 0;
    uint32_t acc_phase = 0;
    const int rows_per_img = p.hb * p.wb;
    for (int t = blockIdx.x; t < g.total; t += gridDim.x) {
      const Tile x = decode_tile(t, p, g);
      // Which output position does this accumulator row hold?
      bool valid;
      size_t obase;  // element offset of (n, h, w, 0) / row start
      int grow = 0;
      if (p.plain) {
        grow = x.w0 + row;
        valid = grow < g.count;
        obase = static_cast<size_t>(grow) * p.Cout;
      } else {
        const int j = row / rows_per_img;
        const int pix = row % rows_per_img;
        const int h = x.h0 + pix / p.wb;
        const int w = x.w0 + pix % p.wb;
        const int idx = x.grp * p.ipt + j;
        valid = (idx < g.count) && (h < p.Ho) && (w < p.Wo);
        const int n = valid ? image_of(p, idx) : 0;
        obase = ((static_cast<size_t>(n) * p.Ho + h) * p.Wo + w) * p.Cout;
      }
      mbar_wait(tfull0 + 8 * acc, acc_phase);
      tc_fence_after();
      const uint32_t t_row = tmem_base + (static_cast<uint32_t>(quad * 32) << 16) + acc * BN;
#pragma unroll 1
      for (int c16 = 0; c16 < BN / 16; ++c16) {
        float v[16];
        tmem_ld16(t_row + c16 * 16, v);
        if (!valid) continue;
        const int co = x.tn * BN + c16 * 16;
        if (p.mode == 1) {
          float4* dst = reinterpret_cast<float4*>(
              p.out_f32 + (static_cast<size_t>(x.ks) * p.rows_total + grow) * p.Cout + co);
#pragma unroll
          for (int q = 0; q < 4; ++q) dst[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
          continue;
        }
        if (p.scale) {
          const float4* sc = reinterpret_cast<const float4*>(p.scale + co);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float4 s4 = __ldg(sc + q);
            v[4 * q] *= s4.x;
            v[4 * q + 1] *= s4.y;
            v[4 * q + 2] *= s4.z;
            v[4 * q + 3] *= s4.w;
          }
        }
        if (p.shift) {
          const float4* sh = reinterpret_cast<const float4*>(p.shift + co);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float4 s4 = __ldg(sh + q);
            v[4 * q] += s4.x;
            v[4 * q + 1] += s4.y;
            v[4 * q + 2] += s4.z;
            v[4 * q + 3] += s4.w;
          }
        }
        const size_t off = obase + co;
        if (p.res_hi) {
          const uint4* rh = reinterpret_cast<const uint4*>(p.res_hi + off);
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const uint4 u = rh[q];
            const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float2 f = __bfloat1622float2(b2[e]);
              v[8 * q + 2 * e] += f.x;
              v[8 * q + 2 * e + 1] += f.y;
            }
          }
          if (p.res_lo) {
            const uint4* rl = reinterpret_cast<const uint4*>(p.res_lo + off);
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              const uint4 u = rl[q];
              const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const float2 f = __bfloat1622float2(b2[e]);
                v[8 * q + 2 * e] += f.x;
                v[8 * q + 2 * e + 1] += f.y;
              }
            }
          }
        }
        if (p.relu) {
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] = v[i] > 0.0f ? v[i] : 0.0f;
        }
        uint4 hi[2], lo[2];
        __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(hi);
        __nv_bfloat162* l2 = reinterpret_cast<__nv_bfloat162*>(lo);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const __nv_bfloat162 hh = __floats2bfloat162_rn(v[2 * e], v[2 * e + 1]);
          h2[e] = hh;
          const float2 hf = __bfloat1622float2(hh);
          l2[e] = __floats2bfloat162_rn(v[2 * e] - hf.x, v[2 * e + 1] - hf.y);
        }
        uint4* oh = reinterpret_cast<uint4*>(p.out_hi + off);
        oh[0] = hi[0];
        oh[1] = hi[1];
        if (p.out_lo) {
          uint4* ol = reinterpret_cast<uint4*>(p.out_lo + off);
          ol[0] = lo[0];
          ol[1] = lo[1];
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty0 + 8 * acc);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  }
  __syncthreads();
  if (warp == 0) {
    __syncwarp();
    tmem_dealloc(tmem_base, Cfg::kTmemCols);
  }
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess) {
      fn = reinterpret_cast<EncodeTiledFn>(ptr);
    }
  }
  return fn;
}

template <int BN>
cudaError_t launch_bn(const TcConvParams& p, int num_sms, cudaStream_t stream) {
  using Cfg = TcCfg<BN>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(tc_conv_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmem);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  int tiles = tc_conv_max_tiles(p, BN);
  if (tiles <= 0) return cudaSuccess;
  const int grid = tiles < num_sms ? tiles : num_sms;
  tc_conv_kernel<BN><<<grid, 192, Cfg::kSmem, stream>>>(p);
  return cudaGetLastError();
}

}  // namespace

bool encode_act_map(CUtensorMap* map, const void* base, int C, int W, int H, int N, int P, int wb, int hb) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[5] = {static_cast<cuuint64_t>(C), static_cast<cuuint64_t>(W), static_cast<cuuint64_t>(H),
                        static_cast<cuuint64_t>(N), static_cast<cuuint64_t>(P)};
  cuuint64_t strides[4];
  strides[0] = static_cast<cuuint64_t>(C) * 2;
  strides[1] = strides[0] * W;
  strides[2] = strides[1] * H;
  strides[3] = strides[2] * N;
  cuuint32_t box[5] = {64, static_cast<cuuint32_t>(wb), static_cast<cuuint32_t>(hb), 1, 1};
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool encode_weight_map(CUtensorMap* map, const void* base, int K, int Cout, int BN) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(Cout)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(K) * 2};
  cuuint32_t box[2] = {64, static_cast<cuuint32_t>(BN)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

int tc_conv_pick_bn(int Cout) {
  if (Cout % 256 == 0 && Cout >= 512) return 256;
  if (Cout % 128 == 0) return 128;
  return 64;
}

int tc_conv_max_tiles(const TcConvParams& p, int BN) {
  const int count = p.count_static;
  long long n_groups, tiles_w;
  if (p.plain) {
    n_groups = 1;
    tiles_w = (count + kBM - 1) / kBM;
  } else {
    n_groups = (count + p.ipt - 1) / p.ipt;
    tiles_w = p.tiles_w;
  }
  const long long total = n_groups * p.tiles_h * tiles_w * (p.Cout / BN) * p.ksplit;
  return total > 0x7fffffff ? 0x7fffffff : static_cast<int>(total);
}

cudaError_t tc_conv_launch(const TcConvParams& p, int BN, int num_sms, cudaStream_t stream) {
  switch (BN) {
    case 64:
      return launch_bn<64>(p, num_sms, stream);
    case 128:
      return launch_bn<128>(p, num_sms, stream);
    case 256:
      return launch_bn<256>(p, num_sms, stream);
    default:
      return cudaErrorInvalidValue;
  }
}

}  // namespace lcb
