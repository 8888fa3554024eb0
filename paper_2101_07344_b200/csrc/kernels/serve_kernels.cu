// Serve-path kernels (see serve_kernels.cuh). All cache-head arithmetic is
// fp32 with deterministic (fixed-order) reductions; only the activations are
// bf16 hi (+lo) planes.
#include "gpu_sync.cuh"
#include "pdl.cuh"
#include "serve_kernels.cuh"

#include <cfloat>

namespace lcb {

namespace {

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ float ld_tap(const TapView& t, long long off) {
  float v = __bfloat162float(t.hi[off]);
  if (t.lo) v += __bfloat162float(t.lo[off]);
  return v;
}

// 8 consecutive channels (16 bytes per plane) -> 8 floats.
__device__ __forceinline__ void ld_tap8(const TapView& t, long long off, float (&v)[8]) {
  const uint4 h = *reinterpret_cast<const uint4*>(t.hi + off);
  const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&h);
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const float2 f = __bfloat1622float2(h2[e]);
    v[2 * e] = f.x;
    v[2 * e + 1] = f.y;
  }
  if (t.lo) {
    const uint4 l = *reinterpret_cast<const uint4*>(t.lo + off);
    const __nv_bfloat162* l2 = reinterpret_cast<const __nv_bfloat162*>(&l);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 f = __bfloat1622float2(l2[e]);
      v[2 * e] += f.x;
      v[2 * e + 1] += f.y;
    }
  }
}

__device__ __forceinline__ void split_store(float v, __nv_bfloat16* hi, __nv_bfloat16* lo, long long off) {
  const __nv_bfloat16 h = __float2bfloat16_rn(v);
  hi[off] = h;
  if (lo) lo[off] = __float2bfloat16_rn(v - __bfloat162float(h));
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Block-wide sum with a fixed reduction tree (deterministic). blockDim <= 1024.
__device__ float block_sum(float v, float* scratch) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) scratch[warp] = v;
  __syncthreads();
  float t = 0.0f;
  if (warp == 0) {
    t = lane < nw ? scratch[lane] : 0.0f;
    t = warp_sum(t);
    if (lane == 0) scratch[0] = t;
  }
  __syncthreads();
  const float r = scratch[0];
  __syncthreads();
  return r;
}
__device__ float block_max(float v, float* scratch) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_max(v);
  __syncthreads();
  if (lane == 0) scratch[warp] = v;
  __syncthreads();
  if (warp == 0) {
    float t = lane < nw ? scratch[lane] : -FLT_MAX;
    t = warp_max(t);
    if (lane == 0) scratch[0] = t;
  }
  __syncthreads();
  const float r = scratch[0];
  __syncthreads();
  return r;
}

// ------------------------------------------------------------------ pooling
// Reference AvgPool (network.cpp:130-138) over the NCHW-flat tap: bin o is
// the mean of flat elements [o*win, (o+1)*win).
// Case A: win divides HW -> bins are channel strips; each thread owns whole
// strips of 8 channels and streams them (16-byte loads).
__global__ void pool_strips_kernel(TapView t, int win, int width, float inv, float* bins) {
  pdl_wait();
  pdl_trigger();
  const int r = blockIdx.x;
  if (r >= *t.count) return;
  const long long n = t.data_idx ? t.data_idx[r] : r;
  const int cs = blockIdx.y * 64;
  const int g = threadIdx.x & 7, q = threadIdx.x >> 3;
  const int spc = t.HW / win;
  const int per = (spc + 31) / 32;
  const long long base = n * t.row_stride + cs + g * 8;
  for (int wi = q * per; wi < (q + 1) * per && wi < spc; ++wi) {
    float s[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int p = wi * win; p < (wi + 1) * win; ++p) {
      float v[8];
      ld_tap8(t, base + static_cast<long long>(p) * t.C, v);
#pragma unroll
      for (int e = 0; e < 8; ++e) s[e] += v[e];
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) bins[static_cast<long long>(r) * width + static_cast<long long>(cs + g * 8 + e) * spc + wi] = s[e] * inv;
  }
}

// Case B: win = gch * HW (gch divides 64): per-channel totals over 32 pixel
// ranges, combined in a fixed order, then gch channels per bin.
__global__ void pool_channels_kernel(TapView t, int gch, int width, float inv, float* bins) {
  pdl_wait();
  pdl_trigger();
  __shared__ float part[32][65];
  __shared__ float tot[64];
  const int r = blockIdx.x;
  if (r >= *t.count) return;
  const long long n = t.data_idx ? t.data_idx[r] : r;
  const int cs = blockIdx.y * 64;
  const int g = threadIdx.x & 7, q = threadIdx.x >> 3;
  const int R = (t.HW + 31) / 32;
  const long long base = n * t.row_stride + cs + g * 8;
  float s[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int p = q * R; p < (q + 1) * R && p < t.HW; ++p) {
    float v[8];
    ld_tap8(t, base + static_cast<long long>(p) * t.C, v);
#pragma unroll
    for (int e = 0; e < 8; ++e) s[e] += v[e];
  }
#pragma unroll
  for (int e = 0; e < 8; ++e) part[q][g * 8 + e] = s[e];
  __syncthreads();
  if (threadIdx.x < 64) {
    float a = 0.0f;
    for (int k = 0; k < 32; ++k) a += part[k][threadIdx.x];
    tot[threadIdx.x] = a;
  }
  __syncthreads();
  const int nb = 64 / gch;
  if (threadIdx.x < nb) {
    float a = 0.0f;
    for (int k = 0; k < gch; ++k) a += tot[threadIdx.x * gch + k];
    bins[static_cast<long long>(r) * width + cs / gch + threadIdx.x] = a * inv;
  }
}

// ------------------------------------------------------------------ GAP reductions
// Lookup kernels run one CTA of kLk threads per request row; the reductions
// below keep many independent 16-byte loads in flight per thread (the
// surviving-row counts are small, so latency, not bandwidth, is the enemy)
// and combine partial sums in a fixed order (deterministic).
constexpr int kLk = 512;

__device__ __forceinline__ void add4(float4& a, const float4 b) {
  a.x += b.x;
  a.y += b.y;
  a.z += b.z;
  a.w += b.w;
}

// feat[c] = inv * sum_seg src[seg][c] for one image's fused GAP partials
// (tc_conv epilogue, [segs][C] fp32, C % 4 == 0). Thread layout: float4
// column j, segment group g; 4 interleaved chains per thread, then the groups
// in ascending order. red: kLk float4 of shared scratch. Ends with a barrier.
template <int kT = kLk>
__device__ void gap_feats_block(const float* __restrict__ src, int segs, int C, float inv, float* feat, float4* red) {
  constexpr int kLk = kT;  // threads of the calling CTA
  const int tid = threadIdx.x;
  const int C4 = C >> 2;
  const float4* s4 = reinterpret_cast<const float4*>(src);
  if (C4 >= kLk) {
    for (int j = tid; j < C4; j += kLk) {
      float4 a0 = make_float4(0.f, 0.f, 0.f, 0.f), a1 = a0, a2 = a0, a3 = a0;
      int sg = 0;
      for (; sg + 4 <= segs; sg += 4) {
        add4(a0, __ldg(s4 + static_cast<long long>(sg) * C4 + j));
        add4(a1, __ldg(s4 + static_cast<long long>(sg + 1) * C4 + j));
        add4(a2, __ldg(s4 + static_cast<long long>(sg + 2) * C4 + j));
        add4(a3, __ldg(s4 + static_cast<long long>(sg + 3) * C4 + j));
      }
      for (; sg < segs; ++sg) add4(a0, __ldg(s4 + static_cast<long long>(sg) * C4 + j));
      add4(a0, a1);
      add4(a2, a3);
      add4(a0, a2);
      feat[4 * j] = a0.x * inv;
      feat[4 * j + 1] = a0.y * inv;
      feat[4 * j + 2] = a0.z * inv;
      feat[4 * j + 3] = a0.w * inv;
    }
  } else {
    const int G = kLk / C4;
    const int j = tid % C4, g = tid / C4;
    float4 a0 = make_float4(0.f, 0.f, 0.f, 0.f), a1 = a0, a2 = a0, a3 = a0;
    if (g < G) {
      int sg = g;
      for (; sg + 3 * G < segs; sg += 4 * G) {
        add4(a0, __ldg(s4 + static_cast<long long>(sg) * C4 + j));
        add4(a1, __ldg(s4 + static_cast<long long>(sg + G) * C4 + j));
        add4(a2, __ldg(s4 + static_cast<long long>(sg + 2 * G) * C4 + j));
        add4(a3, __ldg(s4 + static_cast<long long>(sg + 3 * G) * C4 + j));
      }
      for (; sg < segs; sg += G) add4(a0, __ldg(s4 + static_cast<long long>(sg) * C4 + j));
    }
    add4(a0, a1);
    add4(a2, a3);
    add4(a0, a2);
    red[tid] = a0;
    __syncthreads();
    if (tid < C4) {
      float4 t = red[tid];
      for (int q = 1; q < G; ++q) add4(t, red[q * C4 + tid]);
      feat[4 * tid] = t.x * inv;
      feat[4 * tid + 1] = t.y * inv;
      feat[4 * tid + 2] = t.z * inv;
      feat[4 * tid + 3] = t.w * inv;
    }
  }
  __syncthreads();
}

// feat[c] = (1/HW) * sum_pixel tap[pixel][c] over one image's NHWC tap
// (hi + lo bf16, C % 8 == 0): 8 channels per 16-byte load, pixel groups of
// threads with 2 chains each, groups combined in ascending order. red: kLk*8
// floats of shared scratch. Ends with a barrier.
__device__ void tap_gap_block(const TapView& t, long long rowb, int C, int HW, float* feat, float* red) {
  const int tid = threadIdx.x;
  const int C8 = C >> 3;
  const float inv = 1.0f / HW;
  if (C8 >= kLk) {
    for (int j = tid; j < C8; j += kLk) {
      float a[8] = {0, 0, 0, 0, 0, 0, 0, 0}, b[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      int q = 0;
      for (; q + 2 <= HW; q += 2) {
        float v[8], w[8];
        ld_tap8(t, rowb + static_cast<long long>(q) * C + 8 * j, v);
        ld_tap8(t, rowb + static_cast<long long>(q + 1) * C + 8 * j, w);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          a[e] += v[e];
          b[e] += w[e];
        }
      }
      if (q < HW) {
        float v[8];
        ld_tap8(t, rowb + static_cast<long long>(q) * C + 8 * j, v);
#pragma unroll
        for (int e = 0; e < 8; ++e) a[e] += v[e];
      }
#pragma unroll
      for (int e = 0; e < 8; ++e) feat[8 * j + e] = (a[e] + b[e]) * inv;
    }
  } else {
    const int G = kLk / C8;
    const int j = tid % C8, g = tid / C8;
    float a[8] = {0, 0, 0, 0, 0, 0, 0, 0}, b[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (g < G) {
      int q = g;
      for (; q + G < HW; q += 2 * G) {
        float v[8], w[8];
        ld_tap8(t, rowb + static_cast<long long>(q) * C + 8 * j, v);
        ld_tap8(t, rowb + static_cast<long long>(q + G) * C + 8 * j, w);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          a[e] += v[e];
          b[e] += w[e];
        }
      }
      if (q < HW) {
        float v[8];
        ld_tap8(t, rowb + static_cast<long long>(q) * C + 8 * j, v);
#pragma unroll
        for (int e = 0; e < 8; ++e) a[e] += v[e];
      }
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) red[tid * 8 + e] = a[e] + b[e];
    __syncthreads();
    if (tid < C8) {
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        float s = red[tid * 8 + e];
        for (int q = 1; q < G; ++q) s += red[(q * C8 + tid) * 8 + e];
        feat[8 * tid + e] = s * inv;
      }
    }
  }
  __syncthreads();
}

// Fused-GAP bins for heads that need them in global memory (classes > 32:
// the batched logits GEMM reads them): bins[r][c], one CTA per row.
constexpr int kGapBinsThreads = 1024;
__global__ void __launch_bounds__(kGapBinsThreads) gap_bins_kernel(const float* gap, int segs, int C, float inv,
                                                                   const int* data_idx, const int* count, float* bins) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ float feat_s[];
  __shared__ float4 red[kGapBinsThreads];
  const int r = blockIdx.x;
  if (r >= *count) return;
  const long long n = data_idx ? data_idx[r] : r;
  gap_feats_block<kGapBinsThreads>(gap + n * segs * C, segs, C, inv, feat_s, red);
  for (int c = threadIdx.x; c < C; c += kGapBinsThreads) bins[static_cast<long long>(r) * C + c] = feat_s[c];
}

// Generic: one thread per bin, sequential over its flat window.
__global__ void pool_generic_kernel(TapView t, int win, int width, float inv, float* bins) {
  pdl_wait();
  pdl_trigger();
  const int r = blockIdx.x;
  if (r >= *t.count) return;
  const long long n = t.data_idx ? t.data_idx[r] : r;
  for (int o = blockIdx.y * blockDim.x + threadIdx.x; o < width; o += gridDim.y * blockDim.x) {
    float s = 0.0f;
    for (long long f = static_cast<long long>(o) * win; f < static_cast<long long>(o + 1) * win; ++f) {
      const long long off = (f % t.HW) * t.C + f / t.HW;
      s += ld_tap(t, n * t.row_stride + off);
    }
    bins[static_cast<long long>(r) * width + o] = s * inv;
  }
}

// ------------------------------------------------------------------ conv1d
// Reference Conv(k,s) predictor (cache.cpp:126-131): y[o] = relu(b1 +
// sum_t w1[t] x[o*s+t]) over the flat tap, then logits = W2 y + b2. Each CTA
// stages a chunk of the flat tap (plus a k-1 halo) in shared memory and
// emits per-chunk partial logits (summed in a fixed order by the head).
__global__ void conv1d_partials_kernel(TapView t, long long D, int kernel, int stride, int out_dim, const float* w1,
                                       float b1, const float* W2, int classes, int chunk_elems, int nchunks,
                                       float* partials) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ float xs[];
  __shared__ float red[32];
  const int r = blockIdx.x;
  if (r >= *t.count) return;
  const long long n = t.data_idx ? t.data_idx[r] : r;
  const int chunk = blockIdx.y;
  const long long f0 = static_cast<long long>(chunk) * chunk_elems;
  const long long f1 = f0 + chunk_elems < D ? f0 + chunk_elems : D;
  const long long fe = f1 + kernel - 1 < D ? f1 + kernel - 1 : D;
  const long long len = fe - f0;
  const long long rowb = n * t.row_stride;
  if (t.HW == 1) {
    for (long long i = threadIdx.x; i < len; i += blockDim.x) xs[i] = ld_tap(t, rowb + f0 + i);
  } else {
    // chunk_elems is a whole number of channels: walk (pixel, channel) with
    // the channel fastest so consecutive threads read consecutive addresses.
    const long long c0 = f0 / t.HW;
    const long long cb = (f1 - f0 + t.HW - 1) / t.HW;
    const long long body = cb * t.HW;
    for (long long i = threadIdx.x; i < body; i += blockDim.x) {
      const long long cl = i % cb, p = i / cb;
      const long long f = (c0 + cl) * t.HW + p;
      if (f < f1) xs[f - f0] = ld_tap(t, rowb + p * t.C + c0 + cl);
    }
    for (long long f = f1 + threadIdx.x; f < fe; f += blockDim.x) {
      xs[f - f0] = ld_tap(t, rowb + (f % t.HW) * t.C + f / t.HW);
    }
  }
  __syncthreads();
  const long long ob = (f0 + stride - 1) / stride;
  long long oe = (f1 + stride - 1) / stride;
  if (oe > out_dim) oe = out_dim;
  for (int k0 = 0; k0 < classes; k0 += 16) {
    float acc[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) acc[k] = 0.0f;
    for (long long o = ob + threadIdx.x; o < oe; o += blockDim.x) {
      float y = b1;
      const long long xb = o * stride - f0;
      for (int tt = 0; tt < kernel; ++tt) y += w1[tt] * xs[xb + tt];
      y = y > 0.0f ? y : 0.0f;
#pragma unroll
      for (int k = 0; k < 16; ++k)
        if (k0 + k < classes) acc[k] += W2[static_cast<long long>(k0 + k) * out_dim + o] * y;
    }
    for (int k = 0; k < 16 && k0 + k < classes; ++k) {
      const float s = block_sum(acc[k], red);
      if (threadIdx.x == 0) partials[(static_cast<long long>(r) * nchunks + chunk) * classes + k0 + k] = s;
    }
  }
}

// ------------------------------------------------------------------ batched FC
// part[z][r][k] = sum_{o in K-slice z} A(r, o) * W[k][o] over the surviving
// rows: the reference FC (network.cpp:116-126) as a split-K batched GEMM; the
// consumer adds b[k] + sum_z part[z][r][k] in ascending z (fixed order). A is
// a dense fp32 [rows][feat] matrix (kMode 0) or the FC(h) cache hidden layer
// relu(b1[o] + sum_s partials[s][r][o]) (kMode 1, split-K partials of the
// tensor-core GEMM). CTA tile 32 rows x 128 classes x 32-deep K chunks staged
// in shared memory (k-major, so each thread's 4 rows and 4 classes are one
// 16-byte load each); 4 x 4 register micro-tile per thread. Every row tile
// reads its W slice once: the logits GEMM of heads with many classes.
constexpr int kFcBM = 32, kFcBN = 128, kFcBK = 32;

__host__ __device__ inline int rows_fc_slice(int feat) { return feat <= 512 ? 64 : (feat <= 1024 ? 128 : 256); }

// One K-chunk of the A and W tiles into registers: A row tid/8, W classes
// tid/8 + 32 i, 4 consecutive o at (tid % 8) * 4.
template <int kMode>
__device__ __forceinline__ void rows_fc_load(const float* __restrict__ A, long long lda, int ks, long long part_stride,
                                             const float* __restrict__ b1, int feat, const float* __restrict__ W,
                                             int classes, int n, int r0, int k0, int o0, int oz1, bool vec,
                                             float (&va)[4], float (&vw)[4][4]) {
  const int tid = threadIdx.x;
  const int oo = (tid & 7) * 4;
  {
    const int r = r0 + (tid >> 3);
#pragma unroll
    for (int e = 0; e < 4; ++e) va[e] = 0.0f;
    if (r < n) {
      if (vec && o0 + oo + 4 <= oz1) {
        if (kMode == 0) {
          const float4 f = __ldg(reinterpret_cast<const float4*>(A + static_cast<long long>(r) * lda + o0 + oo));
          va[0] = f.x, va[1] = f.y, va[2] = f.z, va[3] = f.w;
        } else {
          const float4 bb = __ldg(reinterpret_cast<const float4*>(b1 + o0 + oo));
          va[0] = bb.x, va[1] = bb.y, va[2] = bb.z, va[3] = bb.w;
          for (int s = 0; s < ks; ++s) {
            const float4 f = __ldg(reinterpret_cast<const float4*>(A + static_cast<long long>(s) * part_stride +
                                                                   static_cast<long long>(r) * lda + o0 + oo));
            va[0] += f.x, va[1] += f.y, va[2] += f.z, va[3] += f.w;
          }
#pragma unroll
          for (int e = 0; e < 4; ++e) va[e] = va[e] > 0.0f ? va[e] : 0.0f;
        }
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int o = o0 + oo + e;
          if (o < oz1) {
            if (kMode == 0) {
              va[e] = A[static_cast<long long>(r) * lda + o];
            } else {
              float a = b1[o];
              for (int s = 0; s < ks; ++s)
                a += A[static_cast<long long>(s) * part_stride + static_cast<long long>(r) * lda + o];
              va[e] = a > 0.0f ? a : 0.0f;
            }
          }
        }
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int k = k0 + (tid >> 3) + 32 * i;
#pragma unroll
    for (int e = 0; e < 4; ++e) vw[i][e] = 0.0f;
    if (k < classes) {
      if (vec && o0 + oo + 4 <= oz1) {
        const float4 f = __ldg(reinterpret_cast<const float4*>(W + static_cast<long long>(k) * feat + o0 + oo));
        vw[i][0] = f.x, vw[i][1] = f.y, vw[i][2] = f.z, vw[i][3] = f.w;
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (o0 + oo + e < oz1) vw[i][e] = W[static_cast<long long>(k) * feat + o0 + oo + e];
      }
    }
  }
}

template <int kMode>
__global__ void __launch_bounds__(256) rows_fc_kernel(const float* __restrict__ A, long long lda, int ks,
                                                      long long part_stride, const float* __restrict__ b1, int feat,
                                                      int kslice, const float* __restrict__ W, int classes,
                                                      const int* count, long long max_rows, float* out) {
  {
    // the weight slice this CTA multiplies does not depend on upstream
    // kernels: pull it into L2 while the producer of A drains (one row of W
    // per thread, 16-byte aligned rows only)
    const int k = blockIdx.x * kFcBN + static_cast<int>(threadIdx.x);
    const int oz0 = blockIdx.z * kslice, oz1 = oz0 + kslice < feat ? oz0 + kslice : feat;
    if (threadIdx.x < kFcBN && k < classes && (feat & 3) == 0 && oz1 > oz0)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(W + static_cast<long long>(k) * feat + oz0),
                   "r"(static_cast<unsigned>((oz1 - oz0) * 4))
                   : "memory");
  }
  pdl_wait();
  pdl_trigger();
  __shared__ __align__(16) float As[kFcBK][kFcBM + 4];
  __shared__ __align__(16) float Ws[kFcBK][kFcBN + 4];
  const int n = *count;
  const int r0 = blockIdx.y * kFcBM, k0 = blockIdx.x * kFcBN;
  if (r0 >= n) return;
  const int z = blockIdx.z;
  const int oz0 = z * kslice, oz1 = oz0 + kslice < feat ? oz0 + kslice : feat;
  const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5;
  const bool vec = (feat & 3) == 0 && (lda & 3) == 0;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0f;
  float va[4], vw[4][4];
  // register double buffering: chunk c+1 is in flight while chunk c is multiplied
  rows_fc_load<kMode>(A, lda, ks, part_stride, b1, feat, W, classes, n, r0, k0, oz0, oz1, vec, va, vw);
  for (int o0 = oz0; o0 < oz1; o0 += kFcBK) {
    {
      const int rr = tid >> 3, oo = (tid & 7) * 4;
#pragma unroll
      for (int e = 0; e < 4; ++e) As[oo + e][rr] = va[e];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int e = 0; e < 4; ++e) Ws[oo + e][rr + 32 * i] = vw[i][e];
    }
    __syncthreads();
    if (o0 + kFcBK < oz1)
      rows_fc_load<kMode>(A, lda, ks, part_stride, b1, feat, W, classes, n, r0, k0, o0 + kFcBK, oz1, vec, va, vw);
    const int olim = oz1 - o0 < kFcBK ? oz1 - o0 : kFcBK;
#pragma unroll 4
    for (int o = 0; o < olim; ++o) {
      const float4 a = *reinterpret_cast<const float4*>(&As[o][ty * 4]);
      const float4 w = *reinterpret_cast<const float4*>(&Ws[o][tx * 4]);
      const float av[4] = {a.x, a.y, a.z, a.w}, wv[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] += av[i] * wv[j];
    }
    __syncthreads();
  }
  float* outz = out + static_cast<long long>(z) * max_rows * classes;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = r0 + ty * 4 + i;
    if (r >= n) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int k = k0 + tx * 4 + j;
      if (k < classes) outz[static_cast<long long>(r) * classes + k] = acc[i][j];
    }
  }
}

__device__ __forceinline__ float fc_logit(const float* part, int nz, long long zstride, const float* b, int r,
                                          int classes, int k) {
  float a = b[k];
#pragma unroll 8  // loads of 8 slices in flight; adds stay in ascending z
  for (int z = 0; z < nz; ++z) a += __ldg(part + z * zstride + static_cast<long long>(r) * classes + k);
  return a;
}

// Global average pool of the surviving images' final activations (NHWC,
// image ids[r]) -> feats [rows][C] (the base head's GAP), one CTA per row.
__global__ void __launch_bounds__(kLk) gap_rows_kernel(const __nv_bfloat16* hi, const __nv_bfloat16* lo, int C, int HW,
                                                       const int* ids, const int* count, float* feats) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ float feat_s[];
  __shared__ float red[kLk * 8];
  const int r = blockIdx.x;
  if (r >= *count) return;
  TapView t;
  t.hi = hi;
  t.lo = lo;
  tap_gap_block(t, static_cast<long long>(ids[r]) * HW * C, C, HW, feat_s, red);
  for (int c = threadIdx.x; c < C; c += kLk) feats[static_cast<long long>(r) * C + c] = feat_s[c];
}

// logits[k] = b[k] + W[k] . feat for k < classes: warp per class, lanes
// strided over the features (4 independent chains), fixed combination order.
template <bool kSmemW = false>
__device__ void block_logits(const float* __restrict__ W, const float* __restrict__ b, int classes, int nf,
                             const float* feat, float* logits) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int k = warp; k < classes; k += kLk / 32) {
    const float* wr = W + static_cast<long long>(k) * nf;
    float a0 = 0.0f, a1 = 0.0f, a2 = 0.0f, a3 = 0.0f;
    int o = lane;
#pragma unroll 4
    for (; o + 96 < nf; o += 128) {
      a0 += (kSmemW ? wr[o] : __ldg(wr + o)) * feat[o];
      a1 += (kSmemW ? wr[o + 32] : __ldg(wr + o + 32)) * feat[o + 32];
      a2 += (kSmemW ? wr[o + 64] : __ldg(wr + o + 64)) * feat[o + 64];
      a3 += (kSmemW ? wr[o + 96] : __ldg(wr + o + 96)) * feat[o + 96];
    }
    for (; o < nf; o += 32) a0 += (kSmemW ? wr[o] : __ldg(wr + o)) * feat[o];
    const float a = warp_sum((a0 + a1) + (a2 + a3));
    if (lane == 0) logits[k] = a + b[k];
  }
}

// Fused-GAP and direct-row heads stage W2 + Ws1 in shared memory when they
// fit (48 KB). Heads that do not stage W2 still stage the selector's first
// layer (16 x C) before the wait when it fits (<= 64 KB): one L2 round trip
// off the tail.
__host__ __device__ inline bool head_stages_ws1(const CacheHeadParams& p);
#ifndef LCB_FC_NO_STAGE
#define LCB_FC_NO_STAGE 0
#endif
// columns of W2 [classes][cols]: the Conv(k,s) head of a direct row reads its own conv outputs
__host__ __device__ inline int head_w2_cols(const CacheHeadParams& p) {
  return (p.row_hi && p.family == 2) ? p.out_dim : p.feat;
}
__host__ __device__ inline bool head_stages_weights(const CacheHeadParams& p) {
  // (FC(h) heads: batch-sized launches only, whose copy overlaps the hidden-layer GEMM)
  return (p.gap != nullptr || p.row_hi != nullptr || (p.family == 0 && p.rows_total >= 32 && !LCB_FC_NO_STAGE)) &&
         !p.pre_logits && p.classes * (head_w2_cols(p) + 16) <= 12288;
}
// floats of the head's feature region (after the logits): direct rows hold
// [features][row] there; launch_cache_head sizes the same extent
__host__ __device__ inline int head_feat_len(const CacheHeadParams& p) {
  if (p.row_hi) {
    const int nf = head_w2_cols(p);
    return (nf > p.classes ? nf : p.classes) + p.D;
  }
  return (p.family == 2 || p.pre_logits) ? p.classes : (p.feat > p.classes ? p.feat : p.classes);
}
__host__ __device__ inline bool head_stages_ws1(const CacheHeadParams& p) {
  // batch-sized launches only: with a handful of rows the copy is not hidden
  // behind the upstream kernel and the selector reads L2 directly anyway.
  // rows_total is the engine's capacity (max_batch), fixed when the graph is
  // captured — not the live count: an engine built for >= 32 rows stages even
  // when it serves one request (the batch-1 saving needs max_batch < 32)
  return !head_stages_weights(p) && p.classes <= 1024 && p.rows_total >= 32 && !p.row_hi;
}

// Shared scratch of one row's head.
struct HeadSmem {
  float bv[32];
  int bi[32];
  float part[32 * 17];  // per warp: 16 selector sums + the softmax denominator
  float S;
};

// softmax(logits) (losses.cpp:35-46), selector FC(C,16)+ReLU+FC(16,1),
// branch-stable sigmoid (losses.cpp:26-33), inclusive p >= delta
// (cache.cpp:259-265), argmax(pr) with the lowest index on ties
// (tensor.hpp:57-63). logits complete in shared memory.
// ws1: the selector's first layer [16][classes] (shared-memory copy or p.Ws1).
// Two passes over the classes: (1) max and argmax of the logits (softmax is
// monotonic: argmax(pr) = argmax(logits), lowest index on ties); (2) e_k =
// exp(l_k - max), S = sum e_k and the 16 selector sums sum_k Ws1[j][k] e_k in
// one sweep, since sum_k Ws1[j][k] pr_k = (sum_k Ws1[j][k] e_k) / S. Two block
// reductions instead of one per softmax/selector step.
__device__ void head_block(const CacheHeadParams& p, int r, const float* logits, float* /*pr scratch*/, HeadSmem& hs,
                           const float* ws1, const float* bs1, const float* ws2) {
  const int C = p.classes;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = kLk / 32;
  float bv = -FLT_MAX;
  int bi = 0x7fffffff;
  for (int k = tid; k < C; k += kLk)
    if (logits[k] > bv) {  // ascending k: the lowest index wins within the thread
      bv = logits[k];
      bi = k;
    }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > bv || (ov == bv && oi < bi)) {
      bv = ov;
      bi = oi;
    }
  }
  if (lane == 0) {
    hs.bv[warp] = bv;
    hs.bi[warp] = bi;
  }
  __syncthreads();
  float m = hs.bv[0];
  int arg = hs.bi[0];
  for (int w = 1; w < nw; ++w)
    if (hs.bv[w] > m || (hs.bv[w] == m && hs.bi[w] < arg)) {
      m = hs.bv[w];
      arg = hs.bi[w];
    }
  float acc[17];
#pragma unroll
  for (int j = 0; j < 17; ++j) acc[j] = 0.0f;
  for (int k = tid; k < C; k += kLk) {
    const float e = expf(logits[k] - m);
    acc[16] += e;
#pragma unroll
    for (int j = 0; j < 16; ++j) acc[j] += ws1[j * C + k] * e;
  }
#pragma unroll
  for (int j = 0; j < 17; ++j) acc[j] = warp_sum(acc[j]);
  if (lane < 17) {
    float v = acc[0];
#pragma unroll
    for (int j = 1; j < 17; ++j) v = lane == j ? acc[j] : v;
    hs.part[warp * 17 + lane] = v;
  }
  __syncthreads();
  if (warp == 0) {
    // lane j < 17: the warps' partials of sum j in ascending warp order
    float t = 0.0f;
    if (lane < 17)
      for (int w = 0; w < nw; ++w) t += hs.part[w * 17 + lane];
    const float S = __shfl_sync(0xffffffffu, t, 16);
    float h = 0.0f;
    if (lane < 16) {
      const float a = t / S + bs1[lane];
      h = (a > 0.0f ? a : 0.0f) * ws2[lane];
    }
    // z = bs2 + sum_j ws2[j] * relu(hidden_j), j ascending
    float hj[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) hj[j] = __shfl_sync(0xffffffffu, h, j);
    if (lane == 0) {
      float z = p.bs2;
#pragma unroll
      for (int j = 0; j < 16; ++j) z += hj[j];
      float q;
      if (z >= 0.0f) {
        q = 1.0f / (1.0f + expf(-z));
      } else {
        const float e = expf(z);
        q = e / (1.0f + e);
      }
      p.prob[r] = q;
      p.hit[r] = static_cast<double>(q) >= p.delta ? 1 : 0;
      p.label[r] = arg;
      hs.S = S;
    }
  }
  if (p.pr_out) {
    __syncthreads();
    const float S = hs.S;
    for (int k = tid; k < C; k += kLk) p.pr_out[static_cast<long long>(r) * C + k] = expf(logits[k] - m) / S;
  }
  if (p.logits_out)
    for (int k = tid; k < C; k += kLk) p.logits_out[static_cast<long long>(r) * C + k] = logits[k];
}

// Arrival of every CTA of a head launch; the LAST one records first hits and
// compacts the surviving rows in order (warp ballot + block prefix sum):
// exit_compact of serve_one (serving.cpp:112-121) without its own launch.
__device__ void exit_tail(const ExitParams& e, int n, const float* prob, const int* hit, const int* label) {
  __shared__ int last_s, base_s;
  __shared__ int warp_tot[32];
  __syncthreads();  // the CTA's head results before its (acq_rel) arrival
  if (threadIdx.x == 0) last_s = (atom_add_acq_rel_gpu(e.arrive, 1) == static_cast<int>(gridDim.x) - 1) ? 1 : 0;
  __syncthreads();
  if (!last_s) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  if (tid == 0) {
    base_s = 0;
    *e.arrive = 0;
  }
  __syncthreads();
  const unsigned long long now = globaltimer();
  for (int c0 = 0; c0 < n; c0 += blockDim.x) {
    const int r = c0 + tid;
    const bool valid = r < n;
    const bool h = valid && __ldcg(hit + r);
    const int id = valid ? e.ids_in[r] : -1;
    if (valid) {
      if (e.probs_out) e.probs_out[id] = __ldcg(prob + r);
      if (e.labels_out) e.labels_out[id] = __ldcg(label + r);
      if (h && e.exit_layer[id] == 0) {
        e.exit_layer[id] = e.layer;
        e.served[id] = __ldcg(label + r);
        e.exit_ns[id] = now;
      }
    }
    const bool keep = valid && (e.shadow || !h);
    const unsigned mask = __ballot_sync(0xffffffffu, keep);
    const int pos_in_warp = __popc(mask & ((1u << lane) - 1u));
    if (lane == 0) warp_tot[warp] = __popc(mask);
    __syncthreads();
    if (warp == 0) {
      int v = lane < nw ? warp_tot[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += u;
      }
      if (lane < nw) warp_tot[lane] = v;  // inclusive prefix
    }
    __syncthreads();
    const int pos = base_s + (warp == 0 ? 0 : warp_tot[warp - 1]) + pos_in_warp;
    if (keep) {
      e.ids_out[pos] = id;
      if (e.src_rows_out) e.src_rows_out[pos] = r;
    }
    __syncthreads();
    if (tid == 0) base_s += warp_tot[nw - 1];
    __syncthreads();
  }
  if (tid == 0) *e.count_out = base_s;
}

// First-hit exit of row r by its own CTA (serve_one, serving.cpp:112-121) with
// atomic-position compaction of the row-compacted activations (ExitParams::
// rows_dst_hi): a miss is appended to ids_out and its activation row copied.
// use_held: the row's 16-byte vectors already in registers (held), thread t <
// nv the hi plane's vector t, nv <= t < 2 nv the lo plane's vector t - nv (the
// copy is then stores only: no second read of the row after the atomic).
__device__ void row_exit_append(const ExitParams& e, int n, int r, const float* prob, const int* hit,
                                const int* label, bool use_held = false, uint4 held = uint4{}, int nv_held = 0) {
  __shared__ int pos_s;
  __syncthreads();  // the row's head results (written by thread 0)
  if (r >= n) return;
  if (threadIdx.x == 0) {
    const int id = e.ids_in[r];
    const bool h = hit[r] != 0;
    const int lab = label[r];
    if (e.probs_out) e.probs_out[id] = prob[r];
    if (e.labels_out) e.labels_out[id] = lab;
    int pos = -1;
    if (h) {
      if (e.exit_layer[id] == 0) {
        e.exit_layer[id] = e.layer;
        e.served[id] = lab;
        e.exit_ns[id] = globaltimer();
      }
    } else {
      pos = atomicAdd(e.count_out, 1);
      e.ids_out[pos] = id;
      if (e.src_rows_out) e.src_rows_out[pos] = r;
    }
    pos_s = pos;
  }
  __syncthreads();
  const int pos = pos_s;
  if (pos < 0) return;
  if (use_held) {
    const int t = threadIdx.x;
    if (t < nv_held)
      reinterpret_cast<uint4*>(e.rows_dst_hi + static_cast<long long>(pos) * e.row_elems)[t] = held;
    else if (e.rows_src_lo && t < 2 * nv_held)
      reinterpret_cast<uint4*>(e.rows_dst_lo + static_cast<long long>(pos) * e.row_elems)[t - nv_held] = held;
    return;
  }
  const long long nv = e.row_elems / 8;  // 16-byte vectors per plane row
  const uint4* sh = reinterpret_cast<const uint4*>(e.rows_src_hi + static_cast<long long>(r) * e.row_elems);
  uint4* dh = reinterpret_cast<uint4*>(e.rows_dst_hi + static_cast<long long>(pos) * e.row_elems);
  for (long long i = threadIdx.x; i < nv; i += blockDim.x) dh[i] = __ldg(sh + i);
  if (e.rows_src_lo) {
    const uint4* sl = reinterpret_cast<const uint4*>(e.rows_src_lo + static_cast<long long>(r) * e.row_elems);
    uint4* dl = reinterpret_cast<uint4*>(e.rows_dst_lo + static_cast<long long>(pos) * e.row_elems);
    for (long long i = threadIdx.x; i < nv; i += blockDim.x) dl[i] = __ldg(sl + i);
  }
}

// ------------------------------------------------------------------ head
// Reference lookup (cache.cpp:259-265): pr = softmax(pred(tap)),
// p = sigmoid(sel(pr)), hit = p >= delta (inclusive); label = argmax(pr).
// One CTA per row. Logits come from (in order of precedence) the batched
// split-K GEMM partials, the fused GAP partials (Pool(C), classes <= 32),
// the Conv(k,s) chunk partials, or the pooled bins / FC(h) hidden partials.
// With p.ex.arrive the last CTA also runs the exit + compaction.
// Global -> shared copy of n floats by one kLk-thread CTA: 16-byte loads, 4 in
// flight per thread (a scalar loop is a chain of L2 round trips when the copy
// lands on the critical path, e.g. batch-1 serving).
__device__ __forceinline__ void stage_floats(float* dst, const float* __restrict__ src, int n, int tid) {
  const int n4 = (reinterpret_cast<uintptr_t>(src) & 15) == 0 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0 ? n / 4 : 0;
  const float4* s4 = reinterpret_cast<const float4*>(src);
  float4* d4 = reinterpret_cast<float4*>(dst);
#pragma unroll 4
  for (int i = tid; i < n4; i += kLk) d4[i] = __ldg(s4 + i);
  for (int i = 4 * n4 + tid; i < n; i += kLk) dst[i] = __ldg(src + i);
}

__global__ void __launch_bounds__(kLk) cache_head_kernel(CacheHeadParams p) {
  extern __shared__ float sm[];
  __shared__ HeadSmem hs;
  __shared__ float4 red4[kLk];
  __shared__ float sel_s[32];  // selector: bs1[16], ws2[16]
  const int r = blockIdx.x;
  const int C = p.classes;
  float* logits = sm;    // [C]
  float* feat = sm + C;  // [head_feat_len]
  const int tid = threadIdx.x;
  // fused-GAP and direct-row heads (<= 32 classes): the static head weights
  // are staged in shared memory BEFORE the programmatic-launch wait, i.e.
  // while the tap's producer is still draining (launch_cache_head sizes the region)
  const bool stage_w = head_stages_weights(p);
  const int w2c = head_w2_cols(p);
  float* w2s = feat + head_feat_len(p);             // [C][w2c]
  const bool stage_s = head_stages_ws1(p);
  float* ws1s = stage_w ? w2s + C * w2c : w2s;  // [16][C]
  if (stage_w) stage_floats(w2s, p.W2, C * w2c, tid);
  if (stage_w || stage_s) stage_floats(ws1s, p.Ws1, 16 * C, tid);
  if (p.row_hi) {  // (direct rows: the whole head reads shared memory after the wait)
    if (tid < 16) sel_s[tid] = __ldg(p.bs1 + tid);
    else if (tid < 32) sel_s[tid] = __ldg(p.ws2 + tid - 16);
  }
  // direct rows in 16-byte vectors (thread t < nv: hi vector t; nv <= t < 2 nv:
  // lo vector t - nv), kept in registers for the row append's copy
  const int nv = p.D / 8;
  const bool rvec = p.row_hi && (p.D & 7) == 0 && (p.row_stride & 7) == 0 &&
                    (reinterpret_cast<uintptr_t>(p.row_hi) & 15) == 0 &&
                    (reinterpret_cast<uintptr_t>(p.row_lo) & 15) == 0 && 2 * nv <= kLk;
  pdl_wait();
  pdl_trigger();
  uint4 held = make_uint4(0u, 0u, 0u, 0u);
  if (rvec) {  // issued with the count's load (rows up to max_rows are allocated; r >= n is discarded)
    const long long rb = static_cast<long long>(r) * p.row_stride;
    if (tid < nv)
      held = __ldg(reinterpret_cast<const uint4*>(p.row_hi + rb) + tid);
    else if (p.row_lo && tid < 2 * nv)
      held = __ldg(reinterpret_cast<const uint4*>(p.row_lo + rb) + tid - nv);
  }
  const int n = *p.count;
  if (r < n && p.row_hi) {
    // direct row mode: x = the request's row; Pool(w) bins (AvgPool over flat
    // windows times 1/w, network.cpp:130-138) or Conv(k,s) + ReLU
    // (network.cpp:127-148) into feat, then the FC(.,C) logits
    float* x = feat + (p.family == 2 ? p.out_dim : p.feat);  // [D]
    if (rvec) {
      // x = hi + lo (the lo plane parked in red4 first)
      float* lo_s = reinterpret_cast<float*>(red4);
      // bf16 -> fp32 is the 16-bit pattern shifted up (no address taken: held stays in registers)
      const uint32_t hw[4] = {held.x, held.y, held.z, held.w};
      float* dst = tid < nv ? x + 8 * tid : lo_s + 8 * (tid - nv);
      if (tid < nv || (p.row_lo && tid < 2 * nv)) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          dst[2 * e] = __uint_as_float(hw[e] << 16);
          dst[2 * e + 1] = __uint_as_float(hw[e] & 0xffff0000u);
        }
      }
      if (p.row_lo) {
        __syncthreads();
        for (int i = tid; i < p.D; i += kLk) x[i] += lo_s[i];
      }
    } else {
      const long long rb = static_cast<long long>(r) * p.row_stride;
      for (int i = tid; i < p.D; i += kLk) {
        float v = __bfloat162float(p.row_hi[rb + i]);
        if (p.row_lo) v += __bfloat162float(p.row_lo[rb + i]);
        x[i] = v;
      }
    }
    __syncthreads();
    int nf;
    if (p.family == 1) {
      nf = p.feat;
      for (int o = tid; o < nf; o += kLk) {
        float a = 0.0f;
        for (int t = 0; t < p.win; ++t) a += x[o * p.win + t];
        feat[o] = a * p.pool_inv;
      }
    } else {
      nf = p.out_dim;
      for (int o = tid; o < nf; o += kLk) {
        float y = p.b1c;
        for (int t = 0; t < p.kernel; ++t) y += __ldg(p.w1 + t) * x[o * p.stride + t];
        feat[o] = y > 0.0f ? y : 0.0f;
      }
    }
    __syncthreads();
    if (stage_w)
      block_logits<true>(w2s, p.b2, C, nf, feat, logits);
    else
      block_logits(p.W2, p.b2, C, nf, feat, logits);
    __syncthreads();
    head_block(p, r, logits, feat, hs, stage_w ? ws1s : p.Ws1, sel_s, sel_s + 16);
  } else if (r < n) {
    if (p.pre_logits) {
      for (int k = tid; k < C; k += kLk) logits[k] = fc_logit(p.pre_logits, p.pre_nz, p.pre_zstride, p.b2, r, C, k);
    } else if (p.family == 2) {
      for (int k = tid; k < C; k += kLk) {
        float a = p.b2[k];
        const float* q = p.feats + static_cast<long long>(r) * p.feat * C + k;
#pragma unroll 4
        for (int c = 0; c < p.feat; ++c) a += __ldg(q + static_cast<long long>(c) * C);
        logits[k] = a;
      }
    } else {
      if (p.gap) {
        const long long img = p.gap_ids ? p.gap_ids[r] : r;
        gap_feats_block(p.gap + img * p.gap_segs * p.feat, p.gap_segs, p.feat, p.gap_inv, feat, red4);
      } else if (p.family == 1) {
        for (int o = tid; o < p.feat; o += kLk) feat[o] = __ldg(p.feats + static_cast<long long>(r) * p.feat + o);
      } else {
        // hidden = relu(b1 + sum of the split-K partials, ascending split):
        // 8 splits' loads issued before the adds (a runtime-bounded loop
        // would wait on each load in turn)
        for (int j = tid; j < p.feat; j += kLk) {
          float a = p.b1[j];
          for (int s0 = 0; s0 < p.ks; s0 += 8) {
            float t[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              const int sp = s0 + u < p.ks ? s0 + u : p.ks - 1;
              t[u] = __ldg(p.feats + (static_cast<long long>(sp) * p.rows_total + r) * p.hp + j);
            }
#pragma unroll
            for (int u = 0; u < 8; ++u)
              if (s0 + u < p.ks) a += t[u];
          }
          feat[j] = a > 0.0f ? a : 0.0f;
        }
      }
      __syncthreads();
      if (stage_w)
        block_logits<true>(w2s, p.b2, C, p.feat, feat, logits);
      else
        block_logits(p.W2, p.b2, C, p.feat, feat, logits);
    }
    __syncthreads();
    head_block(p, r, logits, feat, hs, (stage_w || stage_s) ? ws1s : p.Ws1, p.bs1, p.ws2);
  }
  if (p.ex.arrive) {
    if (p.ex.rows_dst_hi && !p.ex.shadow) {
      // the held vectors are the whole row to copy when the tap is the compacted row itself
      const bool use_held = rvec && p.ex.rows_src_hi == p.row_hi && p.ex.rows_src_lo == p.row_lo &&
                            p.ex.row_elems == p.D && p.row_stride == p.ex.row_elems;
      row_exit_append(p.ex, n, r, p.prob, p.hit, p.label, use_held, held, nv);
    } else {
      exit_tail(p.ex, n, p.prob, p.hit, p.label);
    }
  }
}

// ------------------------------------------------------- warp-per-row head
// The same lookup (cache.cpp:259-265) for heads with <= 32 classes whose
// features come from the request's own row (block-MLP Pool(w) / Conv(k,s)),
// from FC(h) split-K partials or from pooled bins: one WARP per row, 8 rows
// per CTA, no block barriers after the staging. W2 is staged transposed
// ([feature][class]) so lane k accumulates class k from shared memory
// without bank conflicts; softmax, argmax (lowest index on ties), the
// selector FC(C,16)+ReLU+FC(16,1) and the branch-stable sigmoid are warp
// reductions. The block-per-row kernel above costs a 512-thread CTA per row:
// latency-bound at a few hundred rows and ~50x slower per row at 16K rows.
constexpr int kWhWarps = 8;

__host__ __device__ inline int warp_head_nf(const CacheHeadParams& p) {
  return (p.row_hi && p.family == 2) ? p.out_dim : p.feat;
}
__host__ __device__ inline int warp_head_dx(const CacheHeadParams& p) { return p.row_hi ? ((p.D + 3) & ~3) : 0; }
// floats of shared memory: W2 [C][nf + 1] (odd row pitch: lane k reading
// W2[k][o] hits bank (k (nf + 1) + o) mod 32, distinct over the classes),
// Ws1 [16][C], bs1|ws2 [32], b2 [32], per warp x [dx] + feat [nf]
__host__ __device__ inline size_t warp_head_smem_floats(const CacheHeadParams& p) {
  const size_t nf = static_cast<size_t>(warp_head_nf(p)), C = static_cast<size_t>(p.classes);
  return (nf + 1) * C + 16 * C + 64 + static_cast<size_t>(kWhWarps) * (static_cast<size_t>(warp_head_dx(p)) + nf);
}

__global__ void __launch_bounds__(kWhWarps * 32) warp_head_kernel(CacheHeadParams p) {
  extern __shared__ __align__(16) float whs[];
  const int C = p.classes, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool direct = p.row_hi != nullptr;
  const int nf = warp_head_nf(p), dx = warp_head_dx(p);
  const int pw = nf + 1;       // W2 row pitch in shared memory
  float* w2s = whs;            // [C][nf + 1]
  float* ws1 = w2s + pw * C;   // [16][C]
  float* sel = ws1 + 16 * C;   // bs1[16], ws2[16]
  float* b2s = sel + 32;       // [C]
  float* x = b2s + 32 + warp * (dx + nf);  // this warp's row [dx]
  float* feat = x + dx;                    // and features [nf]
  // static head weights, before the programmatic-launch wait
  // 16-byte loads of W2's rows, 4 per thread in flight per round (W2 rows are
  // 16-byte aligned when nf % 4 == 0), scattered into the padded rows
  if ((nf & 3) == 0 && (reinterpret_cast<uintptr_t>(p.W2) & 15) == 0) {
    const int n4 = nf * C / 4;
    for (int b0 = 0; b0 < n4; b0 += 4 * kWhWarps * 32) {
      float4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i4 = b0 + u * kWhWarps * 32 + tid;
        v[u] = i4 < n4 ? __ldg(reinterpret_cast<const float4*>(p.W2) + i4) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i4 = b0 + u * kWhWarps * 32 + tid;
        if (i4 < n4) {
          const int k = (4 * i4) / nf, o = 4 * i4 - k * nf;
          float* d = w2s + k * pw + o;
          d[0] = v[u].x;
          d[1] = v[u].y;
          d[2] = v[u].z;
          d[3] = v[u].w;
        }
      }
    }
  } else {
    for (int i = tid; i < nf * C; i += blockDim.x) {
      const int k = i / nf, o = i - k * nf;
      w2s[k * pw + o] = __ldg(p.W2 + i);
    }
  }
  for (int i = tid; i < 16 * C; i += blockDim.x) ws1[i] = __ldg(p.Ws1 + i);
  if (tid < 16)
    sel[tid] = __ldg(p.bs1 + tid);
  else if (tid < 32)
    sel[tid] = __ldg(p.ws2 + tid - 16);
  else if (tid < 32 + C)
    b2s[tid - 32] = __ldg(p.b2 + tid - 32);
  pdl_wait();
  pdl_trigger();
  const int n = *p.count;
  __syncthreads();
  const int r = blockIdx.x * kWhWarps + warp;
  // direct rows as 16-byte vectors (lane j holds vectors j, j + 32, ...), kept for the row append's copy
  const int nv = direct ? p.D / 8 : 0;
  const bool rvec = direct && (p.D & 7) == 0 && (p.row_stride & 7) == 0 &&
                    (reinterpret_cast<uintptr_t>(p.row_hi) & 15) == 0 &&
                    (reinterpret_cast<uintptr_t>(p.row_lo) & 15) == 0 && nv <= 32 * 4;
  uint4 hv[4], lv[4];
  float q = 0.0f;
  int hit = 0, am = 0;
  if (r < n) {
    if (direct) {
      const long long rb = static_cast<long long>(r) * p.row_stride;
      if (rvec) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int vi = lane + 32 * j;
          hv[j] = lv[j] = make_uint4(0u, 0u, 0u, 0u);
          if (vi < nv) {
            hv[j] = __ldg(reinterpret_cast<const uint4*>(p.row_hi + rb) + vi);
            if (p.row_lo) lv[j] = __ldg(reinterpret_cast<const uint4*>(p.row_lo + rb) + vi);
          }
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int vi = lane + 32 * j;
          if (vi < nv) {
            const uint32_t hw[4] = {hv[j].x, hv[j].y, hv[j].z, hv[j].w};
            const uint32_t lw[4] = {lv[j].x, lv[j].y, lv[j].z, lv[j].w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              // bf16 -> fp32: the pattern shifted up; x = hi + lo as the reference-width value
              float a = __uint_as_float(hw[e] << 16), b = __uint_as_float(hw[e] & 0xffff0000u);
              if (p.row_lo) {
                a += __uint_as_float(lw[e] << 16);
                b += __uint_as_float(lw[e] & 0xffff0000u);
              }
              x[8 * vi + 2 * e] = a;
              x[8 * vi + 2 * e + 1] = b;
            }
          }
        }
      } else {
        for (int i = lane; i < p.D; i += 32) {
          float v = __bfloat162float(p.row_hi[rb + i]);
          if (p.row_lo) v += __bfloat162float(p.row_lo[rb + i]);
          x[i] = v;
        }
      }
      __syncwarp();
      if (p.family == 1) {  // Pool(w): AvgPool over flat windows times 1/w (network.cpp:130-138)
        for (int o = lane; o < nf; o += 32) {
          float a = 0.0f;
          for (int t = 0; t < p.win; ++t) a += x[o * p.win + t];
          feat[o] = a * p.pool_inv;
        }
      } else {  // Conv(k,s) + ReLU (network.cpp:127-148)
        for (int o = lane; o < nf; o += 32) {
          float y = p.b1c;
          for (int t = 0; t < p.kernel; ++t) y += __ldg(p.w1 + t) * x[o * p.stride + t];
          feat[o] = y > 0.0f ? y : 0.0f;
        }
      }
    } else if (p.gap) {  // Pool(C) = GAP from the conv's fused partials gap[image][segs][C], C % 4 == 0
      const long long img = p.gap_ids ? p.gap_ids[r] : r;
      const float4* s4 = reinterpret_cast<const float4*>(p.gap + img * p.gap_segs * nf);
      const int C4 = nf >> 2;
      for (int j = lane; j < C4; j += 32) {
        float4 a0 = make_float4(0.f, 0.f, 0.f, 0.f), a1 = a0, a2 = a0, a3 = a0;
        int sg = 0;
        for (; sg + 4 <= p.gap_segs; sg += 4) {
          add4(a0, __ldg(s4 + static_cast<long long>(sg) * C4 + j));
          add4(a1, __ldg(s4 + static_cast<long long>(sg + 1) * C4 + j));
          add4(a2, __ldg(s4 + static_cast<long long>(sg + 2) * C4 + j));
          add4(a3, __ldg(s4 + static_cast<long long>(sg + 3) * C4 + j));
        }
        for (; sg < p.gap_segs; ++sg) add4(a0, __ldg(s4 + static_cast<long long>(sg) * C4 + j));
        add4(a0, a1);
        add4(a2, a3);
        add4(a0, a2);
        feat[4 * j] = a0.x * p.gap_inv;
        feat[4 * j + 1] = a0.y * p.gap_inv;
        feat[4 * j + 2] = a0.z * p.gap_inv;
        feat[4 * j + 3] = a0.w * p.gap_inv;
      }
    } else if (p.family == 1) {  // pooled bins [rows][feat]
      for (int o = lane; o < nf; o += 32) feat[o] = __ldg(p.feats + static_cast<long long>(r) * nf + o);
    } else {  // FC(h): hidden = relu(b1 + sum of the split-K partials, ascending split)
      // 4 hidden units per lane x 4 splits per round: 16 loads in flight
      for (int j0 = lane; j0 < nf; j0 += 4 * 32) {
        float a[4];
#pragma unroll
        for (int v = 0; v < 4; ++v) a[v] = j0 + 32 * v < nf ? p.b1[j0 + 32 * v] : 0.0f;
        for (int s0 = 0; s0 < p.ks; s0 += 4) {
          float t[4][4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int sp = s0 + u < p.ks ? s0 + u : p.ks - 1;
            const float* src = p.feats + (static_cast<long long>(sp) * p.rows_total + r) * p.hp;
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              const int j = j0 + 32 * v < nf ? j0 + 32 * v : j0;
              t[u][v] = __ldg(src + j);
            }
          }
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (s0 + u < p.ks) {
#pragma unroll
              for (int v = 0; v < 4; ++v) a[v] += t[u][v];
            }
        }
#pragma unroll
        for (int v = 0; v < 4; ++v)
          if (j0 + 32 * v < nf) feat[j0 + 32 * v] = a[v] > 0.0f ? a[v] : 0.0f;
      }
    }
    __syncwarp();
    // logits: lane = (class k, slice g), G = 32 / C slices of the features
    // (every lane busy for C <= 16), 2 chains per lane; the slices' sums are
    // gathered into lane k in ascending g (fixed order)
    float l = -FLT_MAX;
    {
      const int G = 32 / C;
      const int k = lane % C, g = lane / C;
      float a0 = 0.0f, a1 = 0.0f;
      if (g < G) {
        const int o0 = (nf * g) / G, o1 = (nf * (g + 1)) / G;
        const float* wr = w2s + k * pw;
        int o = o0;
        for (; o + 1 < o1; o += 2) {
          a0 += wr[o] * feat[o];
          a1 += wr[o + 1] * feat[o + 1];
        }
        if (o < o1) a0 += wr[o] * feat[o];
      }
      float part = a0 + a1;
      float sum = part;
      for (int gg = 1; gg < G; ++gg) sum += __shfl_sync(0xffffffffu, part, lane + gg * C < 32 ? lane + gg * C : lane);
      if (lane < C) l = sum + b2s[lane];
    }
    // argmax(pr) = argmax(logits), lowest index on ties (tensor.hpp:57-63)
    float m = l;
    am = lane < C ? lane : 0x7fffffff;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, m, o);
      const int oa = __shfl_xor_sync(0xffffffffu, am, o);
      if (ov > m || (ov == m && oa < am)) {
        m = ov;
        am = oa;
      }
    }
    // softmax (losses.cpp:35-46) and the selector: sum_k Ws1[j][k] pr_k = (sum_k Ws1[j][k] e_k) / S
    const float e = lane < C ? expf(l - m) : 0.0f;
    const float S = warp_sum(e);
    float t = 0.0f;
    for (int k = 0; k < C; ++k) {
      const float ek = __shfl_sync(0xffffffffu, e, k);
      if (lane < 16) t += ws1[lane * C + k] * ek;
    }
    float h = 0.0f;
    if (lane < 16) {
      const float a = t / S + sel[lane];
      h = (a > 0.0f ? a : 0.0f) * sel[16 + lane];
    }
    float hj[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) hj[j] = __shfl_sync(0xffffffffu, h, j);
    if (lane == 0) {
      float z = p.bs2;
#pragma unroll
      for (int j = 0; j < 16; ++j) z += hj[j];
      if (z >= 0.0f) {  // branch-stable sigmoid (losses.cpp:26-33)
        q = 1.0f / (1.0f + expf(-z));
      } else {
        const float ez = expf(z);
        q = ez / (1.0f + ez);
      }
      hit = static_cast<double>(q) >= p.delta ? 1 : 0;  // inclusive threshold
      p.prob[r] = q;
      p.hit[r] = hit;
      p.label[r] = am;
    }
    if (p.pr_out && lane < C) p.pr_out[static_cast<long long>(r) * C + lane] = e / S;
    if (p.logits_out && lane < C) p.logits_out[static_cast<long long>(r) * C + lane] = l;
  }
  if (!p.ex.arrive) return;
  const ExitParams& ex = p.ex;
  if (!ex.rows_dst_hi && ex.scan_agg && !ex.unordered && !ex.shadow && gridDim.x <= kScanMaxCtas) {
    // ordered compaction in one pass: this CTA's rows are positions
    // [prefix, prefix + misses) where prefix = the misses of CTAs 0..b-1
    // (all co-resident: the grid is at most 2 CTAs per SM)
    __shared__ int miss_s[kWhWarps], red_s[kWhWarps], tot_s;
    const bool miss = r < n && !__shfl_sync(0xffffffffu, hit, 0);
    int id = 0;
    if (lane == 0) {
      if (r < n) {
        id = ex.ids_in[r];
        if (ex.probs_out) ex.probs_out[id] = q;
        if (ex.labels_out) ex.labels_out[id] = am;
        if (hit && ex.exit_layer[id] == 0) {
          ex.exit_layer[id] = ex.layer;
          ex.served[id] = am;
          ex.exit_ns[id] = globaltimer();
        }
      }
      miss_s[warp] = miss ? 1 : 0;
    }
    __syncthreads();
    const unsigned long long ep = static_cast<unsigned long long>(static_cast<unsigned>(*ex.epoch)) << 32;
    if (tid == 0) {
      int tot = 0;
      for (int w = 0; w < kWhWarps; ++w) tot += miss_s[w];
      tot_s = tot;
      st_release_u64(ex.scan_agg + blockIdx.x, ep | static_cast<unsigned long long>(tot + 1));
    }
    int acc = 0;
    for (int j = tid; j < static_cast<int>(blockIdx.x); j += blockDim.x) {
      unsigned long long v;
      do {
        v = ld_acquire_u64(ex.scan_agg + j);
      } while ((v & 0xffffffff00000000ull) != ep);
      acc += static_cast<int>(v & 0xffffffffull) - 1;
    }
    acc = __reduce_add_sync(0xffffffffu, acc);
    if (lane == 0) red_s[warp] = acc;
    __syncthreads();
    int prefix = 0;
    for (int w = 0; w < kWhWarps; ++w) prefix += red_s[w];
    if (miss && lane == 0) {
      int pos = prefix;
      for (int w = 0; w < warp; ++w) pos += miss_s[w];
      ex.ids_out[pos] = id;
      if (ex.src_rows_out) ex.src_rows_out[pos] = r;
    }
    if (blockIdx.x == gridDim.x - 1 && tid == 0) *ex.count_out = prefix + tot_s;
    return;
  }
  if (!ex.rows_dst_hi && ex.unordered && !ex.shadow) {
    // first-hit records per row; the CTA's misses take one atomic for their positions
    __shared__ int miss_s[kWhWarps], base_s;
    const bool miss = r < n && !__shfl_sync(0xffffffffu, hit, 0);
    int id = 0;
    if (lane == 0) {
      if (r < n) {
        id = ex.ids_in[r];
        if (ex.probs_out) ex.probs_out[id] = q;
        if (ex.labels_out) ex.labels_out[id] = am;
        if (hit && ex.exit_layer[id] == 0) {
          ex.exit_layer[id] = ex.layer;
          ex.served[id] = am;
          ex.exit_ns[id] = globaltimer();
        }
      }
      miss_s[warp] = miss ? 1 : 0;
    }
    __syncthreads();
    if (tid == 0) {
      int tot = 0;
      for (int w = 0; w < kWhWarps; ++w) tot += miss_s[w];
      base_s = tot ? atomicAdd(ex.count_out, tot) : 0;
    }
    __syncthreads();
    if (miss && lane == 0) {
      int pos = base_s;
      for (int w = 0; w < warp; ++w) pos += miss_s[w];
      ex.ids_out[pos] = id;
      if (ex.src_rows_out) ex.src_rows_out[pos] = r;
    }
    return;
  }
  if (!(ex.rows_dst_hi && !ex.shadow)) {
    exit_tail(ex, n, p.prob, p.hit, p.label);  // ordered compaction by the last CTA (every thread)
    return;
  }
  // block-MLP compact mode: the row's warp records a first hit or appends the
  // miss at an atomic position and copies its activations (serving.cpp:112-121)
  if (r >= n) return;
  int pos = -1;
  if (lane == 0) {
    const int id = ex.ids_in[r];
    if (ex.probs_out) ex.probs_out[id] = q;
    if (ex.labels_out) ex.labels_out[id] = am;
    if (hit) {
      if (ex.exit_layer[id] == 0) {
        ex.exit_layer[id] = ex.layer;
        ex.served[id] = am;
        ex.exit_ns[id] = globaltimer();
      }
    } else {
      pos = atomicAdd(ex.count_out, 1);
      ex.ids_out[pos] = id;
      if (ex.src_rows_out) ex.src_rows_out[pos] = r;
    }
  }
  pos = __shfl_sync(0xffffffffu, pos, 0);
  if (pos < 0) return;
  const bool held = rvec && ex.rows_src_hi == p.row_hi && ex.rows_src_lo == p.row_lo && ex.row_elems == p.D &&
                    p.row_stride == ex.row_elems;
  if (held) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int vi = lane + 32 * j;
      if (vi < nv) {
        reinterpret_cast<uint4*>(ex.rows_dst_hi + static_cast<long long>(pos) * ex.row_elems)[vi] = hv[j];
        if (ex.rows_src_lo) reinterpret_cast<uint4*>(ex.rows_dst_lo + static_cast<long long>(pos) * ex.row_elems)[vi] = lv[j];
      }
    }
    return;
  }
  const long long nvr = ex.row_elems / 8;
  const uint4* sh = reinterpret_cast<const uint4*>(ex.rows_src_hi + static_cast<long long>(r) * ex.row_elems);
  uint4* dh = reinterpret_cast<uint4*>(ex.rows_dst_hi + static_cast<long long>(pos) * ex.row_elems);
  for (long long i = lane; i < nvr; i += 32) dh[i] = __ldg(sh + i);
  if (ex.rows_src_lo) {
    const uint4* sl = reinterpret_cast<const uint4*>(ex.rows_src_lo + static_cast<long long>(r) * ex.row_elems);
    uint4* dl = reinterpret_cast<uint4*>(ex.rows_dst_lo + static_cast<long long>(pos) * ex.row_elems);
    for (long long i = lane; i < nvr; i += 32) dl[i] = __ldg(sl + i);
  }
}

// ------------------------------------------------------------ wide lookup
// Pool(C) caches with many classes (ImageNet heads: C up to 2048, 1000
// classes) in ONE persistent launch instead of three (GAP bins, logits GEMM,
// per-row head): every CTA of the grid is resident (one per SM), and two grid
// barriers separate the phases.
//   pre-wait: the CTA's slice of W2 (classes [k0, k1)) and the selector's
//             first layer Ws1 are staged in shared memory (static weights)
//   phase 1 : feats[r][c] = inv * sum_seg gap[img(r)][seg][c] (units of one
//             row x 64 channels; the segments split over 8 thread groups and
//             combined in fixed order: deterministic)
//   phase 2 : logits[r][k] = b2[k] + W2[k] . feats[r] for the CTA's classes,
//             every row (W2 read from HBM/L2 once per launch)
//   phase 3 : per row (CTA-strided): softmax, argmax, selector, sigmoid,
//             inclusive threshold (head_block: cache.cpp:259-265)
//   exit    : the last CTA records first hits and compacts (exit_tail)
struct WideLookupParams {
  CacheHeadParams h;  // classes, feat (= C), W2, b2, Ws1, bs1, ws2, bs2, delta, count, gap, gap_segs, gap_inv, gap_ids,
                      // prob, hit, label, pr_out, logits_out, ex
  float* feats;       // [max_rows][C] scratch
  float* logits;      // [max_rows][grid][kWideRec] per-row, per-CTA softmax records (scratch)
  unsigned* gsync;    // arrival counter of the grid barriers (zero-initialised once)
  int kpc;            // classes per CTA (phase 2)
  unsigned long long* stamps;  // nullable: CTA 0's %globaltimer at each phase boundary [8]
};

// Grid barrier over a monotonic arrival counter (one thread per CTA; every
// CTA resident). Each launch adds exactly kWideSyncPeriod to the counter (2 x
// gridDim.x arrivals, then CTA 0 pads to the period), so the launch's base is
// the counter rounded down to the period: u32 wrap-around is harmless since
// the period divides 2^32. Arrivals are fire-and-forget releases (no
// round trip to learn who was last); every CTA polls with acquire loads.
constexpr unsigned kWideSyncPeriod = 512;  // >= 2 * grid
__device__ __forceinline__ void grid_arrive(unsigned* cnt) {
  asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(cnt) : "memory");
}
__device__ __forceinline__ void grid_barrier(unsigned* cnt, unsigned base, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    grid_arrive(cnt);
    while (ld_acquire_u32(cnt) - base < target) __nanosleep(20);
  }
  __syncthreads();
}

// One halving step of a reduce-scatter over the lanes: lanes whose bit `o`
// is set keep the upper kN/2 values (adding the partner's), the others the lower.
template <int kN>
__device__ __forceinline__ void rs_halve(float (&v)[32], int o, int lane) {
  const bool up = (lane & o) != 0;
#pragma unroll
  for (int e = 0; e < kN / 2; ++e) {
    const float send = up ? v[e] : v[e + kN / 2];
    const float keep = up ? v[e + kN / 2] : v[e];
    v[e] = keep + __shfl_xor_sync(0xffffffffu, send, o);
  }
}

constexpr int kWideSegGroups = kLk / 16;  // 16 float4 columns (64 channels) x 32 segment groups
constexpr int kWideFeatChunk = 4096;      // largest feature width (C) of a wide lookup
constexpr int kWideScratch = 4 * kLk * 4;  // floats of phase-1 scratch (4 float4 per thread)
constexpr int kWideRec = 20;              // record of one (row, CTA): max, argmax, sum e, 16 selector sums, pad

// Group of 8 lanes (lane bits 0-2) reductions of the split softmax.
__device__ __forceinline__ float g8_max(float v) {
#pragma unroll
  for (int o = 4; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float g8_sum(float v) {
#pragma unroll
  for (int o = 4; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__global__ void __launch_bounds__(kLk, 1) wide_lookup_kernel(WideLookupParams q) {
  extern __shared__ __align__(16) float wsm[];
  __shared__ HeadSmem hs;
  __shared__ float wpart[64 * 32];  // phase-2 partial sums [row block x slice][32]
  const CacheHeadParams& p = q.h;
#define STAMP(i) \
  if (q.stamps && blockIdx.x == 0 && threadIdx.x == 0) q.stamps[i] = globaltimer();
  STAMP(0);
  const int C = p.feat, K = p.classes, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int G = gridDim.x;
  const int k0 = blockIdx.x * q.kpc;
  const int k1 = k0 + q.kpc < K ? k0 + q.kpc : K;
  const int nk = k1 > k0 ? k1 - k0 : 0;
  float* w2s = wsm;                                    // [kpc][C]  the CTA's classes of W2
  float* ws1c = w2s + static_cast<size_t>(q.kpc) * C;  // [16][8]   their selector columns
  float* fst = ws1c + 16 * 8;                          // [kWideScratch] phase-1 scratch
  if (nk > 0) stage_floats(w2s, p.W2 + static_cast<long long>(k0) * C, nk * C, tid);
  if (tid < 16 * 8) {
    const int j = tid >> 3, k = tid & 7;
    ws1c[tid] = k < nk ? __ldg(p.Ws1 + j * K + k0 + k) : 0.0f;
  }
  pdl_wait();
  STAMP(1);
  const int n = *p.count;
  // this launch's barrier base: no CTA can have passed barrier 1 yet, so the
  // counter lies in [base, base + gridDim.x)
  const unsigned sync_base = tid == 0 ? (ld_acquire_u32(q.gsync) & ~(kWideSyncPeriod - 1u)) : 0u;
  // ---- phase 1: GAP features of every row. Unit = (row, 64 channels); the
  // CTA takes 4 of its units at once (all their loads in flight), threads =
  // 16 float4 columns x 32 segment groups, groups combined in fixed order.
  {
    const int C4 = C >> 2;
    const int col_units = (C4 + 15) / 16, total = n * col_units;
    const int j = tid & 15, g = tid >> 4;
    float4* scr = reinterpret_cast<float4*>(fst);  // [4][kLk]
    for (int ub = blockIdx.x; ub < total; ub += 4 * gridDim.x) {
      const float4* base[4];
      bool ok[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int uu = ub + u * gridDim.x;
        const int r = uu / col_units, c4 = (uu % col_units) * 16 + j;
        ok[u] = uu < total && c4 < C4;
        const long long img = ok[u] ? (p.gap_ids ? p.gap_ids[r] : r) : 0;
        base[u] = reinterpret_cast<const float4*>(p.gap + img * p.gap_segs * C) + (ok[u] ? c4 : 0);
      }
      float4 a[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) a[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int sg = g; sg < p.gap_segs; sg += kWideSegGroups) {
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (ok[u]) add4(a[u], __ldcg(base[u] + static_cast<long long>(sg) * C4));
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) scr[u * kLk + tid] = a[u];
      __syncthreads();
      if (tid < 64) {
        const int u = tid >> 4, jj = tid & 15;
        const int uu = ub + u * gridDim.x;
        const int r = uu / col_units, c4 = (uu % col_units) * 16 + jj;
        if (uu < total && c4 < C4) {
          float4 t = scr[u * kLk + jj];
          for (int q2 = 1; q2 < kWideSegGroups; ++q2) add4(t, scr[u * kLk + q2 * 16 + jj]);
          const float inv = p.gap_inv;
          reinterpret_cast<float4*>(q.feats + static_cast<long long>(r) * C)[c4] =
              make_float4(t.x * inv, t.y * inv, t.z * inv, t.w * inv);
        }
      }
      __syncthreads();
    }
  }
  grid_barrier(q.gsync, sync_base, gridDim.x);
  // ---- phase 2: logits of the CTA's classes for every row, then the row's
  // split-softmax record over those classes, by chunks of rows. A warp owns a block of 4
  // rows x the CTA's <= 8 classes over a slice of the channels: 32
  // accumulators per lane, reduce-scattered across the lanes (31 shuffles),
  // slices added in fixed order. Record of (row, CTA): m = max logit, the
  // lowest class index attaining it, S = sum e^(l - m), sel_j = sum Ws1[j][k]
  // e^(l_k - m) — softmax + selector FC(C,16) reassociate exactly over CTAs
  // (losses.cpp:35-46, cache.cpp:259-265).
  STAMP(2);
  {
    constexpr int R = 256;  // rows per pass (<= 64 row blocks of partial sums)
    for (int r0 = 0; r0 < n; r0 += R) {
      const int rn = n - r0 < R ? n - r0 : R;
      const int nb = (rn + 3) >> 2;  // row blocks
      int wpb = 1;                   // warps per row block (channel slices of >= 32)
      while (wpb * 2 * nb <= kLk / 32 && C / (wpb * 2) >= 32) wpb *= 2;
      const int per = (kLk / 32) / wpb;  // row blocks in flight
      if (nk > 0) {
        for (int rb = warp / wpb; rb < nb; rb += per) {
          const int sub = warp % wpb;
          const int c0 = (C * sub) / wpb, c1 = (C * (sub + 1)) / wpb;
          float v[32];
#pragma unroll
          for (int e = 0; e < 32; ++e) v[e] = 0.0f;
          const float* f[4];
#pragma unroll
          for (int i = 0; i < 4; ++i)
            f[i] = q.feats + static_cast<long long>(r0 + (rb * 4 + i < rn ? rb * 4 + i : rb * 4)) * C;
#pragma unroll 4
          for (int c = c0 + lane; c < c1; c += 32) {
            float x[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) x[i] = __ldcg(f[i] + c);
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              const float w = k < nk ? w2s[k * C + c] : 0.0f;
#pragma unroll
              for (int i = 0; i < 4; ++i) v[i * 8 + k] += x[i] * w;
            }
          }
          // lane l ends with the full sum of accumulator l = (row i = l / 8, class k = l % 8)
          rs_halve<32>(v, 16, lane);
          rs_halve<16>(v, 8, lane);
          rs_halve<8>(v, 4, lane);
          rs_halve<4>(v, 2, lane);
          rs_halve<2>(v, 1, lane);
          wpart[(rb * wpb + sub) * 32 + lane] = v[0];
        }
      }
      __syncthreads();
      // records: warp w handles row blocks w, w + 16, ...; lanes 8i..8i+7 = row i's classes
      for (int rb = warp; rb < nb; rb += kLk / 32) {
        const int i = lane >> 3, k = lane & 7, rr = rb * 4 + i;
        const bool kin = k < nk;
        float l = -FLT_MAX;
        if (kin) {
          float a = wpart[(rb * wpb) * 32 + lane];
          for (int sb = 1; sb < wpb; ++sb) a += wpart[(rb * wpb + sb) * 32 + lane];
          l = a + __ldg(p.b2 + k0 + k);
        }
        const float m = g8_max(l);
        // lowest class index attaining the max (softmax is monotonic: argmax(pr) = argmax(logits))
        int am = kin && l == m ? k : 8;
#pragma unroll
        for (int o = 4; o > 0; o >>= 1) am = min(am, __shfl_xor_sync(0xffffffffu, am, o));
        const float e = kin ? expf(l - m) : 0.0f;
        const float S = g8_sum(e);
        // 16 selector sums reduce-scattered over the 8 lanes: lane k ends with j = 2k, 2k + 1
        float sv[16];
#pragma unroll
        for (int jj = 0; jj < 16; ++jj) sv[jj] = ws1c[jj * 8 + k] * e;
#pragma unroll
        for (int o = 4, h = 8; o > 0; o >>= 1, h >>= 1) {
          const bool up = (lane & o) != 0;
#pragma unroll
          for (int t = 0; t < 8; ++t) {
            if (t < h) {
              const float send = up ? sv[t] : sv[t + h];
              const float keep = up ? sv[t + h] : sv[t];
              sv[t] = keep + __shfl_xor_sync(0xffffffffu, send, o);
            }
          }
        }
        if (rr < rn && nk > 0) {
          float* rec = q.logits + (static_cast<long long>(r0 + rr) * G + blockIdx.x) * kWideRec;
          if (k == 0) {
            rec[0] = m;
            rec[1] = __int_as_float(k0 + am);
            rec[2] = S;
          }
          rec[3 + 2 * k] = sv[0];
          rec[4 + 2 * k] = sv[1];
        }
      }
      __syncthreads();  // wpart reused by the next chunk
    }
  }
  STAMP(3);
  grid_barrier(q.gsync, sync_base, 2 * gridDim.x);
  if (blockIdx.x == 0 && tid == 0)  // every CTA has arrived twice: pad to the period
    asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(q.gsync), "r"(kWideSyncPeriod - 2 * gridDim.x)
                 : "memory");
  STAMP(4);
  pdl_trigger();
  // ---- phase 3: each row combines its G records (fixed CTA order):
  // M = max m_c, label = the lowest CTA's argmax attaining M, S = sum S_c
  // e^(m_c - M), sel_j = sum sel_c,j e^(m_c - M); then the selector head.
  const int nwarps = kLk / 32;
  for (int r = blockIdx.x; r < n; r += gridDim.x) {
    const bool has = tid < G && (tid * q.kpc < K);  // CTAs that own classes wrote records
    float rv[kWideRec];
    if (has) {
      const float4* src = reinterpret_cast<const float4*>(q.logits + (static_cast<long long>(r) * G + tid) * kWideRec);
#pragma unroll
      for (int u = 0; u < kWideRec / 4; ++u) {
        const float4 t = __ldcg(src + u);
        rv[4 * u] = t.x;
        rv[4 * u + 1] = t.y;
        rv[4 * u + 2] = t.z;
        rv[4 * u + 3] = t.w;
      }
    } else {
      rv[0] = -FLT_MAX;
      rv[1] = __int_as_float(0x7fffffff);
    }
    // block max with the lowest CTA index on ties (CTAs own ascending class ranges)
    float bv = rv[0];
    int bc = has ? tid : 0x7fffffff;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oc = __shfl_xor_sync(0xffffffffu, bc, o);
      if (ov > bv || (ov == bv && oc < bc)) {
        bv = ov;
        bc = oc;
      }
    }
    if (lane == 0) {
      hs.bv[warp] = bv;
      hs.bi[warp] = bc;
    }
    __syncthreads();
    float M = hs.bv[0];
    int cm = hs.bi[0];
    for (int w = 1; w < nwarps; ++w)
      if (hs.bv[w] > M || (hs.bv[w] == M && hs.bi[w] < cm)) {
        M = hs.bv[w];
        cm = hs.bi[w];
      }
    const float wt = has ? expf(rv[0] - M) : 0.0f;
    float acc[17];
    acc[16] = has ? rv[2] * wt : 0.0f;
#pragma unroll
    for (int j = 0; j < 16; ++j) acc[j] = has ? rv[3 + j] * wt : 0.0f;
#pragma unroll
    for (int j = 0; j < 17; ++j) acc[j] = warp_sum(acc[j]);
    if (lane < 17) {
      float v = acc[0];
#pragma unroll
      for (int j = 1; j < 17; ++j) v = lane == j ? acc[j] : v;
      hs.part[warp * 17 + lane] = v;
    }
    if (tid == cm) hs.S = rv[1];  // the label: argmax of the CTA holding the maximum (int bits)
    __syncthreads();
    if (warp == 0) {
      float t = 0.0f;
      if (lane < 17)
        for (int w = 0; w < nwarps; ++w) t += hs.part[w * 17 + lane];
      const float S = __shfl_sync(0xffffffffu, t, 16);
      float h = 0.0f;
      if (lane < 16) {
        const float a = t / S + p.bs1[lane];
        h = (a > 0.0f ? a : 0.0f) * p.ws2[lane];
      }
      float hj[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) hj[j] = __shfl_sync(0xffffffffu, h, j);
      if (lane == 0) {
        float z = p.bs2;
#pragma unroll
        for (int j = 0; j < 16; ++j) z += hj[j];
        float qv;
        if (z >= 0.0f) {
          qv = 1.0f / (1.0f + expf(-z));
        } else {
          const float ez = expf(z);
          qv = ez / (1.0f + ez);
        }
        p.prob[r] = qv;
        p.hit[r] = static_cast<double>(qv) >= p.delta ? 1 : 0;
        p.label[r] = __float_as_int(hs.S);
      }
    }
    __syncthreads();  // hs reused by the next row
  }
  STAMP(5);
  if (p.ex.arrive) exit_tail(p.ex, n, p.prob, p.hit, p.label);
  STAMP(6);
#undef STAMP
}

__global__ void gather_rows_kernel(const __nv_bfloat16* src_hi, const __nv_bfloat16* src_lo, __nv_bfloat16* dst_hi,
                                   __nv_bfloat16* dst_lo, long long row_elems, const int* src_rows, const int* count) {
  pdl_wait();
  pdl_trigger();
  const int j = blockIdx.x;
  if (j >= *count) return;
  const long long s = src_rows[j];
  const uint4* sh = reinterpret_cast<const uint4*>(src_hi + s * row_elems);
  uint4* dh = reinterpret_cast<uint4*>(dst_hi + static_cast<long long>(j) * row_elems);
  const long long nv = row_elems / 8;
  for (long long i = blockIdx.y * blockDim.x + threadIdx.x; i < nv; i += gridDim.y * blockDim.x) dh[i] = sh[i];
  if (src_lo) {
    const uint4* sl = reinterpret_cast<const uint4*>(src_lo + s * row_elems);
    uint4* dl = reinterpret_cast<uint4*>(dst_lo + static_cast<long long>(j) * row_elems);
    for (long long i = blockIdx.y * blockDim.x + threadIdx.x; i < nv; i += gridDim.y * blockDim.x) dl[i] = sl[i];
  }
}

__global__ void split_rows_kernel(const float* x, int in_dim, int dp, const int* ids, const int* count,
                                  __nv_bfloat16* hi, __nv_bfloat16* lo) {
  pdl_wait();
  pdl_trigger();
  const int j = blockIdx.x;
  if (j >= *count) return;
  const long long src = ids ? ids[j] : j;
  const float* xr = x + src * in_dim;
  const long long ob = static_cast<long long>(j) * dp;
  if ((in_dim & 3) == 0 && (dp & 3) == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0) {
    // 16-byte loads, kSplitVec per thread issued before any use (the row is
    // usually cold in HBM: one round trip per batch of loads, not per element)
    constexpr int kSplitVec = 4;
    const int n4 = dp >> 2, in4 = in_dim >> 2;
    for (int base = 0; base < n4; base += kSplitVec * blockDim.x) {
      float4 v[kSplitVec];
#pragma unroll
      for (int u = 0; u < kSplitVec; ++u) {
        const int i4 = base + u * blockDim.x + threadIdx.x;
        v[u] = i4 < in4 ? __ldg(reinterpret_cast<const float4*>(xr) + i4) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < kSplitVec; ++u) {
        const int i4 = base + u * blockDim.x + threadIdx.x;
        if (i4 < n4) {
          const float f[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
          __nv_bfloat16 h[4], l[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            h[e] = __float2bfloat16_rn(f[e]);
            l[e] = __float2bfloat16_rn(f[e] - __bfloat162float(h[e]));
          }
          uint2 hp, lp;
          hp.x = (static_cast<uint32_t>(__bfloat16_as_ushort(h[1])) << 16) | __bfloat16_as_ushort(h[0]);
          hp.y = (static_cast<uint32_t>(__bfloat16_as_ushort(h[3])) << 16) | __bfloat16_as_ushort(h[2]);
          lp.x = (static_cast<uint32_t>(__bfloat16_as_ushort(l[1])) << 16) | __bfloat16_as_ushort(l[0]);
          lp.y = (static_cast<uint32_t>(__bfloat16_as_ushort(l[3])) << 16) | __bfloat16_as_ushort(l[2]);
          *reinterpret_cast<uint2*>(hi + ob + 4 * i4) = hp;
          if (lo) *reinterpret_cast<uint2*>(lo + ob + 4 * i4) = lp;
        }
      }
    }
    return;
  }
  for (int i = threadIdx.x; i < dp; i += blockDim.x) {
    const float v = i < in_dim ? xr[i] : 0.0f;
    split_store(v, hi, lo, ob + i);
  }
}

__global__ void split_taps_nchw_kernel(const float* x, int C, int HW, long long row_stride, __nv_bfloat16* hi,
                                       __nv_bfloat16* lo) {
  pdl_wait();
  pdl_trigger();
  const int r = blockIdx.x;
  const long long D = static_cast<long long>(C) * HW;
  for (long long i = blockIdx.y * blockDim.x + threadIdx.x; i < row_stride; i += gridDim.y * blockDim.x) {
    // storage index i = p*C + c  <-  flat f = c*HW + p
    float v = 0.0f;
    if (i < D) {
      const long long p = i / C, c = i % C;
      v = x[r * D + c * HW + p];
    }
    split_store(v, hi, lo, r * row_stride + i);
  }
}

// Read-back of a stored tap as the reference sees it: fp32 hi + lo, NCHW-flat.
__global__ void planes_to_nchw_kernel(const __nv_bfloat16* hi, const __nv_bfloat16* lo, long long row_stride, int C,
                                      int HW, float* out) {
  pdl_wait();
  pdl_trigger();
  const int r = blockIdx.x;
  const long long D = static_cast<long long>(C) * HW;
  for (long long f = blockIdx.y * blockDim.x + threadIdx.x; f < D; f += gridDim.y * blockDim.x) {
    const long long i = r * row_stride + (f % HW) * C + f / HW;
    float v = __bfloat162float(hi[i]);
    if (lo) v += __bfloat162float(lo[i]);
    out[r * D + f] = v;
  }
}

// Base head (base_model.cpp:48-49): logits -> softmax -> argmax (serving.cpp:108).
template <bool kGap>
__global__ void __launch_bounds__(kLk) base_head_kernel(const __nv_bfloat16* hi, const __nv_bfloat16* lo,
                                                        long long row_stride, int C, int HW, const float* W,
                                                        const float* b, int classes, const int* ids, const int* count,
                                                        int* base_pred, float* logits_out, int* exit_layer, int* served,
                                                        unsigned long long* exit_ns, const float* pre_logits,
                                                        int pre_nz, long long pre_zstride) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ float sm[];
  __shared__ float red[kLk * 8];
  __shared__ int bi_s[32];
  __shared__ float bv_s[32];
  const int r = blockIdx.x;
  if (r >= *count) return;
  const int id = ids[r];
  const long long n = kGap ? id : r;
  float* feat = sm;          // [C]
  float* logits = sm + C;    // [classes]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = kLk / 32;
  TapView t;
  t.hi = hi;
  t.lo = lo;
  if (pre_logits) {
    for (int k = tid; k < classes; k += kLk) logits[k] = fc_logit(pre_logits, pre_nz, pre_zstride, b, r, classes, k);
  } else {
    if (kGap) {
      tap_gap_block(t, n * row_stride, C, HW, feat, red);
    } else {
      for (int c = tid; c < C; c += kLk) feat[c] = ld_tap(t, n * row_stride + c);
      __syncthreads();
    }
    block_logits(W, b, classes, C, feat, logits);
  }
  __syncthreads();
  float m = -FLT_MAX;
  for (int k = tid; k < classes; k += kLk) m = fmaxf(m, logits[k]);
  m = block_max(m, red);
  float part = 0.0f;
  for (int k = tid; k < classes; k += kLk) part += expf(logits[k] - m);
  const float sum = block_sum(part, red);
  float bv = -FLT_MAX;
  int bi = 0x7fffffff;
  for (int k = tid; k < classes; k += kLk) {
    const float pk = expf(logits[k] - m) / sum;
    if (pk > bv) {
      bv = pk;
      bi = k;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > bv || (ov == bv && oi < bi)) {
      bv = ov;
      bi = oi;
    }
  }
  if (lane == 0) {
    bv_s[warp] = bv;
    bi_s[warp] = bi;
  }
  __syncthreads();
  if (tid == 0) {
    float v = bv_s[0];
    int i = bi_s[0];
    for (int w = 1; w < nw; ++w)
      if (bv_s[w] > v || (bv_s[w] == v && bi_s[w] < i)) {
        v = bv_s[w];
        i = bi_s[w];
      }
    base_pred[id] = i;
    if (exit_layer[id] == 0) {
      served[id] = i;
      exit_ns[id] = globaltimer();
    }
  }
  if (logits_out)
    for (int k = tid; k < classes; k += kLk) logits_out[static_cast<long long>(id) * classes + k] = logits[k];
}

// One thread per (output pixel, 8 consecutive K entries): 16-byte stores.
__global__ void stem_im2col_kernel(const float* x, const int* count, int C, int H, int W, int k, int stride, int pad,
                                   int Ho, int Wo, int Kp, __nv_bfloat16* hi, __nv_bfloat16* lo) {
  pdl_wait();
  pdl_trigger();
  const int kg = Kp / 8;
  const int pix = Ho * Wo;
  const long long total = static_cast<long long>(*count) * pix * kg;
  const int K = k * k * C;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int g8 = static_cast<int>(i % kg);
    const long long m = i / kg;
    const int n = static_cast<int>(m / pix);
    const int rem = static_cast<int>(m - static_cast<long long>(n) * pix);
    const int oh = rem / Wo, ow = rem - (rem / Wo) * Wo;
    const float* xn = x + static_cast<long long>(n) * C * H * W;
    float v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int kk = g8 * 8 + e;
      float val = 0.0f;
      if (kk < K) {
        const int c = kk % C, rs = kk / C, s2 = rs % k, r = rs / k;
        const int ih = oh * stride + r - pad, iw = ow * stride + s2 - pad;
        if (ih >= 0 && ih < H && iw >= 0 && iw < W) val = xn[(c * H + ih) * W + iw];
      }
      v[e] = val;
    }
    uint4 h4, l4;
    __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&h4);
    __nv_bfloat162* l2 = reinterpret_cast<__nv_bfloat162*>(&l4);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const __nv_bfloat162 hh = __floats2bfloat162_rn(v[2 * e], v[2 * e + 1]);
      h2[e] = hh;
      const float2 hf = __bfloat1622float2(hh);
      l2[e] = __floats2bfloat162_rn(v[2 * e] - hf.x, v[2 * e + 1] - hf.y);
    }
    reinterpret_cast<uint4*>(hi)[i] = h4;
    if (lo) reinterpret_cast<uint4*>(lo)[i] = l4;
  }
}

__global__ void phase_split_kernel(const __nv_bfloat16* hi, const __nv_bfloat16* lo, int H, int W, int C, int N,
                                   int Hs, int Ws, const int* ids, const int* count, __nv_bfloat16* ohi,
                                   __nv_bfloat16* olo) {
  pdl_wait();
  pdl_trigger();
  const int j = blockIdx.x;
  if (j >= *count) return;
  const long long n = ids[j];
  const int cv = C / 8;
  const long long per = 4LL * Hs * Ws * cv;
  for (long long i = blockIdx.y * blockDim.x + threadIdx.x; i < per; i += gridDim.y * blockDim.x) {
    const int c8 = static_cast<int>(i % cv);
    long long rest = i / cv;
    const int jj = static_cast<int>(rest % Ws);
    rest /= Ws;
    const int ii = static_cast<int>(rest % Hs);
    const int ph = static_cast<int>(rest / Hs);
    const int h = 2 * ii + (ph >> 1), w = 2 * jj + (ph & 1);
    const long long dst = ((((static_cast<long long>(ph) * N + n) * Hs + ii) * Ws + jj) * C) + c8 * 8;
    uint4 vh = make_uint4(0, 0, 0, 0), vl = make_uint4(0, 0, 0, 0);
    if (h < H && w < W) {
      const long long src = ((n * H + h) * W + w) * C + c8 * 8;
      vh = *reinterpret_cast<const uint4*>(hi + src);
      if (lo) vl = *reinterpret_cast<const uint4*>(lo + src);
    }
    *reinterpret_cast<uint4*>(ohi + dst) = vh;
    if (olo) *reinterpret_cast<uint4*>(olo + dst) = vl;
  }
}

// Max-pool (the ResNet stem's 3x3 s2 pool) over the surviving images, NHWC
// hi (+lo): one thread per (output pixel, 8 channels), 16-byte loads/stores;
// per channel the first maximum in (r, s) order wins (hi and lo move
// together). kK > 0: compile-time window (all k*k loads in flight at once).
template <int kK>
__global__ void maxpool_kernel(const __nv_bfloat16* hi, const __nv_bfloat16* lo, int H, int W, int C, int k_rt,
                               int stride, int pad, int Ho, int Wo, const int* ids, const int* count,
                               __nv_bfloat16* ohi, __nv_bfloat16* olo) {
  pdl_wait();
  pdl_trigger();
  const int k = kK > 0 ? kK : k_rt;
  const int j = blockIdx.x;
  if (j >= *count) return;
  const long long n = ids[j];
  const int c8n = C / 8;
  const int per = Ho * Wo * c8n;  // (32-bit index math per element)
  for (int i = blockIdx.y * blockDim.x + threadIdx.x; i < per; i += gridDim.y * blockDim.x) {
    const int pix = i / c8n, c8 = i - pix * c8n;
    const int oh = pix / Wo, ow = pix - oh * Wo;
    float best[8];
    uint4 bh = make_uint4(0, 0, 0, 0), bl = make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int e = 0; e < 8; ++e) best[e] = -FLT_MAX;
#pragma unroll
    for (int r = 0; r < (kK > 0 ? kK : 1); ++r) {
#pragma unroll
      for (int s2 = 0; s2 < (kK > 0 ? kK : 1); ++s2) {
        for (int rr = r; rr < (kK > 0 ? r + 1 : k); ++rr) {
          for (int ss = s2; ss < (kK > 0 ? s2 + 1 : k); ++ss) {
            const int ih = oh * stride + rr - pad, iw = ow * stride + ss - pad;
            if (ih < 0 || ih >= H || iw < 0 || iw >= W) continue;
            const long long src = ((n * H + ih) * W + iw) * C + c8 * 8;
            const uint4 vh = __ldg(reinterpret_cast<const uint4*>(hi + src));
            const uint4 vl = lo ? __ldg(reinterpret_cast<const uint4*>(lo + src)) : make_uint4(0, 0, 0, 0);
            const __nv_bfloat16* h8 = reinterpret_cast<const __nv_bfloat16*>(&vh);
            const __nv_bfloat16* l8 = reinterpret_cast<const __nv_bfloat16*>(&vl);
            __nv_bfloat16* bh8 = reinterpret_cast<__nv_bfloat16*>(&bh);
            __nv_bfloat16* bl8 = reinterpret_cast<__nv_bfloat16*>(&bl);
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              const float v = __bfloat162float(h8[e]) + __bfloat162float(l8[e]);
              if (v > best[e]) {
                best[e] = v;
                bh8[e] = h8[e];
                bl8[e] = l8[e];
              }
            }
          }
        }
      }
    }
    const long long dst = ((n * Ho + oh) * Wo + ow) * C + c8 * 8;
    *reinterpret_cast<uint4*>(ohi + dst) = bh;
    if (olo) *reinterpret_cast<uint4*>(olo + dst) = bl;
  }
}

__global__ void set_int_kernel(int* p, int v) {
  pdl_wait();
  pdl_trigger();
  *p = v;
}

__global__ void stamp_kernel(unsigned long long* t0) {
  pdl_wait();
  pdl_trigger(); *t0 = globaltimer(); }

// B is a kernel argument: a captured graph's node is updated in place when
// the batch size changes (Engine::serve_mode), so no separate launch writes
// it; batch_out keeps a device copy for later kernels (confusion counts).
__global__ void init_batch_kernel(int B, int* batch_out, int max_batch, int* ids0, int* count0, int* rows_out,
                                  int rows_mult, int* exit_layer, int* served, int* base_pred,
                                  unsigned long long* exit_ns, float* probs, int L, unsigned long long* t0) {
  pdl_wait();
  pdl_trigger();
  if (t0 && blockIdx.x == 0 && threadIdx.x == 0) *t0 = globaltimer();  // batch start (latency origin)
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < max_batch; i += gridDim.x * blockDim.x) {
    ids0[i] = i;
    exit_layer[i] = 0;
    served[i] = -1;
    base_pred[i] = -1;
    exit_ns[i] = 0;
    for (int l = 0; l < L; ++l) probs[static_cast<long long>(l) * max_batch + i] = __int_as_float(0x7fc00000);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *count0 = B;
    if (batch_out) *batch_out = B;
    if (rows_out) *rows_out = B * rows_mult;
  }
  // per-layer survivor counts start at zero (atomic row compaction appends to them);
  // count0[L + 2] is the serve epoch that tags the heads' look-back scan records
  if (blockIdx.x == 0 && threadIdx.x >= 1 && threadIdx.x <= L) count0[threadIdx.x] = 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) count0[L + 2] += 1;
}

__global__ void __launch_bounds__(256) confusion_kernel(const float* probs, const int* labels, const int* base_pred,
                                                       int max_batch, const int* batch, const double* grid, int G,
                                                       unsigned long long* counts) {
  pdl_wait();
  pdl_trigger();
  __shared__ unsigned int cnt[64][4];
  const int l = blockIdx.x;
  for (int i = threadIdx.x; i < 64 * 4; i += blockDim.x) cnt[i / 4][i % 4] = 0u;
  __syncthreads();
  const int B = *batch;
  for (int i = threadIdx.x; i < B; i += blockDim.x) {
    const float p = probs[static_cast<long long>(l) * max_batch + i];
    if (p != p) continue;  // not probed
    const bool agree = labels[static_cast<long long>(l) * max_batch + i] == base_pred[i];
    for (int g = 0; g < G; ++g) {
      const bool hit = static_cast<double>(p) >= grid[g];
      atomicAdd(&cnt[g][hit ? (agree ? 0 : 1) : (agree ? 3 : 2)], 1u);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < G * 4; i += blockDim.x)
    counts[(static_cast<long long>(l) * G + i / 4) * 4 + i % 4] = cnt[i / 4][i % 4];
}

}  // namespace

void launch_confusion(const float* probs, const int* labels, const int* base_pred, int max_batch, const int* batch,
                      int L, const double* grid, int G, unsigned long long* counts, cudaStream_t s) {
  if (L <= 0 || G <= 0) return;
  launch_pdl(confusion_kernel, dim3(L), dim3(256), 0, s, probs, labels, base_pred, max_batch, batch, grid, G, counts);
}

void launch_pool_bins(const TapView& tap, int max_rows, int win, int width, float* bins, cudaStream_t s) {
  const float inv = static_cast<float>(1.0 / win);
  if (max_rows <= 0) return;
  if (tap.HW > 1 && tap.C % 64 == 0 && win <= tap.HW && tap.HW % win == 0 && tap.HW / win >= 32) {
    launch_pdl(pool_strips_kernel, dim3(dim3(max_rows, tap.C / 64)), dim3(256), 0, s, tap, win, width, inv, bins);
  } else if (tap.HW > 1 && tap.C % 64 == 0 && win % tap.HW == 0 && 64 % (win / tap.HW) == 0) {
    launch_pdl(pool_channels_kernel, dim3(dim3(max_rows, tap.C / 64)), dim3(256), 0, s, tap, win / tap.HW, width, inv, bins);
  } else {
    const int gy = (width + 255) / 256 < 64 ? (width + 255) / 256 : 64;
    launch_pdl(pool_generic_kernel, dim3(dim3(max_rows, gy)), dim3(256), 0, s, tap, win, width, inv, bins);
  }
}

void launch_gap_bins(const float* gap, int segs, int C, int HW, const int* data_idx, const int* count, int max_rows,
                     float* bins, cudaStream_t s) {
  if (max_rows <= 0) return;
  const float inv = static_cast<float>(1.0 / HW);
  launch_pdl(gap_bins_kernel, dim3(max_rows), dim3(kGapBinsThreads), static_cast<size_t>(C) * sizeof(float), s, gap, segs, C, inv, data_idx, count,
                                                                                 bins);
}

void launch_conv1d_partials(const TapView& tap, int max_rows, long long D, int kernel, int stride, int out_dim,
                            const float* w1, float b1, const float* W2, int classes, int chunk_elems, int nchunks,
                            float* partials, cudaStream_t s) {
  if (max_rows <= 0) return;
  const size_t smem = static_cast<size_t>(chunk_elems + kernel) * sizeof(float);
  static std::atomic<unsigned long long> attr{0};
  if (first_on_device(attr))
    cudaFuncSetAttribute(conv1d_partials_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  launch_pdl(conv1d_partials_kernel, dim3(dim3(max_rows, nchunks)), dim3(256), smem, s, tap, D, kernel, stride, out_dim, w1, b1, W2,
                                                                    classes, chunk_elems, nchunks, partials);
}

int rows_fc_splits(int feat) {
  const int sl = rows_fc_slice(feat);
  return (feat + sl - 1) / sl;
}

void launch_rows_fc(const float* A, long long lda, int ks, long long part_stride, const float* b1, int feat,
                    const float* W, int classes, const int* count, int max_rows, float* out, cudaStream_t s) {
  if (max_rows <= 0) return;
  const dim3 grid((classes + kFcBN - 1) / kFcBN, (max_rows + kFcBM - 1) / kFcBM, rows_fc_splits(feat));
  if (ks > 0)
    launch_pdl(rows_fc_kernel<1>, dim3(grid), dim3(256), 0, s, A, lda, ks, part_stride, b1, feat, rows_fc_slice(feat), W, classes, count,
                                           max_rows, out);
  else
    launch_pdl(rows_fc_kernel<0>, dim3(grid), dim3(256), 0, s, A, lda, 0, 0, nullptr, feat, rows_fc_slice(feat), W, classes, count,
                                           max_rows, out);
}

size_t wide_lookup_smem(int classes, int C, int grid) {
  const int kpc = (classes + grid - 1) / grid;
  return (static_cast<size_t>(kpc) * C + 16 * 8 + kWideScratch) * sizeof(float);
}

constexpr size_t kWideSmemMax = 200 * 1024;
bool wide_lookup_supported(int classes, int C, int num_sms) {
  const int grid = num_sms < static_cast<int>(kWideSyncPeriod / 2) ? num_sms : static_cast<int>(kWideSyncPeriod / 2);
  return classes > 32 && C % 4 == 0 && C <= kWideFeatChunk && (classes + grid - 1) / grid <= 8 &&
         grid <= kLk && wide_lookup_smem(classes, C, num_sms) <= kWideSmemMax;
}


static unsigned long long* g_wide_stamps = nullptr;
void set_wide_lookup_stamps(unsigned long long* stamps) { g_wide_stamps = stamps; }

void launch_wide_lookup(const CacheHeadParams& h, float* feats, float* logits, int* gsync, int num_sms,
                        cudaStream_t s) {
  WideLookupParams q{};
  q.stamps = g_wide_stamps;
  q.h = h;
  q.feats = feats;
  q.logits = logits;
  q.gsync = reinterpret_cast<unsigned*>(gsync);
  const int grid = num_sms < static_cast<int>(kWideSyncPeriod / 2) ? num_sms : static_cast<int>(kWideSyncPeriod / 2);
  q.kpc = (h.classes + grid - 1) / grid;
  const size_t smem = wide_lookup_smem(h.classes, h.feat, grid);
  static std::atomic<unsigned long long> attr{0};
  if (first_on_device(attr))
    cudaFuncSetAttribute(wide_lookup_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kWideSmemMax);
  launch_pdl(wide_lookup_kernel, dim3(grid), dim3(kLk), smem, s, q);
}

// Warp-per-row head eligibility: <= 32 classes, features from the row, FC(h)
// partials or pooled bins (not the fused GAP partials, not the Conv(k,s)
// chunk partials), shared memory within bounds; LCB_BLOCK_HEADS=1 keeps the
// block-per-row kernel (A/B).
static bool warp_head_ok(const CacheHeadParams& p, int max_rows) {
  const char* env = std::getenv("LCB_BLOCK_HEADS");  // (read per launch build: tests switch it)
  const int mode = env ? std::atoi(env) : 0;
  if (mode == 1 || p.classes > 32 || p.pre_logits) return false;
  if (p.gap && (p.family != 1 || (p.feat & 3) != 0)) return false;
  const bool direct = p.row_hi != nullptr;
  if (!direct && p.family == 2) return false;
  if (direct && p.family == 0) return false;
  // a warp per row has a longer per-row latency than 16 warps per row: it wins
  // once there are more rows than a CTA-per-row launch keeps resident (C1:
  // b256 202 vs 204 us/step, b512 226 vs 214, b16384 2329 vs 533; LCB_BLOCK_HEADS=2 forces it)
  // (fused-GAP heads read a few KB per row: the warp wins at any batch — R18 b256 355.8K -> 360.7K req/s)
  if (max_rows < 512 && !p.gap && mode != 2) return false;
  if (direct && p.D > 8192) return false;
  return warp_head_smem_floats(p) * sizeof(float) <= 160 * 1024;
}

void launch_cache_head(const CacheHeadParams& p_in, int max_rows, cudaStream_t s) {
  if (max_rows <= 0) return;
  CacheHeadParams p = p_in;
  if (warp_head_ok(p, max_rows)) {
    // the look-back scan needs every CTA of the grid resident: <= 2 per SM by shared memory
    if (warp_head_smem_floats(p) * sizeof(float) > 100 * 1024) p.ex.scan_agg = nullptr;
    static std::atomic<unsigned long long> wattr{0};
    if (first_on_device(wattr))
      cudaFuncSetAttribute(warp_head_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    launch_pdl(warp_head_kernel, dim3((max_rows + kWhWarps - 1) / kWhWarps), dim3(kWhWarps * 32),
               warp_head_smem_floats(p) * sizeof(float), s, p);
    return;
  }
  if (p.classes > 32 && p.family != 2 && p.fc_scratch) {
    // Many classes: one batched split-K logits GEMM, then the per-row head.
    if (p.family == 1)
      launch_rows_fc(p.feats, p.feat, 0, 0, nullptr, p.feat, p.W2, p.classes, p.count, max_rows, p.fc_scratch, s);
    else
      launch_rows_fc(p.feats, p.hp, p.ks, p.rows_total * p.hp, p.b1, p.feat, p.W2, p.classes, p.count, max_rows,
                     p.fc_scratch, s);
    p.pre_logits = p.fc_scratch;
    p.pre_nz = rows_fc_splits(p.feat);
    p.pre_zstride = static_cast<long long>(max_rows) * p.classes;
    p.gap = nullptr;
  }
  size_t smem = static_cast<size_t>(p.classes + head_feat_len(p)) * sizeof(float);
  if (head_stages_weights(p)) smem += static_cast<size_t>(p.classes) * (head_w2_cols(p) + 16) * sizeof(float);  // W2 + Ws1
  else if (head_stages_ws1(p)) smem += static_cast<size_t>(p.classes) * 16 * sizeof(float);          // Ws1
  static std::atomic<unsigned long long> attr{0};
  if (first_on_device(attr))
    cudaFuncSetAttribute(cache_head_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  launch_pdl(cache_head_kernel, dim3(max_rows), dim3(kLk), smem, s, p);
}

bool fused_lookup_supported(int classes, int C, int max_rows) {
  return classes <= 32 && C % 4 == 0 && C <= 16384 && max_rows > 0;
}

void launch_gather_rows(const __nv_bfloat16* src_hi, const __nv_bfloat16* src_lo, __nv_bfloat16* dst_hi,
                        __nv_bfloat16* dst_lo, long long row_elems, const int* src_rows, const int* count, int max_rows,
                        cudaStream_t s) {
  if (max_rows <= 0) return;
  const long long nv = row_elems / 8;
  int gy = static_cast<int>((nv + 255) / 256);
  if (gy > 64) gy = 64;
  launch_pdl(gather_rows_kernel, dim3(dim3(max_rows, gy)), dim3(256), 0, s, src_hi, src_lo, dst_hi, dst_lo, row_elems, src_rows, count);
}

void launch_split_rows(const float* x, int in_dim, int dp, const int* ids, const int* count, int max_rows,
                       __nv_bfloat16* hi, __nv_bfloat16* lo, cudaStream_t s) {
  if (max_rows <= 0) return;
  launch_pdl(split_rows_kernel, dim3(max_rows), dim3(256), 0, s, x, in_dim, dp, ids, count, hi, lo);
}

void launch_split_taps_nchw(const float* x, int C, int HW, int rows, long long row_stride, __nv_bfloat16* hi,
                            __nv_bfloat16* lo, cudaStream_t s) {
  if (rows <= 0) return;
  int gy = static_cast<int>((row_stride + 255) / 256);
  if (gy > 128) gy = 128;
  launch_pdl(split_taps_nchw_kernel, dim3(dim3(rows, gy)), dim3(256), 0, s, x, C, HW, row_stride, hi, lo);
}

void launch_planes_to_nchw(const __nv_bfloat16* hi, const __nv_bfloat16* lo, long long row_stride, int C, int HW,
                           int rows, float* out, cudaStream_t s) {
  if (rows <= 0) return;
  const long long D = static_cast<long long>(C) * HW;
  int gy = static_cast<int>((D + 255) / 256);
  if (gy > 128) gy = 128;
  launch_pdl(planes_to_nchw_kernel, dim3(rows, gy), dim3(256), 0, s, hi, lo, row_stride, C, HW, out);
}

void launch_mlp_head(const __nv_bfloat16* hi, const __nv_bfloat16* lo, int dp, int dim, const float* W, const float* b,
                     int classes, const int* ids, const int* count, int max_rows, int* base_pred, float* logits_out,
                     int* exit_layer, int* served, unsigned long long* exit_ns, cudaStream_t s) {
  if (max_rows <= 0) return;
  const size_t smem = static_cast<size_t>(dim + classes) * sizeof(float);
  launch_pdl(base_head_kernel<false>, dim3(max_rows), dim3(kLk), smem, s, hi, lo, dp, dim, 1, W, b, classes, ids, count, base_pred,
                                                      logits_out, exit_layer, served, exit_ns, nullptr, 0, 0);
}

void launch_cnn_head(const __nv_bfloat16* hi, const __nv_bfloat16* lo, int C, int HW, const float* W, const float* b,
                     int classes, const int* ids, const int* count, int max_rows, int* base_pred, float* logits_out,
                     int* exit_layer, int* served, unsigned long long* exit_ns, float* feats_scratch,
                     float* logits_scratch, cudaStream_t s) {
  if (max_rows <= 0) return;
  const float* pre = nullptr;
  if (classes > 32 && feats_scratch && logits_scratch) {
    // Many classes: GAP rows, one batched logits GEMM, then the per-row softmax/argmax.
    launch_pdl(gap_rows_kernel, dim3(max_rows), dim3(kLk), static_cast<size_t>(C) * sizeof(float), s, hi, lo, C, HW, ids, count,
                                                                                  feats_scratch);
    launch_rows_fc(feats_scratch, C, 0, 0, nullptr, C, W, classes, count, max_rows, logits_scratch, s);
    pre = logits_scratch;
  }
  const size_t smem = static_cast<size_t>(C + classes) * sizeof(float);
  launch_pdl(base_head_kernel<true>, dim3(max_rows), dim3(kLk), smem, s, hi, lo, static_cast<long long>(C) * HW, C, HW, W, b, classes, ids,
                                                     count, base_pred, logits_out, exit_layer, served, exit_ns, pre,
                                                     rows_fc_splits(C), static_cast<long long>(max_rows) * classes);
}

void launch_stem_im2col(const float* x, const int* count, int max_n, int C, int H, int W, int k, int stride, int pad,
                        int Ho, int Wo, int Kp, __nv_bfloat16* hi, __nv_bfloat16* lo, cudaStream_t s) {
  const long long total = static_cast<long long>(max_n) * Ho * Wo * (Kp / 8);
  long long blocks = (total + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  if (blocks < 1) blocks = 1;
  launch_pdl(stem_im2col_kernel, dim3(static_cast<int>(blocks)), dim3(256), 0, s, x, count, C, H, W, k, stride, pad, Ho, Wo, Kp, hi, lo);
}

void launch_phase_split(const __nv_bfloat16* hi, const __nv_bfloat16* lo, int H, int W, int C, int N, int Hs, int Ws,
                        const int* ids, const int* count, int max_rows, __nv_bfloat16* ohi, __nv_bfloat16* olo,
                        cudaStream_t s) {
  if (max_rows <= 0) return;
  const long long per = 4LL * Hs * Ws * (C / 8);
  int gy = static_cast<int>((per + 255) / 256);
  if (gy > 64) gy = 64;
  launch_pdl(phase_split_kernel, dim3(dim3(max_rows, gy)), dim3(256), 0, s, hi, lo, H, W, C, N, Hs, Ws, ids, count, ohi, olo);
}

void launch_maxpool(const __nv_bfloat16* hi, const __nv_bfloat16* lo, int H, int W, int C, int k, int stride, int pad,
                    int Ho, int Wo, const int* ids, const int* count, int max_rows, __nv_bfloat16* ohi,
                    __nv_bfloat16* olo, cudaStream_t s) {
  if (max_rows <= 0) return;
  const long long per = static_cast<long long>(Ho) * Wo * (C / 8);
  int gy = static_cast<int>((per + 255) / 256);
  if (gy > 128) gy = 128;
  if (k == 3)
    launch_pdl(maxpool_kernel<3>, dim3(max_rows, gy), dim3(256), 0, s, hi, lo, H, W, C, k, stride, pad, Ho, Wo, ids,
               count, ohi, olo);
  else
    launch_pdl(maxpool_kernel<0>, dim3(max_rows, gy), dim3(256), 0, s, hi, lo, H, W, C, k, stride, pad, Ho, Wo, ids,
               count, ohi, olo);
}

void launch_set_int(int* p, int v, cudaStream_t s) { launch_pdl(set_int_kernel, dim3(1), dim3(1), 0, s, p, v); }

void launch_stamp_start(unsigned long long* t0, cudaStream_t s) { launch_pdl(stamp_kernel, dim3(1), dim3(1), 0, s, t0); }

void launch_init_batch(int B, int* batch_out, int max_batch, int* ids0, int* count0, int* rows_out, int rows_mult,
                       int* exit_layer, int* served, int* base_pred, unsigned long long* exit_ns, float* probs, int L,
                       unsigned long long* t0, cudaStream_t s) {
  const int blocks = (max_batch + 255) / 256 > 0 ? (max_batch + 255) / 256 : 1;
  launch_pdl(init_batch_kernel, dim3(blocks), dim3(256), 0, s, B, batch_out, max_batch, ids0, count0, rows_out,
             rows_mult, exit_layer, served, base_pred, exit_ns, probs, L, t0);
}

const void* init_batch_kernel_fn() { return reinterpret_cast<const void*>(&init_batch_kernel); }

}  // namespace lcb
