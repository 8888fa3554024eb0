// Serve-path kernels (see serve_kernels.cuh). All cache-head arithmetic is
// fp32 with deterministic (fixed-order) reductions; only the activations are
// bf16 hi (+lo) planes.
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

// Fused-GAP bins: bin c = (sum over the tap conv's segment partials, fixed
// order) x 1/HW; the partials were written by tc_conv's epilogue.
__global__ void gap_bins_kernel(const float* gap, int segs, int C, float inv, const int* data_idx, const int* count,
                                float* bins) {
  const int r = blockIdx.x;
  if (r >= *count) return;
  const long long n = data_idx ? data_idx[r] : r;
  const float* src = gap + n * segs * C;
  for (int c = blockIdx.y * blockDim.x + threadIdx.x; c < C; c += gridDim.y * blockDim.x) {
    float a = 0.0f;
    for (int sg = 0; sg < segs; ++sg) a += src[static_cast<long long>(sg) * C + c];
    bins[static_cast<long long>(r) * C + c] = a * inv;
  }
}

// Generic: one thread per bin, sequential over its flat window.
__global__ void pool_generic_kernel(TapView t, int win, int width, float inv, float* bins) {
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
// tensor-core GEMM). Every 16-row tile reads its W slice once instead of
// once per row: the logits GEMM of heads with many classes (ImageNet).
constexpr int kFcBM = 16, kFcBN = 64, kFcBK = 32;

template <int kMode>
__global__ void __launch_bounds__(256) rows_fc_kernel(const float* A, long long lda, int ks, long long part_stride,
                                                      const float* b1, int feat, int kslice, const float* W,
                                                      int classes, const int* count, long long max_rows, float* out) {
  __shared__ float As[kFcBM][kFcBK + 1];
  __shared__ float Ws[kFcBN][kFcBK + 1];
  const int n = *count;
  const int r0 = blockIdx.y * kFcBM, k0 = blockIdx.x * kFcBN;
  if (r0 >= n) return;
  const int z = blockIdx.z;
  const int oz0 = z * kslice, oz1 = oz0 + kslice < feat ? oz0 + kslice : feat;
  const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5;
  float acc[2][2] = {{0.0f, 0.0f}, {0.0f, 0.0f}};
  for (int o0 = oz0; o0 < oz1; o0 += kFcBK) {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int idx = tid + i * 256, rr = idx >> 5, oo = idx & 31;
      const int r = r0 + rr, o = o0 + oo;
      float v = 0.0f;
      if (r < n && o < oz1) {
        if (kMode == 0) {
          v = A[static_cast<long long>(r) * lda + o];
        } else {
          float a = b1[o];
          for (int s = 0; s < ks; ++s) a += A[static_cast<long long>(s) * part_stride + static_cast<long long>(r) * lda + o];
          v = a > 0.0f ? a : 0.0f;
        }
      }
      As[rr][oo] = v;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int idx = tid + i * 256, kk = idx >> 5, oo = idx & 31;
      const int k = k0 + kk, o = o0 + oo;
      Ws[kk][oo] = (k < classes && o < oz1) ? W[static_cast<long long>(k) * feat + o] : 0.0f;
    }
    __syncthreads();
    const int olim = oz1 - o0 < kFcBK ? oz1 - o0 : kFcBK;
    for (int o = 0; o < olim; ++o) {
      const float a0 = As[2 * ty][o], a1 = As[2 * ty + 1][o];
      const float w0 = Ws[tx][o], w1 = Ws[tx + 32][o];
      acc[0][0] += a0 * w0;
      acc[0][1] += a0 * w1;
      acc[1][0] += a1 * w0;
      acc[1][1] += a1 * w1;
    }
    __syncthreads();
  }
  float* outz = out + static_cast<long long>(z) * max_rows * classes;
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int r = r0 + 2 * ty + i;
    if (r >= n) continue;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int k = k0 + tx + 32 * j;
      if (k < classes) outz[static_cast<long long>(r) * classes + k] = acc[i][j];
    }
  }
}

__device__ __forceinline__ float fc_logit(const float* part, int nz, long long zstride, const float* b, int r,
                                          int classes, int k) {
  float a = b[k];
  for (int z = 0; z < nz; ++z) a += part[z * zstride + static_cast<long long>(r) * classes + k];
  return a;
}

// Global average pool of the surviving images' final activations (NHWC,
// image ids[r]) -> feats [rows][C]; per channel a sequential pixel sum, then
// x (1/HW) as the base head's GAP.
__global__ void gap_rows_kernel(const __nv_bfloat16* hi, const __nv_bfloat16* lo, int C, int HW, const int* ids,
                                const int* count, float* feats) {
  const int r = blockIdx.x;
  if (r >= *count) return;
  const long long n = ids[r];
  TapView t;
  t.hi = hi;
  t.lo = lo;
  const float inv = 1.0f / HW;
  for (int c = blockIdx.y * blockDim.x + threadIdx.x; c < C; c += gridDim.y * blockDim.x) {
    float a = 0.0f;
    for (int q = 0; q < HW; ++q) a += ld_tap(t, (n * HW + q) * C + c);
    feats[static_cast<long long>(r) * C + c] = a * inv;
  }
}

// ------------------------------------------------------------------ head
// Reference lookup (cache.cpp:259-265): pr = softmax(pred(tap)),
// p = sigmoid(sel(pr)), hit = p >= delta (inclusive); label = argmax(pr).
__global__ void cache_head_kernel(CacheHeadParams p) {
  extern __shared__ float sm[];
  __shared__ float red[32];
  __shared__ float hsel[16];
  __shared__ int best_idx_s[4];
  __shared__ float best_val_s[4];
  const int r = blockIdx.x;
  if (r >= *p.count) return;
  const int C = p.classes;
  float* logits = sm;        // [C]
  float* feat = sm + C;      // [feat]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;

  if (p.pre_logits) {
    for (int k = tid; k < C; k += blockDim.x) logits[k] = fc_logit(p.pre_logits, p.pre_nz, p.pre_zstride, p.b2, r, C, k);
  } else if (p.family == 2) {
    for (int k = tid; k < C; k += blockDim.x) {
      float a = p.b2[k];
      for (int c = 0; c < p.feat; ++c) a += p.feats[(static_cast<long long>(r) * p.feat + c) * C + k];
      logits[k] = a;
    }
  } else {
    if (p.family == 1) {
      for (int o = tid; o < p.feat; o += blockDim.x) feat[o] = p.feats[static_cast<long long>(r) * p.feat + o];
    } else {
      for (int j = tid; j < p.feat; j += blockDim.x) {
        float a = p.b1[j];
        for (int s = 0; s < p.ks; ++s) a += p.feats[(static_cast<long long>(s) * p.rows_total + r) * p.hp + j];
        feat[j] = a > 0.0f ? a : 0.0f;
      }
    }
    __syncthreads();
    for (int k = warp; k < C; k += nw) {
      const float* wr = p.W2 + static_cast<long long>(k) * p.feat;
      float a = 0.0f;
      for (int o = lane; o < p.feat; o += 32) a += wr[o] * feat[o];
      a = warp_sum(a);
      if (lane == 0) logits[k] = a + p.b2[k];
    }
  }
  __syncthreads();
  // softmax (losses.cpp:35-46)
  float m = -FLT_MAX;
  for (int k = tid; k < C; k += blockDim.x) m = fmaxf(m, logits[k]);
  m = block_max(m, red);
  float part = 0.0f;
  for (int k = tid; k < C; k += blockDim.x) part += expf(logits[k] - m);
  const float sum = block_sum(part, red);
  float* pr = feat;  // reuse
  __syncthreads();
  for (int k = tid; k < C; k += blockDim.x) pr[k] = expf(logits[k] - m) / sum;
  __syncthreads();
  // selector FC(C,16) + ReLU
  for (int j = warp; j < 16; j += nw) {
    const float* wr = p.Ws1 + j * C;
    float a = 0.0f;
    for (int k = lane; k < C; k += 32) a += wr[k] * pr[k];
    a = warp_sum(a);
    if (lane == 0) {
      a += p.bs1[j];
      hsel[j] = a > 0.0f ? a : 0.0f;
    }
  }
  // argmax(pr), lowest index on ties (tensor.hpp:57-63)
  float bv = -FLT_MAX;
  int bi = 0x7fffffff;
  for (int k = tid; k < C; k += blockDim.x) {
    if (pr[k] > bv) {
      bv = pr[k];
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
    best_val_s[warp] = bv;
    best_idx_s[warp] = bi;
  }
  __syncthreads();
  if (tid == 0) {
    float v = best_val_s[0];
    int i = best_idx_s[0];
    for (int w = 1; w < nw; ++w)
      if (best_val_s[w] > v || (best_val_s[w] == v && best_idx_s[w] < i)) {
        v = best_val_s[w];
        i = best_idx_s[w];
      }
    float z = p.bs2;
    for (int j = 0; j < 16; ++j) z += p.ws2[j] * hsel[j];
    float q;
    if (z >= 0.0f) {
      q = 1.0f / (1.0f + expf(-z));
    } else {
      const float e = expf(z);
      q = e / (1.0f + e);
    }
    p.prob[r] = q;
    p.hit[r] = static_cast<double>(q) >= p.delta ? 1 : 0;
    p.label[r] = i;
  }
  if (p.pr_out)
    for (int k = tid; k < C; k += blockDim.x) p.pr_out[static_cast<long long>(r) * C + k] = pr[k];
  if (p.logits_out)
    for (int k = tid; k < C; k += blockDim.x) p.logits_out[static_cast<long long>(r) * C + k] = logits[k];
}

// Warp-per-row form of the same head for classes <= 32 (no block barriers):
// lane k owns class k; features are streamed lane-strided.
__global__ void cache_head_warp_kernel(CacheHeadParams p) {
  extern __shared__ float smw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = blockIdx.x * (blockDim.x >> 5) + warp;
  if (r >= *p.count) return;
  const int C = p.classes;
  float logit = -FLT_MAX;
  if (p.family == 2) {
    if (lane < C) {
      float a = p.b2[lane];
      for (int c = 0; c < p.feat; ++c) a += p.feats[(static_cast<long long>(r) * p.feat + c) * C + lane];
      logit = a;
    }
  } else {
    float* feat = smw + warp * p.feat;
    if (p.family == 1) {
      for (int o = lane; o < p.feat; o += 32) feat[o] = p.feats[static_cast<long long>(r) * p.feat + o];
    } else {
      for (int j = lane; j < p.feat; j += 32) {
        float a = p.b1[j];
        for (int s = 0; s < p.ks; ++s) a += p.feats[(static_cast<long long>(s) * p.rows_total + r) * p.hp + j];
        feat[j] = a > 0.0f ? a : 0.0f;
      }
    }
    __syncwarp();
    for (int k = 0; k < C; ++k) {
      const float* wr = p.W2 + static_cast<long long>(k) * p.feat;
      float a = 0.0f;
      for (int o = lane; o < p.feat; o += 32) a += wr[o] * feat[o];
      a = warp_sum(a);
      if (lane == k) logit = a + p.b2[k];
    }
  }
  const float m = warp_max(lane < C ? logit : -FLT_MAX);
  const float e = lane < C ? expf(logit - m) : 0.0f;
  const float sum = warp_sum(e);
  const float pr = lane < C ? e / sum : 0.0f;
  // selector FC(C,16) + ReLU: lane j < 16 owns hidden unit j
  float h = 0.0f;
  {
    float a = lane < 16 ? p.bs1[lane] : 0.0f;
    for (int k = 0; k < C; ++k) {
      const float pk = __shfl_sync(0xffffffffu, pr, k);
      if (lane < 16) a += p.Ws1[lane * C + k] * pk;
    }
    h = (lane < 16 && a > 0.0f) ? a : 0.0f;
  }
  const float z = warp_sum(lane < 16 ? p.ws2[lane] * h : 0.0f) + p.bs2;
  // argmax(pr), lowest index on ties
  float bv = lane < C ? pr : -FLT_MAX;
  int bi = lane < C ? lane : 0x7fffffff;
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
    float q;
    if (z >= 0.0f) {
      q = 1.0f / (1.0f + expf(-z));
    } else {
      const float ez = expf(z);
      q = ez / (1.0f + ez);
    }
    p.prob[r] = q;
    p.hit[r] = static_cast<double>(q) >= p.delta ? 1 : 0;
    p.label[r] = bi;
  }
  if (lane < C) {
    if (p.pr_out) p.pr_out[static_cast<long long>(r) * C + lane] = pr;
    if (p.logits_out) p.logits_out[static_cast<long long>(r) * C + lane] = logit;
  }
}

// ------------------------------------------------------------------ fused lookup + exit
// One launch per cache layer for Pool(C) = GAP caches with <= 32 classes:
// every warp owns rows (bins from tc_conv's fused GAP partials, FC(C,classes),
// softmax, selector FC(C,16)+ReLU+FC(16,1), sigmoid, >= delta, argmax — the
// arithmetic and summation order of gap_bins_kernel + cache_head_warp_kernel);
// per-row decisions go to global scratch and the LAST CTA to finish (arrival
// counter) runs the first-hit record + stable compaction of exit_compact_kernel.
constexpr int kFusedMaxC = 1024;

__global__ void __launch_bounds__(512) gap_lookup_exit_kernel(FusedLookupParams p) {
  __shared__ int warp_tot[32];
  __shared__ int base_s;
  __shared__ int last_s;
  const int n_rows = *p.count_in;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int C = p.C, K = p.classes;
  for (int r = blockIdx.x * nw + warp; r < n_rows; r += gridDim.x * nw) {
    const long long n = p.ids_in[r];
    const float* src = p.gap + n * p.segs * C;
    // bins (gap_bins_kernel order), lane-strided channels
    // 4 independent partial sums over the segments (fixed combination order)
    float f[kFusedMaxC / 32];
#pragma unroll
    for (int j = 0; j < kFusedMaxC / 32; ++j) {
      const int c = lane + 32 * j;
      float a = 0.0f;
      if (c < C) {
        float a0 = 0.0f, a1 = 0.0f, a2 = 0.0f, a3 = 0.0f;
        int sg = 0;
        for (; sg + 4 <= p.segs; sg += 4) {
          const float* q = src + static_cast<long long>(sg) * C + c;
          a0 += __ldg(q);
          a1 += __ldg(q + C);
          a2 += __ldg(q + 2 * C);
          a3 += __ldg(q + 3 * C);
        }
        for (; sg < p.segs; ++sg) a0 += __ldg(src + static_cast<long long>(sg) * C + c);
        a = ((a0 + a1) + (a2 + a3)) * p.inv;
      }
      f[j] = a;
    }
    // logits (cache_head_warp_kernel order)
    float logit = -FLT_MAX;
    for (int k = 0; k < K; ++k) {
      const float* wr = p.W2 + static_cast<long long>(k) * C;
      float a = 0.0f;
#pragma unroll
      for (int j = 0; j < kFusedMaxC / 32; ++j) {
        const int c = lane + 32 * j;
        if (c < C) a += wr[c] * f[j];
      }
      a = warp_sum(a);
      if (lane == k) logit = a + p.b2[k];
    }
    const float m = warp_max(lane < K ? logit : -FLT_MAX);
    const float e = lane < K ? expf(logit - m) : 0.0f;
    const float sum = warp_sum(e);
    const float pr = lane < K ? e / sum : 0.0f;
    float h = 0.0f;
    {
      float a = lane < 16 ? p.bs1[lane] : 0.0f;
      for (int k = 0; k < K; ++k) {
        const float pk = __shfl_sync(0xffffffffu, pr, k);
        if (lane < 16) a += p.Ws1[lane * K + k] * pk;
      }
      h = (lane < 16 && a > 0.0f) ? a : 0.0f;
    }
    const float z = warp_sum(lane < 16 ? p.ws2[lane] * h : 0.0f) + p.bs2;
    float bv = lane < K ? pr : -FLT_MAX;
    int bi = lane < K ? lane : 0x7fffffff;
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
      float q;
      if (z >= 0.0f) {
        q = 1.0f / (1.0f + expf(-z));
      } else {
        const float ez = expf(z);
        q = ez / (1.0f + ez);
      }
      p.prob[r] = q;
      p.hit[r] = static_cast<double>(q) >= p.delta ? 1 : 0;
      p.label[r] = bi;
    }
  }
  // last CTA: first-hit records + stable compaction over all rows
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last_s = (atomicAdd(p.arrive, 1) == static_cast<int>(gridDim.x) - 1) ? 1 : 0;
  __syncthreads();
  if (!last_s) return;
  __threadfence();
  if (threadIdx.x == 0) {
    base_s = 0;
    *p.arrive = 0;
  }
  __syncthreads();
  const unsigned long long now = globaltimer();
  const int tid = threadIdx.x;
  for (int c0 = 0; c0 < n_rows; c0 += blockDim.x) {
    const int r = c0 + tid;
    const bool valid = r < n_rows;
    const bool hit = valid && __ldcg(p.hit + r);
    const int id = valid ? p.ids_in[r] : -1;
    if (valid) {
      if (p.probs_out) p.probs_out[id] = __ldcg(p.prob + r);
      if (hit && p.exit_layer[id] == 0) {
        p.exit_layer[id] = p.layer;
        p.served[id] = __ldcg(p.label + r);
        p.exit_ns[id] = now;
      }
    }
    const bool keep = valid && (p.shadow || !hit);
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
      if (lane < nw) warp_tot[lane] = v;
    }
    __syncthreads();
    const int warp_off = warp == 0 ? 0 : warp_tot[warp - 1];
    const int base = base_s;
    if (keep) p.ids_out[base + warp_off + pos_in_warp] = id;
    __syncthreads();
    if (tid == 0) base_s = base + warp_tot[nw - 1];
    __syncthreads();
  }
  if (tid == 0) *p.count_out = base_s;
}

// ------------------------------------------------------------------ exit
__global__ void exit_compact_kernel(int layer, const int* count_in, const int* ids_in, const int* hit, const int* label,
                                    const float* prob, int* exit_layer, int* served, unsigned long long* exit_ns,
                                    float* probs_out, int* ids_out, int* src_rows_out, int* count_out, int shadow) {
  __shared__ int warp_tot[32];
  __shared__ int base_s;
  const int n = *count_in;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) base_s = 0;
  __syncthreads();
  const unsigned long long now = globaltimer();
  for (int c0 = 0; c0 < n; c0 += blockDim.x) {
    const int r = c0 + tid;
    const bool valid = r < n;
    const bool h = valid && hit[r];
    const int id = valid ? ids_in[r] : -1;
    if (valid) {
      if (probs_out) probs_out[id] = prob[r];
      if (h && exit_layer[id] == 0) {
        exit_layer[id] = layer;
        served[id] = label[r];
        exit_ns[id] = now;
      }
    }
    const bool keep = valid && (shadow || !h);
    const unsigned mask = __ballot_sync(0xffffffffu, keep);
    const int pos_in_warp = __popc(mask & ((1u << lane) - 1u));
    if (lane == 0) warp_tot[warp] = __popc(mask);
    __syncthreads();
    if (warp == 0) {
      const int nw = blockDim.x >> 5;
      int v = lane < nw ? warp_tot[lane] : 0;
      // inclusive scan
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += u;
      }
      if (lane < nw) warp_tot[lane] = v;  // inclusive prefix
    }
    __syncthreads();
    const int warp_off = warp == 0 ? 0 : warp_tot[warp - 1];
    const int base = base_s;
    if (keep) {
      ids_out[base + warp_off + pos_in_warp] = id;
      if (src_rows_out) src_rows_out[base + warp_off + pos_in_warp] = r;
    }
    __syncthreads();
    if (tid == 0) base_s = base + warp_tot[(blockDim.x >> 5) - 1];
    __syncthreads();
  }
  if (tid == 0) *count_out = base_s;
}

__global__ void gather_rows_kernel(const __nv_bfloat16* src_hi, const __nv_bfloat16* src_lo, __nv_bfloat16* dst_hi,
                                   __nv_bfloat16* dst_lo, long long row_elems, const int* src_rows, const int* count) {
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
  const int j = blockIdx.x;
  if (j >= *count) return;
  const long long src = ids ? ids[j] : j;
  for (int i = threadIdx.x; i < dp; i += blockDim.x) {
    const float v = i < in_dim ? x[src * in_dim + i] : 0.0f;
    split_store(v, hi, lo, static_cast<long long>(j) * dp + i);
  }
}

__global__ void split_taps_nchw_kernel(const float* x, int C, int HW, long long row_stride, __nv_bfloat16* hi,
                                       __nv_bfloat16* lo) {
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

// Base head (base_model.cpp:48-49): logits -> softmax -> argmax (serving.cpp:108).
template <bool kGap>
__global__ void base_head_kernel(const __nv_bfloat16* hi, const __nv_bfloat16* lo, long long row_stride, int C, int HW,
                                 const float* W, const float* b, int classes, const int* ids, const int* count,
                                 int* base_pred, float* logits_out, int* exit_layer, int* served,
                                 unsigned long long* exit_ns, const float* pre_logits, int pre_nz,
                                 long long pre_zstride) {
  extern __shared__ float sm[];
  __shared__ float red[32];
  __shared__ int bi_s[32];
  __shared__ float bv_s[32];
  const int r = blockIdx.x;
  if (r >= *count) return;
  const int id = ids[r];
  const long long n = kGap ? id : r;
  float* feat = sm;          // [C]
  float* logits = sm + C;    // [classes]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  TapView t;
  t.hi = hi;
  t.lo = lo;
  if (pre_logits) {
    for (int k = tid; k < classes; k += blockDim.x) logits[k] = fc_logit(pre_logits, pre_nz, pre_zstride, b, r, classes, k);
  }
  for (int c = tid; c < C && !pre_logits; c += blockDim.x) {
    if (kGap) {
      float a = 0.0f;
      for (int q = 0; q < HW; ++q) a += ld_tap(t, n * row_stride + static_cast<long long>(q) * C + c);
      feat[c] = a * (1.0f / HW);
    } else {
      feat[c] = ld_tap(t, n * row_stride + c);
    }
  }
  __syncthreads();
  for (int k = warp; k < classes && !pre_logits; k += nw) {
    const float* wr = W + static_cast<long long>(k) * C;
    float a = 0.0f;
    for (int c = lane; c < C; c += 32) a += wr[c] * feat[c];
    a = warp_sum(a);
    if (lane == 0) logits[k] = a + b[k];
  }
  __syncthreads();
  float m = -FLT_MAX;
  for (int k = tid; k < classes; k += blockDim.x) m = fmaxf(m, logits[k]);
  m = block_max(m, red);
  float part = 0.0f;
  for (int k = tid; k < classes; k += blockDim.x) part += expf(logits[k] - m);
  const float sum = block_sum(part, red);
  float bv = -FLT_MAX;
  int bi = 0x7fffffff;
  for (int k = tid; k < classes; k += blockDim.x) {
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
    for (int k = tid; k < classes; k += blockDim.x) logits_out[static_cast<long long>(id) * classes + k] = logits[k];
}

// One thread per (output pixel, 8 consecutive K entries): 16-byte stores.
__global__ void stem_im2col_kernel(const float* x, const int* count, int C, int H, int W, int k, int stride, int pad,
                                   int Ho, int Wo, int Kp, __nv_bfloat16* hi, __nv_bfloat16* lo) {
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

__global__ void maxpool_kernel(const __nv_bfloat16* hi, const __nv_bfloat16* lo, int H, int W, int C, int k, int stride,
                               int pad, int Ho, int Wo, const int* ids, const int* count, __nv_bfloat16* ohi,
                               __nv_bfloat16* olo) {
  // One thread per (output pixel, 8 channels): 16-byte loads/stores; per
  // channel the first maximum in (r, s) order wins (hi and lo move together).
  const int j = blockIdx.x;
  if (j >= *count) return;
  const long long n = ids[j];
  const int c8n = C / 8;
  const long long per = static_cast<long long>(Ho) * Wo * c8n;
  for (long long i = blockIdx.y * blockDim.x + threadIdx.x; i < per; i += gridDim.y * blockDim.x) {
    const int c8 = static_cast<int>(i % c8n);
    const long long pix = i / c8n;
    const int ow = static_cast<int>(pix % Wo), oh = static_cast<int>(pix / Wo);
    float best[8];
    uint4 bh = make_uint4(0, 0, 0, 0), bl = make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int e = 0; e < 8; ++e) best[e] = -FLT_MAX;
    for (int r = 0; r < k; ++r) {
      const int ih = oh * stride + r - pad;
      if (ih < 0 || ih >= H) continue;
      for (int s2 = 0; s2 < k; ++s2) {
        const int iw = ow * stride + s2 - pad;
        if (iw < 0 || iw >= W) continue;
        const long long src = ((n * H + ih) * W + iw) * C + c8 * 8;
        const uint4 vh = *reinterpret_cast<const uint4*>(hi + src);
        const uint4 vl = lo ? *reinterpret_cast<const uint4*>(lo + src) : make_uint4(0, 0, 0, 0);
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
    const long long dst = ((n * Ho + oh) * Wo + ow) * C + c8 * 8;
    *reinterpret_cast<uint4*>(ohi + dst) = bh;
    if (olo) *reinterpret_cast<uint4*>(olo + dst) = bl;
  }
}

__global__ void stamp_kernel(unsigned long long* t0) { *t0 = globaltimer(); }

__global__ void init_batch_kernel(const int* batch, int max_batch, int* ids0, int* count0, int* rows_out, int rows_mult,
                                  int* exit_layer, int* served, int* base_pred, unsigned long long* exit_ns,
                                  float* probs, int L) {
  const int B = *batch;
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
    if (rows_out) *rows_out = B * rows_mult;
  }
}

}  // namespace

void launch_pool_bins(const TapView& tap, int max_rows, int win, int width, float* bins, cudaStream_t s) {
  const float inv = static_cast<float>(1.0 / win);
  if (max_rows <= 0) return;
  if (tap.HW > 1 && tap.C % 64 == 0 && win <= tap.HW && tap.HW % win == 0 && tap.HW / win >= 32) {
    pool_strips_kernel<<<dim3(max_rows, tap.C / 64), 256, 0, s>>>(tap, win, width, inv, bins);
  } else if (tap.HW > 1 && tap.C % 64 == 0 && win % tap.HW == 0 && 64 % (win / tap.HW) == 0) {
    pool_channels_kernel<<<dim3(max_rows, tap.C / 64), 256, 0, s>>>(tap, win / tap.HW, width, inv, bins);
  } else {
    const int gy = (width + 255) / 256 < 64 ? (width + 255) / 256 : 64;
    pool_generic_kernel<<<dim3(max_rows, gy), 256, 0, s>>>(tap, win, width, inv, bins);
  }
}

void launch_gap_bins(const float* gap, int segs, int C, int HW, const int* data_idx, const int* count, int max_rows,
                     float* bins, cudaStream_t s) {
  if (max_rows <= 0) return;
  const float inv = static_cast<float>(1.0 / HW);
  gap_bins_kernel<<<dim3(max_rows, (C + 255) / 256), 256, 0, s>>>(gap, segs, C, inv, data_idx, count, bins);
}

void launch_conv1d_partials(const TapView& tap, int max_rows, long long D, int kernel, int stride, int out_dim,
                            const float* w1, float b1, const float* W2, int classes, int chunk_elems, int nchunks,
                            float* partials, cudaStream_t s) {
  if (max_rows <= 0) return;
  const size_t smem = static_cast<size_t>(chunk_elems + kernel) * sizeof(float);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(conv1d_partials_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  conv1d_partials_kernel<<<dim3(max_rows, nchunks), 256, smem, s>>>(tap, D, kernel, stride, out_dim, w1, b1, W2,
                                                                    classes, chunk_elems, nchunks, partials);
}

int rows_fc_splits(int feat) { return (feat + kRowsFcSlice - 1) / kRowsFcSlice; }

void launch_rows_fc(const float* A, long long lda, int ks, long long part_stride, const float* b1, int feat,
                    const float* W, int classes, const int* count, int max_rows, float* out, cudaStream_t s) {
  if (max_rows <= 0) return;
  const dim3 grid((classes + kFcBN - 1) / kFcBN, (max_rows + kFcBM - 1) / kFcBM, rows_fc_splits(feat));
  if (ks > 0)
    rows_fc_kernel<1><<<grid, 256, 0, s>>>(A, lda, ks, part_stride, b1, feat, kRowsFcSlice, W, classes, count,
                                           max_rows, out);
  else
    rows_fc_kernel<0><<<grid, 256, 0, s>>>(A, lda, 0, 0, nullptr, feat, kRowsFcSlice, W, classes, count, max_rows,
                                           out);
}

void launch_cache_head(const CacheHeadParams& p_in, int max_rows, cudaStream_t s) {
  if (max_rows <= 0) return;
  CacheHeadParams p = p_in;
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
  }
  if (!p.pre_logits && p.classes <= 32 && (p.family == 2 || p.feat <= 4096)) {
    const int warps = 4;
    const size_t smem = p.family == 2 ? 0 : static_cast<size_t>(warps) * p.feat * sizeof(float);
    static bool wattr = false;
    if (!wattr) {
      cudaFuncSetAttribute(cache_head_warp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      wattr = true;
    }
    cache_head_warp_kernel<<<(max_rows + warps - 1) / warps, 32 * warps, smem, s>>>(p);
    return;
  }
  const int feat_len = (p.family == 2 || p.pre_logits) ? p.classes : (p.feat > p.classes ? p.feat : p.classes);
  const size_t smem = static_cast<size_t>(p.classes + feat_len) * sizeof(float);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(cache_head_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  cache_head_kernel<<<max_rows, 128, smem, s>>>(p);
}

bool fused_lookup_supported(int classes, int C, int max_rows) {
  return classes <= 32 && C <= kFusedMaxC && max_rows > 0;
}

void launch_gap_lookup_exit(const FusedLookupParams& p, int max_rows, cudaStream_t s) {
  const int warps = 16;
  int grid = (max_rows + warps - 1) / warps;
  if (grid > 148) grid = 148;
  gap_lookup_exit_kernel<<<grid, warps * 32, 0, s>>>(p);
}

void launch_exit_compact(int layer, const int* count_in, const int* ids_in, const int* hit, const int* label,
                         const float* prob, int* exit_layer, int* served, unsigned long long* exit_ns, float* probs_out,
                         int* ids_out, int* src_rows_out, int* count_out, int shadow, cudaStream_t s) {
  exit_compact_kernel<<<1, 1024, 0, s>>>(layer, count_in, ids_in, hit, label, prob, exit_layer, served, exit_ns,
                                         probs_out, ids_out, src_rows_out, count_out, shadow);
}

void launch_gather_rows(const __nv_bfloat16* src_hi, const __nv_bfloat16* src_lo, __nv_bfloat16* dst_hi,
                        __nv_bfloat16* dst_lo, long long row_elems, const int* src_rows, const int* count, int max_rows,
                        cudaStream_t s) {
  if (max_rows <= 0) return;
  const long long nv = row_elems / 8;
  int gy = static_cast<int>((nv + 255) / 256);
  if (gy > 64) gy = 64;
  gather_rows_kernel<<<dim3(max_rows, gy), 256, 0, s>>>(src_hi, src_lo, dst_hi, dst_lo, row_elems, src_rows, count);
}

void launch_split_rows(const float* x, int in_dim, int dp, const int* ids, const int* count, int max_rows,
                       __nv_bfloat16* hi, __nv_bfloat16* lo, cudaStream_t s) {
  if (max_rows <= 0) return;
  split_rows_kernel<<<max_rows, 256, 0, s>>>(x, in_dim, dp, ids, count, hi, lo);
}

void launch_split_taps_nchw(const float* x, int C, int HW, int rows, long long row_stride, __nv_bfloat16* hi,
                            __nv_bfloat16* lo, cudaStream_t s) {
  if (rows <= 0) return;
  int gy = static_cast<int>((row_stride + 255) / 256);
  if (gy > 128) gy = 128;
  split_taps_nchw_kernel<<<dim3(rows, gy), 256, 0, s>>>(x, C, HW, row_stride, hi, lo);
}

void launch_mlp_head(const __nv_bfloat16* hi, const __nv_bfloat16* lo, int dp, int dim, const float* W, const float* b,
                     int classes, const int* ids, const int* count, int max_rows, int* base_pred, float* logits_out,
                     int* exit_layer, int* served, unsigned long long* exit_ns, cudaStream_t s) {
  if (max_rows <= 0) return;
  const size_t smem = static_cast<size_t>(dim + classes) * sizeof(float);
  base_head_kernel<false><<<max_rows, 128, smem, s>>>(hi, lo, dp, dim, 1, W, b, classes, ids, count, base_pred,
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
    int gy = (C + 255) / 256;
    gap_rows_kernel<<<dim3(max_rows, gy), 256, 0, s>>>(hi, lo, C, HW, ids, count, feats_scratch);
    launch_rows_fc(feats_scratch, C, 0, 0, nullptr, C, W, classes, count, max_rows, logits_scratch, s);
    pre = logits_scratch;
  }
  const size_t smem = static_cast<size_t>(C + classes) * sizeof(float);
  base_head_kernel<true><<<max_rows, 256, smem, s>>>(hi, lo, static_cast<long long>(C) * HW, C, HW, W, b, classes, ids,
                                                     count, base_pred, logits_out, exit_layer, served, exit_ns, pre,
                                                     rows_fc_splits(C), static_cast<long long>(max_rows) * classes);
}

void launch_stem_im2col(const float* x, const int* count, int max_n, int C, int H, int W, int k, int stride, int pad,
                        int Ho, int Wo, int Kp, __nv_bfloat16* hi, __nv_bfloat16* lo, cudaStream_t s) {
  const long long total = static_cast<long long>(max_n) * Ho * Wo * (Kp / 8);
  long long blocks = (total + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  if (blocks < 1) blocks = 1;
  stem_im2col_kernel<<<static_cast<int>(blocks), 256, 0, s>>>(x, count, C, H, W, k, stride, pad, Ho, Wo, Kp, hi, lo);
}

void launch_phase_split(const __nv_bfloat16* hi, const __nv_bfloat16* lo, int H, int W, int C, int N, int Hs, int Ws,
                        const int* ids, const int* count, int max_rows, __nv_bfloat16* ohi, __nv_bfloat16* olo,
                        cudaStream_t s) {
  if (max_rows <= 0) return;
  const long long per = 4LL * Hs * Ws * (C / 8);
  int gy = static_cast<int>((per + 255) / 256);
  if (gy > 64) gy = 64;
  phase_split_kernel<<<dim3(max_rows, gy), 256, 0, s>>>(hi, lo, H, W, C, N, Hs, Ws, ids, count, ohi, olo);
}

void launch_maxpool(const __nv_bfloat16* hi, const __nv_bfloat16* lo, int H, int W, int C, int k, int stride, int pad,
                    int Ho, int Wo, const int* ids, const int* count, int max_rows, __nv_bfloat16* ohi,
                    __nv_bfloat16* olo, cudaStream_t s) {
  if (max_rows <= 0) return;
  const long long per = static_cast<long long>(Ho) * Wo * (C / 8);
  int gy = static_cast<int>((per + 255) / 256);
  if (gy > 128) gy = 128;
  maxpool_kernel<<<dim3(max_rows, gy), 256, 0, s>>>(hi, lo, H, W, C, k, stride, pad, Ho, Wo, ids, count, ohi, olo);
}

void launch_stamp_start(unsigned long long* t0, cudaStream_t s) { stamp_kernel<<<1, 1, 0, s>>>(t0); }

void launch_init_batch(const int* batch, int max_batch, int* ids0, int* count0, int* rows_out, int rows_mult,
                       int* exit_layer, int* served, int* base_pred, unsigned long long* exit_ns, float* probs, int L,
                       cudaStream_t s) {
  const int blocks = (max_batch + 255) / 256 > 0 ? (max_batch + 255) / 256 : 1;
  init_batch_kernel<<<blocks, 256, 0, s>>>(batch, max_batch, ids0, count0, rows_out, rows_mult, exit_layer, served,
                                           base_pred, exit_ns, probs, L);
}

}  // namespace lcb
