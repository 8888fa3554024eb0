// fp64 SGD kernels for cache retraining — see train_kernels.cuh.
//
// Rounding: wherever the reference accumulates serially (backward()'s input
// gradients, accumulate_grads over a minibatch, the SGD update, the loss
// sums) the kernels keep its order with explicit __dmul_rn/__dadd_rn so nvcc
// cannot contract to FMA (the reference's x86-64 build has no FMA). The
// forward dot products and the Conv1d weight gradient use tree reductions
// (different order); exp/log/pow are CUDA's. Results therefore agree with
// the reference to rounding (~1e-12 relative), not bit for bit.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "kernels/train_kernels.cuh"

namespace lcb {
namespace {

constexpr int kFwdRows = 8;  // samples per register block in the FC forward
constexpr double kTinyProb = 1e-300;

__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }

// std::max(a, b) == (a < b) ? b : a — NaN in `a` propagates (unlike fmax),
// which is how the reference's divergence check sees a NaN loss.
__device__ __forceinline__ double std_max(double a, double b) { return a < b ? b : a; }

__device__ __forceinline__ long long row_of(const int* rows, int k) { return rows ? rows[k] : k; }

// y[k][o] = b[o] + <W[o], x[k]>: one warp per output, lanes over the input
// (coalesced W row), kFwdRows samples per pass.
__global__ void fc_forward_kernel(const double* __restrict__ x, long long ld, const int* __restrict__ rows, int nb,
                                  const double* __restrict__ w, const double* __restrict__ b, int in, int out,
                                  double* __restrict__ y) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= out) return;
  const double* wr = w + static_cast<long long>(warp) * in;
  for (int k0 = 0; k0 < nb; k0 += kFwdRows) {
    const int kn = nb - k0 < kFwdRows ? nb - k0 : kFwdRows;
    const double* xr[kFwdRows];
#pragma unroll
    for (int s = 0; s < kFwdRows; ++s) xr[s] = x + row_of(rows, k0 + (s < kn ? s : 0)) * ld;
    double acc[kFwdRows];
#pragma unroll
    for (int s = 0; s < kFwdRows; ++s) acc[s] = 0.0;
    for (int j = lane; j < in; j += 32) {
      const double wj = wr[j];
#pragma unroll
      for (int s = 0; s < kFwdRows; ++s) acc[s] += wj * xr[s][j];
    }
#pragma unroll
    for (int s = 0; s < kFwdRows; ++s) {
#pragma unroll
      for (int off = 16; off; off >>= 1) acc[s] += __shfl_xor_sync(0xffffffffu, acc[s], off);
    }
    if (lane == 0) {
      for (int s = 0; s < kn; ++s) y[static_cast<long long>(k0 + s) * out + warp] = dadd(b[warp], acc[s]);
    }
  }
}

// Wide-input FC forward: a CTA owns 32 outputs (4 per warp) x one 256-wide
// slice of the input (blockIdx.y); the slice of 16 samples is staged in
// shared memory once and reused by all 32 outputs.
constexpr int kSplitRows = 16;
constexpr int kSplitChunk = 256;
constexpr int kSplitOuts = 32;
__global__ void __launch_bounds__(256) fc_forward_split_kernel(const double* __restrict__ x, long long ld,
                                                               const int* __restrict__ rows, int nb,
                                                               const double* __restrict__ w, int in, int out,
                                                               double* __restrict__ part) {
  __shared__ double xs[kSplitRows][kSplitChunk];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int j0 = blockIdx.y * kSplitChunk;
  const int jn = min(kSplitChunk, in - j0);
  for (int k0 = 0; k0 < nb; k0 += kSplitRows) {
    const int kn = min(kSplitRows, nb - k0);
    __syncthreads();
    for (int e = threadIdx.x; e < kSplitRows * kSplitChunk; e += blockDim.x) {
      const int q = e / kSplitChunk, j = e % kSplitChunk;
      xs[q][j] = (q < kn && j < jn) ? x[row_of(rows, k0 + q) * ld + j0 + j] : 0.0;
    }
    __syncthreads();
#pragma unroll 1
    for (int t = 0; t < kSplitOuts / 8; ++t) {
      const int o = blockIdx.x * kSplitOuts + warp * (kSplitOuts / 8) + t;
      if (o >= out) break;
      const double* wr = w + static_cast<long long>(o) * in + j0;
      double acc[kSplitRows];
#pragma unroll
      for (int q = 0; q < kSplitRows; ++q) acc[q] = 0.0;
#pragma unroll 4
      for (int j = lane; j < jn; j += 32) {
        const double wj = wr[j];
#pragma unroll
        for (int q = 0; q < kSplitRows; ++q) acc[q] += wj * xs[q][j];
      }
#pragma unroll
      for (int q = 0; q < kSplitRows; ++q) {
#pragma unroll
        for (int off = 16; off; off >>= 1) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], off);
      }
      if (lane < kn) {
        double v = acc[0];
#pragma unroll
        for (int q = 1; q < kSplitRows; ++q)
          if (lane == q) v = acc[q];
        part[(static_cast<long long>(blockIdx.y) * nb + k0 + lane) * out + o] = v;
      }
    }
  }
}

__global__ void fc_forward_reduce_kernel(const double* __restrict__ part, int ksplit, int nb, int out,
                                         const double* __restrict__ b, double* __restrict__ y) {
  const long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (e >= static_cast<long long>(nb) * out) return;
  const int o = static_cast<int>(e % out);
  double acc = 0.0;
  for (int s = 0; s < ksplit; ++s) acc += part[static_cast<long long>(s) * nb * out + e];
  y[e] = dadd(b[o], acc);
}

// ReLU / AvgPool / Conv1d forward: one thread per (sample, output).
__global__ void elem_forward_kernel(TrainLayer L, const double* __restrict__ x, long long ld,
                                    const int* __restrict__ rows, int nb, double* __restrict__ y) {
  const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (i >= static_cast<long long>(nb) * L.out) return;
  const int k = static_cast<int>(i / L.out), o = static_cast<int>(i % L.out);
  const double* xr = x + row_of(rows, k) * ld;
  double v;
  if (L.kind == 1) {
    v = xr[o] > 0.0 ? xr[o] : 0.0;
  } else if (L.kind == 2) {  // network.cpp:130-138
    double acc = 0.0;
    for (int t = 0; t < L.window; ++t) acc = dadd(acc, xr[static_cast<long long>(o) * L.window + t]);
    v = dmul(acc, 1.0 / L.window);
  } else {  // Conv1d, network.cpp:139-148
    double acc = L.b[0];
    for (int t = 0; t < L.kernel; ++t) acc = dadd(acc, dmul(L.w[t], xr[static_cast<long long>(o) * L.stride + t]));
    v = acc;
  }
  y[i] = v;
}

// Input gradient (network.cpp:166-232), serial in the reference's order.
__global__ void backward_data_kernel(TrainLayer L, const double* __restrict__ x, const double* __restrict__ g, int nb,
                                     double* __restrict__ gx) {
  const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (i >= static_cast<long long>(nb) * L.in) return;
  const int k = static_cast<int>(i / L.in), j = static_cast<int>(i % L.in);
  const double* gk = g + static_cast<long long>(k) * L.out;
  double v = 0.0;
  if (L.kind == 0) {
    for (int o = 0; o < L.out; ++o) v = dadd(v, dmul(L.w[static_cast<long long>(o) * L.in + j], gk[o]));
  } else if (L.kind == 1) {
    v = x[i] > 0.0 ? gk[j] : 0.0;
  } else if (L.kind == 2) {
    v = dmul(gk[j / L.window], 1.0 / L.window);
  } else {
    // contributions (o, t) with o*stride + t == j, o ascending
    int o_lo = j - L.kernel + 1;
    o_lo = o_lo <= 0 ? 0 : (o_lo + L.stride - 1) / L.stride;
    int o_hi = j / L.stride;
    if (o_hi > L.out - 1) o_hi = L.out - 1;
    for (int o = o_lo; o <= o_hi; ++o) v = dadd(v, dmul(L.w[j - o * L.stride], gk[o]));
  }
  gx[i] = v;
}

__device__ __forceinline__ void sgd_update(double* w, double* v, double grad, double lr, double mom) {
  const double vn = dadd(dmul(mom, *v), grad);
  *v = vn;
  *w = __dsub_rn(*w, dmul(lr, vn));
}

// FC weight gradient over the minibatch in sample order, then SGD.
__global__ void fc_wgrad_sgd_kernel(TrainLayer L, const double* __restrict__ x, long long ld,
                                    const int* __restrict__ rows, const double* __restrict__ g,
                                    const double* __restrict__ scale, int nb, double lr, double mom) {
  const long long nw = static_cast<long long>(L.out) * L.in;
  const long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (e >= nw + L.out) return;
  double acc = 0.0;
  if (e < nw) {
    const int o = static_cast<int>(e / L.in), j = static_cast<int>(e % L.in);
    for (int k = 0; k < nb; ++k) {
      const double gk = dmul(g[static_cast<long long>(k) * L.out + o], x[row_of(rows, k) * ld + j]);
      acc = dadd(acc, dmul(scale[k], gk));
    }
    sgd_update(L.w + e, L.vw + e, acc, lr, mom);
  } else {
    const int o = static_cast<int>(e - nw);
    for (int k = 0; k < nb; ++k) acc = dadd(acc, dmul(scale[k], g[static_cast<long long>(k) * L.out + o]));
    sgd_update(L.b + o, L.vb + o, acc, lr, mom);
  }
}

// Same, two adjacent weights per thread (16-byte loads/stores; even `in`).
__global__ void fc_wgrad_sgd2_kernel(TrainLayer L, const double* __restrict__ x, long long ld,
                                     const int* __restrict__ rows, const double* __restrict__ g,
                                     const double* __restrict__ scale, int nb, double lr, double mom) {
  const long long nw2 = static_cast<long long>(L.out) * L.in / 2;
  const long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (e >= nw2 + L.out) return;
  if (e < nw2) {
    const int o = static_cast<int>(2 * e / L.in), j = static_cast<int>(2 * e % L.in);
    double a0 = 0.0, a1 = 0.0;
    for (int k = 0; k < nb; ++k) {
      const double gk = g[static_cast<long long>(k) * L.out + o], sk = scale[k];
      const double2 xv = *reinterpret_cast<const double2*>(x + row_of(rows, k) * ld + j);
      a0 = dadd(a0, dmul(sk, dmul(gk, xv.x)));
      a1 = dadd(a1, dmul(sk, dmul(gk, xv.y)));
    }
    double2* wp = reinterpret_cast<double2*>(L.w) + e;
    double2* vp = reinterpret_cast<double2*>(L.vw) + e;
    double2 wv = *wp, vv = *vp;
    sgd_update(&wv.x, &vv.x, a0, lr, mom);
    sgd_update(&wv.y, &vv.y, a1, lr, mom);
    *wp = wv;
    *vp = vv;
  } else {
    const int o = static_cast<int>(e - nw2);
    double acc = 0.0;
    for (int k = 0; k < nb; ++k) acc = dadd(acc, dmul(scale[k], g[static_cast<long long>(k) * L.out + o]));
    sgd_update(L.b + o, L.vb + o, acc, lr, mom);
  }
}

// Same, a 4-output x 2-input block per thread: each x pair loaded once for
// four outputs (out % 4 == 0, even `in`).
__global__ void fc_wgrad_sgd42_kernel(TrainLayer L, const double* __restrict__ x, long long ld,
                                      const int* __restrict__ rows, const double* __restrict__ g,
                                      const double* __restrict__ scale, int nb, double lr, double mom) {
  const int in2 = L.in / 2;
  const long long nblk = static_cast<long long>(L.out / 4) * in2;
  const long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (e >= nblk + L.out) return;
  if (e < nblk) {
    const int o0 = static_cast<int>(e / in2) * 4, j = static_cast<int>(e % in2) * 2;
    double a[4][2] = {};
    for (int k = 0; k < nb; ++k) {
      const double sk = scale[k];
      const double2 xv = *reinterpret_cast<const double2*>(x + row_of(rows, k) * ld + j);
      const double* gk = g + static_cast<long long>(k) * L.out + o0;
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        a[r][0] = dadd(a[r][0], dmul(sk, dmul(gk[r], xv.x)));
        a[r][1] = dadd(a[r][1], dmul(sk, dmul(gk[r], xv.y)));
      }
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const long long idx = (static_cast<long long>(o0 + r) * L.in + j) / 2;
      double2* wp = reinterpret_cast<double2*>(L.w) + idx;
      double2* vp = reinterpret_cast<double2*>(L.vw) + idx;
      double2 wv = *wp, vv = *vp;
      sgd_update(&wv.x, &vv.x, a[r][0], lr, mom);
      sgd_update(&wv.y, &vv.y, a[r][1], lr, mom);
      *wp = wv;
      *vp = vv;
    }
  } else {
    const int o = static_cast<int>(e - nblk);
    double acc = 0.0;
    for (int k = 0; k < nb; ++k) acc = dadd(acc, dmul(scale[k], g[static_cast<long long>(k) * L.out + o]));
    sgd_update(L.b + o, L.vb + o, acc, lr, mom);
  }
}

// Conv1d weight gradient: one block per kernel tap (+1 for the bias).
__global__ void conv_wgrad_sgd_kernel(TrainLayer L, const double* __restrict__ x, long long ld,
                                      const int* __restrict__ rows, const double* __restrict__ g,
                                      const double* __restrict__ scale, int nb, double lr, double mom) {
  __shared__ double red[32];
  const int t = blockIdx.x;  // t == kernel: bias
  double acc = 0.0;
  for (int k = 0; k < nb; ++k) {
    const double* gk = g + static_cast<long long>(k) * L.out;
    const double* xr = x + row_of(rows, k) * ld;
    double part = 0.0;
    for (int o = threadIdx.x; o < L.out; o += blockDim.x)
      part += t < L.kernel ? gk[o] * xr[static_cast<long long>(o) * L.stride + t] : gk[o];
#pragma unroll
    for (int off = 16; off; off >>= 1) part += __shfl_xor_sync(0xffffffffu, part, off);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = part;
    __syncthreads();
    if (threadIdx.x == 0) {
      double sum = 0.0;
      for (int q = 0; q < static_cast<int>(blockDim.x >> 5); ++q) sum += red[q];
      acc = dadd(acc, dmul(scale[k], sum));
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    if (t < L.kernel)
      sgd_update(L.w + t, L.vw + t, acc, lr, mom);
    else
      sgd_update(L.b, L.vb, acc, lr, mom);
  }
}

// Per-sample distillation gradient (losses.cpp:72-101); serial sums in
// thread 0 keep the reference's order.
__global__ void distill_grad_kernel(const double* __restrict__ logits, const double* __restrict__ p_tau,
                                    const int* __restrict__ hard, const int* __restrict__ rows, int C, double tau,
                                    double beta, double* __restrict__ g, int* bad) {
  extern __shared__ double sm[];
  double* q = sm;
  double* qt = sm + C;
  __shared__ double stat[4];
  const int k = blockIdx.x;
  const long long r = row_of(rows, k);
  const double* l = logits + static_cast<long long>(k) * C;
  const double* pt = p_tau + r * C;
  if (threadIdx.x == 0) {
    double m = l[0], mt = l[0] / tau;
    for (int i = 1; i < C; ++i) {
      m = std_max(m, l[i]);
      mt = std_max(mt, l[i] / tau);
    }
    stat[0] = m;
    stat[1] = mt;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < C; i += blockDim.x) {
    q[i] = exp(__dsub_rn(l[i], stat[0]));
    qt[i] = exp(__dsub_rn(__ddiv_rn(l[i], tau), stat[1]));
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0, st = 0.0;
    for (int i = 0; i < C; ++i) s = dadd(s, q[i]);
    for (int i = 0; i < C; ++i) st = dadd(st, qt[i]);
    stat[2] = s;
    stat[3] = st;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < C; i += blockDim.x) {
    q[i] = __ddiv_rn(q[i], stat[2]);
    qt[i] = __ddiv_rn(qt[i], stat[3]);
  }
  __syncthreads();
  const int h = hard[r];
  for (int i = threadIdx.x; i < C; i += blockDim.x) {
    const double hd = dmul(beta, __dsub_rn(q[i], i == h ? 1.0 : 0.0));
    const double sf = dmul(dmul(__dsub_rn(1.0, beta), tau), __dsub_rn(qt[i], pt[i]));
    g[static_cast<long long>(k) * C + i] = dadd(hd, sf);
  }
  if (threadIdx.x == 0) {
    const double ce = -log(std_max(q[h], kTinyProb));
    double kl = 0.0;
    for (int i = 0; i < C; ++i)
      if (pt[i] > 0.0) kl = dadd(kl, dmul(pt[i], __dsub_rn(log(pt[i]), log(std_max(qt[i], kTinyProb)))));
    kl = std_max(kl, 0.0);
    const double loss = beta * ce + (1.0 - beta) * tau * tau * kl;
    if (!isfinite(loss)) atomicOr(bad, 1);
  }
}

__global__ void soften_kernel(const double* __restrict__ y, int N, int C, double tau, double* __restrict__ p_tau,
                              int* __restrict__ hard, int* bad) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= N) return;
  const double* yr = y + static_cast<long long>(n) * C;
  double* o = p_tau + static_cast<long long>(n) * C;
  double sum = 0.0;
  int best = 0;
  for (int i = 0; i < C; ++i) {
    if (yr[i] < 0.0) atomicOr(bad, 2);
    o[i] = yr[i] > 0.0 ? pow(yr[i], 1.0 / tau) : 0.0;
    sum = dadd(sum, o[i]);
    if (yr[i] > yr[best]) best = i;
  }
  if (!(sum > 0.0)) atomicOr(bad, 2);
  for (int i = 0; i < C; ++i) o[i] = __ddiv_rn(o[i], sum);
  hard[n] = best;
}

__device__ __forceinline__ double softplus(double x) { return x > 30.0 ? x : log1p(exp(x)); }

// weighted_selector_loss (losses.cpp:103-116) with the branch-stable sigmoid (losses.cpp:26-33).
__global__ void selector_grad_kernel(const double* __restrict__ logit, const int* __restrict__ target,
                                     const int* __restrict__ rows, int nb, double w_fp, double w_fn,
                                     double* __restrict__ g, int* bad) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nb) return;
  const double x = logit[k];
  double s;
  if (x >= 0.0) {
    s = __ddiv_rn(1.0, dadd(1.0, exp(-x)));
  } else {
    const double z = exp(x);
    s = __ddiv_rn(z, dadd(1.0, z));
  }
  double loss;
  if (target[row_of(rows, k)] == 1) {
    loss = w_fn * softplus(-x);
    g[k] = dmul(-w_fn, __dsub_rn(1.0, s));
  } else {
    loss = w_fp * softplus(x);
    g[k] = dmul(w_fp, s);
  }
  if (!isfinite(loss)) atomicOr(bad, 1);
}

__global__ void softmax_labels_kernel(double* __restrict__ x, int N, int C, const int* __restrict__ hard,
                                      int* __restrict__ agree) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= N) return;
  double* r = x + static_cast<long long>(n) * C;
  int best = 0;
  double m = r[0];
  for (int i = 1; i < C; ++i) {
    if (r[i] > r[best]) best = i;
    m = std_max(m, r[i]);
  }
  agree[n] = best == hard[n] ? 1 : 0;
  double sum = 0.0;
  for (int i = 0; i < C; ++i) {
    r[i] = exp(__dsub_rn(r[i], m));
    sum = dadd(sum, r[i]);
  }
  for (int i = 0; i < C; ++i) r[i] = __ddiv_rn(r[i], sum);
}

__device__ __forceinline__ double plane_val(const __nv_bfloat16* hi, const __nv_bfloat16* lo, long long i) {
  double v = __bfloat162float(hi[i]);
  if (lo) v += __bfloat162float(lo[i]);
  return v;
}

__global__ void planes_to_f64_kernel(const __nv_bfloat16* __restrict__ hi, const __nv_bfloat16* __restrict__ lo,
                                     long long ld, long long D, int B, double* __restrict__ out) {
  const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (i >= D * B) return;
  const long long r = i / D, f = i % D;
  out[i] = plane_val(hi, lo, r * ld + f);
}

__global__ void head_logits_kernel(const __nv_bfloat16* __restrict__ hi, const __nv_bfloat16* __restrict__ lo,
                                   long long ld, int D, const float* __restrict__ W, const float* __restrict__ b,
                                   int C, int B, double* __restrict__ logits) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= B * C) return;
  const int r = warp / C, c = warp % C;
  double acc = 0.0;
  for (int j = lane; j < D; j += 32)
    acc += static_cast<double>(W[static_cast<long long>(c) * D + j]) * plane_val(hi, lo, r * ld + j);
#pragma unroll
  for (int off = 16; off; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if (lane == 0) logits[warp] = acc + static_cast<double>(b[c]);
}

__global__ void softmax_rows_kernel(const double* __restrict__ x, int N, int C, double* __restrict__ y) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= N) return;
  const double* r = x + static_cast<long long>(n) * C;
  double* o = y + static_cast<long long>(n) * C;
  double m = r[0];
  for (int i = 1; i < C; ++i) m = std_max(m, r[i]);
  double sum = 0.0;
  for (int i = 0; i < C; ++i) {
    o[i] = exp(r[i] - m);
    sum += o[i];
  }
  for (int i = 0; i < C; ++i) o[i] /= sum;
}

constexpr int kFusedThreads = 1024;
constexpr int kFusedMaxC = 64;  // distillation classes handled by the fused schedule
constexpr int kLossWarps = 16;  // warps computing per-sample distillation gradients

// Layer view inside the fused kernel: every array is a 32-bit offset into
// the dynamic shared memory (LDS/STS addressing, no generic pointers).
struct FusedLayerOff {
  int kind, in, out, window, kernel, stride;
  int ws;                 // FC weight row stride: odd, so lanes over outputs hit distinct banks
  int w, b, vw, vb, act;  // act = this layer's output [rows_cap][out]
};

__global__ void __launch_bounds__(kFusedThreads, 1)
    sgd_fused_kernel(FusedNet gnet, const double* __restrict__ x, long long ld, const int* __restrict__ rows_all,
                     const double* __restrict__ scale_all, const int* __restrict__ boff, const int* __restrict__ bnb,
                     int nbatches, FusedLoss loss, double lr, double mom, int rows_cap, int max_dim, int* bad) {
  // Everything but the records lives in shared memory for the whole
  // schedule: weights, momentum, activations, gradients and each batch's
  // staged input rows.
  __shared__ double lsm[kLossWarps][3 * kFusedMaxC];
  __shared__ FusedLayerOff fl[kFusedMaxLayers];
  __shared__ int offs[5];  // g, gx, xs, ss, conv per-sample weight-gradient sums
  extern __shared__ double dsm[];
  const int tid = threadIdx.x, nt = blockDim.x, nl = gnet.nl;
  if (tid == 0) {
    int p = 0;
    for (int i = 0; i < nl; ++i) {
      const TrainLayer& G = gnet.L[i];
      FusedLayerOff& L = fl[i];
      L.kind = G.kind;
      L.in = G.in;
      L.out = G.out;
      L.window = G.window;
      L.kernel = G.kernel;
      L.stride = G.stride;
      L.ws = G.in | 1;
      L.w = L.b = L.vw = L.vb = 0;
      if (G.kind == 0 || G.kind == 3) {
        const int nw = G.kind == 0 ? G.out * L.ws : G.kernel, nbias = G.kind == 0 ? G.out : 1;
        L.w = p;
        L.b = p + nw;
        L.vw = p + nw + nbias;
        L.vb = p + 2 * nw + nbias;
        p += 2 * (nw + nbias);
      }
    }
    for (int i = 0; i < nl; ++i) {
      fl[i].act = p;
      p += rows_cap * gnet.L[i].out;
    }
    offs[0] = p;
    offs[1] = p + rows_cap * max_dim;
    offs[2] = p + 2 * rows_cap * max_dim;
    offs[3] = offs[2] + rows_cap * gnet.L[0].in;
    offs[4] = offs[3] + rows_cap;
  }
  __syncthreads();
  for (int i = 0; i < nl; ++i) {
    const TrainLayer& G = gnet.L[i];
    if (G.kind == 0 || G.kind == 3) {
      const FusedLayerOff L = fl[i];
      const int nw = G.kind == 0 ? G.out * G.in : G.kernel, nbias = G.kind == 0 ? G.out : 1;
      for (int e = tid; e < nw; e += nt) {
        const int d = G.kind == 0 ? (e / G.in) * L.ws + e % G.in : e;
        dsm[L.w + d] = G.w[e];
        dsm[L.vw + d] = G.vw[e];
      }
      for (int e = tid; e < nbias; e += nt) {
        dsm[L.b + e] = G.b[e];
        dsm[L.vb + e] = G.vb[e];
      }
    }
  }
  const int in0 = gnet.L[0].in;
  const int xs = offs[2], ss = offs[3];
  __syncthreads();
  for (int bi = 0; bi < nbatches; ++bi) {
    const int off = boff[bi], nb = bnb[bi];
    const int* rows = rows_all + off;
    for (int e = tid; e < nb * in0; e += nt) {
      const int k = e / in0, j = e - k * in0;
      dsm[xs + e] = __ldg(x + static_cast<long long>(__ldg(rows + k)) * ld + j);
    }
    for (int k = tid; k < nb; k += nt) dsm[ss + k] = __ldg(scale_all + off + k);
    __syncthreads();
    // ---- forward (network.cpp:104-164), serial dots in the reference's order
    for (int i = 0; i < nl; ++i) {
      const FusedLayerOff L = fl[i];
      const int in = i == 0 ? xs : fl[i - 1].act;
      for (int e = tid; e < nb * L.out; e += nt) {
        const int k = e / L.out, o = e - k * L.out;
        const int xr = in + k * L.in;
        double v;
        if (L.kind == 0) {
          v = dsm[L.b + o];
          const int wr = L.w + o * L.ws;
#pragma unroll 8
          for (int j = 0; j < L.in; ++j) v = dadd(v, dmul(dsm[wr + j], dsm[xr + j]));
        } else if (L.kind == 1) {
          const double u = dsm[xr + o];
          v = u > 0.0 ? u : 0.0;
        } else if (L.kind == 2) {
          double acc = 0.0;
          for (int t = 0; t < L.window; ++t) acc = dadd(acc, dsm[xr + o * L.window + t]);
          v = dmul(acc, 1.0 / L.window);
        } else {
          v = dsm[L.b];
          for (int t = 0; t < L.kernel; ++t) v = dadd(v, dmul(dsm[L.w + t], dsm[xr + o * L.stride + t]));
        }
        dsm[L.act + e] = v;
      }
      __syncthreads();
    }
    // ---- loss gradient into g: distillation one warp per sample (exps in
    // parallel across lanes, sums serial in lane 0), selector one thread per sample
    const int outp = fl[nl - 1].act;
    const int g0 = offs[0];
    if (loss.kind == 0) {
      const int C = loss.C, warp = tid >> 5, lane = tid & 31;
      const double tau = loss.a, beta = loss.b;
      // per-class values computed across lanes; every order-sensitive step
      // (max chains, sums, the kl accumulation) stays serial in class order
      for (int k = warp; k < nb && warp < kLossWarps; k += kLossWarps) {
        const long long r = rows[k];
        const int l = outp + k * C;
        const double* pt = loss.p_tau + r * C;
        double* eq = lsm[warp];
        double* et = lsm[warp] + kFusedMaxC;
        double* kt = lsm[warp] + 2 * kFusedMaxC;
        for (int i = lane; i < C; i += 32) et[i] = __ddiv_rn(dsm[l + i], tau);
        __syncwarp();
        double m = dsm[l], mt = et[0];
        for (int i = 1; i < C; ++i) {
          m = std_max(m, dsm[l + i]);
          mt = std_max(mt, et[i]);
        }
        for (int i = lane; i < C; i += 32) {
          eq[i] = exp(__dsub_rn(dsm[l + i], m));
          et[i] = exp(__dsub_rn(et[i], mt));
        }
        __syncwarp();
        double sm = 0.0, st = 0.0;
        for (int i = 0; i < C; ++i) sm = dadd(sm, eq[i]);
        for (int i = 0; i < C; ++i) st = dadd(st, et[i]);
        const int h = loss.hard[r];
        for (int i = lane; i < C; i += 32) {
          const double q = __ddiv_rn(eq[i], sm);
          const double qt = __ddiv_rn(et[i], st);
          const double hd = dmul(beta, __dsub_rn(q, i == h ? 1.0 : 0.0));
          const double sf = dmul(dmul(__dsub_rn(1.0, beta), tau), __dsub_rn(qt, pt[i]));
          dsm[g0 + k * C + i] = dadd(hd, sf);
          kt[i] = pt[i] > 0.0 ? dmul(pt[i], __dsub_rn(log(pt[i]), log(std_max(qt, kTinyProb)))) : 0.0;
        }
        __syncwarp();
        if (lane == 0) {
          double kl = 0.0;
          for (int i = 0; i < C; ++i)
            if (pt[i] > 0.0) kl = dadd(kl, kt[i]);
          kl = std_max(kl, 0.0);
          const double lossv =
              beta * -log(std_max(__ddiv_rn(eq[h], sm), kTinyProb)) + (1.0 - beta) * tau * tau * kl;
          if (!isfinite(lossv)) atomicOr(bad, 1);
        }
        __syncwarp();
      }
    } else {
      for (int k = tid; k < nb; k += nt) {
        const long long r = rows[k];
        const double z = dsm[outp + k];
        double sg;
        if (z >= 0.0) {
          sg = __ddiv_rn(1.0, dadd(1.0, exp(-z)));
        } else {
          const double ez = exp(z);
          sg = __ddiv_rn(ez, dadd(1.0, ez));
        }
        double lossv;
        if (loss.target[r] == 1) {
          lossv = loss.b * softplus(-z);
          dsm[g0 + k] = dmul(-loss.b, __dsub_rn(1.0, sg));
        } else {
          lossv = loss.a * softplus(z);
          dsm[g0 + k] = dmul(loss.a, sg);
        }
        if (!isfinite(lossv)) atomicOr(bad, 1);
      }
    }
    __syncthreads();
    // ---- backward + SGD, last layer first
    int gc = offs[0], gn = offs[1];
    for (int i = nl - 1; i >= 0; --i) {
      const FusedLayerOff L = fl[i];
      const int in = i == 0 ? xs : fl[i - 1].act;
      if (i > 0) {
        for (int e = tid; e < nb * L.in; e += nt) {
          const int k = e / L.in, j = e - k * L.in;
          const int gk = gc + k * L.out;
          double v = 0.0;
          if (L.kind == 0) {
#pragma unroll 4
            for (int o = 0; o < L.out; ++o) v = dadd(v, dmul(dsm[L.w + o * L.ws + j], dsm[gk + o]));
          } else if (L.kind == 1) {
            v = dsm[in + e] > 0.0 ? dsm[gk + j] : 0.0;
          } else if (L.kind == 2) {
            v = dmul(dsm[gk + j / L.window], 1.0 / L.window);
          } else {
            int o_lo = j - L.kernel + 1;
            o_lo = o_lo <= 0 ? 0 : (o_lo + L.stride - 1) / L.stride;
            int o_hi = j / L.stride;
            if (o_hi > L.out - 1) o_hi = L.out - 1;
            for (int o = o_lo; o <= o_hi; ++o) v = dadd(v, dmul(dsm[L.w + j - o * L.stride], dsm[gk + o]));
          }
          dsm[gn + e] = v;
        }
        __syncthreads();
      }
      if (L.kind == 0) {
        const int nw = L.out * L.in;
        for (int e = tid; e < nw + L.out; e += nt) {
          double acc = 0.0;
          if (e < nw) {
            const int o = e / L.in, j = e - o * L.in;
#pragma unroll 4
            for (int k = 0; k < nb; ++k)
              acc = dadd(acc, dmul(dsm[ss + k], dmul(dsm[gc + k * L.out + o], dsm[in + k * L.in + j])));
            const int d = o * L.ws + j;
            const double vn = dadd(dmul(mom, dsm[L.vw + d]), acc);
            dsm[L.vw + d] = vn;
            dsm[L.w + d] = __dsub_rn(dsm[L.w + d], dmul(lr, vn));
          } else {
            const int o = e - nw;
            for (int k = 0; k < nb; ++k) acc = dadd(acc, dmul(dsm[ss + k], dsm[gc + k * L.out + o]));
            const double vn = dadd(dmul(mom, dsm[L.vb + o]), acc);
            dsm[L.vb + o] = vn;
            dsm[L.b + o] = __dsub_rn(dsm[L.b + o], dmul(lr, vn));
          }
        }
      } else if (L.kind == 3) {
        // backward(): per sample lg.w[t] += go * x[o*stride + t] over o in
        // order (one thread per (sample, tap)), then accumulate_grads over the
        // samples in order (one thread per tap)
        const int sk = offs[4], K1 = L.kernel + 1;
        for (int e = tid; e < nb * K1; e += nt) {
          const int k = e / K1, t = e - k * K1;
          const int gk = gc + k * L.out, xr = in + k * L.in;
          double v = 0.0;
          if (t < L.kernel) {
            for (int o = 0; o < L.out; ++o) v = dadd(v, dmul(dsm[gk + o], dsm[xr + o * L.stride + t]));
          } else {
            for (int o = 0; o < L.out; ++o) v = dadd(v, dsm[gk + o]);
          }
          dsm[sk + e] = v;
        }
        __syncthreads();
        for (int t = tid; t < K1; t += nt) {
          double acc = 0.0;
          for (int k = 0; k < nb; ++k) acc = dadd(acc, dmul(dsm[ss + k], dsm[sk + k * K1 + t]));
          const int wi = t < L.kernel ? L.w + t : L.b, vi = t < L.kernel ? L.vw + t : L.vb;
          const double vn = dadd(dmul(mom, dsm[vi]), acc);
          dsm[vi] = vn;
          dsm[wi] = __dsub_rn(dsm[wi], dmul(lr, vn));
        }
      }
      __syncthreads();
      if (i > 0) {
        const int tmp = gc;
        gc = gn;
        gn = tmp;
      }
    }
  }
  for (int i = 0; i < nl; ++i) {
    const TrainLayer& G = gnet.L[i];
    if (G.kind == 0 || G.kind == 3) {
      const FusedLayerOff L = fl[i];
      const int nw = G.kind == 0 ? G.out * G.in : G.kernel, nbias = G.kind == 0 ? G.out : 1;
      for (int e = tid; e < nw; e += nt) G.w[e] = dsm[L.w + (G.kind == 0 ? (e / G.in) * L.ws + e % G.in : e)];
      for (int e = tid; e < nbias; e += nt) G.b[e] = dsm[L.b + e];
    }
  }
}

inline unsigned blocks_for(long long n, int t) { return static_cast<unsigned>((n + t - 1) / t); }

}  // namespace

int train_fc_ksplit(int in) { return in < 2048 ? 1 : (in + kSplitChunk - 1) / kSplitChunk; }

void launch_train_forward(const TrainLayer& L, const double* act_in, long long in_ld, const int* rows, int nb,
                          double* act_out, cudaStream_t s) {
  if (L.kind == 0 && L.ksplit > 1 && L.part) {
    fc_forward_split_kernel<<<dim3((L.out + kSplitOuts - 1) / kSplitOuts, L.ksplit), 256, 0, s>>>(
        act_in, in_ld, rows, nb, L.w, L.in, L.out, L.part);
    fc_forward_reduce_kernel<<<blocks_for(static_cast<long long>(nb) * L.out, 256), 256, 0, s>>>(
        L.part, L.ksplit, nb, L.out, L.b, act_out);
  } else if (L.kind == 0) {
    fc_forward_kernel<<<blocks_for(static_cast<long long>(L.out) * 32, 256), 256, 0, s>>>(act_in, in_ld, rows, nb, L.w,
                                                                                          L.b, L.in, L.out, act_out);
  } else {
    elem_forward_kernel<<<blocks_for(static_cast<long long>(nb) * L.out, 256), 256, 0, s>>>(L, act_in, in_ld, rows, nb,
                                                                                            act_out);
  }
}

void launch_train_backward_data(const TrainLayer& L, const double* act_in, const double* g, int nb, double* gx,
                                cudaStream_t s) {
  backward_data_kernel<<<blocks_for(static_cast<long long>(nb) * L.in, 256), 256, 0, s>>>(L, act_in, g, nb, gx);
}

void launch_train_wgrad_sgd(const TrainLayer& L, const double* act_in, long long in_ld, const int* rows,
                            const double* g, const double* scale, int nb, double lr, double momentum, cudaStream_t s) {
  if (L.kind == 0 && L.in % 2 == 0 && in_ld % 2 == 0 && L.out % 4 == 0 && L.in >= 512) {
    const long long n = static_cast<long long>(L.out / 4) * (L.in / 2) + L.out;
    fc_wgrad_sgd42_kernel<<<blocks_for(n, 256), 256, 0, s>>>(L, act_in, in_ld, rows, g, scale, nb, lr, momentum);
  } else if (L.kind == 0 && L.in % 2 == 0 && in_ld % 2 == 0) {
    const long long n = static_cast<long long>(L.out) * L.in / 2 + L.out;
    fc_wgrad_sgd2_kernel<<<blocks_for(n, 256), 256, 0, s>>>(L, act_in, in_ld, rows, g, scale, nb, lr, momentum);
  } else if (L.kind == 0) {
    const long long n = static_cast<long long>(L.out) * L.in + L.out;
    fc_wgrad_sgd_kernel<<<blocks_for(n, 256), 256, 0, s>>>(L, act_in, in_ld, rows, g, scale, nb, lr, momentum);
  } else if (L.kind == 3) {
    conv_wgrad_sgd_kernel<<<L.kernel + 1, 256, 0, s>>>(L, act_in, in_ld, rows, g, scale, nb, lr, momentum);
  }
}

void launch_distill_grad(const double* logits, const double* p_tau, const int* hard, const int* rows, int nb, int C,
                         double tau, double beta, double* g, int* bad, cudaStream_t s) {
  distill_grad_kernel<<<nb, 128, 2 * C * sizeof(double), s>>>(logits, p_tau, hard, rows, C, tau, beta, g, bad);
}

void launch_soften(const double* y, int N, int C, double tau, double* p_tau, int* hard, int* bad, cudaStream_t s) {
  soften_kernel<<<blocks_for(N, 128), 128, 0, s>>>(y, N, C, tau, p_tau, hard, bad);
}

void launch_selector_grad(const double* logit, const int* target, const int* rows, int nb, double w_fp, double w_fn,
                          double* g, int* bad, cudaStream_t s) {
  selector_grad_kernel<<<blocks_for(nb, 128), 128, 0, s>>>(logit, target, rows, nb, w_fp, w_fn, g, bad);
}

void launch_softmax_labels(double* x, int N, int C, const int* hard, int* agree, cudaStream_t s) {
  softmax_labels_kernel<<<blocks_for(N, 128), 128, 0, s>>>(x, N, C, hard, agree);
}

size_t sgd_fused_smem_bytes(const FusedNet& net, int rows_cap, int max_dim) {
  size_t n = 0;
  for (int i = 0; i < net.nl; ++i) {
    const TrainLayer& L = net.L[i];
    if (L.kind == 0) n += 2 * (static_cast<size_t>(L.out) * (L.in | 1) + L.out);
    if (L.kind == 3) n += 2 * (static_cast<size_t>(L.kernel) + 1);
    n += static_cast<size_t>(rows_cap) * L.out;
  }
  n += 2 * static_cast<size_t>(rows_cap) * max_dim;
  n += static_cast<size_t>(rows_cap) * (net.L[0].in + 1);  // staged input rows + scales
  int kmax = 0;
  for (int i = 0; i < net.nl; ++i)
    if (net.L[i].kind == 3 && net.L[i].kernel > kmax) kmax = net.L[i].kernel;
  n += static_cast<size_t>(rows_cap) * (kmax + 1);  // conv per-sample weight-gradient sums
  return n * sizeof(double);
}

cudaError_t launch_sgd_fused(const FusedNet& net, const double* x, long long ld, const int* rows, const double* scale,
                             const int* batch_off, const int* batch_nb, int nbatches, const FusedLoss& loss,
                             double lr, double momentum, int rows_cap, int max_dim, int* bad, cudaStream_t s) {
  const size_t smem = sgd_fused_smem_bytes(net, rows_cap, max_dim);
  const cudaError_t e =
      cudaFuncSetAttribute(sgd_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  sgd_fused_kernel<<<1, kFusedThreads, smem, s>>>(net, x, ld, rows, scale, batch_off, batch_nb, nbatches, loss, lr,
                                                  momentum, rows_cap, max_dim, bad);
  return cudaGetLastError();
}

void launch_planes_to_f64(const void* hi, const void* lo, long long ld, long long D, int B, double* out,
                          cudaStream_t s) {
  planes_to_f64_kernel<<<blocks_for(D * B, 256), 256, 0, s>>>(static_cast<const __nv_bfloat16*>(hi),
                                                               static_cast<const __nv_bfloat16*>(lo), ld, D, B, out);
}

void launch_head_probs_f64(const void* hi, const void* lo, long long ld, int D, const float* W, const float* b, int C,
                           int B, double* logits_scratch, double* y, cudaStream_t s) {
  head_logits_kernel<<<blocks_for(static_cast<long long>(B) * C * 32, 256), 256, 0, s>>>(
      static_cast<const __nv_bfloat16*>(hi), static_cast<const __nv_bfloat16*>(lo), ld, D, W, b, C, B, logits_scratch);
  softmax_rows_kernel<<<blocks_for(B, 128), 128, 0, s>>>(logits_scratch, B, C, y);
}

}  // namespace lcb
