// Persistent tcgen05 implicit-GEMM kernel: base-model convolutions (NHWC,
// 3x3/1x1, stride via phase split), dense FC layers (plain GEMM mode) and the
// FC(h) cache predictor GEMMs (split-K fp32 partials).
//
// A operand: activations as a 5-D TMA tensor (C, W, H, N, P) in bf16, C
// innermost; each K-step loads one 64-channel slice of one filter tap for the
// 128 output pixels of a tile (ipt images x hb x wb box), zero padding comes
// from TMA out-of-bounds fill. B operand: weights [Cout, taps*C] K-major.
// Accumulators live in TMEM (double-buffered, 2*BN columns).
//
// Precision: segs == 1 -> plain bf16 x bf16 -> fp32. segs == 3 -> "bf16x3":
// every operand is stored as hi + lo bf16 planes and the kernel accumulates
// hi*hi + hi*lo + lo*hi, which is fp32-class (~2^-16 relative per product);
// this is the parity tier the reference oracle is compared against.
#pragma once

#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace lcb {

constexpr int kMaxTaps = 64;

struct TcConvParams {
  CUtensorMap tmA[2];  // activation planes hi, lo (5-D: C, W, H, N, P)
  CUtensorMap tmB[2];  // weight planes hi, lo (2-D: K, Cout)
  int plain;           // 1: plain GEMM over rows (A = [rows, K], count = rows)
  int Ho, Wo;          // output spatial dims
  int hb, wb, ipt;     // A box geometry: ipt images x hb x wb = 128 rows
  int tiles_h, tiles_w;
  int C;               // input channels per tap (multiple of 64)
  int ntaps;
  int segs;            // 1 or 3
  int Cout;            // output channels (multiple of BN)
  int ksplit;          // split-K factor (mode 1 only)
  const int* surv;     // survivor image list (nullptr = identity)
  const int* count;    // device-side image/row count (nullptr -> count_static)
  int count_static;
  int mode;            // 0: bf16 NHWC out (+lo), 1: fp32 partials [ksplit][rows_total][Cout]
  int rows_total;      // mode 1 row stride
  const float* scale;  // per-Cout multiplier (nullable = 1)
  const float* shift;  // per-Cout bias (nullable = 0)
  const __nv_bfloat16* res_hi;
  const __nv_bfloat16* res_lo;
  int relu;
  __nv_bfloat16* out_hi;
  __nv_bfloat16* out_lo;
  float* out_f32;
  signed char tap_phase[kMaxTaps];
  signed char tap_dh[kMaxTaps];
  signed char tap_dw[kMaxTaps];
};

// Host helpers (tc_conv.cu).
bool encode_act_map(CUtensorMap* map, const void* base, int C, int W, int H, int N, int P, int wb, int hb);
bool encode_weight_map(CUtensorMap* map, const void* base, int K, int Cout, int BN);
int tc_conv_pick_bn(int Cout);
// Upper bound on the tile count at count_static (used to size the grid).
int tc_conv_max_tiles(const TcConvParams& p, int BN);
cudaError_t tc_conv_launch(const TcConvParams& p, int BN, int num_sms, cudaStream_t stream);

}  // namespace lcb
