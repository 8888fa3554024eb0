// Stem convolution (the first conv of every CNN family, input = the request's
// fp32 NCHW image, C_in = 3) on tcgen05 without an im2col buffer.
//
// The image is rewritten once as X: zero-padded, space-to-depth by the conv
// stride (stride 2: 2x2 blocks -> 4*C_in channels; stride 1: identity), 16
// channels (zero-filled), stored per image as [2 channel groups][Hx*Wx][8]
// bf16 hi (+lo). The stem is then a valid stride-1 k' x k' conv over X. With
// output anchors on X's own row pitch (m = oh*Wx + ow; anchors with ow >= Wo
// are computed and discarded), filter tap (r', s') of every anchor in a tile
// of 128 consecutive anchors reads the contiguous X range m + r'*Wx + s':
// ONE slab of X per tile (one bulk copy per group and plane) feeds all k'^2
// taps as shifted shared-memory descriptors (no-swizzle K-major layout, 8-row
// x 16-byte core matrices, so any row shift is a valid operand start).
// K = 16 per tap = one MMA per tap (x3 in the parity tier). The weights
// (taps x 64 x 16, hi/lo) stay resident in shared memory.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace lcb {

struct StemParams {
  const __nv_bfloat16* x_hi;  // [N][2][Hx*Wx][8]
  const __nv_bfloat16* x_lo;  // nullable (bf16 tier)
  const __nv_bfloat16* w_hi;  // bf16: [taps][2][64][8]; bf16x3: stacked [taps][2][hi 64 | lo 64][8]
  const __nv_bfloat16* w_lo;  // unused (kept for the ABI of the parameter block)
  int Hx, Wx, Ho, Wo;
  int kk;                     // k' (taps per dimension over X)
  int tiles_per_img;          // ceil(Ho * Wx / 128)
  const int* count;           // images in the batch (device)
  int count_static;           // max images (grid sizing)
  const float* scale;         // unused (BN scale is folded into the weights)
  const float* shift;         // [64]
  int relu;
  __nv_bfloat16* out_hi;      // NHWC [N][Ho][Wo][64] (hpool: [N][Ho][Wp][64])
  __nv_bfloat16* out_lo;      // nullable
  // hpool = 1: the ResNet stem's 3x3/s2/p1 max-pool, horizontal half, fused
  // into the epilogue: one output row per tile (tiles_per_img = Ho, Wx <= 128),
  // out[n][oh][j] = max over ow in {2j-1, 2j, 2j+1} of the stem output (the
  // vertical half is launch_stem_vpool). The full-resolution stem output never
  // reaches HBM.
  int hpool;
  int Wp;                     // pooled width (Wo - 1) / 2 + 1
};

// Vertical half of the 3x3/s2/p1 max-pool over the hpool stem output:
// out[n][i][j] = max over r in {2i-1, 2i, 2i+1} of in[n][r][j] (per channel the
// first maximum in r order; hi and lo move together), surviving images ids.
void launch_stem_vpool(const __nv_bfloat16* in_hi, const __nv_bfloat16* in_lo, int Hi, int Wp, int C, int Hp,
                       const int* ids, const int* count, int max_rows, __nv_bfloat16* out_hi, __nv_bfloat16* out_lo,
                       cudaStream_t s);

// X geometry for a stem of kernel k, stride s (1 or 2), padding pad over H x W.
struct StemGeom {
  int Hx, Wx, kk, Ho, Wo;
};
StemGeom stem_geom(int H, int W, int k, int stride, int pad);

// fp32 NCHW images [count][C][H][W] -> X hi/lo (see above).
void launch_stem_s2d(const float* x, const int* count, int max_n, int C, int H, int W, int stride, int pad,
                     const StemGeom& g, __nv_bfloat16* x_hi, __nv_bfloat16* x_lo, cudaStream_t s);
// Host: conv weights [64][C][k][k] (double) -> X-space weights [taps][2][64][8] (float, before the hi/lo split).
void stem_weights(const double* w, int Cout, int C, int k, int stride, const StemGeom& g, float* out);
cudaError_t tc_stem_launch(const StemParams& p, int num_sms, cudaStream_t stream);

}  // namespace lcb
