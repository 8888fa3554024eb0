// Persistent tcgen05 implicit-GEMM kernel: base-model convolutions (NHWC,
// any k x k, stride 1 or 2 through TMA traversal strides), dense FC layers
// (plain GEMM mode) and the FC(h) cache predictor GEMMs (split-K fp32 partials).
//
// A operand: activations as a 5-D TMA tensor (C, W, H, N, P) in bf16, C
// innermost; each K-step loads one 64-channel slice of one filter tap for the
// 128 output pixels of a tile (ipt images x hb x wb box), zero padding comes
// from TMA out-of-bounds fill. B operand: weights [Cout, taps*C] K-major.
// Accumulators live in TMEM (double-buffered, 2*BN columns).
//
// Precision: segs == 1 -> plain bf16 x bf16 -> fp32. segs == 3 -> "bf16x3":
// every operand is stored as hi + lo bf16 planes; one pipeline stage carries
// A_hi, A_lo, B_hi, B_lo and the MMA warp accumulates hi*hi + hi*lo + lo*hi
// (fp32-class, ~2^-16 relative per product) — the parity tier.
//
// Split-K (mode 0, ks_max > 1): the split factor is chosen ON DEVICE from the
// surviving-request count so the grid stays full as requests exit
// (ks = floor(grid / tiles), so every split unit runs in the single resident
// wave). Partial tiles go to an fp32 workspace; the ks CTAs of a tile meet at
// a per-tile arrival counter and each reduces 1/ks of the tile in a fixed k
// order before running the epilogue on it (deterministic, parallel). The
// wait requires all CTAs of a launch to be co-resident: one CTA per SM,
// grid <= SM count, and launches on one device must not run concurrently
// (the engine uses one stream per device).
#pragma once

#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace lcb {

constexpr int kMaxTaps = 64;

// Lookup fused into the producing conv (the learned cache's Pool(C) = GAP
// predictor, cache.cpp:104-140 with window H*W, on the tap this conv
// writes). Every tile's epilogue writes GAP partials; per survivor row an
// arrival counter finds the CTA that finishes the row's last tile, and that
// CTA's epilogue warps sum the row's partials (fixed order) into the GAP
// features. With classes > 0 (<= 32) they also run the cache head — logits =
// W2 feat + b2, softmax (losses.cpp:35-46), selector FC(C,16)+ReLU+FC(16,1),
// branch-stable sigmoid (losses.cpp:26-33), inclusive p >= delta
// (cache.cpp:259-265), argmax(pr) with the lowest index on ties — and the CTA
// finishing the LAST row's head records first hits and compacts the survivors
// (serve_one, serving.cpp:112-121): no separate lookup launch.
struct TcGapHead {
  int* row_tiles;          // nullptr = off; [max_rows] per-row tile arrivals (zeroed, reset by the finisher)
  // post = 1: no per-tile arrivals. After the CTA's last tile every CTA of the
  // launch (all resident: persistent grid) meets at a grid barrier on gsync,
  // then the rows' GAP features and heads are computed by CTAs in row-strided
  // order, and the CTA finishing the last head runs the exit + compaction.
  int post;
  unsigned* gsync;         // monotonic grid-barrier counter (zeroed once)
  float inv;               // 1 / (Ho * Wo)
  float* feat;             // nullable: [max_rows][Cout] fp32 GAP features by row (for a separate head)
  int classes;             // 0 = features only; else <= 32: fused head + exit
  const float* W2;         // [classes][Cout]
  const float* b2;         // [classes]
  const float* Ws1;        // [16][classes]
  const float* bs1;        // [16]
  const float* ws2;        // [16]
  float bs2;
  double delta;
  float* prob;             // row-indexed outputs
  int* hit;
  int* label;
  int* heads_done;         // arrival counter over rows (zeroed, reset by the last)
  int layer, shadow;
  const int* ids_in;       // row -> request id
  int* exit_layer;
  int* served;
  unsigned long long* exit_ns;
  float* probs_out;        // by request id (nullable)
  int* labels_out;         // by request id (nullable)
  int* ids_out;
  int* src_rows_out;       // nullable
  int* count_out;
};

struct TcConvParams {
  CUtensorMap tmA[2];  // activation planes hi, lo (5-D: C, W, H, N, P)
  CUtensorMap tmB[2];  // weight planes hi, lo (2-D: K, Cout)
  CUtensorMap tmR[2];  // residual planes as an A operand (nres > 0): 5-D NHWC at the output resolution
  CUtensorMap tmE;     // identity matrix [256][256] bf16 as the B operand of the residual K-steps
  // ipt > 1 (several small images per tile): the same maps with box N-extent
  // ipt, used when the tile's ipt image ids are consecutive (always at full
  // batch / shadow mode, often in early compacted layers): one TMA box per
  // plane instead of ipt (per-box cost dominates 4x4 / 8x8 images)
  CUtensorMap tmAm[2];
  CUtensorMap tmRm[2];
  // Fused 1x1 projection shortcut (res_proj = 1): the residual K-steps are the
  // projection conv of the block input instead of residual x identity — A =
  // tmR/tmRm over the block input at traversal stride res_stride, B = tmP
  // (projection weights [Cout][Cx], BN scale folded, hi/lo planes), nres =
  // Cx / 64; both convs accumulate in one TMEM tile and the epilogue adds the
  // summed shift. The projection's output never exists in HBM.
  CUtensorMap tmP[2];
  int res_proj;
  int res_stride;
  int multi_img;       // 1: tmAm (and tmRm when nres > 0) are valid
  int stacked;         // bf16x3: hi*hi + hi*lo as one N = 2*BN MMA (see tc_conv.cu TcCfg)
  int nres;            // residual K-steps per tile (BN/64): out = conv + residual computed by the MMA
  // Halo mode (stride-1 k x k conv, one image per tile): 128 output anchors on
  // the padded row pitch Pw = W + k - 1 (tiles_h = tiles per image, hb = wb = 1,
  // ipt = 1); per 64-channel chunk ONE slab of halo_rows padded rows (tmA box
  // {64, Pw, halo_rows}) feeds all k*k taps as row-shifted SW128 descriptors.
  int halo;
  int halo_pw, halo_rows, halo_res_rows;
  unsigned halo_aplane;  // bytes per plane of an A-slab slot (1024-aligned)
  int halo_sb;           // B ring depth (2 A-slab slots)
  int dbg;               // measurement-only bits: 1 no TMA loads, 2 no MMAs, 4 no epilogue stores
  int staged_store;    // 1: epilogue stages 32x32 sub-tiles in shared memory and writes full sectors (mode 0, no split)
  int plain;           // 1: plain GEMM over rows (A = [rows, K], count = rows)
  int Ho, Wo;          // output spatial dims
  int hb, wb, ipt;     // output tile geometry: ipt images x hb x wb = 128 rows
  int tiles_h, tiles_w;
  int conv_stride;     // input coordinate = output * conv_stride + tap offset
  int C;               // input channels per tap (multiple of 64)
  int ntaps;
  int segs;            // 1 (bf16) or 3 (bf16x3)
  int Cout;            // output channels (multiple of BN)
  int ksplit;          // mode 1: static split-K factor
  int ks_max;          // mode 0: dynamic split-K upper bound (1 = off)
  int ks_min_steps;  // split-K: at least this many K-steps per split (0 = fill the grid)
  // plain mode, two outputs from one GEMM over shared rows (block-MLP: the next
  // block's FC and an FC(h) cache's hidden layer): output columns >= mix_n1 (a
  // multiple of BN) are written as fp32 to out_f32 [rows][mix_ld] at column
  // (c - mix_n1), like mode 1; columns < mix_n1 take the mode-0 epilogue with
  // output rows of out_ld elements. 0 = off.
  int mix_n1, mix_ld;
  int out_ld;        // plain mode-0 output row stride in elements (0 = Cout)
  float* ws;           // mode 0 split-K workspace (fp32 partial tiles)
  int* ws_counters;    // per output tile arrival counters (zeroed; reset by the last CTA unless ctr_zero)
  int* ctr_zero;       // nullable: the counter set of the NEXT split-K launch, zeroed by this launch after its
                       // upstream wait (the previous user of that set has completed); then no reset arrival
  int ctr_len;         // ints in ctr_zero
  const int* surv;     // survivor image list (nullptr = identity)
  const int* count;    // device-side image/row count (nullptr -> count_static)
  int count_static;
  int mode;            // 0: NHWC out (+lo), 1: fp32 partials [ksplit][rows_total][Cout]
  int rows_total;      // mode 1 row stride
  const float* scale;  // per-Cout multiplier (nullable = 1)
  const float* shift;  // per-Cout bias (nullable = 0)
  const __nv_bfloat16* res_hi;
  const __nv_bfloat16* res_lo;
  int relu;
  __nv_bfloat16* out_hi;
  __nv_bfloat16* out_lo;
  float* out_f32;
  float* gap_out;      // nullable: fused GAP partials [image][gap_segs][Cout] (NHWC conv mode only)
  int gap_segs;        // segments per image = tiles_h * tiles_w * max(1, hb*wb/32)
  TcGapHead gh;        // fused lookup on the GAP partials (gh.row_tiles != nullptr)
  unsigned long long* trace;  // nullable debug: clock64 stamps [8 CTAs][32 units][8]
  // Weight planes to pull into L2 before the programmatic-launch wait (they do
  // not depend on upstream kernels): each CTA prefetches 1/grid of each plane.
  const void* wpre[2];
  long long wpre_bytes;        // bytes per plane (0 = off)
  signed char tap_phase[kMaxTaps];
  signed char tap_dh[kMaxTaps];
  signed char tap_dw[kMaxTaps];
};

// Host helpers (tc_conv.cu).
bool encode_act_map(CUtensorMap* map, const void* base, int C, int W, int H, int N, int P, int wb, int hb,
                    int stride = 1, int nbox = 1);
bool encode_weight_map(CUtensorMap* map, const void* base, int K, int Cout, int BN);
int tc_conv_pick_bn(int Cout, int segs = 1);
// Halo-mode geometry for a stride-1 k x k conv over an H x W image; BN may be
// lowered to 64 so the B ring keeps >= 3 slots. False if it does not apply.
struct HaloPlan {
  int pw, rows, res_rows, tiles_per_img, sb;
  unsigned aplane;
};
bool tc_conv_halo_plan(int H, int W, int k, int stride, int pad, int Cout, bool x3, int& BN, HaloPlan& hp);
int tc_conv_ring_bytes(int BN, bool x3);

// Segments per image of the fused GAP partials for a conv tile geometry.
inline int tc_conv_gap_segs(int tiles_h, int tiles_w, int hb, int wb) {
  return tiles_h * tiles_w * (hb * wb > 32 ? hb * wb / 32 : 1);
}
// Upper bound on the tile count at count_static (used to size the grid).
int tc_conv_max_tiles(const TcConvParams& p, int BN);
// Workspace floats needed for mode-0 split-K with `max_ctas` CTAs.
size_t tc_conv_ws_floats(int BN, int max_ctas);
cudaError_t tc_conv_launch(const TcConvParams& p, int BN, int num_sms, cudaStream_t stream);

}  // namespace lcb
