// Serve-path kernels other than the tensor-core contractions: the learned-cache
// lookup heads (reference lookup(), cache.cpp:259-265), the first-hit exit
// and stream compaction (serve_one, serving.cpp:112-121), and the CNN glue
// (stem im2col, stride-2 phase split, max-pool, GAP+FC head).
//
// Tap addressing: every tap is an activation stored hi (+lo) bf16 with
// `row_stride` elements per request and, inside a row, NHWC order (C
// innermost). The reference's caches see the NCHW-flattened vector, so flat
// index f maps to storage offset (f % HW) * C + f / HW (for MLP taps HW == 1,
// which is the identity).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace lcb {

struct TapView {
  const __nv_bfloat16* hi;
  const __nv_bfloat16* lo;  // nullable (bf16 tier)
  long long row_stride;     // elements per request row
  int C, HW;                // channels, pixels (MLP: C = dim, HW = 1)
  const int* data_idx;      // row r -> storage row (nullable = r)
  const int* count;         // rows in this layer
};

// First-hit exit + stable stream compaction fused into the LAST CTA of a
// lookup head launch (arrival counter): rows with hit leave; ids_in[r] is the
// original request id of row r; kept rows go to ids_out (and their row index
// to src_rows_out, nullable), their number to count_out. shadow != 0: every
// row stays (probing continues) but only the first hit of a request is
// recorded (serve_one, serving.cpp:112-121).
struct ExitParams {
  int* arrive;               // nullptr = no exit/compaction (lookup-only)
  int layer, shadow;
  const int* ids_in;
  int* exit_layer;
  int* served;
  unsigned long long* exit_ns;
  float* probs_out;          // [B] this layer's probabilities by request id (nullable)
  int* labels_out;           // [B] this layer's argmax(pr) by request id (nullable)
  int* ids_out;
  int* src_rows_out;         // nullable
  int* count_out;
  // Row-compacted activations (block-MLP compact mode): the row's own CTA
  // appends a kept row at an atomic position of ids_out (count_out zeroed at
  // batch start) and copies its activation row there — no last-CTA scan, no
  // separate gather launch. The survivors' order then varies from run to run;
  // no request's values do (the next layer's rows are independent).
  const __nv_bfloat16* rows_src_hi;  // nullptr: ordered compaction by the last CTA (exit_tail)
  const __nv_bfloat16* rows_src_lo;
  __nv_bfloat16* rows_dst_hi;
  __nv_bfloat16* rows_dst_lo;
  long long row_elems;
  // compact mode without row copies (CNN taps): 1 = the warp-per-row head
  // appends misses at atomic positions (one atomic per CTA) instead of the
  // last CTA's ordered scan; survivors' order then varies, no request's values do
  int unordered;
  // compact mode without row copies, warp heads: ordered compaction by a
  // single-pass look-back scan (each CTA publishes its miss count tagged with
  // the serve's epoch, then sums its predecessors') instead of the last CTA's
  // scan; nullable. scan_agg: [head grid] per cache layer (grid <= kScanMaxCtas)
  unsigned long long* scan_agg;
  const int* epoch;
};
constexpr int kScanMaxCtas = 296;  // = 2 CTAs per SM: every CTA of the head grid co-resident

// Per-row cache head inputs (one of three predictor families).
struct CacheHeadParams {
  int family;              // 0 = FC(h), 1 = Pool(width), 2 = Conv(k,s)
  int classes;
  int feat;                // pool: width; fc: hidden h; conv: number of chunks
  const float* feats;      // pool: bins [rows][feat]; fc: partials [ks][rows_total][hp]; conv: partials [rows][chunks][classes]
  int ks;                  // fc split-K factor
  int hp;                  // fc padded hidden stride
  long long rows_total;    // fc partial row stride
  const float* b1;         // fc: hidden bias [h]
  const float* W2;         // pool: [classes][width]; fc: [classes][h]
  const float* b2;         // [classes]
  const float* Ws1;        // selector FC(C,16): [16][classes]
  const float* bs1;        // [16]
  const float* ws2;        // FC(16,1): [16]
  float bs2;
  double delta;
  const int* count;
  // Pool(C) = GAP from tc_conv's fused partials gap[image][gap_segs][feat]
  // (nullable): the head sums them itself (classes <= 32) instead of reading feats.
  const float* gap;
  int gap_segs;
  float gap_inv;           // 1 / (H*W)
  const int* gap_ids;      // row r -> image id
  // outputs (row-indexed)
  float* prob;             // [rows] selector probability
  int* hit;                // [rows]
  int* label;              // [rows] argmax(pr)
  float* pr_out;           // nullable [rows][classes]
  float* logits_out;       // nullable [rows][classes]
  float* fc_scratch;       // nullable: [rows_fc_splits(feat)][max_rows][classes]; enables the
                           // batched logits GEMM for classes > 32
  // set by launch_cache_head: split-K logit partials (logit = b2 + sum_z part[z])
  const float* pre_logits;
  int pre_nz;
  long long pre_zstride;
  ExitParams ex;           // ex.arrive != nullptr: fused first-hit exit + compaction
  // Direct row mode (block-MLP taps, one contiguous row per request): the head
  // reads its row (hi + lo) and computes the Pool(w) bins or the Conv(k,s)
  // layer itself — no separate predictor launch. row_hi == nullptr: off.
  const __nv_bfloat16* row_hi;
  const __nv_bfloat16* row_lo;
  long long row_stride;
  int D;                   // tap length
  int win;                 // pool window (family 1)
  float pool_inv;          // 1 / win
  int kernel, stride, out_dim;  // conv (family 2)
  const float* w1;         // conv kernel [kernel]
  float b1c;               // conv bias
};

int rows_fc_splits(int feat);

void launch_pool_bins(const TapView& tap, int max_rows, int win, int width, float* bins, cudaStream_t s);
// Pool(C) bins from tc_conv's fused GAP partials gap[image][segs][C].
void launch_gap_bins(const float* gap, int segs, int C, int HW, const int* data_idx, const int* count, int max_rows,
                     float* bins, cudaStream_t s);
void launch_conv1d_partials(const TapView& tap, int max_rows, long long D, int kernel, int stride, int out_dim,
                            const float* w1, float b1, const float* W2, int classes, int chunk_elems, int nchunks,
                            float* partials, cudaStream_t s);
// Head (+ batched logits GEMM for classes > 32) and, with p.ex.arrive, the
// fused exit/compaction: one or two launches per cache layer.
void launch_cache_head(const CacheHeadParams& p, int max_rows, cudaStream_t s);
// out[z][r][k] = sum_{o in slice z} A(r,o) W[k][o] for r < *count, z < rows_fc_splits(feat)
// (ascending o inside a slice; out z-stride = max_rows*classes).
// ks == 0: A dense [rows][lda]; ks > 0: A(r,o) = relu(b1[o] + sum_s A[s*part_stride + r*lda + o]).
void launch_rows_fc(const float* A, long long lda, int ks, long long part_stride, const float* b1, int feat,
                    const float* W, int classes, const int* count, int max_rows, float* out, cudaStream_t s);

// Confusion counts of measure_metrics (cache.cpp:316-335) for every probed
// layer at every threshold of `grid` (device, G <= 64): counts[l][g] =
// {tp, fp, tn, fn} over the requests whose layer-l probability was recorded
// (probs not NaN); agree = (label == base_pred), hit = (double)p >= grid[g].
void launch_confusion(const float* probs, const int* labels, const int* base_pred, int max_batch, const int* batch,
                      int L, const double* grid, int G, unsigned long long* counts, cudaStream_t s);

// Pool(C) caches whose head reads the GAP partials directly (one launch per layer).
bool fused_lookup_supported(int classes, int C, int max_rows);

// Pool(C) caches with > 32 classes over tc_conv's fused GAP partials: GAP
// features, logits, head and (h.ex.arrive) the exit in ONE persistent launch
// of num_sms CTAs (grid barriers; needs every CTA resident: one per SM).
// feats [max_rows][C], logits [max_rows][classes] scratch; gsync: 2 ints,
// zero-initialised once (self-resetting).
bool wide_lookup_supported(int classes, int C, int num_sms);
size_t wide_lookup_smem(int classes, int C, int grid);
void launch_wide_lookup(const CacheHeadParams& h, float* feats, float* logits, int* gsync, int num_sms,
                        cudaStream_t s);
// Measurement only (tests/cuda/wide_bench): CTA 0 of later wide-lookup launches
// writes %globaltimer at its phase boundaries into stamps[0..7] (nullptr: off).
void set_wide_lookup_stamps(unsigned long long* stamps);

// Copies rows src_rows[j] of src into row j of dst (hi and lo planes).
void launch_gather_rows(const __nv_bfloat16* src_hi, const __nv_bfloat16* src_lo, __nv_bfloat16* dst_hi,
                        __nv_bfloat16* dst_lo, long long row_elems, const int* src_rows, const int* count,
                        int max_rows, cudaStream_t s);

// fp32 rows [rows][in_dim] (row stride in_dim) -> hi/lo bf16 [rows][dp],
// zero padded; row j comes from src row ids[j] (nullable = j).
void launch_split_rows(const float* x, int in_dim, int dp, const int* ids, const int* count, int max_rows,
                       __nv_bfloat16* hi, __nv_bfloat16* lo, cudaStream_t s);
// fp32 NCHW-flat taps -> hi/lo NHWC storage (lookup-only entry point).
void launch_split_taps_nchw(const float* x, int C, int HW, int rows, long long row_stride, __nv_bfloat16* hi,
                            __nv_bfloat16* lo, cudaStream_t s);

// Stored tap rows [rows][row_stride] (NHWC, hi + lo) -> fp32 NCHW-flat [rows][C*HW].
void launch_planes_to_nchw(const __nv_bfloat16* hi, const __nv_bfloat16* lo, long long row_stride, int C, int HW,
                           int rows, float* out, cudaStream_t s);

// MLP head: logits = W [classes][dim] . act + b, softmax, argmax -> base_pred.
void launch_mlp_head(const __nv_bfloat16* hi, const __nv_bfloat16* lo, int dp, int dim, const float* W, const float* b,
                     int classes, const int* ids, const int* count, int max_rows, int* base_pred, float* logits_out,
                     int* exit_layer, int* served, unsigned long long* exit_ns, cudaStream_t s);
// CNN head: GAP over HW then FC [classes][C] + b, softmax, argmax.
// feats_scratch [max_rows][C] / logits_scratch [rows_fc_splits(C)][max_rows][classes] (nullable)
// enable the batched path (GAP rows + logits GEMM) used for classes > 32.
void launch_cnn_head(const __nv_bfloat16* hi, const __nv_bfloat16* lo, int C, int HW, const float* W, const float* b,
                     int classes, const int* ids, const int* count, int max_rows, int* base_pred, float* logits_out,
                     int* exit_layer, int* served, unsigned long long* exit_ns, float* feats_scratch,
                     float* logits_scratch, cudaStream_t s);

// Stem: NCHW fp32 images -> im2col rows [(n*Ho+oh)*Wo+ow][Kp] hi/lo with K
// order (r, s, c), zero padded to Kp.
void launch_stem_im2col(const float* x, const int* count, int max_n, int C, int H, int W, int k, int stride, int pad,
                        int Ho, int Wo, int Kp, __nv_bfloat16* hi, __nv_bfloat16* lo, cudaStream_t s);
// Stride-2 phase split of survivors: [N,H,W,C] -> [4][N][Hs][Ws][C].
void launch_phase_split(const __nv_bfloat16* hi, const __nv_bfloat16* lo, int H, int W, int C, int N, int Hs, int Ws,
                        const int* ids, const int* count, int max_rows, __nv_bfloat16* ohi, __nv_bfloat16* olo,
                        cudaStream_t s);
void launch_maxpool(const __nv_bfloat16* hi, const __nv_bfloat16* lo, int H, int W, int C, int k, int stride, int pad,
                    int Ho, int Wo, const int* ids, const int* count, int max_rows, __nv_bfloat16* ohi,
                    __nv_bfloat16* olo, cudaStream_t s);

void launch_stamp_start(unsigned long long* t0, cudaStream_t s);
// *p = v as a stream-ordered kernel (the value travels in the launch parameters,
// so back-to-back submissions never race on a host staging word).
void launch_set_int(int* p, int v, cudaStream_t s);
// Batch prologue: ids0 = identity, count0 = B (and *batch_out), rows_out = B *
// rows_mult (stem GEMM rows, nullable), outputs reset, probs [L][max_batch] =
// NaN, *t0 = %globaltimer (batch start, nullable).
void launch_init_batch(int B, int* batch_out, int max_batch, int* ids0, int* count0, int* rows_out, int rows_mult,
                       int* exit_layer, int* served, int* base_pred, unsigned long long* exit_ns, float* probs, int L,
                       unsigned long long* t0, cudaStream_t s);
// host stub of the batch-init kernel (locates its node in a captured graph) and its argument count
const void* init_batch_kernel_fn();
constexpr int kInitBatchArgs = 14;

}  // namespace lcb
