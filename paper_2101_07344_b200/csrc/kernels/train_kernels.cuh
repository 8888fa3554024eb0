// fp64 minibatch-SGD kernels for the cache networks (online adaptation,
// SURVEY §8f rank 3): the B200 form of train_predictor / train_selector
// (reference cache.cpp:179-257) over the reference's layer set
// (network.cpp:104-164 forward, 166-232 backward, 234-262 SGD with momentum).
// Everything is double, like the reference; rows of one minibatch run in
// parallel, and every per-parameter gradient is accumulated over the
// minibatch's samples in the reference's order (accumulate_grads,
// network.cpp:274-279) with unfused multiply/add roundings.
#pragma once

#include <cuda_runtime.h>

namespace lcb {

// Layer kinds match host LayerKind (lcb_host.hpp).
struct TrainLayer {
  int kind = 0;  // 0 FC, 1 ReLU, 2 AvgPool, 3 Conv1d
  int in = 0, out = 0, window = 0, kernel = 0, stride = 0;
  double* w = nullptr;   // FC [out][in]; Conv1d [kernel]
  double* b = nullptr;   // FC [out]; Conv1d [1]
  double* vw = nullptr;  // momentum buffers (zero at start, SgdOptimizer ctor)
  double* vb = nullptr;
  // FC with a wide input: the forward splits the input range over `ksplit`
  // CTAs per output group and reduces the partials ([ksplit][rows][out]) in
  // a second pass (deterministic order).
  int ksplit = 1;
  double* part = nullptr;
};
// ksplit for an FC of input width `in` (1 = single-pass kernel).
int train_fc_ksplit(int in);

// act_out[k][:] = layer(act_in[k][:]) for k < nb. When rows != nullptr the
// input row of sample k is act_in[rows[k]] (records gathered in place).
void launch_train_forward(const TrainLayer& L, const double* act_in, long long in_ld, const int* rows, int nb,
                          double* act_out, cudaStream_t s);
// gx[k][:] = dL/dx of the layer for output gradient g (reference backward()).
void launch_train_backward_data(const TrainLayer& L, const double* act_in, const double* g, int nb, double* gx,
                                cudaStream_t s);
// Weight gradient of the minibatch, sum_k scale[k] * grad_k in sample order,
// then the SGD-with-momentum step: v = m*v + g; w -= lr*v.
void launch_train_wgrad_sgd(const TrainLayer& L, const double* act_in, long long in_ld, const int* rows,
                            const double* g, const double* scale, int nb, double lr, double momentum, cudaStream_t s);
// Distillation loss gradient (losses.cpp:72-101) per sample: logits [nb][C],
// p_tau = soften(y, tau) of each record [N][C], hard = argmax(y) per record.
// bad is set when a sample's loss is not finite.
void launch_distill_grad(const double* logits, const double* p_tau, const int* hard, const int* rows, int nb, int C,
                         double tau, double beta, double* g, int* bad, cudaStream_t s);
// p_tau[n] = soften(y[n], tau) (losses.cpp:58-70); hard[n] = argmax(y[n]).
void launch_soften(const double* y, int N, int C, double tau, double* p_tau, int* hard, int* bad, cudaStream_t s);
// Selector loss gradient (losses.cpp:103-116) per sample.
void launch_selector_grad(const double* logit, const int* target, const int* rows, int nb, double w_fp, double w_fn,
                          double* g, int* bad, cudaStream_t s);
// Row softmax in place [N][C] plus the agreement label argmax(logits) == hard
// (selector_labels, cache.cpp:210-218).
void launch_softmax_labels(double* x, int N, int C, const int* hard, int* agree, cudaStream_t s);

// Whole-schedule SGD in ONE thread block for small networks (the
// reference's MLP-tap caches: a few thousand parameters): every minibatch's
// forward, loss gradient, backward and update run back to back inside the
// block with __syncthreads between phases — no launches, and every sum is
// serial in the reference's order (forward dots included).
constexpr int kFusedMaxLayers = 4;
struct FusedNet {
  int nl = 0;
  TrainLayer L[kFusedMaxLayers];
  double* act[kFusedMaxLayers + 1] = {};  // act[i + 1] = output of layer i, [batch][out]
};
struct FusedLoss {
  int kind = 0;  // 0 distillation (predictor), 1 weighted selector loss
  int C = 0;
  double a = 0.0, b = 0.0;  // (tau, beta) or (w_fp, w_fn)
  const double* p_tau = nullptr;
  const int* hard = nullptr;    // distillation hard labels
  const int* target = nullptr;  // selector agreement labels
};
// Shared memory the fused schedule needs: weights + momentum + activations
// of rows_cap samples + two gradient buffers of rows_cap x max_dim.
size_t sgd_fused_smem_bytes(const FusedNet& net, int rows_cap, int max_dim);
constexpr size_t kFusedSmemMax = 190 * 1024;
cudaError_t launch_sgd_fused(const FusedNet& net, const double* x, long long ld, const int* rows, const double* scale,
                             const int* batch_off, const int* batch_nb, int nbatches, const FusedLoss& loss,
                             double lr, double momentum, int rows_cap, int max_dim, int* bad, cudaStream_t s);

// Tap readback for retraining records: rows [B] of hi(+lo) bf16 planes
// (row stride `ld`, D features) as doubles.
void launch_planes_to_f64(const void* hi, const void* lo, long long ld, long long D, int B, double* out,
                          cudaStream_t s);
// Base-model output distribution y = softmax(W . tap + b) per row (the MLP
// head, base_model.cpp:51-52) from the last tap's planes; W fp32 [C][D].
void launch_head_probs_f64(const void* hi, const void* lo, long long ld, int D, const float* W, const float* b, int C,
                           int B, double* logits_scratch, double* y, cudaStream_t s);

}  // namespace lcb
