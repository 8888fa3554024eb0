/* latecache-b200: C-ABI boundary of the B200-native learned-cache serve path.
 *
 * The reference (latecache, /root/reference/proj) exposes this path only as a
 * C++ library API in namespace latecache. Each entry point
 * below replaces one reference interface; the cited file:line is the
 * function it stands in for. Plain pointers and sizes only; all handles are
 * opaque. Every function returns LC_OK or an error code, with a message in
 * lc_last_error() (thread-local). Codes map 1:1 onto the reference's
 * exception types: LC_ERR_INVALID_ARGUMENT = std::invalid_argument,
 * LC_ERR_RUNTIME = std::runtime_error (malformed artifacts),
 * LC_ERR_INFEASIBLE_PLAN = the invalid_argument simulate_model throws for a
 * plan that fails check_constraints (serving.cpp:23-29), LC_ERR_CUDA = device
 * failure. There is no CPU fallback: engine calls fail with LC_ERR_CUDA when
 * no sm_100 device is present.
 */
#ifndef LATECACHE_B200_H
#define LATECACHE_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define LC_API __attribute__((visibility("default")))
#else
#define LC_API
#endif

#ifdef __cplusplus
extern "C" {
#pragma GCC visibility push(default)
#endif

#define LC_OK 0
#define LC_ERR_INVALID_ARGUMENT 1
#define LC_ERR_RUNTIME 2
#define LC_ERR_INFEASIBLE_PLAN 3
#define LC_ERR_CUDA 4

/* Precision tiers of the tensor-core contractions. */
#define LC_PREC_BF16X3 0 /* hi/lo bf16 split, fp32-class: the parity tier */
#define LC_PREC_BF16 1   /* plain bf16 operands, fp32 accumulate */

/* lc_serve_* flags */
#define LC_SERVE_SHADOW 1u   /* no compaction: every request runs full depth (base_pred for all) */
#define LC_SERVE_NO_GRAPH 2u /* launch kernels directly instead of replaying the CUDA graph */

typedef struct lc_model lc_model;     /* latecache::BaseModel   (base_model.hpp:31-39) */
typedef struct lc_variant lc_variant; /* latecache::CacheVariant (cache.hpp:57-64) */
typedef struct lc_engine lc_engine;   /* latecache::Deployment   (serving.hpp:61-69), resident on one GPU */

const char* lc_last_error(void);
const char* lc_version(void);
void lc_free(void* p); /* frees strings returned by the *_save functions */

/* ------------------------------------------------------------ base models */
/* make_base_model (base_model.cpp:30-54) */
int lc_model_make_mlp(int input_dim, int num_classes, const int* widths, int n_widths, int blocks, uint64_t seed,
                      lc_model** out);
/* load_base_model (base_model.cpp:156-175), "latecache-model v1" text */
int lc_model_load(const char* text, size_t len, lc_model** out);
/* save_base_model (base_model.cpp:143-154) */
int lc_model_save(const lc_model* m, char** text, size_t* len);
/* CNN families of BASELINE.json (no reference counterpart): "resnet18_cifar",
 * "resnet50", "resnet152", "vgg16_cifar"; synthetic weights from `seed`. */
int lc_model_make_cnn(const char* arch, int num_classes, uint64_t seed, lc_model** out);
/* Binary checkpoints: the text formats' content with raw
 * little-endian doubles (no decimal round trip; multi-GB weights), plus the
 * CNN op list. save: *data malloc'd (free with lc_free); load: LC_ERR_RUNTIME
 * on a truncated / malformed buffer (the reference's malformed-file errors). */
int lc_model_save_binary(const lc_model* m, char** data, size_t* len);
int lc_model_load_binary(const char* data, size_t len, lc_model** out);
int lc_variant_save_binary(const lc_variant* v, char** data, size_t* len);
int lc_variant_load_binary(const char* data, size_t len, lc_variant** out);
int lc_model_info(const lc_model* m, int* blocks, int* classes, long long* input_dim);
/* Tap geometry of block `layer` (1-based), NCHW: dim = C*H*W (mlp: C = width, H = W = 1). */
int lc_model_tap(const lc_model* m, int layer, int* C, int* H, int* W);
/* Base multiply-accumulates per request up to and including `block` (0 = none, blocks = full). */
long long lc_model_macs(const lc_model* m, int block);
void lc_model_free(lc_model* m);

/* CNN op list (for the CPU oracle's restatement of the same network). */
typedef struct {
  int kind; /* 0 stem conv, 1 conv, 2 max-pool, 3 GAP + FC head */
  int in, out, res; /* activation slots (-1 = network input / none) */
  int C, H, W, Cout, k, stride, pad, relu, tap;
  const double* w; /* conv OIHW [Cout][C][k][k]; head [classes][C] */
  long long w_len;
  const double* scale; /* folded batch-norm, per Cout (conv) */
  const double* shift; /* folded batch-norm shift (conv) / head bias */
} lc_cnn_op_desc;
int lc_model_cnn_ops(const lc_model* m, int* n_ops, int* n_slots);
int lc_model_cnn_op(const lc_model* m, int i, lc_cnn_op_desc* out);

/* ------------------------------------------------------------ cache variants */
/* build_variant (cache.cpp:104-140); arch = "FC(h)" | "Pool(w)" | "Conv(k,s)" (ArchSpec::parse, cache.cpp:80-97) */
int lc_variant_build(int layer, int variant_idx, const char* arch, long long tap_dim, int num_classes, uint64_t seed,
                     lc_variant** out);
/* load_variant / save_variant (cache.cpp:464-489 / :452-462), "latecache-variant v1" text */
int lc_variant_load(const char* text, size_t len, lc_variant** out);
int lc_variant_save(const lc_variant* v, char** text, size_t* len);
/* CacheVariant::delta (cache.hpp:63) */
int lc_variant_set_delta(lc_variant* v, double delta);
int lc_variant_info(const lc_variant* v, int* layer, int* variant_idx, double* delta, char* arch, int arch_len);
/* predictor_macs + selector_macs (cache.cpp:307-308) */
long long lc_variant_macs(const lc_variant* v);
/* Layer `idx` of the predictor (which = 0) or selector (which = 1): kind as
 * network.hpp:14 (0 FC, 1 ReLU, 2 AvgPool, 3 Conv1d, 4 Softmax) and borrowed
 * weight pointers (valid while the variant lives). Returns LC_ERR_INVALID_ARGUMENT past the end. */
int lc_variant_layer(const lc_variant* v, int which, int idx, int* kind, int* in_dim, int* out_dim, int* pool_window,
                     int* kernel, int* stride, const double** w, long long* w_len, const double** b, long long* b_len);
/* force_selector (test_serving.cpp:123-129) generalised: selector output weights *= gain, final bias = bias. */
int lc_variant_set_selector_out(lc_variant* v, double gain, double bias);
void lc_variant_free(lc_variant* v);

/* ------------------------------------------------------------ plan checks */
/* load_metrics + load_plan + check_constraints (cache.cpp:424-450, composer.cpp:330-365, :128-160).
 * profile_ms[blocks]. *feasible = 1/0; *report (nullable, free with lc_free) = violations, one per line.
 * Plan-file choices are written to chosen_layers/chosen_variants (capacity cap, count in *n_chosen). */
int lc_plan_check(const char* metrics_text, const char* plan_text, const double* profile_ms, int blocks,
                  double accuracy_threshold, double memory_budget_mb, int* feasible, int* chosen_layers,
                  int* chosen_variants, int cap, int* n_chosen, char** report);

/* ------------------------------------------------------------ workload / summary */
/* gen_workload (serving.cpp:61-91) over per-sample labels of the test split. */
int lc_gen_workload(int num_classes, double zipf_alpha, double rotation_period_min, double requests_per_sec,
                    double duration_min, uint64_t seed, const int* labels, long long n_labels, int dataset_classes,
                    long long* n_out, long long* sample_idx, int* true_class, double* time_min, long long cap);
/* Nearest-rank percentile (serving.cpp:361-365). */
double lc_nearest_rank(const double* v, long long n, double q);

/* ------------------------------------------------------------ engine */
/* Deployment on `device`: the base model plus the plan's chosen variants
 * (any order; probed in ascending layer; at most one per layer, as
 * make_plan, composer.cpp:65-89). Weights are copied to HBM. */
int lc_engine_create(int device, const lc_model* m, const lc_variant* const* variants, int n_variants, int precision,
                     int max_batch, lc_engine** out);
int lc_engine_destroy(lc_engine* e);
int lc_engine_set_delta(lc_engine* e, int layer, double delta);
int lc_engine_set_selector_out(lc_engine* e, int layer, double gain, double bias);
/* Device input buffer [max_batch][input_dim] fp32 (images: NCHW). */
int lc_engine_input(lc_engine* e, float** device_ptr);
/* Copy B requests' inputs into that buffer (on the engine stream, synchronous);
 * src is a device pointer when on_device != 0, else host memory. */
int lc_engine_stage_input(lc_engine* e, const float* src, int B, int on_device);

/* simulate_model -> serve_one (serving.cpp:97-158) for one batch of B requests,
 * end to end from HOST buffers: inputs [B][input_dim] fp32 in; per request
 * exit_layer (0 = miss, served by the base model), served label, base label
 * (-1 where compaction skipped the full pass), selector probability per
 * probed layer probs [blocks][B] (NaN = not probed), the base model's logits
 * [B][classes] (pre-softmax head output, the reference's
 * forward().activations[size-2], network.hpp:57-60; NaN rows where compaction
 * skipped the full pass), device-timed latency (ms from batch start to the
 * request's exit). Output pointers are nullable. */
int lc_serve_batch(lc_engine* e, const float* inputs, int B, unsigned flags, int* exit_layer, int* served,
                   int* base_pred, float* probs, float* logits, double* latency_ms);
/* Pipelined form of lc_serve_batch (two slots): submit enqueues the H2D copy
 * of `inputs` (pinned host memory for a truly asynchronous copy) on a copy
 * stream, the serve and the result D2H on the engine stream, and returns at
 * once with a ticket; the next submit's upload overlaps this batch's
 * compute. collect waits for the ticket's batch and returns the lc_serve_batch
 * outputs. A slot must be collected before its next reuse: a third submit
 * drops the uncollected batch and its ticket then fails with
 * LC_ERR_INVALID_ARGUMENT. */
int lc_serve_submit(lc_engine* e, const float* inputs, int B, unsigned flags, int* ticket);
int lc_serve_collect(lc_engine* e, int ticket, int B, int* exit_layer, int* served, int* base_pred, float* probs,
                     float* logits, double* latency_ms);
/* Same, input already in lc_engine_input(); enqueued asynchronously. */
int lc_serve_device(lc_engine* e, int B, unsigned flags);
int lc_engine_sync(lc_engine* e);
int lc_engine_results(lc_engine* e, int B, int* exit_layer, int* served, int* base_pred, float* probs, float* logits,
                      double* latency_ms);
/* forward_with_taps (base_model.cpp:56-63) tap read-back: runs the B host
 * requests in shadow mode up to block `layer` and returns that block's tap
 * as the reference's caches see it, out [B][tap_dim] fp32 NCHW-flat (the
 * device's hi + lo planes summed). */
int lc_engine_read_tap(lc_engine* e, const float* inputs, int B, int layer, float* out);
/* Surviving requests after each block: counts[0..blocks] (counts[0] = B). */
int lc_engine_counts(lc_engine* e, int* counts);

/* lookup (cache.cpp:259-265) batched: taps [B][tap_dim] fp32 NCHW-flat (host);
 * hit[B], label = argmax(pr) [B], prob = selector probability [B],
 * pr [B][classes], logits [B][classes] (nullable). */
int lc_lookup_batch(lc_engine* e, int layer, const float* taps, int B, int* hit, int* label, float* prob, float* pr,
                    float* logits);

/* measure_metrics (cache.cpp:316-335) for every attached cache at every
 * threshold of grid[G] (G <= 64), batched: one shadow serve of the B host
 * requests (every cache probed, full base pass), then confusion counts per
 * layer and threshold, counts [blocks][G][4] = {tp, fp, tn, fn}: hit = selector
 * probability >= threshold, agree = argmax(pr) == base prediction. Layers
 * without a cache get zeros. Replaces the per-record lookup loop of
 * measure_metrics / explore_variants (cache.cpp:316-335, 337-...). */
int lc_measure_metrics(lc_engine* e, const float* inputs, int B, const double* grid, int G, long long* counts);
/* tune_delta (cache.cpp:267-307) for every attached cache over the same batch:
 * deltas[blocks] (NaN where no cache); apply != 0 sets the engine thresholds. */
int lc_tune_delta(lc_engine* e, const float* inputs, int B, double target_accuracy, const double* grid, int G,
                  double* deltas, int apply);

/* Cache retraining on the GPU (reference cache.hpp:113-125):
 * train_predictor (cache.cpp:179-208, distillation loss with tau/beta) and
 * train_selector (cache.cpp:220-257, weighted selector loss with w_fp/w_fn),
 * fp64 minibatch SGD with momentum on `device`. Records: taps [N][tap_dim] at
 * the variant's layer (tap_of, cache.cpp:172-177), y [N][classes] base-model
 * output distributions, weights [N] or NULL (= 1.0 each). TrainConfig fields
 * (network.hpp:70-76) are passed as scalars. On success v holds the trained
 * networks; LC_ERR_RUNTIME "... loss diverged" (the reference's runtime_error)
 * leaves v unchanged; bad sizes are LC_ERR_INVALID_ARGUMENT. */
int lc_train_predictor(int device, lc_variant* v, const double* taps, long long tap_dim, const double* y, int classes,
                       int N, const double* weights, double learning_rate, double momentum, int epochs, int batch_size,
                       uint64_t seed, double tau, double beta);
int lc_train_selector(int device, lc_variant* v, const double* taps, long long tap_dim, const double* y, int classes,
                      int N, const double* weights, double learning_rate, double momentum, int epochs, int batch_size,
                      uint64_t seed, double w_fp, double w_fn);
/* Swap a retrained variant into a running engine (run_adaptation's atomic
 * swap, serving.cpp:301-315): uploads v's networks and threshold over the
 * cache attached at v's layer, stream-ordered after every batch already
 * enqueued. v must have the attached variant's architecture. */
int lc_engine_update_variant(lc_engine* e, const lc_variant* v);

/* Online adaptation: run_adaptation (serving.cpp:213-340)
 * over a running engine. AdaptationConfig (serving.hpp:85-94) plus the
 * CacheTrainConfig fields the retrain uses (tau, beta, w_fp, w_fn). */
typedef struct lc_adapt_config {
  double sample_rate, window_min, retrain_interval_min, recency_decay, mixin_fraction;
  int epochs;
  double learning_rate, retrain_pause_ms;
  double tau, beta, w_fp, w_fn;
} lc_adapt_config;
/* RetrainEvent (serving.hpp:96-103). */
typedef struct lc_retrain_event {
  int interval;
  double time_min;
  long long window_size, mixin_size;
  int applied;
  char note[160];
} lc_retrain_event;
/* Request i (time-ordered) serves samples[req_sample[i]] (inputs [n_samples][input_dim]). Serving runs in shadow batches of up to max_batch
 * requests between swap/retrain points; sampled requests' taps at the attached
 * caches' layers and base distributions come back from the device as the
 * window records. original_taps[k] = [N0][tap_dim of attached cache k] (probe
 * order: ascending layer, as make_plan sorts), original_y [N0][classes]: the original training records (mix-in).
 * Retrains run on the GPU (lc_train_predictor/selector) and swap in with
 * lc_engine_update_variant. Outputs per request: hit_layer (0 = miss), served,
 * base_pred, latency_ms (device time within its batch); events[<= events_cap],
 * *n_events = total retrain events. The engine ends holding the final
 * variants (lc_engine_variant). MLP base family only (the reference's). */
int lc_run_adaptation(lc_engine* e, const float* inputs, int n_samples, const double* req_time,
                      const int* req_sample, int R, const lc_adapt_config* cfg, const double* const* original_taps,
                      const double* original_y, int N0, uint64_t seed, int adapt_on, int* hit_layer, int* served,
                      int* base_pred, double* latency_ms, lc_retrain_event* events, int events_cap, int* n_events);
/* Copy of the engine's k-th attached variant (probe order: ascending layer), e.g. the final
 * variants after lc_run_adaptation. */
int lc_engine_variant(lc_engine* e, int k, lc_variant** out);

/* Swap observer for lc_run_adaptation (replaces nothing in the reference: its
 * single-process loop swaps `live = *pending` in place, serving.cpp:303-315).
 * hook(ctx, t) runs on the calling thread right after a pending retrain has
 * landed in the engine: requests at time >= t are served by the new caches,
 * which lc_engine_variant() returns at that moment. A trainer replica uses it
 * to broadcast each swap to the request-sharded replicas. hook == NULL clears. */
typedef void (*lc_swap_hook)(void* ctx, double swap_time_min);
int lc_engine_set_swap_hook(lc_engine* e, lc_swap_hook hook, void* ctx);

/* Hardware-aware costs (replaces CostModel::lookup_ms, cache.hpp:46-55, and the
 * modeled LayerProfile, composer.hpp): one batch of the B host requests through
 * the graph with device timestamps at every block boundary: flags
 * LC_SERVE_SHADOW = every request runs every block (the reference's
 * LayerProfile semantics), 0 = the compacted step (survivors only).
 * block_ms[blocks] = base-model device time per block (block 1 includes the
 * stem, the last block the head) — the LayerProfile for check_constraints /
 * compose; lookup_ms[blocks] = cache lookup + exit time at each layer (0 where
 * no cache is attached) — the VariantMetrics::lookup_ms column. */
int lc_engine_layer_times(lc_engine* e, const float* inputs, int B, unsigned flags, double* block_ms,
                          double* lookup_ms);

/* Device time of `iters` graph replays of a B-request batch (CUDA events on the engine stream). */
int lc_engine_time(lc_engine* e, int B, unsigned flags, int iters, double* ms_per_batch);
/* One batch from lc_engine_input(), CUDA events around it on the engine stream; synchronous. */
int lc_serve_timed(lc_engine* e, int B, unsigned flags, double* ms);
/* Kernel launches per batch of the given kind (-1 all, 1 tensor-core, 2 lookup, 3 exit/compaction). */
int lc_engine_kernel_count(lc_engine* e, unsigned flags, int kind);
/* One batch with CUDA events around every step (no graph): per step its kind,
 * device ms, algorithmic FLOPs and bytes (per-unit figure x surviving units).
 * Writes at most `cap` entries; *n = number of steps. */
int lc_engine_profile(lc_engine* e, int B, unsigned flags, int cap, int* n, int* kinds, double* ms, double* flops,
                      double* bytes);

#ifdef __cplusplus
#pragma GCC visibility pop
}
#endif
#endif
