// Device engine: a Deployment (reference serving.hpp:61-69) resident on one
// B200. Holds the base model and the plan's chosen cache variants in HBM and
// runs the batched serve path — the B200 form of simulate_model ->
// serve_one (serving.cpp:97-158): base forward block by block, the cache
// lookup at every chosen layer, first-hit exit and stream compaction so
// deeper layers only run on the surviving requests.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <functional>
#include <memory>
#include <vector>

#include "host/lcb_host.hpp"
#include "kernels/serve_kernels.cuh"
#include "kernels/tc_conv.cuh"
#include "kernels/tc_stem.cuh"

namespace lcb {

enum Precision { kPrecX3 = 0, kPrecBF16 = 1 };

struct Planes {
  __nv_bfloat16* hi = nullptr;
  __nv_bfloat16* lo = nullptr;
  size_t elems = 0;
};

struct DevCache;  // per chosen layer
struct Step {
  std::function<void(cudaStream_t)> run;
  int kind = 0;      // 0 = other, 1 = tensor-core contraction, 2 = lookup, 3 = exit/compaction
  int launches = 1;  // kernel launches this step enqueues
  // Algorithmic work = per-unit figure x units processed, where units =
  // counts[count_idx] after the batch (surviving requests; -1 = none).
  int count_idx = -1;
  double flops_per_unit = 0.0;
  double bytes_per_unit = 0.0;
};

struct StepProfile {
  int kind;
  double ms, flops, bytes;
};

class Engine {
 public:
  Engine(int device, const BaseModel& model, std::vector<CacheVariant> variants, Precision prec, int max_batch);
  ~Engine();
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;

  // Observer of run_adaptation's swaps (serving.cpp:303-315): called after a
  // pending retrain has landed in the engine, with the swap time (requests at
  // time >= t are served by the new caches). Used to replicate swaps across
  // request-sharded replicas (shard.py).
  using SwapHook = void (*)(void* ctx, double swap_time_min);
  void set_swap_hook(SwapHook hook, void* ctx) {
    swap_hook_ = hook;
    swap_ctx_ = ctx;
  }
  void notify_swap(double swap_time_min) const {
    if (swap_hook_) swap_hook_(swap_ctx_, swap_time_min);
  }

  // ----- serve
  float* input_buffer() { return d_x_; }  // [max_batch][input_dim] fp32 (device)
  long long input_dim() const { return model_.input_dim(); }
  // Enqueue a batch already in input_buffer(). shadow: no compaction (every
  // request runs full depth; base_pred for all; first hit recorded).
  void serve(int B, bool shadow, bool use_graph);
  void serve_host(const float* x, int B, bool shadow, bool use_graph);
  // Pipelined serving from pinned host memory (two slots): the H2D copy of a
  // submitted batch runs on a copy stream while the previous batch computes;
  // results come back by D2H into the slot's pinned buffers. submit returns
  // a ticket ((generation << 1) | slot); collect waits for it and copies the
  // results out, rejecting a ticket whose slot a later submit reused.
  int submit(const float* x_pinned, int B, bool shadow);
  void collect(int slot, int B, int* exit_layer, int* served, int* base, float* probs_LB, float* logits,
               double* latency_ms);
  void synchronize();
  // Results (device pointers, indexed by request id).
  const int* exit_layer() const { return d_exit_; }
  const int* served() const { return d_served_; }
  const int* base_pred() const { return d_base_; }
  const unsigned long long* exit_ns() const { return d_exit_ns_; }
  const unsigned long long* start_ns() const { return d_t0_; }
  const float* probs() const { return d_probs_; }  // [blocks][max_batch]
  const int* layer_counts() const { return d_counts_; }  // [blocks + 1]
  // logits [B][classes]: the base model's pre-softmax output (network.hpp:57-60,
  // activations[size-2]); rows of requests whose full pass compaction skipped are NaN.
  void copy_results(int B, int* exit_layer, int* served, int* base, float* probs_LB, float* logits,
                    double* latency_ms);
  // Tap of block `layer` for requests [0, B) as the reference sees it (fp32,
  // NCHW-flat, hi + lo): runs the batch staged in input_buffer() in shadow
  // mode up to that block (direct launches) and reads the activation back.
  void read_tap_nchw(int layer, int B, float* host_out);

  // ----- lookup only (reference lookup() on caller-provided NCHW-flat taps)
  void lookup(int layer, const float* taps_dev, int B, int* hit, int* label, float* prob, float* pr, float* logits);
  void lookup_host(int layer, const float* taps_host, int B, int* hit, int* label, float* prob, float* pr,
                   float* logits);

  // Batched measure_metrics / tune_delta support (cache.cpp:267-335): a
  // shadow serve of the B staged requests (every cache probed, full base
  // pass), then confusion counts {tp, fp, tn, fn} per layer and threshold.
  // counts: host [blocks][G][4]; rows of layers without a cache are zero.
  void measure(int B, const double* grid, int G, long long* counts);
  // Hardware-aware costs: one shadow batch of the B staged
  // requests through the graph with %globaltimer stamps at every block
  // boundary: block_ms[l] = base-model time of block l (the reference's
  // LayerProfile entries; block 1 includes the stem, the last block the head),
  // lookup_ms[l] = the cache lookup + exit at layer l (0 where none).
  // compact: the same stamps in the compacted step (survivors only).
  void layer_times(int B, double* block_ms, double* lookup_ms, bool compact = false);
  void set_delta(int layer, double delta);
  double delta(int layer) const;
  bool has_cache(int layer) const {
    return layer >= 1 && layer < static_cast<int>(cache_of_layer_.size()) && cache_of_layer_[static_cast<size_t>(layer)] >= 0;
  }
  void set_selector_out(int layer, double gain, double bias);
  // Swap a retrained variant (same architecture) in for the cache at its
  // layer, after every batch already enqueued (run_adaptation's swap,
  // serving.cpp:301-315).
  void update_variant(const CacheVariant& v);
  // Retraining records of the last SHADOW batch (MLP base family): taps of
  // rows [0, B) at `layer` as doubles [B][tap_dim] and the base model's output
  // distribution y [B][classes] (forward_with_taps, base_model.cpp:56-63).
  void read_taps(int layer, int B, double* host_out);
  void read_base_probs(int B, double* host_out);
  const std::vector<CacheVariant>& variants() const { return variants_; }

  // ----- introspection
  int device() const { return device_; }
  int max_batch() const { return max_batch_; }
  int blocks() const { return model_.num_blocks; }
  int classes() const { return model_.num_classes; }
  const BaseModel& model() const { return model_; }
  cudaStream_t stream() const { return stream_; }
  int num_steps(bool shadow) const;
  int count_kernels(bool shadow, int kind);
  // Time `iters` serve() calls (graph replay) with CUDA events on the engine stream.
  double time_serve_ms(int B, bool shadow, int iters);
  // One batch (graph replay), CUDA events on the engine stream around it; synchronous.
  double serve_timed(int B, bool shadow);
  // One batch with CUDA events around every step (no graph) and the
  // algorithmic work each step did.
  std::vector<StepProfile> profile(int B, bool shadow);

 private:
  void build_weights();
  enum { kModeCompact = 0, kModeShadow = 1, kModeCompactStamped = 2, kModes = 3 };
  void build_mlp_steps(std::vector<Step>& steps, bool shadow, bool stamps);
  void build_cnn_steps(std::vector<Step>& steps, bool shadow, bool stamps);
  std::vector<Step>& steps_mode(int mode);
  void serve_mode(int B, int mode, bool use_graph);
  void add_lookup_steps(std::vector<Step>& steps, DevCache& c, const TapView& tap, int max_rows, bool stage_gather,
                        bool fused_gap = false, const ExitParams* ex = nullptr, bool hidden_done = false);
  ExitParams exit_params(int layer, bool shadow, const int* ids_in, int* ids_out, int* src_rows_out, int* count_out);
  void add_stamp(std::vector<Step>& steps, int layer, int which);
  std::vector<Step>& steps_for(bool shadow);
  void* dalloc(size_t bytes);
  void h2d(void* dst, const void* src, size_t bytes);
  Planes alloc_planes(size_t elems, bool zero = true);
  Planes upload_planes(const std::vector<float>& v);
  float* upload_f32(const std::vector<float>& v);

  int device_;
  int num_sms_ = 148;
  Precision prec_;
  int max_batch_;
  BaseModel model_;
  std::vector<CacheVariant> variants_;
  std::vector<std::unique_ptr<DevCache>> caches_;  // by chosen order
  std::vector<int> cache_of_layer_;                // layer -> index or -1
  cudaStream_t stream_ = nullptr;
  std::vector<void*> allocs_;

  // batch state
  float* d_x_ = nullptr;
  int* d_batch_ = nullptr;
  int* h_batch_ = nullptr;  // pinned
  int* d_ids_ = nullptr;    // [blocks + 1][max_batch]
  int* d_src_ = nullptr;    // [blocks + 1][max_batch]
  int* d_counts_ = nullptr; // [blocks + 1] (+1 stem rows)
  int* d_exit_ = nullptr;
  int* d_served_ = nullptr;
  int* d_base_ = nullptr;
  unsigned long long* d_exit_ns_ = nullptr;
  unsigned long long* d_t0_ = nullptr;
  float* d_probs_ = nullptr;
  float* d_logits_ = nullptr;  // [max_batch][classes] base logits by request id
  unsigned long long* d_block_ns_ = nullptr;  // shadow mode: [blocks][2] = {base work done, lookup done}
  int* d_labels_ = nullptr;   // [blocks][max_batch] argmax(pr) of every probed layer
  double* d_grid_ = nullptr;  // measure(): threshold grid (<= 64)
  unsigned long long* d_conf_ = nullptr;  // measure(): [blocks][64][4]

  // MLP weights: per block FC (padded) + head
  struct DevFC {
    int in = 0, out = 0, inp = 0, outp = 0;
    Planes w;
    float* b = nullptr;
  };
  std::vector<DevFC> mlp_fc_;
  std::vector<Planes> mlp_act_;   // [blocks] outputs (taps), [max_batch][outp]
  std::vector<Planes> mlp_cin_;   // [blocks] compacted inputs of block b+1
  Planes mlp_in_;
  float* head_w_ = nullptr;
  float* head_b_ = nullptr;

  // CNN weights/buffers
  struct DevConv {
    Planes w;  // [Cout][k*k*C] (stem: [64][Kp])
    float* scale = nullptr;
    float* shift = nullptr;
    int Kp = 0;
  };
  std::vector<DevConv> cnn_w_;    // by op index
  std::vector<Planes> slot_buf_;  // by slot
  float* ws_ = nullptr;        // split-K workspace shared by all contractions (stream-ordered)
  int* ws_counters_ = nullptr;
  bool gap_fusion_ = true;  // LCB_NO_GAP_FUSION=1 disables the fused Pool(C) partials
  bool staged_store_ = true;  // LCB_DIRECT_STORE=1: per-row 16-byte stores instead of the staged coalesced epilogue
  bool mma_residual_ = true;  // LCB_NO_MMA_RESIDUAL=1: residual added in the epilogue instead of by identity K-steps
  // Fused projection shortcuts (LCB_NO_PROJ_FUSION=1 off): a 1x1 projection
  // conv whose only use is the residual of a later conv runs as that conv's
  // residual K-steps (TcConvParams::res_proj). By op index:
  bool proj_fusion_ = true;
  // block-MLP compact mode: kept rows appended at atomic positions by their own
  // head CTA, which also copies the activation row (LCB_ORDERED_COMPACTION=1:
  // the last CTA's ordered scan + a gather launch)
  bool mlp_row_append_ = true;
  bool direct_rows_ = true;  // block-MLP Pool / Conv caches computed inside the head (no predictor launch)
  // Stem + 3x3/s2 max-pool: the horizontal half of the pool rides the stem's
  // epilogue, the vertical half is a small kernel (LCB_NO_STEM_POOL=1 off).
  bool stem_pool_ = true;
  int stem_pool_op_ = -1;  // the max-pool op fused with the stem (-1: none)
  std::vector<int> proj_into_;  // projection op -> the conv it is fused into (-1: runs on its own)
  std::vector<int> fused_proj_;  // conv op -> its fused projection op (-1: none)
  __nv_bfloat16* identity_ = nullptr;
  bool fused_lookup_ = true;
  bool wide_lookup_ = true;  // LCB_NO_WIDE_LOOKUP=1: GAP bins + logits GEMM + head as three launches
  bool stacked_ = true;
  int ks_min_steps_ = 0;
  bool mlp_fuse_hidden_ = true;  // block-MLP FC(h) hidden layer fused into the next block's GEMM (LCB_MLP_FUSE_HIDDEN)
  bool unordered_ids_ = false;
  bool scan_compaction_ = true;  // warp heads: ordered compaction by look-back scan (LCB_SCAN_COMPACTION=0: last-CTA scan)
  unsigned long long* d_scan_ = nullptr;  // [L + 1][kScanMaxCtas] look-back records  // CNN compact mode: atomic survivor appends in the warp heads (LCB_UNORDERED_IDS)
  int mlp_ks_min_steps_ = 8;  // block-MLP layers: K-steps per split at least (LCB_MLP_KS_MIN_STEPS; C1 sweep 0/2/4/8/12/16/24: 8 best)
  bool wprefetch_ = true;  // LCB_NO_WPREFETCH=1: no L2 prefetch of conv weights before the PDL wait  // LCB_KS_MIN_STEPS: split-K floor of K-steps per split (CNN convs)  // LCB_NO_STACKED=1: three MMAs per bf16x3 K16 group everywhere
  bool halo_ = false;  // LCB_HALO=1: stride-1 convs load one padded-row halo slab per channel chunk  // LCB_UNFUSED_LOOKUP=1: gap_bins + head + exit_compact as three launches
  int* lk_arrive_ = nullptr;
  // lookup fused into the tap conv (TcGapHead): per-row tile arrivals and the
  // head arrival counter (both zeroed, reset in-kernel); LCB_NO_CONV_HEAD=1 off
  int* row_tiles_ = nullptr;
  int* heads_done_ = nullptr;
  int* wide_sync_ = nullptr;
  SwapHook swap_hook_ = nullptr;
  void* swap_ctx_ = nullptr;
  // split-K launches of the step list being built (assign_counter_sets)
  std::vector<std::shared_ptr<TcConvParams>> split_prms_;
  void assign_counter_sets();  // grid barrier of the wide lookup (2 ints, self-resetting)
  // Lookup (<= 32 classes) fused into the tap conv, opt-in (LCB_NO_CONV_HEAD=0):
  // post-phase after a grid barrier (warp per row), or with LCB_CONV_HEAD_TILE=1
  // the older per-tile row arrivals. Both measured slower than the separate
  // head launch on R18 (profiles/r02_fused_head_ab.txt, profiles/r02c/).
  bool conv_head_ = false;
  bool conv_head_post_ = true;
  int tc_dbg_ = 0;
  unsigned* conv_sync_ = nullptr;  // grid-barrier counter of the post-phase (monotonic, zeroed once)
  Planes im2col_buf_;

  std::vector<Step> steps_[kModes];
  std::vector<int> tap_step_end_;  // shadow step list: index one past the op producing tap l (by layer)
  bool built_[kModes] = {false, false, false};
  cudaGraphExec_t graph_[kModes] = {nullptr, nullptr, nullptr};
  cudaGraph_t graph_tmpl_[kModes] = {nullptr, nullptr, nullptr};          // captured template (owns the init node)
  cudaGraphNode_t graph_init_node_[kModes] = {nullptr, nullptr, nullptr};  // batch-init node: B is its argument 0
  int graph_batch_[kModes] = {0, 0, 0};                                     // B the executable graph holds
  int cur_batch_ = 0;  // batch size of the serve being issued (the init step's argument)
  void drop_graph(int mode);
  cudaEvent_t ev0_ = nullptr, ev1_ = nullptr;
  struct Slot {
    float* d_in = nullptr;  // staged input [max_batch][input_dim]
    int* h_exit = nullptr;  // pinned results
    int* h_served = nullptr;
    int* h_base = nullptr;
    float* h_probs = nullptr;  // [blocks][max_batch]
    float* h_logits = nullptr;  // [max_batch][classes]
    unsigned long long* h_ns = nullptr;  // [max_batch + 1]: exit times, then t0
    cudaEvent_t in_done = nullptr, in_free = nullptr, out_done = nullptr;
    int B = 0;
    unsigned gen = 0;  // submit generation: tickets are (gen << 1) | slot
    bool busy = false;
  };
  Slot slots_[2];
  int next_slot_ = 0;
  cudaStream_t copy_stream_ = nullptr;
  void init_slots();

  // lookup-only scratch
  Planes lk_tap_;
  int* d_lk_count_ = nullptr;
  friend struct DevCache;
};

}  // namespace lcb
