// extern "C" boundary (include/latecache_b200.h). Exceptions from the host
// restatement and the engine are mapped to status codes exactly where the
// reference would throw (std::invalid_argument / std::runtime_error).
#include <algorithm>
#include <cmath>
#include <limits>
#include <utility>
#include <vector>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>

#include "../../include/latecache_b200.h"
#include "engine.hpp"
#include "trainer.hpp"
#include "adapt.hpp"
#include "host/lcb_host.hpp"

struct lc_model {
  lcb::BaseModel m;
};
struct lc_variant {
  lcb::CacheVariant v;
};
struct lc_engine {
  std::unique_ptr<lcb::Engine> e;
};

namespace {
thread_local std::string g_err;

template <typename F>
int guard(F&& f) {
  try {
    f();
    return LC_OK;
  } catch (const lcb::InfeasiblePlan& e) {
    g_err = e.what();
    return LC_ERR_INFEASIBLE_PLAN;
  } catch (const lcb::CudaFailure& e) {
    g_err = e.what();
    return LC_ERR_CUDA;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return LC_ERR_INVALID_ARGUMENT;
  } catch (const std::out_of_range& e) {
    g_err = e.what();
    return LC_ERR_INVALID_ARGUMENT;
  } catch (const std::runtime_error& e) {
    g_err = e.what();
    return LC_ERR_RUNTIME;
  } catch (const std::exception& e) {
    g_err = e.what();
    return LC_ERR_RUNTIME;
  }
}

void need(const void* p, const char* what) {
  if (!p) throw std::invalid_argument(std::string(what) + ": null pointer");
}

char* dup(const std::string& s, size_t* len) {
  char* out = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(out, s.data(), s.size());
  out[s.size()] = '\0';
  if (len) *len = s.size();
  return out;
}

lcb::Engine& eng(lc_engine* e) {
  need(e, "engine");
  if (!e->e) throw std::invalid_argument("engine: destroyed handle");
  return *e->e;
}
}  // namespace

extern "C" {

const char* lc_last_error(void) { return g_err.c_str(); }
const char* lc_version(void) { return "latecache-b200 0.1 (sm_100a)"; }
void lc_free(void* p) { std::free(p); }

int lc_model_make_mlp(int input_dim, int num_classes, const int* widths, int n_widths, int blocks, uint64_t seed,
                      lc_model** out) {
  return guard([&] {
    need(out, "out");
    need(widths, "widths");
    auto* m = new lc_model;
    try {
      m->m = lcb::make_base_model(input_dim, num_classes, std::vector<int>(widths, widths + n_widths), blocks, seed);
    } catch (...) {
      delete m;
      throw;
    }
    *out = m;
  });
}

int lc_model_load(const char* text, size_t len, lc_model** out) {
  return guard([&] {
    need(text, "text");
    need(out, "out");
    auto* m = new lc_model;
    try {
      m->m = lcb::load_base_model(std::string(text, len));
    } catch (...) {
      delete m;
      throw;
    }
    *out = m;
  });
}

int lc_model_save(const lc_model* m, char** text, size_t* len) {
  return guard([&] {
    need(m, "model");
    need(text, "text");
    *text = dup(lcb::save_base_model(m->m), len);
  });
}

int lc_model_save_binary(const lc_model* m, char** data, size_t* len) {
  return guard([&] {
    need(m, "model");
    need(data, "data");
    need(len, "len");
    const std::string b = lcb::save_base_model_binary(m->m);
    *data = static_cast<char*>(std::malloc(b.size() ? b.size() : 1));
    std::memcpy(*data, b.data(), b.size());
    *len = b.size();
  });
}

int lc_model_load_binary(const char* data, size_t len, lc_model** out) {
  return guard([&] {
    need(data, "data");
    need(out, "out");
    auto* m = new lc_model;
    try {
      m->m = lcb::load_base_model_binary(std::string(data, len));
    } catch (...) {
      delete m;
      throw;
    }
    *out = m;
  });
}

int lc_variant_save_binary(const lc_variant* v, char** data, size_t* len) {
  return guard([&] {
    need(v, "variant");
    need(data, "data");
    need(len, "len");
    const std::string b = lcb::save_variant_binary(v->v);
    *data = static_cast<char*>(std::malloc(b.size() ? b.size() : 1));
    std::memcpy(*data, b.data(), b.size());
    *len = b.size();
  });
}

int lc_variant_load_binary(const char* data, size_t len, lc_variant** out) {
  return guard([&] {
    need(data, "data");
    need(out, "out");
    auto* v = new lc_variant;
    try {
      v->v = lcb::load_variant_binary(std::string(data, len));
    } catch (...) {
      delete v;
      throw;
    }
    *out = v;
  });
}

int lc_model_make_cnn(const char* arch, int num_classes, uint64_t seed, lc_model** out) {
  return guard([&] {
    need(arch, "arch");
    need(out, "out");
    auto* m = new lc_model;
    try {
      m->m = lcb::make_cnn_model(arch, num_classes, seed);
    } catch (...) {
      delete m;
      throw;
    }
    *out = m;
  });
}

int lc_model_info(const lc_model* m, int* blocks, int* classes, long long* input_dim) {
  return guard([&] {
    need(m, "model");
    if (blocks) *blocks = m->m.num_blocks;
    if (classes) *classes = m->m.num_classes;
    if (input_dim) *input_dim = m->m.input_dim();
  });
}

int lc_model_tap(const lc_model* m, int layer, int* C, int* H, int* W) {
  return guard([&] {
    need(m, "model");
    if (layer < 1 || layer > m->m.num_blocks) throw std::invalid_argument("tap: layer out of range");
    const lcb::TapInfo& t = m->m.taps[static_cast<size_t>(layer - 1)];
    if (C) *C = t.C;
    if (H) *H = t.H;
    if (W) *W = t.W;
  });
}

long long lc_model_macs(const lc_model* m, int block) { return m ? m->m.macs_to_block(block) : -1; }

void lc_model_free(lc_model* m) { delete m; }

int lc_model_cnn_ops(const lc_model* m, int* n_ops, int* n_slots) {
  return guard([&] {
    need(m, "model");
    if (m->m.family != "cnn") throw std::invalid_argument("model: not a CNN");
    if (n_ops) *n_ops = static_cast<int>(m->m.ops.size());
    if (n_slots) *n_slots = m->m.nslots;
  });
}

int lc_model_cnn_op(const lc_model* m, int i, lc_cnn_op_desc* out) {
  return guard([&] {
    need(m, "model");
    need(out, "out");
    if (i < 0 || i >= static_cast<int>(m->m.ops.size())) throw std::invalid_argument("cnn op index out of range");
    const lcb::CnnOp& o = m->m.ops[static_cast<size_t>(i)];
    out->kind = static_cast<int>(o.kind);
    out->in = o.in;
    out->out = o.out;
    out->res = o.res;
    out->C = o.C;
    out->H = o.H;
    out->W = o.W;
    out->Cout = o.Cout;
    out->k = o.k;
    out->stride = o.stride;
    out->pad = o.pad;
    out->relu = o.relu ? 1 : 0;
    out->tap = o.tap;
    out->w = o.w.empty() ? nullptr : o.w.data();
    out->w_len = static_cast<long long>(o.w.size());
    out->scale = o.scale.empty() ? nullptr : o.scale.data();
    out->shift = o.shift.empty() ? nullptr : o.shift.data();
  });
}

int lc_variant_build(int layer, int variant_idx, const char* arch, long long tap_dim, int num_classes, uint64_t seed,
                     lc_variant** out) {
  return guard([&] {
    need(arch, "arch");
    need(out, "out");
    auto* v = new lc_variant;
    try {
      v->v = lcb::build_variant(layer, variant_idx, lcb::ArchSpec::parse(arch), tap_dim, num_classes, seed);
    } catch (...) {
      delete v;
      throw;
    }
    *out = v;
  });
}

int lc_variant_load(const char* text, size_t len, lc_variant** out) {
  return guard([&] {
    need(text, "text");
    need(out, "out");
    auto* v = new lc_variant;
    try {
      v->v = lcb::load_variant(std::string(text, len));
    } catch (...) {
      delete v;
      throw;
    }
    *out = v;
  });
}

int lc_variant_save(const lc_variant* v, char** text, size_t* len) {
  return guard([&] {
    need(v, "variant");
    need(text, "text");
    *text = dup(lcb::save_variant(v->v), len);
  });
}

int lc_variant_set_delta(lc_variant* v, double delta) {
  return guard([&] {
    need(v, "variant");
    v->v.delta = delta;
  });
}

int lc_variant_info(const lc_variant* v, int* layer, int* variant_idx, double* delta, char* arch, int arch_len) {
  return guard([&] {
    need(v, "variant");
    if (layer) *layer = v->v.layer;
    if (variant_idx) *variant_idx = v->v.variant;
    if (delta) *delta = v->v.delta;
    if (arch && arch_len > 0) {
      const std::string a = v->v.arch.to_string();
      std::strncpy(arch, a.c_str(), static_cast<size_t>(arch_len - 1));
      arch[arch_len - 1] = '\0';
    }
  });
}

long long lc_variant_macs(const lc_variant* v) {
  return v ? lcb::mac_count(v->v.predictor) + lcb::mac_count(v->v.selector) : -1;
}

int lc_variant_layer(const lc_variant* v, int which, int idx, int* kind, int* in_dim, int* out_dim, int* pool_window,
                     int* kernel, int* stride, const double** w, long long* w_len, const double** b, long long* b_len) {
  return guard([&] {
    need(v, "variant");
    const lcb::Network& net = which == 0 ? v->v.predictor : v->v.selector;
    if (idx < 0 || idx >= static_cast<int>(net.layers.size())) throw std::invalid_argument("layer index out of range");
    const lcb::LayerSpec& s = net.layers[static_cast<size_t>(idx)];
    const lcb::LayerWeights& lw = net.weights[static_cast<size_t>(idx)];
    if (kind) *kind = static_cast<int>(s.kind);
    if (in_dim) *in_dim = s.in_dim;
    if (out_dim) *out_dim = s.out_dim;
    if (pool_window) *pool_window = s.pool_window;
    if (kernel) *kernel = s.kernel;
    if (stride) *stride = s.stride;
    if (w) *w = lw.w.empty() ? nullptr : lw.w.data();
    if (w_len) *w_len = static_cast<long long>(lw.w.size());
    if (b) *b = lw.b.empty() ? nullptr : lw.b.data();
    if (b_len) *b_len = static_cast<long long>(lw.b.size());
  });
}

int lc_variant_set_selector_out(lc_variant* v, double gain, double bias) {
  return guard([&] {
    need(v, "variant");
    auto& lw = v->v.selector.weights.back();
    for (double& x : lw.w) x *= gain;
    lw.b.back() = bias;
  });
}

void lc_variant_free(lc_variant* v) { delete v; }

int lc_plan_check(const char* metrics_text, const char* plan_text, const double* profile_ms, int blocks,
                  double accuracy_threshold, double memory_budget_mb, int* feasible, int* chosen_layers,
                  int* chosen_variants, int cap, int* n_chosen, char** report) {
  return guard([&] {
    need(metrics_text, "metrics");
    need(plan_text, "plan");
    need(profile_ms, "profile");
    const auto metrics = lcb::load_metrics(metrics_text);
    const auto plan = lcb::load_plan(plan_text, metrics);
    lcb::LayerProfile prof;
    prof.latency_ms.assign(profile_ms, profile_ms + blocks);
    lcb::ComposerConfig cfg;
    cfg.accuracy_threshold = accuracy_threshold;
    cfg.memory_budget_mb = memory_budget_mb;
    for (const auto& m : metrics)
      if (m.layer < 1 || m.layer > blocks)
        throw std::invalid_argument("composer: metrics row at layer " + std::to_string(m.layer) + " outside the profile");
    const lcb::ConstraintReport r = lcb::check_constraints(plan, metrics, prof, cfg);
    if (feasible) *feasible = r.feasible ? 1 : 0;
    if (n_chosen) *n_chosen = static_cast<int>(plan.chosen.size());
    for (size_t k = 0; k < plan.chosen.size() && static_cast<int>(k) < cap; ++k) {
      if (chosen_layers) chosen_layers[k] = metrics[plan.chosen[k]].layer;
      if (chosen_variants) chosen_variants[k] = metrics[plan.chosen[k]].variant;
    }
    if (report) {
      std::string s;
      for (const auto& v : r.violations) s += v + "\n";
      *report = dup(s, nullptr);
    }
  });
}

int lc_gen_workload(int num_classes, double zipf_alpha, double rotation_period_min, double requests_per_sec,
                    double duration_min, uint64_t seed, const int* labels, long long n_labels, int dataset_classes,
                    long long* n_out, long long* sample_idx, int* true_class, double* time_min, long long cap) {
  return guard([&] {
    need(labels, "labels");
    lcb::WorkloadSpec w;
    w.num_classes = num_classes;
    w.zipf_alpha = zipf_alpha;
    w.rotation_period_min = rotation_period_min;
    w.requests_per_sec = requests_per_sec;
    w.duration_min = duration_min;
    w.seed = seed;
    const auto s = lcb::gen_workload(w, std::vector<int>(labels, labels + n_labels), dataset_classes);
    if (n_out) *n_out = static_cast<long long>(s.size());
    for (long long i = 0; i < static_cast<long long>(s.size()) && i < cap; ++i) {
      if (sample_idx) sample_idx[i] = s[static_cast<size_t>(i)].sample_idx;
      if (true_class) true_class[i] = s[static_cast<size_t>(i)].true_class;
      if (time_min) time_min[i] = s[static_cast<size_t>(i)].time_min;
    }
  });
}

double lc_nearest_rank(const double* v, long long n, double q) {
  if (!v || n <= 0) return NAN;
  return lcb::nearest_rank(std::vector<double>(v, v + n), q);
}

int lc_engine_create(int device, const lc_model* m, const lc_variant* const* variants, int n_variants, int precision,
                     int max_batch, lc_engine** out) {
  return guard([&] {
    need(m, "model");
    need(out, "out");
    if (precision != LC_PREC_BF16X3 && precision != LC_PREC_BF16) throw std::invalid_argument("engine: bad precision");
    std::vector<lcb::CacheVariant> vs;
    for (int i = 0; i < n_variants; ++i) {
      need(variants[i], "variant");
      vs.push_back(variants[i]->v);
    }
    auto* e = new lc_engine;
    try {
      e->e = std::make_unique<lcb::Engine>(device, m->m, std::move(vs), static_cast<lcb::Precision>(precision),
                                           max_batch);
    } catch (...) {
      delete e;
      throw;
    }
    *out = e;
  });
}

int lc_engine_destroy(lc_engine* e) {
  return guard([&] {
    if (e) {
      e->e.reset();
      delete e;
    }
  });
}

int lc_engine_set_delta(lc_engine* e, int layer, double delta) {
  return guard([&] { eng(e).set_delta(layer, delta); });
}

int lc_engine_set_selector_out(lc_engine* e, int layer, double gain, double bias) {
  return guard([&] { eng(e).set_selector_out(layer, gain, bias); });
}

int lc_engine_input(lc_engine* e, float** device_ptr) {
  return guard([&] {
    need(device_ptr, "device_ptr");
    *device_ptr = eng(e).input_buffer();
  });
}

int lc_engine_stage_input(lc_engine* e, const float* src, int B, int on_device) {
  return guard([&] {
    need(src, "src");
    lcb::Engine& en = eng(e);
    if (B <= 0 || B > en.max_batch()) throw std::invalid_argument("stage_input: batch outside [1, max_batch]");
    const size_t bytes = static_cast<size_t>(B) * static_cast<size_t>(en.input_dim()) * sizeof(float);
    // a device source was written by the caller's own streams (torch's, say),
    // which the engine's non-blocking stream is not ordered after
    if (on_device && cudaDeviceSynchronize() != cudaSuccess) throw lcb::CudaFailure("stage_input: device sync failed");
    if (cudaSetDevice(en.device()) != cudaSuccess ||
        cudaMemcpyAsync(en.input_buffer(), src, bytes, on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                        en.stream()) != cudaSuccess ||
        cudaStreamSynchronize(en.stream()) != cudaSuccess)
      throw lcb::CudaFailure("stage_input: copy failed");
  });
}

int lc_serve_batch(lc_engine* e, const float* inputs, int B, unsigned flags, int* exit_layer, int* served,
                   int* base_pred, float* probs, float* logits, double* latency_ms) {
  return guard([&] {
    need(inputs, "inputs");
    lcb::Engine& en = eng(e);
    en.serve_host(inputs, B, (flags & LC_SERVE_SHADOW) != 0, (flags & LC_SERVE_NO_GRAPH) == 0);
    en.copy_results(B, exit_layer, served, base_pred, probs, logits, latency_ms);
  });
}

// measure_metrics (cache.cpp:316-335) for every attached cache at every
// threshold of the grid, over one shadow serve of the B host requests.
int lc_measure_metrics(lc_engine* e, const float* inputs, int B, const double* grid, int G, long long* counts) {
  return guard([&] {
    need(inputs, "inputs");
    need(grid, "grid");
    need(counts, "counts");
    lcb::Engine& en = eng(e);
    if (B <= 0 || B > en.max_batch()) throw std::invalid_argument("measure_metrics: batch outside [1, max_batch]");
    if (G <= 0 || G > 64) throw std::invalid_argument("measure_metrics: threshold grid must hold 1..64 values");
    const size_t bytes = static_cast<size_t>(B) * static_cast<size_t>(en.input_dim()) * sizeof(float);
    if (cudaSetDevice(en.device()) != cudaSuccess ||
        cudaMemcpyAsync(en.input_buffer(), inputs, bytes, cudaMemcpyHostToDevice, en.stream()) != cudaSuccess)
      throw lcb::CudaFailure("measure_metrics: input copy failed");
    en.measure(B, grid, G, counts);
  });
}

// ------------------------------------------------------------------ retraining
namespace {
int train_common(int which, int device, lc_variant* v, const double* taps, long long tap_dim, const double* y,
                 int classes, int N, const double* weights, double lr, double momentum, int epochs, int batch_size,
                 uint64_t seed, double a, double b) {
  return guard([&] {
    need(v, "variant");
    need(taps, "taps");
    need(y, "y");
    lcb::TrainRecords r;
    r.taps = taps;
    r.D = tap_dim;
    r.y = y;
    r.C = classes;
    r.N = N;
    if (weights && N > 0) r.weights.assign(weights, weights + N);
    lcb::SgdConfig cfg;
    cfg.learning_rate = lr;
    cfg.momentum = momentum;
    cfg.epochs = epochs;
    cfg.batch_size = batch_size;
    cfg.seed = seed;
    lcb::CacheVariant trained = v->v;  // unchanged on failure
    if (which == 0)
      lcb::gpu_train_predictor(device, trained, r, cfg, a, b);
    else
      lcb::gpu_train_selector(device, trained, r, cfg, a, b);
    v->v = std::move(trained);
  });
}
}  // namespace

int lc_train_predictor(int device, lc_variant* v, const double* taps, long long tap_dim, const double* y, int classes,
                       int N, const double* weights, double learning_rate, double momentum, int epochs, int batch_size,
                       uint64_t seed, double tau, double beta) {
  return train_common(0, device, v, taps, tap_dim, y, classes, N, weights, learning_rate, momentum, epochs, batch_size,
                      seed, tau, beta);
}

int lc_train_selector(int device, lc_variant* v, const double* taps, long long tap_dim, const double* y, int classes,
                      int N, const double* weights, double learning_rate, double momentum, int epochs, int batch_size,
                      uint64_t seed, double w_fp, double w_fn) {
  return train_common(1, device, v, taps, tap_dim, y, classes, N, weights, learning_rate, momentum, epochs, batch_size,
                      seed, w_fp, w_fn);
}

int lc_engine_update_variant(lc_engine* e, const lc_variant* v) {
  return guard([&] {
    need(v, "variant");
    eng(e).update_variant(v->v);
  });
}


int lc_run_adaptation(lc_engine* e, const float* inputs, int n_samples, const double* req_time, const int* req_sample,
                      int R, const lc_adapt_config* cfg, const double* const* original_taps, const double* original_y,
                      int N0, uint64_t seed, int adapt_on, int* hit_layer, int* served, int* base_pred,
                      double* latency_ms, lc_retrain_event* events, int events_cap, int* n_events) {
  return guard([&] {
    need(cfg, "config");
    need(n_events, "n_events");
    lcb::Engine& en = eng(e);
    if (R < 0 || N0 < 0 || n_samples < 0) throw std::invalid_argument("run_adaptation: negative count");
    if (R > 0) {
      need(inputs, "inputs");
      need(req_time, "req_time");
      need(req_sample, "req_sample");
      need(hit_layer, "hit_layer");
      need(served, "served");
      need(base_pred, "base_pred");
      need(latency_ms, "latency_ms");
    }
    const auto& vars = en.variants();
    std::vector<lcb::AdaptRecord> orig(static_cast<size_t>(N0));
    if (N0 > 0) {
      need(original_taps, "original_taps");
      need(original_y, "original_y");
    }
    const int C = en.classes();
    for (int n = 0; n < N0; ++n) {
      lcb::AdaptRecord& r = orig[static_cast<size_t>(n)];
      for (size_t k = 0; k < vars.size(); ++k) {
        const long long D = en.model().tap_dim(vars[k].layer);
        need(original_taps[k], "original_taps[k]");
        const double* src = original_taps[k] + static_cast<size_t>(n) * static_cast<size_t>(D);
        r.taps.emplace_back(src, src + D);
      }
      r.y.assign(original_y + static_cast<size_t>(n) * C, original_y + static_cast<size_t>(n + 1) * C);
    }
    lcb::AdaptOut out{hit_layer, served, base_pred, latency_ms, {}};
    lcb::run_adaptation(en, inputs, n_samples, req_time, req_sample, R, *cfg, orig, seed, adapt_on != 0, out);
    *n_events = static_cast<int>(out.events.size());
    for (int i = 0; i < std::min(events_cap, *n_events); ++i) {
      need(events, "events");
      events[i] = out.events[static_cast<size_t>(i)];
    }
  });
}

int lc_engine_set_swap_hook(lc_engine* e, lc_swap_hook hook, void* ctx) {
  return guard([&] { eng(e).set_swap_hook(hook, ctx); });
}

int lc_engine_variant(lc_engine* e, int k, lc_variant** out) {
  return guard([&] {
    need(out, "out");
    const auto& vars = eng(e).variants();
    if (k < 0 || k >= static_cast<int>(vars.size())) throw std::invalid_argument("engine_variant: index out of range");
    *out = new lc_variant{vars[static_cast<size_t>(k)]};
  });
}

// tune_delta (cache.cpp:267-307) per attached cache from the same counts:
// ascending grid; the first threshold whose hit accuracy tp/(tp+fp) (1 when
// nothing hits) reaches the target wins, else the most accurate one (first
// on ties). deltas[blocks]: NaN where no cache is attached; apply != 0 sets
// the engine's thresholds.
int lc_tune_delta(lc_engine* e, const float* inputs, int B, double target_accuracy, const double* grid, int G,
                  double* deltas, int apply) {
  return guard([&] {
    need(deltas, "deltas");
    need(grid, "grid");
    if (G <= 0 || G > 64) throw std::invalid_argument("tune_delta: empty threshold grid");
    lcb::Engine& en = eng(e);
    std::vector<std::pair<double, int>> sorted;
    for (int g = 0; g < G; ++g) sorted.push_back({grid[g], g});
    std::stable_sort(sorted.begin(), sorted.end(),
                     [](const std::pair<double, int>& a, const std::pair<double, int>& b) { return a.first < b.first; });
    const int L = en.blocks();
    std::vector<long long> counts(static_cast<size_t>(L) * G * 4);
    const int st = lc_measure_metrics(e, inputs, B, grid, G, counts.data());
    if (st != LC_OK) throw std::runtime_error(lc_last_error());
    for (int l = 1; l <= L; ++l) {
      deltas[l - 1] = std::numeric_limits<double>::quiet_NaN();
      if (!en.has_cache(l)) continue;
      double best_delta = sorted.front().first, best_acc = -1.0;
      for (const auto& dg : sorted) {
        const long long* c = &counts[(static_cast<size_t>(l - 1) * G + dg.second) * 4];
        const long long hits = c[0] + c[1];
        const double acc = hits == 0 ? 1.0 : static_cast<double>(c[0]) / static_cast<double>(hits);
        if (acc >= target_accuracy) {
          best_delta = dg.first;  // smallest qualifying threshold maximises the hit rate
          break;
        }
        if (acc > best_acc) {
          best_acc = acc;
          best_delta = dg.first;
        }
      }
      deltas[l - 1] = best_delta;
      if (apply) en.set_delta(l, best_delta);
    }
  });
}

int lc_engine_layer_times(lc_engine* e, const float* inputs, int B, unsigned flags, double* block_ms,
                          double* lookup_ms) {
  return guard([&] {
    need(inputs, "inputs");
    need(block_ms, "block_ms");
    need(lookup_ms, "lookup_ms");
    lcb::Engine& en = eng(e);
    if (B <= 0 || B > en.max_batch()) throw std::invalid_argument("layer_times: batch outside [1, max_batch]");
    const size_t bytes = static_cast<size_t>(B) * static_cast<size_t>(en.input_dim()) * sizeof(float);
    if (cudaSetDevice(en.device()) != cudaSuccess ||
        cudaMemcpyAsync(en.input_buffer(), inputs, bytes, cudaMemcpyHostToDevice, en.stream()) != cudaSuccess)
      throw lcb::CudaFailure("layer_times: input copy failed");
    en.layer_times(B, block_ms, lookup_ms, (flags & LC_SERVE_SHADOW) == 0);
  });
}

int lc_serve_submit(lc_engine* e, const float* inputs, int B, unsigned flags, int* slot) {
  return guard([&] {
    need(inputs, "inputs");
    need(slot, "slot");
    *slot = eng(e).submit(inputs, B, (flags & LC_SERVE_SHADOW) != 0);
  });
}

int lc_serve_collect(lc_engine* e, int slot, int B, int* exit_layer, int* served, int* base_pred, float* probs,
                     float* logits,
                     double* latency_ms) {
  return guard([&] { eng(e).collect(slot, B, exit_layer, served, base_pred, probs, logits, latency_ms); });
}

int lc_serve_device(lc_engine* e, int B, unsigned flags) {
  return guard([&] { eng(e).serve(B, (flags & LC_SERVE_SHADOW) != 0, (flags & LC_SERVE_NO_GRAPH) == 0); });
}

int lc_engine_sync(lc_engine* e) {
  return guard([&] { eng(e).synchronize(); });
}

int lc_engine_results(lc_engine* e, int B, int* exit_layer, int* served, int* base_pred, float* probs, float* logits,
                      double* latency_ms) {
  return guard([&] {
    lcb::Engine& en = eng(e);
    if (B <= 0 || B > en.max_batch()) throw std::invalid_argument("results: batch outside [1, max_batch]");
    en.copy_results(B, exit_layer, served, base_pred, probs, logits, latency_ms);
  });
}

int lc_engine_read_tap(lc_engine* e, const float* inputs, int B, int layer, float* out) {
  return guard([&] {
    need(inputs, "inputs");
    need(out, "out");
    lcb::Engine& en = eng(e);
    if (B <= 0 || B > en.max_batch()) throw std::invalid_argument("read_tap: batch outside [1, max_batch]");
    const size_t bytes = static_cast<size_t>(B) * static_cast<size_t>(en.input_dim()) * sizeof(float);
    if (cudaSetDevice(en.device()) != cudaSuccess ||
        cudaMemcpyAsync(en.input_buffer(), inputs, bytes, cudaMemcpyHostToDevice, en.stream()) != cudaSuccess)
      throw lcb::CudaFailure("read_tap: input upload failed");
    en.read_tap_nchw(layer, B, out);
  });
}

int lc_engine_counts(lc_engine* e, int* counts) {
  return guard([&] {
    need(counts, "counts");
    lcb::Engine& en = eng(e);
    en.synchronize();
    if (cudaMemcpy(counts, en.layer_counts(), static_cast<size_t>(en.blocks() + 1) * sizeof(int),
                   cudaMemcpyDeviceToHost) != cudaSuccess)
      throw lcb::CudaFailure("counts: d2h failed");
  });
}

int lc_lookup_batch(lc_engine* e, int layer, const float* taps, int B, int* hit, int* label, float* prob, float* pr,
                    float* logits) {
  return guard([&] {
    need(taps, "taps");
    lcb::Engine& en = eng(e);
    en.lookup_host(layer, taps, B, hit, label, prob, pr, logits);
  });
}

int lc_engine_time(lc_engine* e, int B, unsigned flags, int iters, double* ms_per_batch) {
  return guard([&] {
    need(ms_per_batch, "ms_per_batch");
    *ms_per_batch = eng(e).time_serve_ms(B, (flags & LC_SERVE_SHADOW) != 0, iters);
  });
}

int lc_serve_timed(lc_engine* e, int B, unsigned flags, double* ms) {
  return guard([&] {
    need(ms, "ms");
    *ms = eng(e).serve_timed(B, (flags & LC_SERVE_SHADOW) != 0);
  });
}

int lc_engine_kernel_count(lc_engine* e, unsigned flags, int kind) {
  if (!e || !e->e) return -1;
  return e->e->count_kernels((flags & LC_SERVE_SHADOW) != 0, kind);
}

int lc_engine_profile(lc_engine* e, int B, unsigned flags, int cap, int* n, int* kinds, double* ms, double* flops,
                      double* bytes) {
  return guard([&] {
    const auto prof = eng(e).profile(B, (flags & LC_SERVE_SHADOW) != 0);
    if (n) *n = static_cast<int>(prof.size());
    for (size_t i = 0; i < prof.size() && static_cast<int>(i) < cap; ++i) {
      if (kinds) kinds[i] = prof[i].kind;
      if (ms) ms[i] = prof[i].ms;
      if (flops) flops[i] = prof[i].flops;
      if (bytes) bytes[i] = prof[i].bytes;
    }
  });
}

}  // extern "C"
