// C++ façade over the C-ABI (latecache_b200.h) with the reference's API shape
// (namespace latecache, /root/reference/proj/include/latecache/*.hpp): same
// function names, argument meaning and exception types, so a caller such as
// cmd_simulate (cli.cpp:742) swaps `latecache::` for `latecache_b200::` on the
// serve path. Header-only; link liblatecache_b200.so.
#pragma once

#include <cstdint>
#include <istream>
#include <iterator>
#include <memory>
#include <ostream>
#include <stdexcept>
#include <string>
#include <vector>

#include "latecache_b200.h"

namespace latecache_b200 {

// Status -> the reference's exception types (SURVEY §8b "Errors").
inline void check(int status) {
  if (status == LC_OK) return;
  const std::string msg = lc_last_error();
  if (status == LC_ERR_INVALID_ARGUMENT || status == LC_ERR_INFEASIBLE_PLAN) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

inline std::string slurp(std::istream& in) {
  return std::string(std::istreambuf_iterator<char>(in), std::istreambuf_iterator<char>());
}

// latecache::BaseModel (base_model.hpp:31-39)
class BaseModel {
 public:
  explicit BaseModel(lc_model* h) : h_(h, &lc_model_free) {
    long long d = 0;
    check(lc_model_info(h, &num_blocks, &num_classes, &d));
    input_dim_ = d;
    for (int l = 1; l <= num_blocks; ++l) {
      int C = 0, H = 0, W = 0;
      check(lc_model_tap(h, l, &C, &H, &W));
      tap_dims.push_back(static_cast<long long>(C) * H * W);
    }
  }
  long long input_dim() const { return input_dim_; }
  const lc_model* handle() const { return h_.get(); }
  int num_blocks = 0;
  int num_classes = 0;
  std::vector<long long> tap_dims;

 private:
  std::shared_ptr<lc_model> h_;
  long long input_dim_ = 0;
};

// make_base_model (base_model.cpp:30-54)
inline BaseModel make_base_model(int input_dim, int num_classes, std::vector<int> widths, int blocks, uint64_t seed) {
  lc_model* h = nullptr;
  check(lc_model_make_mlp(input_dim, num_classes, widths.data(), static_cast<int>(widths.size()), blocks, seed, &h));
  return BaseModel(h);
}
// load_base_model / save_base_model (base_model.cpp:156-175 / 143-154)
inline BaseModel load_base_model(std::istream& in) {
  const std::string t = slurp(in);
  lc_model* h = nullptr;
  check(lc_model_load(t.data(), t.size(), &h));
  return BaseModel(h);
}
inline void save_base_model(std::ostream& out, const BaseModel& m) {
  char* s = nullptr;
  size_t n = 0;
  check(lc_model_save(m.handle(), &s, &n));
  out.write(s, static_cast<std::streamsize>(n));
  lc_free(s);
}

// latecache::CacheVariant (cache.hpp:57-64)
class CacheVariant {
 public:
  explicit CacheVariant(lc_variant* h) : h_(h, &lc_variant_free) {}
  int layer() const { return info().layer; }
  double delta() const { return info().delta; }
  void set_delta(double d) { check(lc_variant_set_delta(h_.get(), d)); }
  std::string arch() const { return info().arch; }
  lc_variant* handle() const { return h_.get(); }

 private:
  struct Info {
    int layer = 0, variant = 0;
    double delta = 0.0;
    std::string arch;
  };
  Info info() const {
    Info i;
    char buf[64] = {0};
    check(lc_variant_info(h_.get(), &i.layer, &i.variant, &i.delta, buf, sizeof buf));
    i.arch = buf;
    return i;
  }
  std::shared_ptr<lc_variant> h_;
};

// build_variant (cache.cpp:104-140)
inline CacheVariant build_variant(int layer, int variant_idx, const std::string& arch, long long tap_dim,
                                  int num_classes, uint64_t global_seed) {
  lc_variant* h = nullptr;
  check(lc_variant_build(layer, variant_idx, arch.c_str(), tap_dim, num_classes, global_seed, &h));
  return CacheVariant(h);
}
// load_variant / save_variant (cache.cpp:464-489 / 452-462)
inline CacheVariant load_variant(std::istream& in) {
  const std::string t = slurp(in);
  lc_variant* h = nullptr;
  check(lc_variant_load(t.data(), t.size(), &h));
  return CacheVariant(h);
}
inline void save_variant(std::ostream& out, const CacheVariant& v) {
  char* s = nullptr;
  size_t n = 0;
  check(lc_variant_save(v.handle(), &s, &n));
  out.write(s, static_cast<std::streamsize>(n));
  lc_free(s);
}

// TrainConfig (network.hpp:70-76).
struct TrainConfig {
  double learning_rate = 0.01;
  double momentum = 0.9;
  int epochs = 20;
  int batch_size = 16;
  uint64_t seed = 1;
};

namespace detail {
inline void flat_records(const std::vector<std::vector<double>>& taps, const std::vector<std::vector<double>>& ys,
                         std::vector<double>& t, std::vector<double>& y, long long& D, int& C) {
  if (taps.empty() || taps.size() != ys.size()) throw std::invalid_argument("train: records/y count mismatch");
  D = static_cast<long long>(taps[0].size());
  C = static_cast<int>(ys[0].size());
  for (size_t i = 0; i < taps.size(); ++i) {
    if (static_cast<long long>(taps[i].size()) != D || static_cast<int>(ys[i].size()) != C)
      throw std::invalid_argument("train: ragged records");
    t.insert(t.end(), taps[i].begin(), taps[i].end());
    y.insert(y.end(), ys[i].begin(), ys[i].end());
  }
}
}  // namespace detail

// train_predictor (cache.cpp:179-208) on the GPU: taps = each record's tap at
// the variant's layer, ys = the base model's output distributions.
inline void train_predictor(CacheVariant& v, const std::vector<std::vector<double>>& taps,
                            const std::vector<std::vector<double>>& ys, const TrainConfig& cfg, double tau, double beta,
                            const std::vector<double>& sample_weights = {}, int device = 0) {
  std::vector<double> t, y;
  long long D = 0;
  int C = 0;
  detail::flat_records(taps, ys, t, y, D, C);
  if (!sample_weights.empty() && sample_weights.size() != taps.size())
    throw std::invalid_argument("train_predictor: sample weight count mismatch");
  check(lc_train_predictor(device, v.handle(), t.data(), D, y.data(), C, static_cast<int>(taps.size()),
                           sample_weights.empty() ? nullptr : sample_weights.data(), cfg.learning_rate, cfg.momentum,
                           cfg.epochs, cfg.batch_size, cfg.seed, tau, beta));
}

// train_selector (cache.cpp:220-257) on the GPU.
inline void train_selector(CacheVariant& v, const std::vector<std::vector<double>>& taps,
                           const std::vector<std::vector<double>>& ys, const TrainConfig& cfg, double w_fp, double w_fn,
                           const std::vector<double>& sample_weights = {}, int device = 0) {
  std::vector<double> t, y;
  long long D = 0;
  int C = 0;
  detail::flat_records(taps, ys, t, y, D, C);
  if (!sample_weights.empty() && sample_weights.size() != taps.size())
    throw std::invalid_argument("train_selector: sample weight count mismatch");
  check(lc_train_selector(device, v.handle(), t.data(), D, y.data(), C, static_cast<int>(taps.size()),
                          sample_weights.empty() ? nullptr : sample_weights.data(), cfg.learning_rate, cfg.momentum,
                          cfg.epochs, cfg.batch_size, cfg.seed, w_fp, w_fn));
}

// latecache::LookupResult (cache.hpp:131-135)
struct LookupResult {
  bool hit = false;
  double selector_prob = 0.0;
  std::vector<double> pr;
};

// latecache::RequestTrace subset produced by the serve path (serving.hpp:48-56).
struct RequestTrace {
  long long id = 0;
  int base_pred = -1;   // -1 when compaction skipped the full pass
  int served_pred = 0;
  int hit_layer = 0;    // 0 = miss
  double latency_ms = 0.0;  // measured device time to the request's exit
};

// latecache::Deployment (serving.hpp:61-69), resident on one GPU.
class Deployment {
 public:
  Deployment(const BaseModel& model, const std::vector<const CacheVariant*>& chosen, int max_batch, int device = 0,
             int precision = LC_PREC_BF16X3)
      : model_(model), max_batch_(max_batch) {
    std::vector<const lc_variant*> hs;
    for (const CacheVariant* v : chosen) hs.push_back(v->handle());
    lc_engine* e = nullptr;
    check(lc_engine_create(device, model.handle(), hs.data(), static_cast<int>(hs.size()), precision, max_batch, &e));
    h_.reset(e, [](lc_engine* p) { lc_engine_destroy(p); });
  }

  // lookup (cache.cpp:259-265), batched.
  std::vector<LookupResult> lookup(int layer, const std::vector<std::vector<double>>& taps) {
    const long long D = model_.tap_dims.at(static_cast<size_t>(layer - 1));
    const int C = model_.num_classes;
    std::vector<LookupResult> out;
    for (size_t s = 0; s < taps.size(); s += static_cast<size_t>(max_batch_)) {
      const int B = static_cast<int>(std::min(taps.size() - s, static_cast<size_t>(max_batch_)));
      std::vector<float> x(static_cast<size_t>(B) * D);
      for (int i = 0; i < B; ++i) {
        if (static_cast<long long>(taps[s + i].size()) != D)
          throw std::invalid_argument("forward: input dim " + std::to_string(taps[s + i].size()) + " != expected " +
                                      std::to_string(D));
        for (long long j = 0; j < D; ++j) x[static_cast<size_t>(i) * D + j] = static_cast<float>(taps[s + i][j]);
      }
      std::vector<int> hit(B), label(B);
      std::vector<float> prob(B), pr(static_cast<size_t>(B) * C);
      check(lc_lookup_batch(h_.get(), layer, x.data(), B, hit.data(), label.data(), prob.data(), pr.data(), nullptr));
      for (int i = 0; i < B; ++i) {
        LookupResult r;
        r.hit = hit[i] != 0;
        r.selector_prob = prob[i];
        r.pr.assign(pr.begin() + static_cast<long>(i) * C, pr.begin() + static_cast<long>(i + 1) * C);
        out.push_back(std::move(r));
      }
    }
    return out;
  }

  // simulate_model (serving.cpp:147-158): request k serves inputs[k].
  // shadow = true keeps the reference's semantics (full pass for every request).
  std::vector<RequestTrace> simulate_model(const std::vector<std::vector<double>>& inputs, bool shadow = true) {
    const long long D = model_.input_dim();
    std::vector<RequestTrace> traces;
    for (size_t s = 0; s < inputs.size(); s += static_cast<size_t>(max_batch_)) {
      const int B = static_cast<int>(std::min(inputs.size() - s, static_cast<size_t>(max_batch_)));
      std::vector<float> x(static_cast<size_t>(B) * D);
      for (int i = 0; i < B; ++i) {
        if (static_cast<long long>(inputs[s + i].size()) != D)
          throw std::invalid_argument("forward: input dim mismatch");
        for (long long j = 0; j < D; ++j) x[static_cast<size_t>(i) * D + j] = static_cast<float>(inputs[s + i][j]);
      }
      std::vector<int> exit_layer(B), served(B), base(B);
      std::vector<double> lat(B);
      check(lc_serve_batch(h_.get(), x.data(), B, shadow ? LC_SERVE_SHADOW : 0u, exit_layer.data(), served.data(),
                           base.data(), nullptr, nullptr, lat.data()));
      for (int i = 0; i < B; ++i) {
        RequestTrace t;
        t.id = static_cast<long long>(s) + i;
        t.base_pred = base[i];
        t.served_pred = served[i];
        t.hit_layer = exit_layer[i];
        t.latency_ms = lat[i];
        traces.push_back(t);
      }
    }
    return traces;
  }

  void set_delta(int layer, double delta) { check(lc_engine_set_delta(h_.get(), layer, delta)); }
  // run_adaptation's swap (serving.cpp:301-315): a retrained variant replaces
  // the attached cache at its layer after the batches already enqueued.
  void swap_in(const CacheVariant& v) { check(lc_engine_update_variant(h_.get(), v.handle())); }

  // measure_metrics (cache.cpp:316-335) of every attached cache at every
  // threshold of `grid`, over the records these inputs make (one batch of at
  // most max_batch): result[layer - 1][g] (zero rows where no cache).
  struct Confusion {
    long long tp = 0, fp = 0, tn = 0, fn = 0;
    double hit_rate() const {
      const long long n = tp + fp + tn + fn;
      return n ? static_cast<double>(tp + fp) / static_cast<double>(n) : 0.0;
    }
    double accuracy() const { return tp + fp ? static_cast<double>(tp) / static_cast<double>(tp + fp) : 1.0; }
  };
  std::vector<std::vector<Confusion>> measure_metrics(const std::vector<std::vector<double>>& inputs,
                                                      const std::vector<double>& grid) {
    const std::vector<float> x = flatten(inputs);
    const int B = static_cast<int>(inputs.size()), G = static_cast<int>(grid.size());
    std::vector<long long> c(static_cast<size_t>(model_.num_blocks) * G * 4);
    check(lc_measure_metrics(h_.get(), x.data(), B, grid.data(), G, c.data()));
    std::vector<std::vector<Confusion>> out(static_cast<size_t>(model_.num_blocks), std::vector<Confusion>(G));
    for (int l = 0; l < model_.num_blocks; ++l)
      for (int g = 0; g < G; ++g) {
        const long long* q = &c[(static_cast<size_t>(l) * G + g) * 4];
        out[l][g] = Confusion{q[0], q[1], q[2], q[3]};
      }
    return out;
  }

  // tune_delta (cache.cpp:267-307) for every attached cache; applies the
  // thresholds to this deployment. result[layer - 1] (NaN where no cache).
  std::vector<double> tune_delta(const std::vector<std::vector<double>>& inputs, double target_accuracy,
                                 const std::vector<double>& grid) {
    const std::vector<float> x = flatten(inputs);
    std::vector<double> d(static_cast<size_t>(model_.num_blocks));
    check(lc_tune_delta(h_.get(), x.data(), static_cast<int>(inputs.size()), target_accuracy, grid.data(),
                        static_cast<int>(grid.size()), d.data(), 1));
    return d;
  }

 private:
  std::vector<float> flatten(const std::vector<std::vector<double>>& inputs) const {
    const long long D = model_.input_dim();
    if (inputs.empty() || static_cast<int>(inputs.size()) > max_batch_)
      throw std::invalid_argument("measure: record count outside [1, max_batch]");
    std::vector<float> x(inputs.size() * static_cast<size_t>(D));
    for (size_t i = 0; i < inputs.size(); ++i) {
      if (static_cast<long long>(inputs[i].size()) != D) throw std::invalid_argument("forward: input dim mismatch");
      for (long long j = 0; j < D; ++j) x[i * D + j] = static_cast<float>(inputs[i][j]);
    }
    return x;
  }

  BaseModel model_;
  int max_batch_;
  std::shared_ptr<lc_engine> h_;
};

}  // namespace latecache_b200
