// Online adaptation loop: run_adaptation
// (reference serving.cpp:213-340) over a device engine.
//
// The reference serves one request at a time and retrains/swaps between
// requests. Here requests between two control points (an interval boundary
// or a pending swap maturing) are served as shadow batches on the GPU — the
// live caches cannot change inside such a run, so the traces are the same —
// and the control flow at the control points is the reference's, step for
// step: the sliding window, recency weights, the mix-in draw, per-variant
// seeds, divergence handling and the swap rule. Retraining is the GPU
// trainer (trainer.cpp); the swap re-uploads the caches in place.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/latecache_b200.h"
#include "adapt.hpp"
#include "trainer.hpp"

namespace lcb {

namespace {

void validate_adaptation(const lc_adapt_config& c) {  // serving.cpp:199-208
  auto req = [](bool ok, const char* m) {
    if (!ok) throw std::invalid_argument(m);
  };
  req(c.sample_rate >= 0.0 && c.sample_rate <= 1.0, "adaptation: sample rate must be in [0, 1]");
  req(c.window_min > 0.0, "adaptation: window must be positive");
  req(c.retrain_interval_min > 0.0, "adaptation: retrain interval must be positive");
  req(c.recency_decay > 0.0 && c.recency_decay <= 1.0, "adaptation: recency decay must be in (0, 1]");
  req(c.mixin_fraction >= 0.0 && c.mixin_fraction < 1.0, "adaptation: mix-in fraction must be in [0, 1)");
  req(c.epochs >= 1, "adaptation: epochs must be positive");
  req(c.learning_rate > 0.0, "adaptation: learning rate must be positive");
  req(c.retrain_pause_ms >= 0.0, "adaptation: retrain pause must be nonnegative");
}

void set_note(lc_retrain_event& ev, const std::string& s) {
  std::memset(ev.note, 0, sizeof(ev.note));
  std::strncpy(ev.note, s.c_str(), sizeof(ev.note) - 1);
}

}  // namespace

void run_adaptation(Engine& en, const float* inputs, int n_samples, const double* req_time,
                    const int* req_sample, int R, const lc_adapt_config& cfg,
                    const std::vector<AdaptRecord>& original_train, uint64_t seed, bool adapt_on, AdaptOut& out) {
  validate_adaptation(cfg);
  const int K = static_cast<int>(en.variants().size());
  const long long in_dim = en.input_dim();
  const int C = en.classes();
  std::vector<int> layers;
  std::vector<long long> dims;
  for (const CacheVariant& v : en.variants()) {
    layers.push_back(v.layer);
    dims.push_back(en.model().tap_dim(v.layer));
  }
  for (const AdaptRecord& r : original_train) {
    if (static_cast<int>(r.taps.size()) != K || static_cast<int>(r.y.size()) != C)
      throw std::invalid_argument("run_adaptation: original record shape mismatch");
  }

  struct WindowSample {
    double time_min;
    AdaptRecord record;
  };
  std::vector<WindowSample> window;
  Rng sample_rng(mix_seed(seed, 0x5a3e));
  std::optional<std::vector<CacheVariant>> pending;
  double swap_time = 0.0;
  int boundary = 1;
  double next_boundary = cfg.retrain_interval_min;

  // ---- batched serving of requests [b0, b1) under the current live caches
  const int maxB = en.max_batch();
  std::vector<float> xb(static_cast<size_t>(maxB) * static_cast<size_t>(in_dim));
  std::vector<int> want;  // batch-relative rows sampled into the window
  std::vector<double> tapbuf, ybuf;
  int b0 = 0;
  std::vector<char> sampled(static_cast<size_t>(R), 0);
  auto flush = [&](int b1) {
    while (b0 < b1) {
      const int B = std::min(maxB, b1 - b0);
      for (int i = 0; i < B; ++i) {
        const int si = req_sample[b0 + i];
        if (si < 0 || si >= n_samples) throw std::invalid_argument("simulate: request points outside the test pool");
        std::memcpy(xb.data() + static_cast<size_t>(i) * in_dim, inputs + static_cast<size_t>(si) * in_dim,
                    static_cast<size_t>(in_dim) * sizeof(float));
      }
      en.serve_host(xb.data(), B, /*shadow=*/true, /*use_graph=*/true);
      en.copy_results(B, out.hit_layer + b0, out.served + b0, out.base_pred + b0, nullptr, nullptr, out.latency_ms + b0);
      want.clear();
      for (int i = 0; i < B; ++i)
        if (sampled[static_cast<size_t>(b0 + i)]) want.push_back(i);
      if (!want.empty()) {
        // full-batch readback (rows are the batch's requests in shadow mode)
        std::vector<std::vector<double>> taps(static_cast<size_t>(K));
        for (int k = 0; k < K; ++k) {
          taps[static_cast<size_t>(k)].resize(static_cast<size_t>(B) * static_cast<size_t>(dims[static_cast<size_t>(k)]));
          en.read_taps(layers[static_cast<size_t>(k)], B, taps[static_cast<size_t>(k)].data());
        }
        ybuf.resize(static_cast<size_t>(B) * C);
        en.read_base_probs(B, ybuf.data());
        for (int i : want) {
          WindowSample w;
          w.time_min = req_time[b0 + i];
          w.record.taps.resize(static_cast<size_t>(K));
          for (int k = 0; k < K; ++k) {
            const size_t D = static_cast<size_t>(dims[static_cast<size_t>(k)]);
            const double* src = taps[static_cast<size_t>(k)].data() + static_cast<size_t>(i) * D;
            w.record.taps[static_cast<size_t>(k)].assign(src, src + D);
          }
          w.record.y.assign(ybuf.begin() + static_cast<long>(i) * C, ybuf.begin() + static_cast<long>(i + 1) * C);
          window.push_back(std::move(w));
        }
      }
      b0 += B;
    }
  };
  auto swap_in = [&]() {
    for (const CacheVariant& v : *pending) en.update_variant(v);
    pending.reset();
    en.notify_swap(swap_time);
  };

  auto retrain_at = [&](double now) {  // serving.cpp:235-298
    lc_retrain_event ev{};
    ev.interval = boundary;
    ev.time_min = now;
    window.erase(std::remove_if(window.begin(), window.end(),
                                [&](const WindowSample& w) { return w.time_min < now - cfg.window_min; }),
                 window.end());
    ev.window_size = static_cast<long long>(window.size());
    if (cfg.sample_rate <= 0.0 || window.empty()) {
      set_note(ev, "skipped: no window samples");
      out.events.push_back(ev);
      return;
    }
    std::vector<const AdaptRecord*> records;
    std::vector<double> weights;
    for (const WindowSample& w : window) {
      const int age = static_cast<int>((now - w.time_min) / cfg.retrain_interval_min);
      records.push_back(&w.record);
      weights.push_back(std::pow(cfg.recency_decay, age));
    }
    Rng mix_rng(mix_seed(mix_seed(seed, static_cast<uint64_t>(boundary)), 0xe7a1));
    size_t mixin = static_cast<size_t>(
        std::llround(static_cast<double>(window.size()) * cfg.mixin_fraction / (1.0 - cfg.mixin_fraction)));
    mixin = std::min(mixin, original_train.size());
    std::vector<size_t> order(original_train.size());
    for (size_t i = 0; i < order.size(); ++i) order[i] = i;
    for (size_t i = 0; i < mixin; ++i) {
      const size_t j = i + static_cast<size_t>(mix_rng.next_int(static_cast<int>(order.size() - i)));
      std::swap(order[i], order[j]);
      records.push_back(&original_train[order[i]]);
      weights.push_back(1.0);
    }
    ev.mixin_size = static_cast<long long>(mixin);

    const int N = static_cast<int>(records.size());
    std::vector<double> ys(static_cast<size_t>(N) * C);
    for (int n = 0; n < N; ++n)
      std::copy(records[static_cast<size_t>(n)]->y.begin(), records[static_cast<size_t>(n)]->y.end(),
                ys.begin() + static_cast<long>(n) * C);
    std::vector<CacheVariant> staged = en.variants();
    std::string note;
    for (int k = 0; k < K; ++k) {
      const size_t D = static_cast<size_t>(dims[static_cast<size_t>(k)]);
      std::vector<double> X(static_cast<size_t>(N) * D);
      for (int n = 0; n < N; ++n)
        std::copy(records[static_cast<size_t>(n)]->taps[static_cast<size_t>(k)].begin(),
                  records[static_cast<size_t>(n)]->taps[static_cast<size_t>(k)].end(), X.begin() + static_cast<long>(n * D));
      TrainRecords tr;
      tr.taps = X.data();
      tr.D = static_cast<long long>(D);
      tr.y = ys.data();
      tr.C = C;
      tr.N = N;
      tr.weights = weights;
      CacheVariant candidate = staged[static_cast<size_t>(k)];
      SgdConfig rc;
      rc.learning_rate = cfg.learning_rate;
      rc.epochs = cfg.epochs;
      const uint64_t vseed = mix_seed(mix_seed(seed, static_cast<uint64_t>(boundary)), static_cast<uint64_t>(k));
      rc.seed = mix_seed(vseed, 1);
      try {
        gpu_train_predictor(en.device(), candidate, tr, rc, cfg.tau, cfg.beta);
        rc.seed = mix_seed(vseed, 2);
        gpu_train_selector(en.device(), candidate, tr, rc, cfg.w_fp, cfg.w_fn);
        staged[static_cast<size_t>(k)] = std::move(candidate);
      } catch (const CudaFailure&) {
        throw;
      } catch (const std::runtime_error&) {
        note += std::string(note.empty() ? "" : "; ") + "layer " + std::to_string(layers[static_cast<size_t>(k)]) +
                " retrain diverged, kept previous networks";
      }
    }
    set_note(ev, note);
    pending = std::move(staged);
    swap_time = now + cfg.retrain_pause_ms / 60000.0;
    ev.applied = 1;
    out.events.push_back(ev);
  };

  for (int i = 0; i < R; ++i) {
    const double t = req_time[i];
    while (t >= next_boundary) {
      flush(i);
      if (pending && next_boundary >= swap_time) swap_in();
      if (adapt_on) retrain_at(next_boundary);
      ++boundary;
      next_boundary = static_cast<double>(boundary) * cfg.retrain_interval_min;
    }
    if (pending && t >= swap_time) {
      flush(i);
      swap_in();
    }
    if (adapt_on && sample_rng.next_double() < cfg.sample_rate) sampled[static_cast<size_t>(i)] = 1;
  }
  flush(R);
}

}  // namespace lcb
