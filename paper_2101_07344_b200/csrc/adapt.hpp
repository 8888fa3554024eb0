// Online adaptation loop over a device engine (adapt.cpp).
#pragma once

#include <cstdint>
#include <vector>

#include "../../include/latecache_b200.h"
#include "engine.hpp"

namespace lcb {

// One retraining record: taps at every attached cache's layer (attach order)
// and the base model's output distribution (reference TapRecord, cache.hpp:76-80).
struct AdaptRecord {
  std::vector<std::vector<double>> taps;
  std::vector<double> y;
};

struct AdaptOut {
  int* hit_layer;
  int* served;
  int* base_pred;
  double* latency_ms;
  std::vector<lc_retrain_event> events;
};

// run_adaptation (serving.cpp:213-340); request i serves inputs[req_sample[i]].
void run_adaptation(Engine& en, const float* inputs, int n_samples, const double* req_time, const int* req_sample,
                    int R, const lc_adapt_config& cfg, const std::vector<AdaptRecord>& original_train, uint64_t seed,
                    bool adapt_on, AdaptOut& out);

}  // namespace lcb
