// Cache retraining on the GPU: train_predictor /
// train_selector (reference cache.cpp:179-257) as fp64 minibatch SGD on one
// B200. The host keeps the reference's control flow — Rng shuffles per epoch,
// minibatch boundaries, per-sample weights scaled by 1/|batch| — and uploads
// it once; every forward/backward/update runs on the device.
#pragma once

#include <cstdint>
#include <vector>

#include "host/lcb_host.hpp"

namespace lcb {

struct SgdConfig {  // reference TrainConfig (network.hpp:70-76)
  double learning_rate = 0.01;
  double momentum = 0.9;
  int epochs = 20;
  int batch_size = 16;
  uint64_t seed = 1;
};

// Records as the variant sees them: taps [N][D] at the variant's layer
// (tap_of, cache.cpp:172-177) and the base model's output distribution
// y [N][C]. weights: empty = 1.0 each (resolve_weights, cache.cpp:35-39).
struct TrainRecords {
  const double* taps = nullptr;
  long long D = 0;
  const double* y = nullptr;
  int C = 0;
  int N = 0;
  std::vector<double> weights;
};

// Both throw std::invalid_argument on bad inputs and std::runtime_error
// ("... loss diverged") when a loss turns non-finite; the variant is left
// unchanged then.
void gpu_train_predictor(int device, CacheVariant& v, const TrainRecords& r, const SgdConfig& cfg, double tau,
                         double beta);
void gpu_train_selector(int device, CacheVariant& v, const TrainRecords& r, const SgdConfig& cfg, double w_fp,
                        double w_fn);

}  // namespace lcb
