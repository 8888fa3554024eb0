// Host-side model of the learned-cache serve path (B200 build).
//
// These are the reference's data types and the non-kernel functions of the
// path, restated in C++ so the product loads the reference's artifacts and
// synthesises identical weights from the same seeds:
//   Rng / mix_seed            include/latecache/rng.hpp:15-98
//   LayerSpec / Network       include/latecache/network.hpp:16-48, src/network.cpp:25-102
//   latecache-network v1      src/network.cpp:301-409
//   BaseModel (MLP family)    src/base_model.cpp:30-54, format :143-175
//   ArchSpec / build_variant  src/cache.cpp:22-140, format :452-489
//   metrics / plan / checks   src/cache.cpp:412-450, src/composer.cpp:65-160, :317-365
//   gen_workload / summarize  src/serving.cpp:31-91, :342-376
// plus the CNN family (ResNet-18/50/152, VGG-16) that BASELINE.json's configs
// name and the reference does not implement (its base layers are "parity
// unpinned by reference"; the caches on its taps are reference-pinned).
#pragma once

#include <cstdint>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

namespace lcb {

// ----------------------------------------------------------------- errors
// Mirrors the reference's exception contract: invalid_argument
// for shapes/args/infeasible plans, runtime_error for malformed artifacts.
struct InfeasiblePlan : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct CudaFailure : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// ----------------------------------------------------------------- RNG
inline uint64_t splitmix64(uint64_t& state) {
  uint64_t z = (state += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
uint64_t mix_seed(uint64_t seed, uint64_t tag);

class Rng {
 public:
  explicit Rng(uint64_t seed);
  uint64_t next_u64();
  double next_double() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * next_double(); }
  int next_int(int n);
  double normal();

 private:
  uint64_t s_[4];
  bool has_spare_ = false;
  double spare_ = 0.0;
};

// ----------------------------------------------------------------- networks
enum class LayerKind { FC = 0, ReLU = 1, Pool = 2, Conv1d = 3, Softmax = 4 };

struct LayerSpec {
  LayerKind kind = LayerKind::ReLU;
  int in_dim = 0, out_dim = 0, pool_window = 0, kernel = 0, stride = 0;
  static LayerSpec fc(int in, int out);
  static LayerSpec relu(int dim);
  static LayerSpec pool(int in, int window);
  static LayerSpec conv1d(int in, int kernel, int stride);
  static LayerSpec softmax(int dim);
};

struct LayerWeights {
  std::vector<double> w;  // FC [out, in]; Conv1d [kernel]
  std::vector<double> b;  // FC [out]; Conv1d [1]
};

struct Network {
  std::vector<LayerSpec> layers;
  std::vector<LayerWeights> weights;
  int input_dim() const { return layers.front().in_dim; }
  int output_dim() const { return layers.back().out_dim; }
};

Network make_network(std::vector<LayerSpec> layers, uint64_t seed);
long long mac_count(const Network& net);
long long parameter_count(const Network& net);
std::string save_network(const Network& net);
Network load_network(const std::string& text, size_t& pos);

std::string fmt_double(double v);
double parse_double(const std::string& s);
long long parse_int(const std::string& s);

// ----------------------------------------------------------------- CNN family
enum class CnnOpKind { Stem = 0, Conv = 1, MaxPool = 2, Head = 3 };

struct CnnOp {
  CnnOpKind kind = CnnOpKind::Conv;
  int in = -1, out = -1, res = -1;  // activation slots (-1: network input)
  int C = 0, H = 0, W = 0;          // input geometry per image
  int Cout = 0, k = 1, stride = 1, pad = 0;
  bool relu = false;
  std::vector<double> w;             // conv: OIHW [Cout][C][k][k]; head: [classes][C]
  std::vector<double> scale, shift;  // folded batch-norm (conv); head bias in shift
  int tap = -1;                      // output is block tap #tap (0-based)
  int Ho() const { return (H + 2 * pad - k) / stride + 1; }
  int Wo() const { return (W + 2 * pad - k) / stride + 1; }
};

struct TapInfo {
  int C = 0, H = 0, W = 0;
  long long dim() const { return static_cast<long long>(C) * H * W; }
};

// ----------------------------------------------------------------- base model
struct BaseModel {
  // family "mlp": the reference's make_base_model network (FC+ReLU blocks,
  // FC+softmax head). family "cnn": op list below.
  std::string family = "mlp";
  std::string arch;  // "mlp", "resnet18_cifar", "resnet50", "resnet152", "vgg16_cifar"
  Network net;
  int num_blocks = 0;
  int num_classes = 0;
  std::vector<int> tap_layer;  // mlp: index of the layer whose output is tap i
  std::vector<TapInfo> taps;   // per block: NCHW geometry of the tap (mlp: C=dim, H=W=1)
  // cnn
  int in_C = 0, in_H = 0, in_W = 0;
  std::vector<CnnOp> ops;
  int nslots = 0;

  long long input_dim() const {
    return family == "mlp" ? net.input_dim() : static_cast<long long>(in_C) * in_H * in_W;
  }
  long long tap_dim(int layer) const { return taps.at(static_cast<size_t>(layer - 1)).dim(); }
  long long macs_to_block(int block) const;  // base MACs up to and including block (0 = none)
};

BaseModel make_base_model(int input_dim, int num_classes, std::vector<int> widths, int blocks, uint64_t seed);
std::string save_base_model(const BaseModel& m);
BaseModel load_base_model(const std::string& text);
// CNN families with synthetic weights (He-normal convs, folded BN with a
// residual-branch scale so activations stay O(1) through depth).
BaseModel make_cnn_model(const std::string& arch, int num_classes, uint64_t seed);

// ----------------------------------------------------------------- caches
enum class ArchFamily { FC = 0, Pool = 1, Conv = 2 };

struct ArchSpec {
  ArchFamily family = ArchFamily::FC;
  int hidden = 0, kernel = 0, stride = 0;
  static ArchSpec parse(const std::string& text);
  std::string to_string() const;
};

int clamp_pool_width(int want, long long dim);

struct CacheVariant {
  int layer = 0;
  int variant = 0;
  ArchSpec arch;
  Network predictor;
  Network selector;
  double delta = 0.5;
};

CacheVariant build_variant(int layer, int variant_idx, const ArchSpec& arch, long long tap_dim, int num_classes,
                           uint64_t global_seed);
std::string save_variant(const CacheVariant& v);
CacheVariant load_variant(const std::string& text);

// Binary mirror of the text checkpoints (host/binfmt.cpp; raw doubles, plus the CNN op list).
std::string save_base_model_binary(const BaseModel& m);
BaseModel load_base_model_binary(const std::string& data);
std::string save_variant_binary(const CacheVariant& v);
CacheVariant load_variant_binary(const std::string& data);

// ----------------------------------------------------------------- plan
struct VariantMetrics {
  int layer = 0, variant = 0;
  ArchSpec arch;
  double hit_rate = 0.0, accuracy = 1.0, lookup_ms = 0.0, memory_mb = 0.0;
  long long tp = 0, fp = 0, tn = 0, fn = 0;
};
struct LayerProfile {
  std::vector<double> latency_ms;
  int blocks() const { return static_cast<int>(latency_ms.size()); }
  double prefix(int k) const;
  double total() const { return prefix(blocks()); }
};
struct ComposerConfig {
  double accuracy_threshold = 0.97;
  double memory_budget_mb = 0.0;
  double alpha = 0.2;
};
struct SelectionPlan {
  std::vector<size_t> chosen;
  std::vector<double> eh;
  std::vector<std::string> notes;
};
struct ConstraintReport {
  bool feasible = true;
  std::vector<std::string> violations;
};

std::vector<VariantMetrics> load_metrics(const std::string& text);
SelectionPlan make_plan(std::vector<size_t> chosen, const std::vector<VariantMetrics>& metrics);
SelectionPlan load_plan(const std::string& text, const std::vector<VariantMetrics>& metrics);
double plan_accuracy(const SelectionPlan& plan, const std::vector<VariantMetrics>& metrics);
double expected_latency(const SelectionPlan& plan, const std::vector<VariantMetrics>& metrics,
                        const LayerProfile& profile);
ConstraintReport check_constraints(const SelectionPlan& plan, const std::vector<VariantMetrics>& metrics,
                                   const LayerProfile& profile, const ComposerConfig& cfg);

// ----------------------------------------------------------------- workload
struct WorkloadSpec {
  int num_classes = 10;
  double zipf_alpha = 1.5, rotation_period_min = 15.0, requests_per_sec = 2.0, duration_min = 60.0;
  uint64_t seed = 1;
};
struct Request {
  long long id = 0;
  double time_min = 0.0;
  int true_class = 0;
  long long sample_idx = 0;
};
// labels: class of each test sample (the per-class request pools).
std::vector<Request> gen_workload(const WorkloadSpec& spec, const std::vector<int>& labels, int dataset_classes);

struct SimSummary {
  long long requests = 0;
  double avg_latency_ms = 0, p50_latency_ms = 0, p99_latency_ms = 0, max_latency_ms = 0;
  double agreement = 1, accuracy = 1, hit_rate = 0, speedup = 1;
  std::map<int, long long> hits_by_layer;
};
struct RequestTrace {
  long long id = 0;
  double time_min = 0;
  int true_class = 0, base_pred = 0, served_pred = 0, hit_layer = 0;
  double latency_ms = 0;
};
SimSummary summarize(const std::vector<RequestTrace>& traces, const LayerProfile& profile);
// Nearest-rank percentile (serving.cpp:361-365) over an unsorted sample.
double nearest_rank(std::vector<double> v, double q);

}  // namespace lcb
