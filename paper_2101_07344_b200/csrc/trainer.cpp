// GPU cache retraining — see trainer.hpp.
#include "trainer.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <utility>

#include "kernels/train_kernels.cuh"

namespace lcb {
namespace {

void tck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaFailure(std::string("train: ") + what + ": " + cudaGetErrorString(e));
}

// Stream-ordered device allocations (the CUDA pool allocator: no device-wide
// sync per retrain), released on scope exit (also on throw).
class Arena {
 public:
  explicit Arena(cudaStream_t s) : s_(s) {}
  ~Arena() {
    for (void* p : ptrs_) cudaFreeAsync(p, s_);
  }
  template <typename T>
  T* alloc(size_t n) {
    void* p = nullptr;
    tck(cudaMallocAsync(&p, std::max<size_t>(n, 1) * sizeof(T), s_), "cudaMallocAsync");
    ptrs_.push_back(p);
    return static_cast<T*>(p);
  }
  template <typename T>
  T* upload(const T* src, size_t n, cudaStream_t s) {
    T* d = alloc<T>(n);
    if (n) tck(cudaMemcpyAsync(d, src, n * sizeof(T), cudaMemcpyHostToDevice, s), "upload");
    return d;
  }

 private:
  cudaStream_t s_;
  std::vector<void*> ptrs_;
};

struct DeviceGuard {
  int prev = 0;
  explicit DeviceGuard(int dev) {
    tck(cudaGetDevice(&prev), "cudaGetDevice");
    tck(cudaSetDevice(dev), "cudaSetDevice");
  }
  ~DeviceGuard() { cudaSetDevice(prev); }
};

// One training stream per device and host thread, created on first use.
cudaStream_t train_stream(int device) {
  thread_local std::vector<cudaStream_t> streams;
  if (static_cast<int>(streams.size()) <= device) streams.resize(static_cast<size_t>(device) + 1, nullptr);
  cudaStream_t& s = streams[static_cast<size_t>(device)];
  if (!s) tck(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "cudaStreamCreate");
  return s;
}

int kind_code(LayerKind k) {
  switch (k) {
    case LayerKind::FC: return 0;
    case LayerKind::ReLU: return 1;
    case LayerKind::Pool: return 2;
    case LayerKind::Conv1d: return 3;
    default: throw std::invalid_argument("train: softmax layers are not trainable here");
  }
}

// A network resident on the device with zeroed momentum (SgdOptimizer ctor,
// network.cpp:234-244) and activation buffers for `rows` samples.
struct DevNet {
  std::vector<TrainLayer> layers;
  std::vector<double*> act;  // act[i + 1] = output of layer i, [rows][out]
  DevNet(const Network& net, int rows, Arena& A, cudaStream_t s) {
    act.push_back(nullptr);
    for (size_t i = 0; i < net.layers.size(); ++i) {
      const LayerSpec& sp = net.layers[i];
      TrainLayer L;
      L.kind = kind_code(sp.kind);
      L.in = sp.in_dim;
      L.out = sp.out_dim;
      L.window = sp.pool_window;
      L.kernel = sp.kernel;
      L.stride = sp.stride;
      const LayerWeights& w = net.weights[i];
      if (L.kind == 0 || L.kind == 3) {
        L.w = A.upload(w.w.data(), w.w.size(), s);
        L.b = A.upload(w.b.data(), w.b.size(), s);
        L.vw = A.alloc<double>(w.w.size());
        L.vb = A.alloc<double>(w.b.size());
        tck(cudaMemsetAsync(L.vw, 0, w.w.size() * sizeof(double), s), "memset");
        tck(cudaMemsetAsync(L.vb, 0, w.b.size() * sizeof(double), s), "memset");
      }
      if (L.kind == 0) {
        L.ksplit = train_fc_ksplit(L.in);
        if (L.ksplit > 1) L.part = A.alloc<double>(static_cast<size_t>(L.ksplit) * rows * L.out);
      }
      layers.push_back(L);
      act.push_back(A.alloc<double>(static_cast<size_t>(rows) * sp.out_dim));
    }
  }
  // Forward of nb samples whose inputs are rows `rows` of x (ld = row stride).
  void forward(const double* x, long long ld, const int* rows, int nb, cudaStream_t s) const {
    for (size_t i = 0; i < layers.size(); ++i) {
      if (i == 0)
        launch_train_forward(layers[0], x, ld, rows, nb, act[1], s);
      else
        launch_train_forward(layers[i], act[i], layers[i].in, nullptr, nb, act[i + 1], s);
    }
  }
  // Backward from the output gradient in g (clobbers g/gx), weights updated
  // after each layer's input gradient is taken (same values as the
  // reference's backward-then-step).
  void backward_step(const double* x, long long ld, const int* rows, int nb, double* g, double* gx,
                     const double* scale, double lr, double mom, cudaStream_t s) const {
    for (int i = static_cast<int>(layers.size()) - 1; i >= 0; --i) {
      const TrainLayer& L = layers[static_cast<size_t>(i)];
      const double* in = i == 0 ? x : act[static_cast<size_t>(i)];
      const long long in_ld = i == 0 ? ld : L.in;
      const int* r = i == 0 ? rows : nullptr;
      if (i > 0) launch_train_backward_data(L, in, g, nb, gx, s);
      launch_train_wgrad_sgd(L, in, in_ld, r, g, scale, nb, lr, mom, s);
      if (i > 0) std::swap(g, gx);
    }
  }
  void download(Network& net, cudaStream_t s) const {
    for (size_t i = 0; i < layers.size(); ++i) {
      const TrainLayer& L = layers[i];
      if (!L.w) continue;
      LayerWeights& w = net.weights[i];
      tck(cudaMemcpyAsync(w.w.data(), L.w, w.w.size() * sizeof(double), cudaMemcpyDeviceToHost, s), "download");
      tck(cudaMemcpyAsync(w.b.data(), L.b, w.b.size() * sizeof(double), cudaMemcpyDeviceToHost, s), "download");
    }
    tck(cudaStreamSynchronize(s), "sync");
  }
  int max_dim() const {
    int m = 0;
    for (const TrainLayer& L : layers) m = std::max({m, L.in, L.out});
    return m;
  }
};

// The reference's epoch/minibatch schedule (cache.cpp:185-205): per epoch
// Rng::shuffle of the record order, then batches of batch_size with
// per-sample gradient scale (1/|batch|) * weight.
struct Schedule {
  std::vector<int> rows;       // [epochs][N]
  std::vector<double> scale;   // [epochs][N]
  std::vector<std::pair<int, int>> batches;  // (offset into rows, nb)
};

Schedule make_schedule(int N, const SgdConfig& cfg, uint64_t tag, const std::vector<double>& weights) {
  if (cfg.batch_size < 1) throw std::invalid_argument("train: batch size must be positive");
  Schedule sc;
  Rng rng(mix_seed(cfg.seed, tag));
  std::vector<int> order(static_cast<size_t>(N));
  for (int i = 0; i < N; ++i) order[static_cast<size_t>(i)] = i;
  for (int e = 0; e < cfg.epochs; ++e) {
    for (int i = N - 1; i > 0; --i) std::swap(order[static_cast<size_t>(i)], order[static_cast<size_t>(rng.next_int(i + 1))]);
    const int base = e * N;
    int pos = 0;
    while (pos < N) {
      const int end = std::min(N, pos + cfg.batch_size);
      const double inv = 1.0 / static_cast<double>(end - pos);
      for (int k = pos; k < end; ++k) {
        const int r = order[static_cast<size_t>(k)];
        sc.rows.push_back(r);
        sc.scale.push_back(inv * weights[static_cast<size_t>(r)]);
      }
      sc.batches.push_back({base + pos, end - pos});
      pos = end;
    }
  }
  return sc;
}

std::vector<double> resolve_weights(const TrainRecords& r, const char* who) {
  if (r.weights.empty()) return std::vector<double>(static_cast<size_t>(r.N), 1.0);
  if (r.weights.size() != static_cast<size_t>(r.N))
    throw std::invalid_argument(std::string(who) + ": sample weight count mismatch");
  return r.weights;
}

void check_records(const CacheVariant& v, const TrainRecords& r, const char* who) {
  if (r.N <= 0) throw std::invalid_argument(std::string(who) + ": no records");
  if (!r.taps || !r.y) throw std::invalid_argument(std::string(who) + ": null records");
  if (r.D != v.predictor.input_dim())
    throw std::invalid_argument(std::string(who) + ": tap dimension does not match the predictor input");
  if (r.C > 3072) throw std::invalid_argument(std::string(who) + ": more than 3072 classes");
  if (r.C != v.predictor.output_dim())
    throw std::invalid_argument(std::string(who) + ": class count does not match the predictor output");
}

struct Uploaded {
  double* X = nullptr;
  double* y = nullptr;
};

Uploaded upload_records(const TrainRecords& r, Arena& A, cudaStream_t s) {
  Uploaded u;
  u.X = A.upload(r.taps, static_cast<size_t>(r.N) * static_cast<size_t>(r.D), s);
  u.y = A.upload(r.y, static_cast<size_t>(r.N) * static_cast<size_t>(r.C), s);
  return u;
}

int read_flag(const int* d, cudaStream_t s) {
  int h = 0;
  tck(cudaMemcpyAsync(&h, d, sizeof(int), cudaMemcpyDeviceToHost, s), "flag");
  tck(cudaStreamSynchronize(s), "sync");
  return h;
}

// Small networks train in one thread block (launch_sgd_fused): the
// reference's MLP-tap caches have a few thousand parameters, where a
// launch per phase would dominate. Bigger ones (CNN-tap caches) run one
// kernel per phase across the GPU, the whole schedule captured as one graph.
FusedNet fused_view(const DevNet& net) {
  FusedNet fn;
  fn.nl = static_cast<int>(net.layers.size());
  for (int i = 0; i < fn.nl && i < kFusedMaxLayers; ++i) {
    fn.L[i] = net.layers[static_cast<size_t>(i)];
    fn.act[i + 1] = net.act[static_cast<size_t>(i) + 1];
  }
  return fn;
}

bool fused_fits(const DevNet& net, const FusedLoss& loss, int batch) {
  if (const char* e = std::getenv("LCB_TRAIN_UNFUSED"); e && e[0] == '1') return false;
  if (net.layers.size() > static_cast<size_t>(kFusedMaxLayers)) return false;
  if (loss.kind == 0 && loss.C > 64) return false;
  long long serial = 0;
  for (const TrainLayer& L : net.layers) {
    if (L.kind == 3) serial = std::max<long long>(serial, static_cast<long long>(L.out) * batch);
    serial = std::max<long long>(serial, L.in);
  }
  return serial <= 8192 && sgd_fused_smem_bytes(fused_view(net), batch, net.max_dim()) <= kFusedSmemMax;
}

// Minibatch SGD over `net` with inputs = rows of x.
void run_sgd(DevNet& net, const double* x, long long ld, const Schedule& sc, const SgdConfig& cfg, Arena& A,
             cudaStream_t s, const FusedLoss& loss, int* bad) {
  int* d_rows = A.upload(sc.rows.data(), sc.rows.size(), s);
  double* d_scale = A.upload(sc.scale.data(), sc.scale.size(), s);
  const size_t gsz = static_cast<size_t>(cfg.batch_size) * static_cast<size_t>(net.max_dim());
  double* g = A.alloc<double>(gsz);
  double* gx = A.alloc<double>(gsz);
  if (fused_fits(net, loss, cfg.batch_size)) {
    std::vector<int> off, nb;
    for (const auto& [o, n] : sc.batches) {
      off.push_back(o);
      nb.push_back(n);
    }
    const int* d_off = A.upload(off.data(), off.size(), s);
    const int* d_nb = A.upload(nb.data(), nb.size(), s);
    tck(launch_sgd_fused(fused_view(net), x, ld, d_rows, d_scale, d_off, d_nb, static_cast<int>(off.size()), loss,
                         cfg.learning_rate, cfg.momentum, cfg.batch_size, net.max_dim(), bad, s),
        "sgd_fused launch");
    tck(cudaStreamSynchronize(s), "train");
    return;
  }
  // One graph for the whole schedule: it is fully known up front.
  cudaGraph_t graph = nullptr;
  tck(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal), "capture");
  for (const auto& [off, nb] : sc.batches) {
    const int* rows = d_rows + off;
    net.forward(x, ld, rows, nb, s);
    if (loss.kind == 0)
      launch_distill_grad(net.act.back(), loss.p_tau, loss.hard, rows, nb, loss.C, loss.a, loss.b, g, bad, s);
    else
      launch_selector_grad(net.act.back(), loss.target, rows, nb, loss.a, loss.b, g, bad, s);
    net.backward_step(x, ld, rows, nb, g, gx, d_scale + off, cfg.learning_rate, cfg.momentum, s);
  }
  tck(cudaStreamEndCapture(s, &graph), "capture end");
  cudaGraphExec_t exec = nullptr;
  const cudaError_t ie = cudaGraphInstantiate(&exec, graph, 0);
  cudaGraphDestroy(graph);
  tck(ie, "graph instantiate");
  const cudaError_t le = cudaGraphLaunch(exec, s);
  const cudaError_t se = cudaStreamSynchronize(s);
  cudaGraphExecDestroy(exec);
  tck(le, "graph launch");
  tck(se, "train");
}

}  // namespace

void gpu_train_predictor(int device, CacheVariant& v, const TrainRecords& r, const SgdConfig& cfg, double tau,
                         double beta) {
  const char* who = "train_predictor";
  check_records(v, r, who);
  if (tau <= 0.0) throw std::invalid_argument("distill_loss: tau must be positive");
  if (beta < 0.0 || beta > 1.0) throw std::invalid_argument("distill_loss: beta must lie in [0, 1]");
  const std::vector<double> weights = resolve_weights(r, who);
  DeviceGuard dg(device);
  cudaStream_t s = train_stream(device);
  Arena A(s);
  const Uploaded u = upload_records(r, A, s);
  double* p_tau = A.alloc<double>(static_cast<size_t>(r.N) * r.C);
  int* hard = A.alloc<int>(r.N);
  int* bad = A.alloc<int>(1);
  tck(cudaMemsetAsync(bad, 0, sizeof(int), s), "memset");
  launch_soften(u.y, r.N, r.C, tau, p_tau, hard, bad, s);
  if (read_flag(bad, s) & 2) throw std::invalid_argument("soften: probabilities must be nonnegative and not all zero");
  DevNet net(v.predictor, cfg.batch_size, A, s);
  const Schedule sc = make_schedule(r.N, cfg, 0x90ed, weights);
  FusedLoss loss;
  loss.kind = 0;
  loss.C = r.C;
  loss.a = tau;
  loss.b = beta;
  loss.p_tau = p_tau;
  loss.hard = hard;
  run_sgd(net, u.X, r.D, sc, cfg, A, s, loss, bad);
  if (read_flag(bad, s)) throw std::runtime_error("train_predictor: loss diverged");
  net.download(v.predictor, s);
}

void gpu_train_selector(int device, CacheVariant& v, const TrainRecords& r, const SgdConfig& cfg, double w_fp,
                        double w_fn) {
  const char* who = "train_selector";
  check_records(v, r, who);
  if (w_fp <= 0.0 || w_fn <= 0.0) throw std::invalid_argument("weighted_selector_loss: weights must be positive");
  const std::vector<double> weights = resolve_weights(r, who);
  DeviceGuard dg(device);
  cudaStream_t s = train_stream(device);
  Arena A(s);
  const Uploaded u = upload_records(r, A, s);
  int* hard = A.alloc<int>(r.N);
  int* agree = A.alloc<int>(r.N);
  int* bad = A.alloc<int>(1);
  double* p_unused = A.alloc<double>(static_cast<size_t>(r.N) * r.C);
  tck(cudaMemsetAsync(bad, 0, sizeof(int), s), "memset");
  launch_soften(u.y, r.N, r.C, 1.0, p_unused, hard, bad, s);  // hard = argmax(y)
  // Frozen predictor: softmax inputs and agreement labels once up front
  // (cache.cpp:223-231).
  constexpr int kChunk = 256;
  double* inputs = A.alloc<double>(static_cast<size_t>(r.N) * r.C);
  {
    DevNet pred(v.predictor, kChunk, A, s);
    for (int n0 = 0; n0 < r.N; n0 += kChunk) {
      const int nb = std::min(kChunk, r.N - n0);
      pred.forward(u.X + static_cast<size_t>(n0) * r.D, r.D, nullptr, nb, s);
      tck(cudaMemcpyAsync(inputs + static_cast<size_t>(n0) * r.C, pred.act.back(), static_cast<size_t>(nb) * r.C * sizeof(double),
                          cudaMemcpyDeviceToDevice, s),
          "copy");
    }
  }
  launch_softmax_labels(inputs, r.N, r.C, hard, agree, s);
  DevNet net(v.selector, cfg.batch_size, A, s);
  const Schedule sc = make_schedule(r.N, cfg, 0x5e1ec7, weights);
  FusedLoss loss;
  loss.kind = 1;
  loss.C = r.C;
  loss.a = w_fp;
  loss.b = w_fn;
  loss.target = agree;
  run_sgd(net, inputs, r.C, sc, cfg, A, s, loss, bad);
  if (read_flag(bad, s)) throw std::runtime_error("train_selector: loss diverged");
  net.download(v.selector, s);
}

}  // namespace lcb
