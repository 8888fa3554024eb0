// Microbenchmark of the wide (> 32 classes) Pool(C) lookup kernel: per-launch
// time back to back (programmatic launches) and CTA 0's phase timestamps.
// Build: nvcc -std=c++17 -O2 -gencode arch=compute_100a,code=sm_100a
//        -I paper_2101_07344_b200/csrc/kernels tests/cuda/wide_bench.cu
//        paper_2101_07344_b200/csrc/kernels/serve_kernels.cu -o tests/cuda/wide_bench
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "serve_kernels.cuh"

using namespace lcb;

#define CK(x)                                                                         \
  do {                                                                                \
    cudaError_t e_ = (x);                                                             \
    if (e_ != cudaSuccess) {                                                          \
      std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      std::exit(1);                                                                   \
    }                                                                                 \
  } while (0)

template <typename T>
static T* dev_fill(size_t n, T v) {
  std::vector<T> h(n, v);
  T* d;
  CK(cudaMalloc(&d, n * sizeof(T)));
  CK(cudaMemcpy(d, h.data(), n * sizeof(T), cudaMemcpyHostToDevice));
  return d;
}

static void run(int B, int n, int C, int segs, int classes, int sms) {
  std::vector<float> g(static_cast<size_t>(B) * segs * C);
  for (size_t i = 0; i < g.size(); ++i) g[i] = static_cast<float>((i * 2654435761u) % 1000) * 1e-3f;
  float* gap;
  CK(cudaMalloc(&gap, g.size() * 4));
  CK(cudaMemcpy(gap, g.data(), g.size() * 4, cudaMemcpyHostToDevice));
  std::vector<int> ids(B);
  for (int i = 0; i < B; ++i) ids[i] = i;
  int* d_ids;
  CK(cudaMalloc(&d_ids, B * 4));
  CK(cudaMemcpy(d_ids, ids.data(), B * 4, cudaMemcpyHostToDevice));
  int* cnt = dev_fill<int>(1, n);
  CacheHeadParams p{};
  p.family = 1;
  p.classes = classes;
  p.feat = C;
  p.rows_total = B;
  p.W2 = dev_fill<float>(static_cast<size_t>(classes) * C, 1e-3f);
  p.b2 = dev_fill<float>(classes, 0.0f);
  p.Ws1 = dev_fill<float>(16 * static_cast<size_t>(classes), 1e-2f);
  p.bs1 = dev_fill<float>(16, 0.0f);
  p.ws2 = dev_fill<float>(16, 1.0f);
  p.bs2 = -0.5f;
  p.delta = 0.5;
  p.count = cnt;
  p.prob = dev_fill<float>(B, 0.0f);
  p.hit = dev_fill<int>(B, 0);
  p.label = dev_fill<int>(B, 0);
  p.gap = gap;
  p.gap_segs = segs;
  p.gap_inv = 1.0f / (segs * 32);
  p.gap_ids = d_ids;
  ExitParams& e = p.ex;
  e.arrive = dev_fill<int>(1, 0);
  e.layer = 1;
  e.shadow = 1;  // every row stays: the count is the same on every launch
  e.ids_in = d_ids;
  e.exit_layer = dev_fill<int>(B, 0);
  e.served = dev_fill<int>(B, 0);
  e.exit_ns = dev_fill<unsigned long long>(B, 0);
  e.ids_out = dev_fill<int>(B, 0);
  e.count_out = dev_fill<int>(1, 0);
  float* feats = dev_fill<float>(static_cast<size_t>(B) * C, 0.0f);
  float* logits = dev_fill<float>(static_cast<size_t>(B) * sms * 20, 0.0f);  // per-row, per-CTA softmax records
  int* gsync = dev_fill<int>(2, 0);
  for (int i = 0; i < 3; ++i) launch_wide_lookup(p, feats, logits, gsync, sms, 0);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 50;
  cudaEventRecord(e0);
  for (int i = 0; i < iters; ++i) launch_wide_lookup(p, feats, logits, gsync, sms, 0);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long* st = dev_fill<unsigned long long>(8, 0ull);
  set_wide_lookup_stamps(st);
  launch_wide_lookup(p, feats, logits, gsync, sms, 0);
  CK(cudaDeviceSynchronize());
  set_wide_lookup_stamps(nullptr);
  unsigned long long h[8];
  CK(cudaMemcpy(h, st, sizeof(h), cudaMemcpyDeviceToHost));
  std::printf("wide n=%3d/%3d C=%4d segs=%3d classes=%d: %7.2f us/launch | CTA0 ns: wait %lld p1 %lld bar1 %lld p2 %lld "
              "bar2 %lld p3 %lld exit %lld\n",
              n, B, C, segs, classes, 1e3 * ms / iters, (long long)(h[1] - h[0]), 0LL, 0LL,
              (long long)(h[3] - h[2]), (long long)(h[4] - h[3]), (long long)(h[5] - h[4]), (long long)(h[6] - h[5]));
  std::printf("      stamps rel entry: %lld %lld %lld %lld %lld %lld\n", (long long)(h[1] - h[0]), (long long)(h[2] - h[0]),
              (long long)(h[3] - h[0]), (long long)(h[4] - h[0]), (long long)(h[5] - h[0]), (long long)(h[6] - h[0]));
}

int main() {
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  const int sms = prop.multiProcessorCount;
  // R50 cache layers at the compacted step's survivor counts (gap_segs: 32-row segments per image)
  run(128, 128, 256, 98, 1000, sms);
  run(128, 70, 512, 25, 1000, sms);
  run(128, 27, 1024, 7, 1000, sms);
  run(128, 13, 1024, 7, 1000, sms);
  run(128, 2, 2048, 2, 1000, sms);
  run(128, 0, 2048, 2, 1000, sms);
  return 0;
}
