// Device engine implementation (see engine.hpp).
#include "engine.hpp"
#include "kernels/train_kernels.cuh"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>

namespace lcb {

namespace {

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaFailure(std::string(what) + ": " + cudaGetErrorString(e));
}
void require(bool ok, const std::string& msg) {
  if (!ok) throw std::invalid_argument(msg);
}
int round_up(long long v, int m) { return static_cast<int>((v + m - 1) / m * m); }

// A tile covers 128 output pixels: ipt images x (hb x wb) boxes. Boxes are a
// multiple of 8 rows so every box starts 1024-byte aligned in shared memory
// (the 128-byte swizzle atom).
void choose_box(int Ho, int Wo, int& hb, int& wb, int& ipt) {
  int w2 = 1;
  while (w2 < Wo) w2 <<= 1;
  int h2 = 1;
  while (h2 < Ho) h2 <<= 1;
  if (w2 > 128) w2 = 128;
  if (h2 * w2 <= 128) {
    hb = h2;
    wb = w2;
    while (hb * wb < 8) wb <<= 1;
    ipt = 128 / (hb * wb);
  } else {
    wb = w2;
    hb = 128 / wb;
    ipt = 1;
  }
}

void split_planes(const std::vector<float>& v, std::vector<__nv_bfloat16>& hi, std::vector<__nv_bfloat16>& lo) {
  hi.resize(v.size());
  lo.resize(v.size());
  for (size_t i = 0; i < v.size(); ++i) {
    const __nv_bfloat16 h = __float2bfloat16_rn(v[i]);
    hi[i] = h;
    lo[i] = __float2bfloat16_rn(v[i] - __bfloat162float(h));
  }
}

std::vector<float> to_f32(const std::vector<double>& v) { return std::vector<float>(v.begin(), v.end()); }

// One stream per device shared by every engine on it: launches of different
// engines never run concurrently, which the split-K reduction in tc_conv
// relies on (all CTAs of a launch co-resident), and graph capture on that
// stream is serialised by the device lock.
struct DevStream {
  std::recursive_mutex mu;
  cudaStream_t stream = nullptr;
};
DevStream& dev_stream(int device) {
  static std::mutex m;
  static std::map<int, std::unique_ptr<DevStream>> streams;
  std::lock_guard<std::mutex> g(m);
  auto& p = streams[device];
  if (!p) {
    p = std::make_unique<DevStream>();
    ck(cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking), "cudaStreamCreate");
  }
  return *p;
}

}  // namespace

struct DevCache {
  int layer = 0, family = 0, classes = 0;
  long long D = 0;
  // pool
  int width = 0, win = 1;
  // conv
  int kernel = 0, stride = 0, out_dim = 0, chunk_elems = 0, nchunks = 0;
  float* w1 = nullptr;
  float b1c = 0.0f;
  // fc
  int h = 0, hp = 0, ks = 1, Dk = 0;
  Planes W1;
  float* b1 = nullptr;
  Planes gather;
  // shared
  float* W2 = nullptr;
  float* b2 = nullptr;
  float* Ws1 = nullptr;
  float* bs1 = nullptr;
  float* ws2 = nullptr;
  float bs2 = 0.0f;
  double delta = 0.5;
  // scratch / outputs (row-indexed)
  float* feats = nullptr;
  int* hit = nullptr;
  int* label = nullptr;
  float* prob = nullptr;
  float* pr_out = nullptr;
  float* logits_out = nullptr;
  float* fc_scratch = nullptr;
  // fused GAP partials written by the tap conv's epilogue (Pool(C) caches)
  float* gap = nullptr;
  int gap_segs = 0;
  // the tap conv also finishes the lookup: features only (conv_feat, the head
  // runs separately on them) or the whole head + exit (conv_head)
  bool conv_feat = false, conv_head = false;
  // block-MLP FC(h) caches: the hidden layer rides the next block's GEMM
  // ([W_next; W1] concatenated along N, one launch over the tap's rows); the
  // next block's output for those rows lands in `spec` and the head's
  // compaction copies the survivors' rows on (Engine::mlp_fuse_hidden_)
  bool fused = false;
  Planes fw;             // [next.outp + hp][next.inp]
  float* fb = nullptr;   // [next.outp + hp]: next block's bias, zeros
  int fn1 = 0, fBN = 64;
  Planes spec;           // [max_batch][next.outp]
  // lookup-only step list
  std::vector<Step> lookup_steps;
};

// ------------------------------------------------------------------ memory
void* Engine::dalloc(size_t bytes) {
  void* p = nullptr;
  ck(cudaMalloc(&p, bytes < 256 ? 256 : bytes), "cudaMalloc");
  allocs_.push_back(p);
  return p;
}
// Every host->device write of the engine is ordered on stream_ (the stream all
// of its kernels run on). Pageable cudaMemcpyAsync stages the source before it
// returns, so the host vectors may die right after the call; the device-side
// copy still lands in stream order, after any memset queued before it and
// before any kernel queued after it.
void Engine::h2d(void* dst, const void* src, size_t bytes) {
  if (bytes) ck(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, stream_), "upload");
}
Planes Engine::alloc_planes(size_t elems, bool zero) {
  Planes p;
  p.elems = elems;
  p.hi = static_cast<__nv_bfloat16*>(dalloc(elems * 2));
  if (zero) ck(cudaMemsetAsync(p.hi, 0, elems * 2, stream_), "memset");
  if (prec_ == kPrecX3) {
    p.lo = static_cast<__nv_bfloat16*>(dalloc(elems * 2));
    if (zero) ck(cudaMemsetAsync(p.lo, 0, elems * 2, stream_), "memset");
  }
  return p;
}
Planes Engine::upload_planes(const std::vector<float>& v) {
  Planes p = alloc_planes(v.size(), false);  // fully overwritten below
  std::vector<__nv_bfloat16> hi, lo;
  split_planes(v, hi, lo);
  h2d(p.hi, hi.data(), v.size() * 2);
  if (p.lo) h2d(p.lo, lo.data(), v.size() * 2);
  return p;
}
float* Engine::upload_f32(const std::vector<float>& v) {
  float* p = static_cast<float*>(dalloc(v.size() * sizeof(float)));
  h2d(p, v.data(), v.size() * sizeof(float));
  return p;
}

// FC(h) cache first layer in the tap's storage order: [hp][Dk] fp32, the
// reference's NCHW-flat feature f at NHWC offset (f % HW) * C + f / HW.
static std::vector<float> fc_w1_layout(const std::vector<double>& w1, const DevCache& c, const TapInfo& ti, bool mlp) {
  std::vector<float> w(static_cast<size_t>(c.hp) * c.Dk, 0.0f);
  const int HW = ti.H * ti.W, Ct = ti.C;
  for (int j = 0; j < c.h; ++j)
    for (long long f = 0; f < c.D; ++f) {
      const long long off = mlp ? f : (f % HW) * Ct + f / HW;
      w[static_cast<size_t>(j) * c.Dk + static_cast<size_t>(off)] =
          static_cast<float>(w1[static_cast<size_t>(j) * c.D + static_cast<size_t>(f)]);
    }
  return w;
}

// ------------------------------------------------------------------ build
Engine::Engine(int device, const BaseModel& model, std::vector<CacheVariant> variants, Precision prec, int max_batch)
    : device_(device), prec_(prec), max_batch_(max_batch), model_(model), variants_(std::move(variants)) {
  require(max_batch > 0, "engine: max_batch must be positive");
  require(model_.num_blocks > 0, "engine: empty base model");
  int ndev = 0;
  ck(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
  require(device >= 0 && device < ndev, "engine: device index out of range");
  ck(cudaSetDevice(device), "cudaSetDevice");
  cudaDeviceProp prop;
  ck(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
  require(prop.major == 10, "engine: requires an sm_100 (B200) device");
  num_sms_ = prop.multiProcessorCount;
  DevStream& ds = dev_stream(device);
  std::lock_guard<std::recursive_mutex> dev_lock(ds.mu);  // build work queues on the shared stream
  stream_ = ds.stream;
  ck(cudaEventCreate(&ev0_), "event");
  ck(cudaEventCreate(&ev1_), "event");

  // make_plan semantics (composer.cpp:65-89): probe order = ascending layer,
  // at most one variant per layer.
  std::stable_sort(variants_.begin(), variants_.end(),
                   [](const CacheVariant& a, const CacheVariant& b) { return a.layer < b.layer; });
  for (size_t k = 1; k < variants_.size(); ++k)
    require(variants_[k - 1].layer != variants_[k].layer,
            "plan: more than one variant at layer " + std::to_string(variants_[k].layer));
  cache_of_layer_.assign(static_cast<size_t>(model_.num_blocks) + 1, -1);
  for (size_t k = 0; k < variants_.size(); ++k) {
    const CacheVariant& v = variants_[k];
    require(v.layer >= 1 && v.layer <= model_.num_blocks,
            "simulate: variant layer " + std::to_string(v.layer) + " outside the model");
    require(v.predictor.input_dim() == model_.tap_dim(v.layer),
            "forward: input dim " + std::to_string(model_.tap_dim(v.layer)) + " != expected " +
                std::to_string(v.predictor.input_dim()));
    require(v.predictor.output_dim() == model_.num_classes && v.selector.input_dim() == model_.num_classes,
            "engine: variant class count does not match the base model");
    cache_of_layer_[static_cast<size_t>(v.layer)] = static_cast<int>(k);
  }
  const char* nf = std::getenv("LCB_NO_GAP_FUSION");
  gap_fusion_ = !(nf && nf[0] == '1');
  const char* nl = std::getenv("LCB_UNFUSED_LOOKUP");
  fused_lookup_ = !(nl && nl[0] == '1');
  if (const char* nc = std::getenv("LCB_NO_CONV_HEAD")) conv_head_ = !(nc[0] == '1');
  if (const char* cm = std::getenv("LCB_CONV_HEAD_TILE")) conv_head_post_ = !(cm[0] == '1');
  if (const char* td = std::getenv("LCB_TC_DBG")) tc_dbg_ = std::atoi(td);
  if (const char* nw = std::getenv("LCB_NO_WIDE_LOOKUP")) wide_lookup_ = !(nw[0] == '1');
  const char* ns = std::getenv("LCB_NO_STACKED");
  stacked_ = !(ns && ns[0] == '1');
  if (const char* km = std::getenv("LCB_KS_MIN_STEPS")) ks_min_steps_ = std::atoi(km);
  if (const char* km = std::getenv("LCB_MLP_KS_MIN_STEPS")) mlp_ks_min_steps_ = std::atoi(km);
  if (const char* u = std::getenv("LCB_UNORDERED_IDS")) unordered_ids_ = std::atoi(u) != 0;
  if (const char* u = std::getenv("LCB_MLP_FUSE_HIDDEN")) mlp_fuse_hidden_ = std::atoi(u) != 0;
  if (const char* u = std::getenv("LCB_SCAN_COMPACTION")) scan_compaction_ = std::atoi(u) != 0;
  if (const char* wp = std::getenv("LCB_NO_WPREFETCH")) wprefetch_ = !(wp[0] == '1');
  const char* nh = std::getenv("LCB_HALO");  // opt-in: not yet faster than the per-tap loads
  halo_ = nh && nh[0] == '1';
  const char* nr = std::getenv("LCB_NO_MMA_RESIDUAL");
  mma_residual_ = !(nr && nr[0] == '1');
  if (const char* np = std::getenv("LCB_NO_PROJ_FUSION")) proj_fusion_ = !(np[0] == '1');
  if (const char* ra = std::getenv("LCB_ORDERED_COMPACTION")) mlp_row_append_ = !(ra[0] == '1');
  if (const char* pl = std::getenv("LCB_PREDICTOR_LAUNCH")) direct_rows_ = !(pl[0] == '1');
  if (const char* sp = std::getenv("LCB_NO_STEM_POOL")) stem_pool_ = !(sp[0] == '1');
  const char* nt = std::getenv("LCB_DIRECT_STORE");
  staged_store_ = !(nt && nt[0] == '1');
  build_weights();
  ck(cudaStreamSynchronize(stream_), "build");
}

void Engine::drop_graph(int mode) {
  if (graph_[mode]) cudaGraphExecDestroy(graph_[mode]);
  if (graph_tmpl_[mode]) cudaGraphDestroy(graph_tmpl_[mode]);
  graph_[mode] = nullptr;
  graph_tmpl_[mode] = nullptr;
  graph_init_node_[mode] = nullptr;
}

Engine::~Engine() {
  if (stream_) cudaStreamSynchronize(stream_);
  for (int m = 0; m < kModes; ++m) drop_graph(m);
  for (void* p : allocs_) cudaFree(p);
  if (h_batch_) cudaFreeHost(h_batch_);
  if (copy_stream_) cudaStreamSynchronize(copy_stream_);
  for (Slot& sl : slots_) {
    if (sl.h_exit) cudaFreeHost(sl.h_exit);
    if (sl.h_served) cudaFreeHost(sl.h_served);
    if (sl.h_base) cudaFreeHost(sl.h_base);
    if (sl.h_probs) cudaFreeHost(sl.h_probs);
    if (sl.h_logits) cudaFreeHost(sl.h_logits);
    if (sl.h_ns) cudaFreeHost(sl.h_ns);
    for (cudaEvent_t e : {sl.in_done, sl.in_free, sl.out_done})
      if (e) cudaEventDestroy(e);
  }
  if (copy_stream_) cudaStreamDestroy(copy_stream_);
  if (ev0_) cudaEventDestroy(ev0_);
  if (ev1_) cudaEventDestroy(ev1_);
}

void Engine::build_weights() {
  const int L = model_.num_blocks;
  const int B = max_batch_;
  // batch state
  d_x_ = static_cast<float*>(dalloc(static_cast<size_t>(B) * model_.input_dim() * sizeof(float)));
  d_batch_ = static_cast<int*>(dalloc(sizeof(int)));
  ck(cudaMallocHost(&h_batch_, sizeof(int)), "cudaMallocHost");
  d_ids_ = static_cast<int*>(dalloc(static_cast<size_t>(L + 1) * B * sizeof(int)));
  d_src_ = static_cast<int*>(dalloc(static_cast<size_t>(L + 1) * B * sizeof(int)));
  d_counts_ = static_cast<int*>(dalloc(static_cast<size_t>(L + 4) * sizeof(int)));  // [L + 2] = serve epoch
  ck(cudaMemsetAsync(d_counts_, 0, static_cast<size_t>(L + 4) * sizeof(int), stream_), "memset");
  d_scan_ = static_cast<unsigned long long*>(dalloc(static_cast<size_t>(L + 1) * kScanMaxCtas * 8));
  ck(cudaMemsetAsync(d_scan_, 0, static_cast<size_t>(L + 1) * kScanMaxCtas * 8, stream_), "memset");
  d_exit_ = static_cast<int*>(dalloc(static_cast<size_t>(B) * sizeof(int)));
  d_served_ = static_cast<int*>(dalloc(static_cast<size_t>(B) * sizeof(int)));
  d_base_ = static_cast<int*>(dalloc(static_cast<size_t>(B) * sizeof(int)));
  d_exit_ns_ = static_cast<unsigned long long*>(dalloc(static_cast<size_t>(B) * 8));
  d_t0_ = static_cast<unsigned long long*>(dalloc(8));
  d_probs_ = static_cast<float*>(dalloc(static_cast<size_t>(L) * B * sizeof(float)));
  d_logits_ = static_cast<float*>(dalloc(static_cast<size_t>(B) * model_.num_classes * sizeof(float)));
  d_block_ns_ = static_cast<unsigned long long*>(dalloc(static_cast<size_t>(L + 1) * 2 * 8));
  d_labels_ = static_cast<int*>(dalloc(static_cast<size_t>(L) * B * sizeof(int)));
  d_grid_ = static_cast<double*>(dalloc(64 * sizeof(double)));
  d_conf_ = static_cast<unsigned long long*>(dalloc(static_cast<size_t>(L) * 64 * 4 * sizeof(unsigned long long)));
  d_lk_count_ = static_cast<int*>(dalloc(sizeof(int)));
  lk_arrive_ = static_cast<int*>(dalloc(sizeof(int)));
  row_tiles_ = static_cast<int*>(dalloc(static_cast<size_t>(B) * sizeof(int)));
  ck(cudaMemsetAsync(row_tiles_, 0, static_cast<size_t>(B) * sizeof(int), stream_), "memset");
  conv_sync_ = static_cast<unsigned*>(dalloc(sizeof(unsigned)));
  ck(cudaMemsetAsync(conv_sync_, 0, sizeof(unsigned), stream_), "memset");
  heads_done_ = static_cast<int*>(dalloc(sizeof(int)));
  ck(cudaMemsetAsync(heads_done_, 0, sizeof(int), stream_), "memset");
  ck(cudaMemsetAsync(lk_arrive_, 0, sizeof(int), stream_), "memset");
  wide_sync_ = static_cast<int*>(dalloc(2 * sizeof(int)));
  ck(cudaMemsetAsync(wide_sync_, 0, 2 * sizeof(int), stream_), "memset");
  ws_ = static_cast<float*>(dalloc(tc_conv_ws_floats(256, num_sms_) * sizeof(float)));
  // three counter sets (split-K launches alternate; see assign_counter_sets)
  ws_counters_ = static_cast<int*>(dalloc(3 * 2 * static_cast<size_t>(num_sms_) * sizeof(int)));
  ck(cudaMemsetAsync(ws_counters_, 0, 3 * 2 * static_cast<size_t>(num_sms_) * sizeof(int), stream_), "memset");

  // ---------------- base model
  long long max_tap_storage = 0;
  if (model_.family == "mlp") {
    const Network& net = model_.net;
    for (int b = 0; b < L; ++b) {
      const LayerSpec& s = net.layers[static_cast<size_t>(2 * b)];
      DevFC f;
      f.in = s.in_dim;
      f.out = s.out_dim;
      f.inp = round_up(s.in_dim, 64);
      f.outp = round_up(s.out_dim, 64);
      std::vector<float> w(static_cast<size_t>(f.outp) * f.inp, 0.0f), bias(static_cast<size_t>(f.outp), 0.0f);
      const LayerWeights& lw = net.weights[static_cast<size_t>(2 * b)];
      for (int o = 0; o < f.out; ++o) {
        for (int i = 0; i < f.in; ++i)
          w[static_cast<size_t>(o) * f.inp + i] = static_cast<float>(lw.w[static_cast<size_t>(o) * f.in + i]);
        bias[static_cast<size_t>(o)] = static_cast<float>(lw.b[static_cast<size_t>(o)]);
      }
      f.w = upload_planes(w);
      f.b = upload_f32(bias);
      mlp_fc_.push_back(f);
      mlp_act_.push_back(alloc_planes(static_cast<size_t>(B) * f.outp));
      mlp_cin_.push_back(alloc_planes(static_cast<size_t>(B) * f.outp));
      max_tap_storage = std::max<long long>(max_tap_storage, f.outp);
    }
    mlp_in_ = alloc_planes(static_cast<size_t>(B) * mlp_fc_[0].inp);
    const LayerWeights& hw = net.weights[static_cast<size_t>(2 * L)];
    head_w_ = upload_f32(to_f32(hw.w));
    head_b_ = upload_f32(to_f32(hw.b));
  } else {
    {
      std::vector<__nv_bfloat16> eye(256 * 256, __float2bfloat16_rn(0.0f));
      for (int i = 0; i < 256; ++i) eye[static_cast<size_t>(i) * 256 + i] = __float2bfloat16_rn(1.0f);
      identity_ = static_cast<__nv_bfloat16*>(dalloc(eye.size() * 2));
      h2d(identity_, eye.data(), eye.size() * 2);
    }
    cnn_w_.resize(model_.ops.size());
    // Projection shortcuts that ride their consumer's residual K-steps: a 1x1,
    // unpadded, ReLU-free conv whose output slot is used exactly once, as the
    // residual of a conv at the same output resolution (the ResNet downsample
    // branch). Not with halo slabs (their producer has no projection path).
    const size_t nops = model_.ops.size();
    proj_into_.assign(nops, -1);
    fused_proj_.assign(nops, -1);
    if (proj_fusion_ && mma_residual_ && !halo_) {
      std::vector<int> uses(static_cast<size_t>(model_.nslots), 0), producer(static_cast<size_t>(model_.nslots), -1);
      for (size_t i = 0; i < nops; ++i) {
        const CnnOp& o = model_.ops[i];
        if (o.in >= 0) ++uses[static_cast<size_t>(o.in)];
        if (o.res >= 0) ++uses[static_cast<size_t>(o.res)];
        if (o.kind != CnnOpKind::Head) producer[static_cast<size_t>(o.out)] = static_cast<int>(i);
      }
      for (size_t i = 0; i < nops; ++i) {
        const CnnOp& o = model_.ops[i];
        if (o.kind != CnnOpKind::Conv || o.res < 0 || uses[static_cast<size_t>(o.res)] != 1) continue;
        const int j = producer[static_cast<size_t>(o.res)];
        if (j < 0 || j >= static_cast<int>(i)) continue;
        const CnnOp& pj = model_.ops[static_cast<size_t>(j)];
        if (pj.kind != CnnOpKind::Conv || pj.k != 1 || pj.pad != 0 || pj.relu || pj.res >= 0 || pj.tap >= 0 ||
            pj.in < 0 || pj.C % 64 != 0 || pj.Cout != o.Cout || pj.Ho() != o.Ho() || pj.Wo() != o.Wo() ||
            (pj.stride != 1 && pj.stride != 2))
          continue;
        proj_into_[static_cast<size_t>(j)] = static_cast<int>(i);
        fused_proj_[i] = j;
      }
    }
    // stem followed by the 3x3/s2/p1 max-pool that is its output's only use
    stem_pool_op_ = -1;
    if (stem_pool_) {
      for (size_t i = 0; i + 1 < nops; ++i) {
        const CnnOp& st = model_.ops[i];
        const CnnOp& mp = model_.ops[i + 1];
        if (st.kind != CnnOpKind::Stem || mp.kind != CnnOpKind::MaxPool || mp.in != st.out || mp.k != 3 ||
            mp.stride != 2 || mp.pad != 1 || !st.relu)
          continue;
        int uses = 0;
        for (const CnnOp& o : model_.ops) uses += (o.in == st.out) + (o.res == st.out);
        const StemGeom sg = stem_geom(st.H, st.W, st.k, st.stride, st.pad);
        if (uses == 1 && sg.Wx <= 128 && mp.Ho() == (sg.Ho - 1) / 2 + 1 && mp.Wo() == (sg.Wo - 1) / 2 + 1)
          stem_pool_op_ = static_cast<int>(i + 1);
      }
    }
    std::vector<long long> slot_elems(static_cast<size_t>(model_.nslots), 0);
    long long im2col_elems = 0;
    for (size_t i = 0; i < model_.ops.size(); ++i) {
      const CnnOp& o = model_.ops[i];
      if (o.kind == CnnOpKind::Stem) {
        require(o.Cout == 64 && (o.stride == 1 || o.stride == 2) && o.C * o.stride * o.stride <= 16,
                "engine: stem must be C_in*stride^2 <= 16 -> 64 channels, stride 1 or 2");
        DevConv dc;
        const StemGeom g = stem_geom(o.H, o.W, o.k, o.stride, o.pad);
        std::vector<float> w(static_cast<size_t>(g.kk) * g.kk * 2 * 64 * 8);
        std::vector<double> ws(o.w);
        const size_t per_out = ws.size() / static_cast<size_t>(o.Cout);
        for (size_t i = 0; i < ws.size(); ++i) ws[i] *= o.scale[i / per_out];  // fold BN scale
        stem_weights(ws.data(), o.Cout, o.C, o.k, o.stride, g, w.data());
        if (prec_ == kPrecX3) {
          // stacked per tap and channel group: 64 hi rows then 64 lo rows (tc_stem's N = 128 MMA)
          std::vector<__nv_bfloat16> hi, lo, st(2 * w.size());
          split_planes(w, hi, lo);
          const size_t groups = w.size() / (64 * 8);  // taps x 2
          for (size_t gi = 0; gi < groups; ++gi)
            for (size_t r = 0; r < 64 * 8; ++r) {
              st[gi * 1024 + r] = hi[gi * 512 + r];
              st[gi * 1024 + 512 + r] = lo[gi * 512 + r];
            }
          dc.w.hi = static_cast<__nv_bfloat16*>(dalloc(st.size() * 2));
          h2d(dc.w.hi, st.data(), st.size() * 2);
          dc.w.lo = nullptr;
        } else {
          dc.w = upload_planes(w);
        }
        dc.scale = nullptr;
        dc.shift = upload_f32(to_f32(o.shift));
        cnn_w_[i] = dc;
        // fused with the max-pool: the stem writes the horizontally pooled rows
        const long long ow = stem_pool_op_ == static_cast<int>(i + 1) ? (o.Wo() - 1) / 2 + 1 : o.Wo();
        slot_elems[static_cast<size_t>(o.out)] = static_cast<long long>(B) * o.Ho() * ow * o.Cout;
        im2col_elems = std::max(im2col_elems, static_cast<long long>(B) * 2 * g.Hx * g.Wx * 8);
      } else if (o.kind == CnnOpKind::Conv) {
        DevConv dc;
        const int K = o.k * o.k * o.C;
        dc.Kp = K;
        require(o.C % 64 == 0, "engine: conv input channels must be a multiple of 64");
        // folded batch-norm scale goes into the weights (W * scale), so the
        // epilogue only adds the shift (and a residual add can ride the MMA)
        std::vector<float> w(static_cast<size_t>(o.Cout) * dc.Kp, 0.0f);
        for (int co = 0; co < o.Cout; ++co)
          for (int c = 0; c < o.C; ++c)
            for (int r = 0; r < o.k; ++r)
              for (int s = 0; s < o.k; ++s)
                w[static_cast<size_t>(co) * dc.Kp + (r * o.k + s) * o.C + c] =
                    static_cast<float>(o.w[((static_cast<size_t>(co) * o.C + c) * o.k + r) * o.k + s] *
                                       o.scale[static_cast<size_t>(co)]);
        dc.w = upload_planes(w);
        dc.scale = nullptr;
        std::vector<double> shift(o.shift);
        if (fused_proj_[i] >= 0) {  // conv + projection accumulate together: one shift
          const CnnOp& pj = model_.ops[static_cast<size_t>(fused_proj_[i])];
          for (size_t c = 0; c < shift.size(); ++c) shift[c] += pj.shift[c];
        }
        dc.shift = upload_f32(to_f32(shift));
        cnn_w_[i] = dc;
        if (proj_into_[i] < 0)
          slot_elems[static_cast<size_t>(o.out)] = static_cast<long long>(B) * o.Ho() * o.Wo() * o.Cout;
      } else if (o.kind == CnnOpKind::MaxPool) {
        slot_elems[static_cast<size_t>(o.out)] = static_cast<long long>(B) * o.Ho() * o.Wo() * o.C;
      } else if (o.kind == CnnOpKind::Head) {
        head_w_ = upload_f32(to_f32(o.w));
        head_b_ = upload_f32(to_f32(o.shift));
      }
    }
    // Liveness-based slot -> buffer assignment.
    std::vector<int> last_use(static_cast<size_t>(model_.nslots), -1);
    for (size_t i = 0; i < model_.ops.size(); ++i) {
      const CnnOp& o = model_.ops[i];
      if (o.in >= 0) last_use[static_cast<size_t>(o.in)] = static_cast<int>(i);
      if (o.res >= 0) last_use[static_cast<size_t>(o.res)] = static_cast<int>(i);
      // a fused projection reads its input when its consumer runs
      if (fused_proj_[i] >= 0) last_use[static_cast<size_t>(model_.ops[static_cast<size_t>(fused_proj_[i])].in)] = static_cast<int>(i);
    }
    slot_buf_.assign(static_cast<size_t>(model_.nslots), Planes{});
    std::multimap<long long, Planes> free_pool;
    for (size_t i = 0; i < model_.ops.size(); ++i) {
      const CnnOp& o = model_.ops[i];
      if (o.kind != CnnOpKind::Head && proj_into_[i] < 0) {
        const long long need = slot_elems[static_cast<size_t>(o.out)];
        auto it = free_pool.find(need);
        if (it != free_pool.end()) {
          slot_buf_[static_cast<size_t>(o.out)] = it->second;
          free_pool.erase(it);
        } else {
          slot_buf_[static_cast<size_t>(o.out)] = alloc_planes(static_cast<size_t>(need));
        }
      }
      for (int s = 0; s < model_.nslots; ++s)
        if (last_use[static_cast<size_t>(s)] == static_cast<int>(i) && slot_buf_[static_cast<size_t>(s)].hi)
          free_pool.emplace(slot_elems[static_cast<size_t>(s)], slot_buf_[static_cast<size_t>(s)]);
    }
    if (im2col_elems) im2col_buf_ = alloc_planes(static_cast<size_t>(im2col_elems));
    for (const TapInfo& t : model_.taps) max_tap_storage = std::max(max_tap_storage, t.dim());
  }

  // ---------------- caches
  for (const CacheVariant& v : variants_) {
    auto c = std::make_unique<DevCache>();
    c->layer = v.layer;
    c->classes = model_.num_classes;
    c->D = model_.tap_dim(v.layer);
    c->delta = v.delta;
    const TapInfo ti = model_.taps[static_cast<size_t>(v.layer - 1)];
    const bool mlp = model_.family == "mlp";
    const long long row_stride = mlp ? mlp_fc_[static_cast<size_t>(v.layer - 1)].outp : c->D;
    const auto& P = v.predictor.layers;
    const auto& PW = v.predictor.weights;
    const int C = c->classes;
    if (P.size() == 2 && P[0].kind == LayerKind::Pool && P[1].kind == LayerKind::FC) {
      c->family = 1;
      c->win = P[0].pool_window;
      c->width = P[0].out_dim;
      c->W2 = upload_f32(to_f32(PW[1].w));
      c->b2 = upload_f32(to_f32(PW[1].b));
      c->feats = static_cast<float*>(dalloc(static_cast<size_t>(B) * c->width * sizeof(float)));
    } else if (P.size() == 3 && P[0].kind == LayerKind::Conv1d && P[1].kind == LayerKind::ReLU &&
               P[2].kind == LayerKind::FC) {
      c->family = 2;
      c->kernel = P[0].kernel;
      c->stride = P[0].stride;
      c->out_dim = P[0].out_dim;
      c->w1 = upload_f32(to_f32(PW[0].w));
      c->b1c = static_cast<float>(PW[0].b[0]);
      c->W2 = upload_f32(to_f32(PW[2].w));
      c->b2 = upload_f32(to_f32(PW[2].b));
      // chunk = whole channels, <= ~24K floats of shared memory
      if (ti.H * ti.W == 1) {
        c->chunk_elems = static_cast<int>(std::min<long long>(c->D, 8192));
      } else {
        const int HW = ti.H * ti.W;
        int cb = std::max(1, 24576 / HW);
        cb = std::min(cb, ti.C);
        c->chunk_elems = cb * HW;
      }
      c->nchunks = static_cast<int>((c->D + c->chunk_elems - 1) / c->chunk_elems);
      c->feats = static_cast<float*>(dalloc(static_cast<size_t>(B) * c->nchunks * C * sizeof(float)));
    } else if (P.size() == 3 && P[0].kind == LayerKind::FC && P[1].kind == LayerKind::ReLU &&
               P[2].kind == LayerKind::FC) {
      c->family = 0;
      c->h = P[0].out_dim;
      c->hp = round_up(c->h, 64);
      c->Dk = static_cast<int>(round_up(row_stride, 64));
      c->W1 = upload_planes(fc_w1_layout(PW[0].w, *c, ti, mlp));
      c->b1 = upload_f32(to_f32(PW[0].b));
      c->W2 = upload_f32(to_f32(PW[2].w));
      c->b2 = upload_f32(to_f32(PW[2].b));
      const int tiles_mn = ((B + 127) / 128) * (c->hp / tc_conv_pick_bn(c->hp, prec_ == kPrecX3 ? 3 : 1));
      const int nk = c->Dk / 64;  // K-steps (one 64-channel slice each; bf16x3 segments share a step)
      c->ks = std::max(1, std::min(nk, num_sms_ / std::max(1, tiles_mn)));
      c->feats = static_cast<float*>(dalloc(static_cast<size_t>(c->ks) * B * c->hp * sizeof(float)));
      if (!mlp) c->gather = alloc_planes(static_cast<size_t>(B) * c->Dk);
    } else {
      throw std::invalid_argument("engine: unsupported predictor architecture at layer " + std::to_string(v.layer));
    }
    const auto& S = v.selector.layers;
    require(S.size() == 3 && S[0].kind == LayerKind::FC && S[0].out_dim == 16 && S[1].kind == LayerKind::ReLU &&
                S[2].kind == LayerKind::FC && S[2].out_dim == 1,
            "engine: selector must be FC(C,16)+ReLU+FC(16,1) (cache.cpp:135-137)");
    c->Ws1 = upload_f32(to_f32(v.selector.weights[0].w));
    c->bs1 = upload_f32(to_f32(v.selector.weights[0].b));
    c->ws2 = upload_f32(to_f32(v.selector.weights[2].w));
    c->bs2 = static_cast<float>(v.selector.weights[2].b[0]);
    c->hit = static_cast<int*>(dalloc(static_cast<size_t>(B) * sizeof(int)));
    c->label = static_cast<int*>(dalloc(static_cast<size_t>(B) * sizeof(int)));
    c->prob = static_cast<float*>(dalloc(static_cast<size_t>(B) * sizeof(float)));
    c->pr_out = static_cast<float*>(dalloc(static_cast<size_t>(B) * C * sizeof(float)));
    c->logits_out = static_cast<float*>(dalloc(static_cast<size_t>(B) * C * sizeof(float)));
    if (C > 32 && c->family != 2) {
      const int feat = c->family == 1 ? c->width : c->h;
      // (also the wide lookup's per-row, per-CTA softmax records: B x grid x 20 floats)
      const size_t sc = std::max(static_cast<size_t>(rows_fc_splits(feat)) * B * C, static_cast<size_t>(B) * num_sms_ * 20);
      c->fc_scratch = static_cast<float*>(dalloc(sc * sizeof(float)));
    }
    caches_.push_back(std::move(c));
  }
  lk_tap_ = alloc_planes(static_cast<size_t>(B) * round_up(max_tap_storage, 64));
  if (model_.family == "mlp" && mlp_fuse_hidden_) {
    for (auto& cp : caches_) {
      DevCache& c = *cp;
      if (c.family != 0 || c.layer >= model_.num_blocks) continue;
      const DevFC& nf = mlp_fc_[static_cast<size_t>(c.layer)];  // the next block's FC
      if (nf.inp != c.Dk) continue;
      const int n1 = nf.outp, nt = n1 + c.hp;
      int bn = tc_conv_pick_bn(nt, prec_ == kPrecX3 ? 3 : 1);
      if (n1 % bn != 0 || c.hp % bn != 0) bn = 64;
      c.fw = alloc_planes(static_cast<size_t>(nt) * nf.inp, false);
      const size_t e1 = static_cast<size_t>(n1) * nf.inp, e2 = static_cast<size_t>(c.hp) * c.Dk;
      ck(cudaMemcpyAsync(c.fw.hi, nf.w.hi, e1 * 2, cudaMemcpyDeviceToDevice, stream_), "fused W");
      ck(cudaMemcpyAsync(c.fw.hi + e1, c.W1.hi, e2 * 2, cudaMemcpyDeviceToDevice, stream_), "fused W");
      if (c.fw.lo) {
        ck(cudaMemcpyAsync(c.fw.lo, nf.w.lo, e1 * 2, cudaMemcpyDeviceToDevice, stream_), "fused W");
        ck(cudaMemcpyAsync(c.fw.lo + e1, c.W1.lo, e2 * 2, cudaMemcpyDeviceToDevice, stream_), "fused W");
      }
      c.fb = static_cast<float*>(dalloc(static_cast<size_t>(nt) * sizeof(float)));
      ck(cudaMemsetAsync(c.fb, 0, static_cast<size_t>(nt) * sizeof(float), stream_), "fused b");
      ck(cudaMemcpyAsync(c.fb, nf.b, static_cast<size_t>(n1) * sizeof(float), cudaMemcpyDeviceToDevice, stream_),
         "fused b");
      c.spec = alloc_planes(static_cast<size_t>(B) * n1, false);
      c.fn1 = n1;
      c.fBN = bn;
      c.ks = 1;  // the hidden layer's partials: one split (K = the tap width)
      c.fused = true;
    }
  }
}

// ------------------------------------------------------------------ lookups
void Engine::add_lookup_steps(std::vector<Step>& steps, DevCache& c, const TapView& tap, int max_rows,
                              bool stage_gather, bool fused_gap, const ExitParams* ex, bool hidden_done) {
  DevCache* cp = &c;
  const long long L2 = model_.num_blocks + 2;
  const int cidx = (tap.count >= d_counts_ && tap.count < d_counts_ + L2) ? static_cast<int>(tap.count - d_counts_) : -1;
  const double eb = prec_ == kPrecX3 ? 4.0 : 2.0;  // bytes per activation element (hi + lo planes)
  const double tap_bytes = static_cast<double>(c.D) * eb;
  // Pool(C) with <= 32 classes: the head itself sums the conv's fused GAP partials.
  const bool head_gap = c.family == 1 && fused_gap && c.gap && fused_lookup_ &&
                        fused_lookup_supported(c.classes, c.width, max_rows);
  // block-MLP taps (one contiguous row per request): the head reads the row and
  // runs the Pool(w) / Conv(k,s) predictor layer itself (LCB_PREDICTOR_LAUNCH=1: separate launch)
  // (Pool(w) heads with > 32 classes take the batched logits GEMM over pooled features instead)
  const bool direct = direct_rows_ && tap.HW == 1 && !tap.data_idx && !fused_gap &&
                      ((c.family == 1 && c.classes <= 32) || c.family == 2) && c.D <= 8192;
  double head_bytes = 0.0;  // per surviving row, beyond the (L2-resident) head weights
  if (head_gap) {
    head_bytes = 4.0 * c.gap_segs * c.width;
  } else if (c.family == 1 && fused_gap && c.gap && c.conv_feat) {
    // the tap conv already wrote the GAP features into c.feats
  } else if (c.family == 1 && fused_gap && c.gap && wide_lookup_ && ex && c.fc_scratch &&
             wide_lookup_supported(c.classes, c.width, num_sms_)) {
    // many classes: GAP features, logits, head and exit in one persistent launch
    const ExitParams exv = *ex;
    const float gap_inv = static_cast<float>(1.0 / tap.HW);
    int* gsync = wide_sync_;
    const int sms = num_sms_;
    steps.push_back({[cp, tap, max_rows, exv, gap_inv, gsync, sms](cudaStream_t s) {
                       CacheHeadParams p{};
                       p.family = 1;
                       p.classes = cp->classes;
                       p.feat = cp->width;
                       p.rows_total = max_rows;
                       p.W2 = cp->W2;
                       p.b2 = cp->b2;
                       p.Ws1 = cp->Ws1;
                       p.bs1 = cp->bs1;
                       p.ws2 = cp->ws2;
                       p.bs2 = cp->bs2;
                       p.delta = cp->delta;
                       p.count = tap.count;
                       p.prob = cp->prob;
                       p.hit = cp->hit;
                       p.label = cp->label;
                       p.gap = cp->gap;
                       p.gap_segs = cp->gap_segs;
                       p.gap_inv = gap_inv;
                       p.gap_ids = tap.data_idx;
                       p.ex = exv;
                       launch_wide_lookup(p, cp->feats, cp->fc_scratch, gsync, sms, s);
                     },
                     2, 1, cidx, 2.0 * c.width * c.classes,
                     4.0 * c.gap_segs * c.width + 4.0 * c.width * c.classes / max_rows});
    return;
  } else if (c.family == 1 && fused_gap && c.gap) {
    steps.push_back({[cp, tap, max_rows](cudaStream_t s) {
                       launch_gap_bins(cp->gap, cp->gap_segs, tap.C, tap.HW, tap.data_idx, tap.count, max_rows,
                                       cp->feats, s);
                     },
                     2, 1, cidx, 0.0, 4.0 * c.gap_segs * c.width + 4.0 * c.width});
  } else if (c.family == 1 && direct) {
    // the head pools its own row (direct row mode)
  } else if (c.family == 1) {
    steps.push_back({[cp, tap, max_rows](cudaStream_t s) {
                       launch_pool_bins(tap, max_rows, cp->win, cp->width, cp->feats, s);
                     },
                     2, 1, cidx, 0.0, tap_bytes + 4.0 * c.width});
  } else if (c.family == 2 && direct) {
    // the head runs the Conv(k,s) layer on its own row (direct row mode)
  } else if (c.family == 2) {
    steps.push_back({[cp, tap, max_rows](cudaStream_t s) {
                       launch_conv1d_partials(tap, max_rows, cp->D, cp->kernel, cp->stride, cp->out_dim, cp->w1,
                                              cp->b1c, cp->W2, cp->classes, cp->chunk_elems, cp->nchunks, cp->feats,
                                              s);
                     },
                     2, 1, cidx, 2.0 * (static_cast<double>(c.out_dim) * c.kernel + static_cast<double>(c.out_dim) * c.classes),
                     tap_bytes});
  } else if (hidden_done) {
    // FC(h) whose hidden layer the next block's GEMM already produced (fused serve)
  } else {
    // FC(h): hidden = W1 . tap as a split-K tensor-core GEMM over the rows.
    const __nv_bfloat16* a_hi = tap.hi;
    const __nv_bfloat16* a_lo = tap.lo;
    if (stage_gather) {
      const long long row_elems = tap.row_stride;
      Planes g = c.gather;
      const int* idx = tap.data_idx;
      const int* cnt = tap.count;
      steps.push_back({[g, tap, row_elems, idx, cnt, max_rows](cudaStream_t s) {
                         launch_gather_rows(tap.hi, tap.lo, g.hi, g.lo, row_elems, idx, cnt, max_rows, s);
                       },
                       3, 1, cidx, 0.0, 2.0 * tap_bytes});
      a_hi = g.hi;
      a_lo = g.lo;
    }
    auto prm = std::make_shared<TcConvParams>();
    std::memset(prm.get(), 0, sizeof(TcConvParams));
    const int BN = tc_conv_pick_bn(c.hp, prec_ == kPrecX3 ? 3 : 1);
    const bool x3 = prec_ == kPrecX3;
    bool ok = encode_act_map(&prm->tmA[0], a_hi, c.Dk, max_rows, 1, 1, 1, 128, 1) &&
              encode_weight_map(&prm->tmB[0], c.W1.hi, c.Dk, c.hp, BN);
    if (x3)
      ok = ok && encode_act_map(&prm->tmA[1], a_lo, c.Dk, max_rows, 1, 1, 1, 128, 1) &&
           encode_weight_map(&prm->tmB[1], c.W1.lo, c.Dk, c.hp, BN);
    if (!ok) throw CudaFailure("engine: TMA descriptor encode failed (FC cache)");
    prm->plain = 1;
    prm->Ho = 1;
    prm->Wo = max_rows;
    prm->hb = 1;
    prm->wb = 128;
    prm->ipt = 1;
    prm->tiles_h = 1;
    prm->C = c.Dk;
    prm->ntaps = 1;
    prm->segs = x3 ? 3 : 1;
    prm->Cout = c.hp;
    prm->ksplit = c.ks;
    prm->count = tap.count;
    prm->count_static = max_rows;
    prm->mode = 1;
    prm->rows_total = max_rows;
    prm->out_f32 = c.feats;
    const int sms = num_sms_;
    steps.push_back({[prm, BN, sms](cudaStream_t s) { ck(tc_conv_launch(*prm, BN, sms, s), "tc_conv (fc cache)"); }, 1,
                     1, cidx, 2.0 * static_cast<double>(c.D) * c.h, tap_bytes});
  }
  const int rows_total = max_rows;
  const ExitParams exv = ex ? *ex : ExitParams{};
  const float gap_inv = head_gap ? static_cast<float>(1.0 / tap.HW) : 0.0f;
  steps.push_back({[cp, tap, max_rows, rows_total, exv, head_gap, gap_inv, direct](cudaStream_t s) {
                     CacheHeadParams p{};
                     if (direct) {
                       p.row_hi = tap.hi;
                       p.row_lo = tap.lo;
                       p.row_stride = tap.row_stride;
                       p.D = static_cast<int>(cp->D);
                       p.win = cp->win;
                       p.pool_inv = static_cast<float>(1.0 / cp->win);
                       p.kernel = cp->kernel;
                       p.stride = cp->stride;
                       p.out_dim = cp->out_dim;
                       p.w1 = cp->w1;
                       p.b1c = cp->b1c;
                     }
                     p.family = cp->family;
                     p.classes = cp->classes;
                     p.feat = cp->family == 1 ? cp->width : (cp->family == 0 ? cp->h : cp->nchunks);
                     p.feats = cp->feats;
                     p.ks = cp->ks;
                     p.hp = cp->hp;
                     p.rows_total = rows_total;
                     p.b1 = cp->b1;
                     p.W2 = cp->W2;
                     p.b2 = cp->b2;
                     p.Ws1 = cp->Ws1;
                     p.bs1 = cp->bs1;
                     p.ws2 = cp->ws2;
                     p.bs2 = cp->bs2;
                     p.delta = cp->delta;
                     p.count = tap.count;
                     p.prob = cp->prob;
                     p.hit = cp->hit;
                     p.label = cp->label;
                     if (!exv.arrive) {  // lookup-only entry point returns pr/logits; serving does not
                       p.pr_out = cp->pr_out;
                       p.logits_out = cp->logits_out;
                     }
                     p.fc_scratch = cp->fc_scratch;
                     if (head_gap) {
                       p.gap = cp->gap;
                       p.gap_segs = cp->gap_segs;
                       p.gap_inv = gap_inv;
                       p.gap_ids = tap.data_idx;
                     }
                     p.ex = exv;
                     launch_cache_head(p, max_rows, s);
                   },
                   2, (c.classes > 32 && c.family != 2) ? 2 : 1, cidx,
                   direct && c.family == 2 ? 2.0 * (static_cast<double>(c.out_dim) * c.kernel +
                                                    static_cast<double>(c.out_dim) * c.classes)
                                           : 0.0,
                   direct ? tap_bytes : head_bytes});
}

ExitParams Engine::exit_params(int layer, bool shadow, const int* ids_in, int* ids_out, int* src_rows_out,
                               int* count_out) {
  ExitParams e{};
  e.arrive = lk_arrive_;
  e.layer = layer;
  e.shadow = shadow ? 1 : 0;
  e.ids_in = ids_in;
  e.exit_layer = d_exit_;
  e.served = d_served_;
  e.exit_ns = d_exit_ns_;
  e.probs_out = d_probs_ + static_cast<size_t>(layer - 1) * max_batch_;
  e.labels_out = d_labels_ + static_cast<size_t>(layer - 1) * max_batch_;
  e.ids_out = ids_out;
  e.src_rows_out = src_rows_out;
  e.count_out = count_out;
  e.unordered = (!shadow && unordered_ids_) ? 1 : 0;
  if (scan_compaction_) {
    e.scan_agg = d_scan_ + static_cast<size_t>(layer) * kScanMaxCtas;
    e.epoch = d_counts_ + model_.num_blocks + 2;
  }
  return e;
}

// %globaltimer stamp into d_block_ns_[layer][which] (shadow step lists only).
void Engine::add_stamp(std::vector<Step>& steps, int layer, int which) {
  unsigned long long* dst = d_block_ns_ + static_cast<size_t>(layer - 1) * 2 + which;
  steps.push_back({[dst](cudaStream_t s) { launch_stamp_start(dst, s); }, 0, 1});
}

void Engine::layer_times(int B, double* block_ms, double* lookup_ms, bool compact) {
  std::lock_guard<std::recursive_mutex> dev_lock(dev_stream(device_).mu);
  const int L = model_.num_blocks;
  ck(cudaMemsetAsync(d_block_ns_, 0, static_cast<size_t>(L + 1) * 2 * 8, stream_), "memset");
  serve_mode(B, compact ? kModeCompactStamped : kModeShadow, true);
  std::vector<unsigned long long> ns(static_cast<size_t>(L + 1) * 2);
  unsigned long long t0 = 0;
  ck(cudaMemcpyAsync(ns.data(), d_block_ns_, ns.size() * 8, cudaMemcpyDeviceToHost, stream_), "d2h");
  ck(cudaMemcpyAsync(&t0, d_t0_, 8, cudaMemcpyDeviceToHost, stream_), "d2h");
  ck(cudaStreamSynchronize(stream_), "layer_times sync");
  unsigned long long prev = t0;
  for (int l = 0; l < L; ++l) {
    const unsigned long long base_end = ns[static_cast<size_t>(l) * 2];
    const unsigned long long lk_end = ns[static_cast<size_t>(l) * 2 + 1];
    block_ms[l] = base_end > prev ? static_cast<double>(base_end - prev) * 1e-6 : 0.0;
    lookup_ms[l] = lk_end > base_end ? static_cast<double>(lk_end - base_end) * 1e-6 : 0.0;
    prev = lk_end > base_end ? lk_end : base_end;
  }
  const unsigned long long head_end = ns[static_cast<size_t>(L) * 2];
  if (head_end > prev) block_ms[L - 1] += static_cast<double>(head_end - prev) * 1e-6;
}

// ------------------------------------------------------------------ MLP serve
void Engine::build_mlp_steps(std::vector<Step>& steps, bool shadow, bool stamps) {
  const int B = max_batch_, L = model_.num_blocks;
  const bool x3 = prec_ == kPrecX3;
  int* ids = d_ids_;
  int* src = d_src_;
  int* counts = d_counts_;
  steps.push_back({[this, L](cudaStream_t s) {
                     launch_init_batch(cur_batch_, d_batch_, max_batch_, d_ids_, d_counts_, nullptr, 0, d_exit_,
                                       d_served_, d_base_, d_exit_ns_, d_probs_, L, d_t0_, s);
                   },
                   0, 1});
  const int in_dim = static_cast<int>(model_.input_dim());
  {
    Planes in = mlp_in_;
    const int inp = mlp_fc_[0].inp;
    steps.push_back({[this, in, in_dim, inp, counts, B](cudaStream_t s) {
                       launch_split_rows(d_x_, in_dim, inp, nullptr, counts, B, in.hi, in.lo, s);
                     },
                     0});
  }
  Planes cur = mlp_in_;
  int* cur_ids = ids;
  int* cur_count = counts;
  // one plain tcgen05 GEMM over the rows: Cout columns of W (K = inp) from A;
  // with fuse != nullptr the columns >= fuse->fn1 are the FC(h) cache's hidden
  // layer (fp32 partials into its feats), the rest the block's output
  auto gemm_step = [&](const Planes& A, int inp, const Planes& W, int cout, int BN, const float* bias,
                       const Planes& out, int out_ld, DevCache* fuse, double flops, double bytes) {
    auto prm = std::make_shared<TcConvParams>();
    std::memset(prm.get(), 0, sizeof(TcConvParams));
    bool ok = encode_act_map(&prm->tmA[0], A.hi, inp, B, 1, 1, 1, 128, 1) &&
              encode_weight_map(&prm->tmB[0], W.hi, inp, cout, BN);
    if (x3)
      ok = ok && encode_act_map(&prm->tmA[1], A.lo, inp, B, 1, 1, 1, 128, 1) &&
           encode_weight_map(&prm->tmB[1], W.lo, inp, cout, BN);
    if (!ok) throw CudaFailure("engine: TMA descriptor encode failed (mlp)");
    prm->plain = 1;
    prm->Ho = 1;
    prm->Wo = B;
    prm->hb = 1;
    prm->wb = 128;
    prm->ipt = 1;
    prm->tiles_h = 1;
    prm->C = inp;
    prm->ntaps = 1;
    prm->segs = x3 ? 3 : 1;
    prm->Cout = cout;
    prm->ksplit = 1;
    if (fuse) {
      prm->ks_max = 1;  // (K = one tap: 1-8 steps)
      prm->mix_n1 = fuse->fn1;
      prm->mix_ld = fuse->hp;
      prm->out_ld = out_ld;
      prm->out_f32 = fuse->feats;
      prm->rows_total = B;
    } else {
      prm->ks_max = 32;
      prm->ks_min_steps = mlp_ks_min_steps_;
      prm->ws = ws_;
      prm->ws_counters = ws_counters_;
      split_prms_.push_back(prm);
    }
    prm->count = cur_count;
    prm->count_static = B;
    prm->mode = 0;
    prm->shift = bias;
    prm->relu = 1;
    prm->out_hi = out.hi;
    prm->out_lo = out.lo;
    prm->staged_store = staged_store_ ? 1 : 0;
    const int sms = num_sms_;
    steps.push_back({[prm, BN, sms](cudaStream_t s) { ck(tc_conv_launch(*prm, BN, sms, s), "tc_conv (mlp)"); }, 1, 1,
                     static_cast<int>(cur_count - d_counts_), flops, bytes});
  };
  std::vector<char> gemm_done(static_cast<size_t>(L), 0);
  for (int b = 0; b < L; ++b) {
    const DevFC& f = mlp_fc_[static_cast<size_t>(b)];
    Planes act = mlp_act_[static_cast<size_t>(b)];
    const int layer = b + 1;
    if (!gemm_done[static_cast<size_t>(b)]) {
      gemm_step(cur, f.inp, f.w, f.outp, tc_conv_pick_bn(f.outp, x3 ? 3 : 1), f.b, act, 0, nullptr,
                2.0 * f.in * f.out, (x3 ? 4.0 : 2.0) * (static_cast<double>(f.inp) + f.outp));
      if (shadow) tap_step_end_[static_cast<size_t>(layer)] = static_cast<int>(steps.size());
    }
    if (stamps) add_stamp(steps, layer, 0);
    const int ci = cache_of_layer_[static_cast<size_t>(layer)];
    if (ci >= 0) {
      DevCache& c = *caches_[static_cast<size_t>(ci)];
      const bool fuse = c.fused && b + 1 < L;
      const Planes next_act = fuse ? mlp_act_[static_cast<size_t>(b + 1)] : Planes{};
      if (fuse) {
        // the next block's FC and this cache's hidden layer in one GEMM over the
        // tap's rows: the next block's rows for requests that exit here are
        // computed and dropped by the compaction below
        const DevFC& nf = mlp_fc_[static_cast<size_t>(b + 1)];
        gemm_step(act, nf.inp, c.fw, c.fn1 + c.hp, c.fBN, c.fb, shadow ? next_act : c.spec, c.fn1, &c,
                  2.0 * nf.in * nf.out + 2.0 * static_cast<double>(c.D) * c.h,
                  (x3 ? 4.0 : 2.0) * (static_cast<double>(nf.inp) + nf.outp) + 4.0 * c.hp);
        gemm_done[static_cast<size_t>(b + 1)] = 1;
        if (shadow) tap_step_end_[static_cast<size_t>(layer + 1)] = static_cast<int>(steps.size());
      }
      TapView tap;
      tap.hi = act.hi;
      tap.lo = act.lo;
      tap.row_stride = f.outp;
      tap.C = f.out;
      tap.HW = 1;
      tap.data_idx = nullptr;
      tap.count = cur_count;
      int* ids_out = ids + static_cast<size_t>(layer) * B;
      int* src_out = src + static_cast<size_t>(layer) * B;
      int* cnt_out = counts + layer;
      ExitParams ex = exit_params(layer, shadow, cur_ids, ids_out, src_out, cnt_out);
      const bool row_append = !shadow && mlp_row_append_ && c.classes <= 32;
      // the rows that continue: this tap's (compacted into cin) or, fused, the next block's output
      const Planes csrc = fuse ? c.spec : act;
      const Planes cdst = fuse ? next_act : mlp_cin_[static_cast<size_t>(b)];
      const long long crow = fuse ? c.fn1 : f.outp;
      if (row_append) {
        // each head appends its kept row and copies the activations (no gather launch)
        ex.rows_src_hi = csrc.hi;
        ex.rows_src_lo = csrc.lo;
        ex.rows_dst_hi = cdst.hi;
        ex.rows_dst_lo = cdst.lo;
        ex.row_elems = crow;
      }
      add_lookup_steps(steps, c, tap, B, false, false, &ex, fuse);
      if (stamps) add_stamp(steps, layer, 1);
      if (!shadow) {
        if (!row_append)
          steps.push_back({[csrc, cdst, crow, src_out, cnt_out, B](cudaStream_t s) {
                             launch_gather_rows(csrc.hi, csrc.lo, cdst.hi, cdst.lo, crow, src_out, cnt_out, B, s);
                           },
                           3});
        cur = cdst;
      } else {
        cur = act;
      }
      cur_ids = ids_out;
      cur_count = cnt_out;
    } else {
      cur = act;
    }
  }
  const DevFC& last = mlp_fc_.back();
  const int classes = model_.num_classes;
  steps.push_back({[this, cur, last, classes, cur_ids, cur_count, B](cudaStream_t s) {
                     launch_mlp_head(cur.hi, cur.lo, last.outp, last.out, head_w_, head_b_, classes, cur_ids,
                                     cur_count, B, d_base_, d_logits_, d_exit_, d_served_, d_exit_ns_, s);
                   },
                   0});
  if (stamps) add_stamp(steps, L + 1, 0);  // after the head (charged to the last block)
}

// ------------------------------------------------------------------ CNN serve
void Engine::build_cnn_steps(std::vector<Step>& steps, bool shadow, bool stamps) {
  const int B = max_batch_, L = model_.num_blocks;
  const bool x3 = prec_ == kPrecX3;
  int* ids = d_ids_;
  int* counts = d_counts_;
  int stem_mult = 1;
  for (const CnnOp& o : model_.ops)
    if (o.kind == CnnOpKind::Stem) stem_mult = o.Ho() * o.Wo();
  int* stem_rows = counts + L + 1;
  steps.push_back({[this, L, stem_rows, stem_mult](cudaStream_t s) {
                     launch_init_batch(cur_batch_, d_batch_, max_batch_, d_ids_, d_counts_, stem_rows, stem_mult,
                                       d_exit_, d_served_, d_base_, d_exit_ns_, d_probs_, L, d_t0_, s);
                   },
                   0, 1});
  int* cur_ids = ids;
  int* cur_count = counts;
  const int sms = num_sms_;
  for (size_t i = 0; i < model_.ops.size(); ++i) {
    const CnnOp& o = model_.ops[i];
    if (o.kind == CnnOpKind::Stem) {
      // Space-to-depth rewrite of the images, then the slab-fed tcgen05 stem.
      const DevConv& dc = cnn_w_[i];
      Planes X = im2col_buf_;
      Planes out = slot_buf_[static_cast<size_t>(o.out)];
      const StemGeom g = stem_geom(o.H, o.W, o.k, o.stride, o.pad);
      steps.push_back({[this, o, g, X, counts, B](cudaStream_t s) {
                         launch_stem_s2d(d_x_, counts, B, o.C, o.H, o.W, o.stride, o.pad, g, X.hi, X.lo, s);
                       },
                       0, 1, 0, 0.0,
                       4.0 * o.C * o.H * o.W + (x3 ? 4.0 : 2.0) * 2.0 * g.Hx * g.Wx * 8});
      StemParams sp{};
      sp.x_hi = X.hi;
      sp.x_lo = x3 ? X.lo : nullptr;
      sp.w_hi = dc.w.hi;
      sp.w_lo = x3 ? dc.w.lo : nullptr;
      sp.Hx = g.Hx;
      sp.Wx = g.Wx;
      sp.Ho = g.Ho;
      sp.Wo = g.Wo;
      sp.kk = g.kk;
      sp.tiles_per_img = (g.Ho * g.Wx + 127) / 128;
      sp.count = counts;
      sp.count_static = B;
      sp.scale = dc.scale;
      sp.shift = dc.shift;
      sp.relu = o.relu ? 1 : 0;
      sp.out_hi = out.hi;
      sp.out_lo = x3 ? out.lo : nullptr;
      const bool hpool = stem_pool_op_ == static_cast<int>(i + 1);
      if (hpool) {
        sp.hpool = 1;
        sp.Wp = (g.Wo - 1) / 2 + 1;
        sp.tiles_per_img = g.Ho;  // one output row per tile
      }
      steps.push_back({[sp, sms](cudaStream_t s) { ck(tc_stem_launch(sp, sms, s), "tc_stem"); }, 1, 1, 0,
                       2.0 * g.Ho * g.Wo * o.Cout * o.k * o.k * o.C,
                       (x3 ? 4.0 : 2.0) * (32.0 * g.Hx * g.Wx / 2.0 +
                                           static_cast<double>(g.Ho) * (hpool ? sp.Wp : g.Wo) * o.Cout)});
    } else if (o.kind == CnnOpKind::MaxPool && stem_pool_op_ == static_cast<int>(i)) {
      // vertical half of the stem's max-pool over the horizontally pooled rows
      Planes in = slot_buf_[static_cast<size_t>(o.in)], out = slot_buf_[static_cast<size_t>(o.out)];
      const int Hi = o.H, Wp = o.Wo(), Hp = o.Ho(), C = o.C;
      steps.push_back({[in, out, Hi, Wp, Hp, C, cur_ids, cur_count, B](cudaStream_t s) {
                         launch_stem_vpool(in.hi, in.lo, Hi, Wp, C, Hp, cur_ids, cur_count, B, out.hi, out.lo, s);
                       },
                       0, 1, static_cast<int>(cur_count - d_counts_), 0.0,
                       (x3 ? 4.0 : 2.0) * (static_cast<double>(Hi) * Wp * C + static_cast<double>(Hp) * Wp * C)});
    } else if (o.kind == CnnOpKind::MaxPool) {
      Planes in = slot_buf_[static_cast<size_t>(o.in)], out = slot_buf_[static_cast<size_t>(o.out)];
      const int Ho = o.Ho(), Wo = o.Wo();
      steps.push_back({[o, in, out, Ho, Wo, cur_ids, cur_count, B](cudaStream_t s) {
                         launch_maxpool(in.hi, in.lo, o.H, o.W, o.C, o.k, o.stride, o.pad, Ho, Wo, cur_ids, cur_count,
                                        B, out.hi, out.lo, s);
                       },
                       0, 1, static_cast<int>(cur_count - d_counts_), 0.0,
                       (x3 ? 4.0 : 2.0) * (static_cast<double>(o.H) * o.W * o.C + static_cast<double>(Ho) * Wo * o.C)});
    } else if (o.kind == CnnOpKind::Conv && proj_into_[i] >= 0) {
      // fused into its consumer's residual K-steps (no launch, no output buffer)
    } else if (o.kind == CnnOpKind::Conv) {
      const DevConv& dc = cnn_w_[i];
      const int pjx = fused_proj_[i];
      const CnnOp* pj = pjx >= 0 ? &model_.ops[static_cast<size_t>(pjx)] : nullptr;
      Planes in = slot_buf_[static_cast<size_t>(o.in)], out = slot_buf_[static_cast<size_t>(o.out)];
      // Stride 2 reads the NHWC input directly through TMA traversal strides.
      require(o.stride == 1 || o.stride == 2, "engine: only stride 1 and 2 convolutions are supported");
      const int Ho = o.Ho(), Wo = o.Wo();
      int hb, wb, ipt;
      choose_box(Ho, Wo, hb, wb, ipt);
      auto prm = std::make_shared<TcConvParams>();
      std::memset(prm.get(), 0, sizeof(TcConvParams));
      int BN = tc_conv_pick_bn(o.Cout, x3 ? 3 : 1);
      HaloPlan hp{};
      const bool halo = halo_ && tc_conv_halo_plan(o.H, o.W, o.k, o.stride, o.pad, o.Cout, x3, BN, hp);
      // box of the A loads: halo = {Pw, rows} padded-row slab; else the tile's image box
      const int abw = halo ? hp.pw : wb, abh = halo ? hp.rows : hb;
      bool ok = encode_act_map(&prm->tmA[0], in.hi, o.C, o.W, o.H, B, 1, abw, abh, o.stride) &&
                encode_weight_map(&prm->tmB[0], dc.w.hi, dc.Kp, o.Cout, BN);
      if (x3)
        ok = ok && encode_act_map(&prm->tmA[1], in.lo, o.C, o.W, o.H, B, 1, abw, abh, o.stride) &&
             encode_weight_map(&prm->tmB[1], dc.w.lo, dc.Kp, o.Cout, BN);
      if (!ok) throw CudaFailure("engine: TMA descriptor encode failed (conv)");
      if (!halo && ipt > 1) {
        bool mok = encode_act_map(&prm->tmAm[0], in.hi, o.C, o.W, o.H, B, 1, abw, abh, o.stride, ipt) &&
                   (!x3 || encode_act_map(&prm->tmAm[1], in.lo, o.C, o.W, o.H, B, 1, abw, abh, o.stride, ipt));
        if (mok && pj) {
          const Planes& xb = slot_buf_[static_cast<size_t>(pj->in)];
          mok = encode_act_map(&prm->tmRm[0], xb.hi, pj->C, pj->W, pj->H, B, 1, wb, hb, pj->stride, ipt) &&
                (!x3 || encode_act_map(&prm->tmRm[1], xb.lo, pj->C, pj->W, pj->H, B, 1, wb, hb, pj->stride, ipt));
        } else if (mok && o.res >= 0 && mma_residual_) {
          const Planes& rb = slot_buf_[static_cast<size_t>(o.res)];
          mok = encode_act_map(&prm->tmRm[0], rb.hi, o.Cout, Wo, Ho, B, 1, wb, hb, 1, ipt) &&
                (!x3 || encode_act_map(&prm->tmRm[1], rb.lo, o.Cout, Wo, Ho, B, 1, wb, hb, 1, ipt));
        }
        prm->multi_img = mok ? 1 : 0;
      }
      if (halo) {
        hb = 1;
        wb = 1;
        ipt = 1;
        prm->halo = 1;
        prm->halo_pw = hp.pw;
        prm->halo_rows = hp.rows;
        prm->halo_res_rows = hp.res_rows;
        prm->halo_aplane = hp.aplane;
        prm->halo_sb = hp.sb;
      }
      prm->plain = 0;
      prm->Ho = Ho;
      prm->Wo = Wo;
      prm->hb = hb;
      prm->wb = wb;
      prm->ipt = ipt;
      prm->tiles_h = halo ? hp.tiles_per_img : (Ho + hb - 1) / hb;
      prm->tiles_w = halo ? 1 : (Wo + wb - 1) / wb;
      prm->conv_stride = o.stride;
      prm->C = o.C;
      prm->ntaps = o.k * o.k;
      prm->segs = x3 ? 3 : 1;
      // many K-steps per tile: MMA-issue bound -> fewer, wider MMAs (the wider
      // accumulator costs epilogue TMEM reads, which only pays for k x k convs)
      prm->stacked = (x3 && o.k > 1 && stacked_) ? 1 : 0;
      prm->Cout = o.Cout;
      prm->ksplit = 1;
      prm->ks_max = 32;
      prm->ks_min_steps = ks_min_steps_;
      if (wprefetch_) {
        prm->wpre[0] = dc.w.hi;
        prm->wpre[1] = dc.w.lo;
        prm->wpre_bytes = static_cast<long long>(o.Cout) * dc.Kp * 2;
      }
      prm->ws = ws_;
      prm->ws_counters = ws_counters_;
      split_prms_.push_back(prm);
      prm->surv = cur_ids;
      prm->count = cur_count;
      prm->count_static = B;
      prm->mode = 0;
      prm->scale = dc.scale;
      prm->shift = dc.shift;
      if (pj) {
        // projection shortcut on the tensor core: K-steps over the block input
        // (stride pj->stride) against the projection weights
        require(!halo, "engine: fused projection with a halo conv");
        const Planes& xb = slot_buf_[static_cast<size_t>(pj->in)];
        const DevConv& pw = cnn_w_[static_cast<size_t>(pjx)];
        bool rok = encode_act_map(&prm->tmR[0], xb.hi, pj->C, pj->W, pj->H, B, 1, wb, hb, pj->stride) &&
                   (!x3 || encode_act_map(&prm->tmR[1], xb.lo, pj->C, pj->W, pj->H, B, 1, wb, hb, pj->stride)) &&
                   encode_weight_map(&prm->tmP[0], pw.w.hi, pw.Kp, o.Cout, BN) &&
                   (!x3 || encode_weight_map(&prm->tmP[1], pw.w.lo, pw.Kp, o.Cout, BN));
        if (!rok) throw CudaFailure("engine: TMA descriptor encode failed (projection)");
        prm->nres = pj->C / 64;
        prm->res_proj = 1;
        prm->res_stride = pj->stride;
      } else if (o.res >= 0) {
        const Planes& rb = slot_buf_[static_cast<size_t>(o.res)];
        if (mma_residual_) {
          // residual add on the tensor core: BN/64 extra K-steps (residual x identity)
          const int rbw = halo ? hp.pw : wb, rbh = halo ? hp.res_rows : hb;
          bool rok = encode_act_map(&prm->tmR[0], rb.hi, o.Cout, Wo, Ho, B, 1, rbw, rbh, 1) &&
                     (!x3 || encode_act_map(&prm->tmR[1], rb.lo, o.Cout, Wo, Ho, B, 1, rbw, rbh, 1)) &&
                     encode_weight_map(&prm->tmE, identity_, 256, 256, BN);
          if (!rok) throw CudaFailure("engine: TMA descriptor encode failed (residual)");
          prm->nres = BN / 64;
        } else {
          prm->res_hi = rb.hi;
          prm->res_lo = rb.lo;
        }
      }
      prm->relu = o.relu ? 1 : 0;
      prm->out_hi = out.hi;
      prm->out_lo = out.lo;
      prm->staged_store = staged_store_ ? 1 : 0;
      prm->dbg = tc_dbg_;  // LCB_TC_DBG: measurement-only kernel bits (wrong results)
      if (o.tap >= 0 && gap_fusion_) {
        // Pool(C) cache on this conv's output: GAP partials from the epilogue.
        const int ci = cache_of_layer_[static_cast<size_t>(o.tap + 1)];
        if (ci >= 0) {
          DevCache& c = *caches_[static_cast<size_t>(ci)];
          if (c.family == 1 && c.win == Ho * Wo && c.width == o.Cout) {
            const int segs = halo ? prm->tiles_h * 4 : tc_conv_gap_segs(prm->tiles_h, prm->tiles_w, hb, wb);
            if (!c.gap) {
              c.gap = static_cast<float*>(dalloc(static_cast<size_t>(B) * segs * o.Cout * sizeof(float)));
              c.gap_segs = segs;
            }
            prm->gap_out = c.gap;
            prm->gap_segs = segs;
            // post-phase mode runs heads with <= 32 classes (the wide ones keep
            // their own persistent launch); per-tile mode (opt-in) also the
            // features of wide heads
            // (post mode stages W2, Ws1 and 8 feature rows in the pipeline ring)
            const long long post_floats = static_cast<long long>(c.classes) * c.width + 16 * 32 + 8LL * c.width;
            const bool post_fits = post_floats * 4 <= tc_conv_ring_bytes(BN, x3);
            if (conv_head_ && fused_lookup_ && c.width % 4 == 0 &&
                (conv_head_post_ ? (c.classes <= 32 && post_fits) : true)) {
              // the lookup rides the conv: every row's GAP features (and, for
              // <= 32 classes, its head and the layer's exit) come from the
              // conv's CTAs — after a grid barrier that follows the last tile
              // (post mode), or from the CTA finishing the row's last tile
              const int layer = o.tap + 1;
              TcGapHead& gh = prm->gh;
              gh.row_tiles = row_tiles_;
              gh.post = conv_head_post_ ? 1 : 0;
              gh.gsync = conv_sync_;
              gh.inv = static_cast<float>(1.0 / (static_cast<double>(Ho) * Wo));
              if (c.classes <= 32) {
                const ExitParams ex = exit_params(layer, shadow, cur_ids, ids + static_cast<size_t>(layer) * B,
                                                  nullptr, counts + layer);
                gh.classes = c.classes;
                gh.W2 = c.W2;
                gh.b2 = c.b2;
                gh.Ws1 = c.Ws1;
                gh.bs1 = c.bs1;
                gh.ws2 = c.ws2;
                gh.bs2 = c.bs2;
                gh.delta = c.delta;
                gh.prob = c.prob;
                gh.hit = c.hit;
                gh.label = c.label;
                gh.heads_done = heads_done_;
                gh.layer = ex.layer;
                gh.shadow = ex.shadow;
                gh.ids_in = ex.ids_in;
                gh.exit_layer = ex.exit_layer;
                gh.served = ex.served;
                gh.exit_ns = ex.exit_ns;
                gh.probs_out = ex.probs_out;
                gh.labels_out = ex.labels_out;
                gh.ids_out = ex.ids_out;
                gh.src_rows_out = ex.src_rows_out;
                gh.count_out = ex.count_out;
                c.conv_head = true;
              } else {
                gh.feat = c.feats;  // [B][width] bins for the separate head
                c.conv_feat = true;
              }
            }
          }
        }
      }
      for (int r = 0; r < o.k; ++r)
        for (int sx = 0; sx < o.k; ++sx) {
          const int t = r * o.k + sx;
          prm->tap_phase[t] = 0;
          prm->tap_dh[t] = static_cast<signed char>(r - o.pad);
          prm->tap_dw[t] = static_cast<signed char>(sx - o.pad);
        }
      DevCache* head_cache = nullptr;  // threshold / selector bias are read at launch (set_delta, swaps)
      if (prm->gh.row_tiles && prm->gh.classes) head_cache = caches_[static_cast<size_t>(cache_of_layer_[static_cast<size_t>(o.tap + 1)])].get();
      steps.push_back({[prm, BN, sms, head_cache](cudaStream_t s) {
                         if (head_cache) {
                           prm->gh.delta = head_cache->delta;
                           prm->gh.bs2 = head_cache->bs2;
                         }
                         ck(tc_conv_launch(*prm, BN, sms, s), "tc_conv (conv)");
                       },
                       1,
                       1, static_cast<int>(cur_count - d_counts_),
                       2.0 * Ho * Wo * o.Cout * (static_cast<double>(o.C) * o.k * o.k + (pj ? pj->C : 0)),
                       (x3 ? 4.0 : 2.0) * (static_cast<double>(o.H) * o.W * o.C +
                                           (pj ? static_cast<double>(pj->H) * pj->W * pj->C / (pj->stride * pj->stride)
                                               : 0.0) +
                                           static_cast<double>(Ho) * Wo * o.Cout * (o.res >= 0 && !pj ? 2 : 1))});
    } else if (o.kind == CnnOpKind::Head) {
      Planes in = slot_buf_[static_cast<size_t>(o.in)];
      const int classes = model_.num_classes, C = o.C, HW = o.H * o.W;
      float* fs = static_cast<float*>(dalloc(static_cast<size_t>(B) * C * sizeof(float)));
      float* ls = static_cast<float*>(dalloc(static_cast<size_t>(rows_fc_splits(C)) * B * classes * sizeof(float)));
      steps.push_back({[this, in, C, HW, classes, cur_ids, cur_count, B, fs, ls](cudaStream_t s) {
                         launch_cnn_head(in.hi, in.lo, C, HW, head_w_, head_b_, classes, cur_ids, cur_count, B,
                                         d_base_, d_logits_, d_exit_, d_served_, d_exit_ns_, fs, ls, s);
                       },
                       0, classes > 32 ? 3 : 1, static_cast<int>(cur_count - d_counts_),
                       2.0 * C * classes, (x3 ? 4.0 : 2.0) * static_cast<double>(C) * HW + 4.0 * classes});
    }
    if (o.tap >= 0) {
      const int layer = o.tap + 1;
      if (shadow) tap_step_end_[static_cast<size_t>(layer)] = static_cast<int>(steps.size());
      if (stamps) add_stamp(steps, layer, 0);
      const int ci = cache_of_layer_[static_cast<size_t>(layer)];
      if (ci >= 0) {
        DevCache& c = *caches_[static_cast<size_t>(ci)];
        const TapInfo& ti = model_.taps[static_cast<size_t>(o.tap)];
        int* ids_out = ids + static_cast<size_t>(layer) * B;
        int* cnt_out = counts + layer;
        Planes tb = slot_buf_[static_cast<size_t>(o.out)];
        TapView tap;
        tap.hi = tb.hi;
        tap.lo = tb.lo;
        tap.row_stride = ti.dim();
        tap.C = ti.C;
        tap.HW = ti.H * ti.W;
        tap.data_idx = cur_ids;
        tap.count = cur_count;
        const ExitParams ex = exit_params(layer, shadow, cur_ids, ids_out, nullptr, cnt_out);
        if (!c.conv_head) add_lookup_steps(steps, c, tap, B, true, c.gap != nullptr, &ex);
        if (stamps) add_stamp(steps, layer, 1);
        cur_ids = ids_out;
        cur_count = cnt_out;
      }
    }
  }
  if (stamps) add_stamp(steps, L + 1, 0);  // after the head (charged to the last block)
}

// Split-K arrival counters without a reset arrival: the step list's split-K
// launches cycle through counter sets so that consecutive ones (cyclically,
// across graph replays) differ, and each launch zeroes the NEXT launch's set
// after its upstream wait, when that set's previous user has completed. Lists
// start on set 0; an odd count ends on set 2. A single launch keeps the
// in-kernel reset (its next launch is itself).
void Engine::assign_counter_sets() {
  const size_t M = split_prms_.size();
  if (M < 2) return;
  std::vector<int> set(M);
  for (size_t j = 0; j < M; ++j) set[j] = static_cast<int>(j % 2);
  if (M % 2) set[M - 1] = 2;
  const int len = 2 * num_sms_;
  for (size_t j = 0; j < M; ++j) {
    split_prms_[j]->ws_counters = ws_counters_ + static_cast<size_t>(set[j]) * len;
    split_prms_[j]->ctr_zero = ws_counters_ + static_cast<size_t>(set[(j + 1) % M]) * len;
    split_prms_[j]->ctr_len = len;
  }
  split_prms_.clear();
}

std::vector<Step>& Engine::steps_for(bool shadow) { return steps_mode(shadow ? kModeShadow : kModeCompact); }

// Step lists: compact (the product), shadow (with block-boundary stamps; also
// the tap read-back prefix), compact with stamps (per-block device times of
// the compacted step, tools/layer_times.py).
std::vector<Step>& Engine::steps_mode(int mode) {
  std::vector<Step>& st = steps_[mode];
  if (!built_[mode]) {
    st.clear();
    const bool shadow = mode == kModeShadow, stamps = mode != kModeCompact;
    if (shadow) tap_step_end_.assign(static_cast<size_t>(model_.num_blocks) + 1, -1);
    split_prms_.clear();
    if (model_.family == "mlp") build_mlp_steps(st, shadow, stamps);
    else build_cnn_steps(st, shadow, stamps);
    assign_counter_sets();
    built_[mode] = true;
  }
  return st;
}

int Engine::num_steps(bool shadow) const {
  return static_cast<int>(steps_[shadow ? kModeShadow : kModeCompact].size());
}

int Engine::count_kernels(bool shadow, int kind) {
  const auto& st = steps_for(shadow);
  int n = 0;
  for (const Step& s : st)
    if (kind < 0 || s.kind == kind) n += s.launches;
  return n;
}

void Engine::serve(int B, bool shadow, bool use_graph) { serve_mode(B, shadow ? kModeShadow : kModeCompact, use_graph); }

void Engine::serve_mode(int B, int mode, bool use_graph) {
  std::lock_guard<std::recursive_mutex> dev_lock(dev_stream(device_).mu);
  require(B > 0 && B <= max_batch_, "serve: batch size " + std::to_string(B) + " outside [1, max_batch]");
  ck(cudaSetDevice(device_), "cudaSetDevice");
  cur_batch_ = B;
  std::vector<Step>& st = steps_mode(mode);
  if (!use_graph) {
    static const bool sync_steps = std::getenv("LCB_SYNC_STEPS") != nullptr;  // debug: locate a failing step
    for (size_t i = 0; i < st.size(); ++i) {
      st[i].run(stream_);
      if (sync_steps) {
        std::fprintf(stderr, "lcb step %zu (kind %d) ...", i, st[i].kind);
        ck(cudaStreamSynchronize(stream_), "step");
        std::fprintf(stderr, " done\n");
      }
    }
    ck(cudaGetLastError(), "serve");
    return;
  }
  cudaGraphExec_t& ge = graph_[mode];
  if (ge && graph_batch_[mode] != B) {
    // the batch size lives in the init node's arguments: update it in place
    // (launches already enqueued keep theirs); re-capture if that fails
    bool ok = graph_init_node_[mode] != nullptr;
    if (ok) {
      cudaKernelNodeParams kp{};
      ok = cudaGraphKernelNodeGetParams(graph_init_node_[mode], &kp) == cudaSuccess && kp.kernelParams;
      if (ok) {
        void* args[kInitBatchArgs];
        for (int i = 0; i < kInitBatchArgs; ++i) args[i] = kp.kernelParams[i];
        int b = B;
        args[0] = &b;
        kp.kernelParams = args;
        kp.extra = nullptr;
        ok = cudaGraphExecKernelNodeSetParams(ge, graph_init_node_[mode], &kp) == cudaSuccess;
      }
    }
    if (ok) {
      graph_batch_[mode] = B;
    } else {
      cudaGetLastError();
      drop_graph(mode);
    }
  }
  if (!ge) {
    cudaGraph_t g;
    ck(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal), "capture");
    try {
      for (Step& s : st) s.run(stream_);
    } catch (...) {
      // a failed launch must not leave the (shared) stream capturing
      cudaGraph_t partial = nullptr;
      cudaStreamEndCapture(stream_, &partial);
      if (partial) cudaGraphDestroy(partial);
      cudaGetLastError();
      throw;
    }
    ck(cudaStreamEndCapture(stream_, &g), "capture end");
    ck(cudaGraphInstantiate(&ge, g, 0), "graph instantiate");
    // keep the template graph: its init node is the handle for batch-size updates
    graph_tmpl_[mode] = g;
    graph_batch_[mode] = B;
    graph_init_node_[mode] = nullptr;
    size_t nn = 0;
    if (cudaGraphGetNodes(g, nullptr, &nn) == cudaSuccess && nn > 0) {
      std::vector<cudaGraphNode_t> nodes(nn);
      if (cudaGraphGetNodes(g, nodes.data(), &nn) == cudaSuccess) {
        for (cudaGraphNode_t nd : nodes) {
          cudaGraphNodeType ty;
          cudaKernelNodeParams kp{};
          if (cudaGraphNodeGetType(nd, &ty) == cudaSuccess && ty == cudaGraphNodeTypeKernel &&
              cudaGraphKernelNodeGetParams(nd, &kp) == cudaSuccess && kp.func == init_batch_kernel_fn()) {
            graph_init_node_[mode] = nd;
            break;
          }
        }
      }
    }
    cudaGetLastError();
  }
  ck(cudaGraphLaunch(ge, stream_), "graph launch");
}

void Engine::serve_host(const float* x, int B, bool shadow, bool use_graph) {
  std::lock_guard<std::recursive_mutex> dev_lock(dev_stream(device_).mu);
  require(B > 0 && B <= max_batch_, "serve: batch size " + std::to_string(B) + " outside [1, max_batch]");
  ck(cudaSetDevice(device_), "cudaSetDevice");
  ck(cudaMemcpyAsync(d_x_, x, static_cast<size_t>(B) * model_.input_dim() * sizeof(float), cudaMemcpyHostToDevice,
                     stream_),
     "input upload");
  serve(B, shadow, use_graph);
}

void Engine::init_slots() {
  if (copy_stream_) return;
  const int L = model_.num_blocks, B = max_batch_;
  ck(cudaStreamCreateWithFlags(&copy_stream_, cudaStreamNonBlocking), "copy stream");
  for (Slot& sl : slots_) {
    sl.d_in = static_cast<float*>(dalloc(static_cast<size_t>(B) * model_.input_dim() * sizeof(float)));
    ck(cudaMallocHost(&sl.h_exit, static_cast<size_t>(B) * sizeof(int)), "cudaMallocHost");
    ck(cudaMallocHost(&sl.h_served, static_cast<size_t>(B) * sizeof(int)), "cudaMallocHost");
    ck(cudaMallocHost(&sl.h_base, static_cast<size_t>(B) * sizeof(int)), "cudaMallocHost");
    ck(cudaMallocHost(&sl.h_probs, static_cast<size_t>(L) * B * sizeof(float)), "cudaMallocHost");
    ck(cudaMallocHost(&sl.h_logits, static_cast<size_t>(B) * model_.num_classes * sizeof(float)), "cudaMallocHost");
    ck(cudaMallocHost(&sl.h_ns, static_cast<size_t>(B + 1) * 8), "cudaMallocHost");
    ck(cudaEventCreateWithFlags(&sl.in_done, cudaEventDisableTiming), "event");
    ck(cudaEventCreateWithFlags(&sl.in_free, cudaEventDisableTiming), "event");
    ck(cudaEventCreateWithFlags(&sl.out_done, cudaEventDisableTiming), "event");
    ck(cudaEventRecord(sl.in_free, stream_), "event");
  }
}

int Engine::submit(const float* x, int B, bool shadow) {
  std::lock_guard<std::recursive_mutex> dev_lock(dev_stream(device_).mu);
  require(B > 0 && B <= max_batch_, "submit: batch size " + std::to_string(B) + " outside [1, max_batch]");
  ck(cudaSetDevice(device_), "cudaSetDevice");
  init_slots();
  const int id = next_slot_;
  next_slot_ ^= 1;
  Slot& sl = slots_[id];
  if (sl.busy) ck(cudaEventSynchronize(sl.out_done), "slot wait");  // uncollected results are dropped
  ++sl.gen;  // tickets of the dropped batch no longer match
  const size_t bytes = static_cast<size_t>(B) * model_.input_dim() * sizeof(float);
  // H2D on the copy stream once the slot's previous staging copy was consumed
  ck(cudaStreamWaitEvent(copy_stream_, sl.in_free, 0), "wait");
  ck(cudaMemcpyAsync(sl.d_in, x, bytes, cudaMemcpyHostToDevice, copy_stream_), "input upload");
  ck(cudaEventRecord(sl.in_done, copy_stream_), "event");
  // compute stream: stage into the graph's input buffer, serve, results to host
  ck(cudaStreamWaitEvent(stream_, sl.in_done, 0), "wait");
  ck(cudaMemcpyAsync(d_x_, sl.d_in, bytes, cudaMemcpyDeviceToDevice, stream_), "input stage");
  ck(cudaEventRecord(sl.in_free, stream_), "event");
  serve(B, shadow, true);
  const int L = model_.num_blocks;
  ck(cudaMemcpyAsync(sl.h_exit, d_exit_, B * sizeof(int), cudaMemcpyDeviceToHost, stream_), "d2h");
  ck(cudaMemcpyAsync(sl.h_served, d_served_, B * sizeof(int), cudaMemcpyDeviceToHost, stream_), "d2h");
  ck(cudaMemcpyAsync(sl.h_base, d_base_, B * sizeof(int), cudaMemcpyDeviceToHost, stream_), "d2h");
  ck(cudaMemcpy2DAsync(sl.h_probs, static_cast<size_t>(B) * sizeof(float), d_probs_,
                       static_cast<size_t>(max_batch_) * sizeof(float), static_cast<size_t>(B) * sizeof(float), L,
                       cudaMemcpyDeviceToHost, stream_),
     "d2h");
  ck(cudaMemcpyAsync(sl.h_logits, d_logits_, static_cast<size_t>(B) * model_.num_classes * sizeof(float),
                     cudaMemcpyDeviceToHost, stream_),
     "d2h");
  ck(cudaMemcpyAsync(sl.h_ns, d_exit_ns_, static_cast<size_t>(B) * 8, cudaMemcpyDeviceToHost, stream_), "d2h");
  ck(cudaMemcpyAsync(sl.h_ns + B, d_t0_, 8, cudaMemcpyDeviceToHost, stream_), "d2h");
  ck(cudaEventRecord(sl.out_done, stream_), "event");
  sl.B = B;
  sl.busy = true;
  return static_cast<int>((sl.gen & 0x3fffffff) << 1) | id;
}

namespace {
// Base logits exist only for requests whose full pass ran (base_pred >= 0).
void mask_logits(float* logits, const int* base, int B, int classes) {
  for (int i = 0; i < B; ++i)
    if (base[i] < 0)
      for (int k = 0; k < classes; ++k) logits[static_cast<size_t>(i) * classes + k] = std::nanf("");
}
}  // namespace

void Engine::collect(int slot, int B, int* exit_layer, int* served, int* base, float* probs_LB, float* logits,
                     double* latency_ms) {
  require(slot >= 0, "collect: bad ticket");
  Slot& sl = slots_[slot & 1];
  require(sl.busy, "collect: slot holds no submitted batch");
  require(static_cast<unsigned>(slot >> 1) == (sl.gen & 0x3fffffff),
          "collect: ticket superseded (its slot was reused by a later submit)");
  require(B == sl.B, "collect: batch size differs from the submitted one");
  ck(cudaEventSynchronize(sl.out_done), "collect");
  const size_t n = static_cast<size_t>(B);
  if (exit_layer) std::memcpy(exit_layer, sl.h_exit, n * sizeof(int));
  if (served) std::memcpy(served, sl.h_served, n * sizeof(int));
  if (base) std::memcpy(base, sl.h_base, n * sizeof(int));
  if (probs_LB) std::memcpy(probs_LB, sl.h_probs, static_cast<size_t>(model_.num_blocks) * n * sizeof(float));
  if (logits) {
    const int C = model_.num_classes;
    std::memcpy(logits, sl.h_logits, n * C * sizeof(float));
    mask_logits(logits, sl.h_base, B, C);
  }
  if (latency_ms)
    for (size_t i = 0; i < n; ++i) latency_ms[i] = static_cast<double>(sl.h_ns[i] - sl.h_ns[n]) * 1e-6;
  sl.busy = false;
}

void Engine::measure(int B, const double* grid, int G, long long* counts) {
  std::lock_guard<std::recursive_mutex> dev_lock(dev_stream(device_).mu);
  require(G > 0 && G <= 64, "measure: threshold grid must hold 1..64 values");
  const int L = model_.num_blocks;
  serve(B, true, true);
  ck(cudaMemcpyAsync(d_grid_, grid, static_cast<size_t>(G) * sizeof(double), cudaMemcpyHostToDevice, stream_),
     "grid h2d");
  launch_confusion(d_probs_, d_labels_, d_base_, max_batch_, d_batch_, L, d_grid_, G, d_conf_, stream_);
  ck(cudaGetLastError(), "confusion");
  std::vector<unsigned long long> h(static_cast<size_t>(L) * G * 4);
  ck(cudaMemcpyAsync(h.data(), d_conf_, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost, stream_),
     "counts d2h");
  ck(cudaStreamSynchronize(stream_), "measure sync");
  for (size_t i = 0; i < h.size(); ++i) counts[i] = static_cast<long long>(h[i]);
}

void Engine::synchronize() { ck(cudaStreamSynchronize(stream_), "synchronize"); }

void Engine::copy_results(int B, int* exit_layer, int* served, int* base, float* probs_LB, float* logits,
                          double* latency_ms) {
  std::lock_guard<std::recursive_mutex> dev_lock(dev_stream(device_).mu);
  ck(cudaSetDevice(device_), "cudaSetDevice");
  std::vector<int> base_tmp;
  if (logits && !base) {
    base_tmp.resize(static_cast<size_t>(B));
    base = base_tmp.data();
  }
  if (exit_layer) ck(cudaMemcpyAsync(exit_layer, d_exit_, B * sizeof(int), cudaMemcpyDeviceToHost, stream_), "d2h");
  if (served) ck(cudaMemcpyAsync(served, d_served_, B * sizeof(int), cudaMemcpyDeviceToHost, stream_), "d2h");
  if (base) ck(cudaMemcpyAsync(base, d_base_, B * sizeof(int), cudaMemcpyDeviceToHost, stream_), "d2h");
  if (logits)
    ck(cudaMemcpyAsync(logits, d_logits_, static_cast<size_t>(B) * model_.num_classes * sizeof(float),
                       cudaMemcpyDeviceToHost, stream_),
       "d2h");
  if (probs_LB)
    for (int l = 0; l < model_.num_blocks; ++l)
      ck(cudaMemcpyAsync(probs_LB + static_cast<size_t>(l) * B, d_probs_ + static_cast<size_t>(l) * max_batch_,
                         B * sizeof(float), cudaMemcpyDeviceToHost, stream_),
         "d2h");
  std::vector<unsigned long long> ns;
  unsigned long long t0 = 0;
  if (latency_ms) {
    ns.resize(static_cast<size_t>(B));
    ck(cudaMemcpyAsync(ns.data(), d_exit_ns_, B * 8, cudaMemcpyDeviceToHost, stream_), "d2h");
    ck(cudaMemcpyAsync(&t0, d_t0_, 8, cudaMemcpyDeviceToHost, stream_), "d2h");
  }
  ck(cudaStreamSynchronize(stream_), "d2h sync");
  if (latency_ms)
    for (int i = 0; i < B; ++i) latency_ms[i] = static_cast<double>(ns[static_cast<size_t>(i)] - t0) * 1e-6;
  if (logits) mask_logits(logits, base, B, model_.num_classes);
}

void Engine::read_tap_nchw(int layer, int B, float* host_out) {
  std::lock_guard<std::recursive_mutex> dev_lock(dev_stream(device_).mu);
  require(layer >= 1 && layer <= model_.num_blocks, "read_tap: layer out of range");
  require(B > 0 && B <= max_batch_, "read_tap: batch outside [1, max_batch]");
  ck(cudaSetDevice(device_), "cudaSetDevice");
  cur_batch_ = B;
  std::vector<Step>& st = steps_for(true);
  const int end = tap_step_end_[static_cast<size_t>(layer)];
  require(end >= 0, "read_tap: no tap recorded for the layer");
  for (int i = 0; i < end; ++i) st[static_cast<size_t>(i)].run(stream_);
  const TapInfo& ti = model_.taps[static_cast<size_t>(layer - 1)];
  Planes p;
  long long row_stride = 0;
  int C = 0, HW = 1;
  if (model_.family == "mlp") {
    p = mlp_act_[static_cast<size_t>(layer - 1)];
    row_stride = mlp_fc_[static_cast<size_t>(layer - 1)].outp;
    C = mlp_fc_[static_cast<size_t>(layer - 1)].out;
  } else {
    int slot = -1;
    for (const CnnOp& o : model_.ops)
      if (o.tap == layer - 1) slot = o.out;
    require(slot >= 0, "read_tap: no op produces the tap");
    p = slot_buf_[static_cast<size_t>(slot)];
    row_stride = ti.dim();
    C = ti.C;
    HW = ti.H * ti.W;
  }
  const size_t n = static_cast<size_t>(B) * C * HW;
  float* d = nullptr;
  ck(cudaMallocAsync(reinterpret_cast<void**>(&d), n * sizeof(float), stream_), "read_tap alloc");
  launch_planes_to_nchw(p.hi, p.lo, row_stride, C, HW, B, d, stream_);
  const cudaError_t e = cudaMemcpyAsync(host_out, d, n * sizeof(float), cudaMemcpyDeviceToHost, stream_);
  cudaFreeAsync(d, stream_);
  ck(e, "read_tap copy");
  ck(cudaStreamSynchronize(stream_), "read_tap");
}

void Engine::lookup(int layer, const float* taps_dev, int B, int* hit, int* label, float* prob, float* pr,
                    float* logits) {
  std::lock_guard<std::recursive_mutex> dev_lock(dev_stream(device_).mu);
  require(layer >= 1 && layer <= model_.num_blocks, "lookup: layer out of range");
  const int ci = cache_of_layer_[static_cast<size_t>(layer)];
  require(ci >= 0, "lookup: no cache attached at layer " + std::to_string(layer));
  require(B > 0 && B <= max_batch_, "lookup: batch outside [1, max_batch]");
  ck(cudaSetDevice(device_), "cudaSetDevice");
  DevCache& c = *caches_[static_cast<size_t>(ci)];
  const TapInfo& ti = model_.taps[static_cast<size_t>(layer - 1)];
  const bool mlp = model_.family == "mlp";
  const long long row_stride = mlp ? mlp_fc_[static_cast<size_t>(layer - 1)].outp : ti.dim();
  if (c.lookup_steps.empty()) {
    TapView tap;
    tap.hi = lk_tap_.hi;
    tap.lo = lk_tap_.lo;
    tap.row_stride = row_stride;
    tap.C = mlp ? ti.C : ti.C;
    tap.HW = mlp ? 1 : ti.H * ti.W;
    tap.data_idx = nullptr;
    tap.count = d_lk_count_;
    add_lookup_steps(c.lookup_steps, c, tap, max_batch_, false);
  }
  launch_set_int(d_lk_count_, B, stream_);
  launch_split_taps_nchw(taps_dev, ti.C, mlp ? 1 : ti.H * ti.W, B, row_stride, lk_tap_.hi, lk_tap_.lo, stream_);
  for (Step& s : c.lookup_steps) s.run(stream_);
  ck(cudaGetLastError(), "lookup");
  const int C = model_.num_classes;
  if (hit) ck(cudaMemcpyAsync(hit, c.hit, B * sizeof(int), cudaMemcpyDeviceToHost, stream_), "d2h");
  if (label) ck(cudaMemcpyAsync(label, c.label, B * sizeof(int), cudaMemcpyDeviceToHost, stream_), "d2h");
  if (prob) ck(cudaMemcpyAsync(prob, c.prob, B * sizeof(float), cudaMemcpyDeviceToHost, stream_), "d2h");
  if (pr) ck(cudaMemcpyAsync(pr, c.pr_out, static_cast<size_t>(B) * C * sizeof(float), cudaMemcpyDeviceToHost, stream_), "d2h");
  if (logits)
    ck(cudaMemcpyAsync(logits, c.logits_out, static_cast<size_t>(B) * C * sizeof(float), cudaMemcpyDeviceToHost, stream_),
       "d2h");
  ck(cudaStreamSynchronize(stream_), "lookup sync");
}

void Engine::lookup_host(int layer, const float* taps_host, int B, int* hit, int* label, float* prob, float* pr,
                         float* logits) {
  std::lock_guard<std::recursive_mutex> dev_lock(dev_stream(device_).mu);
  require(layer >= 1 && layer <= model_.num_blocks, "lookup: layer out of range");
  require(B > 0 && B <= max_batch_, "lookup: batch outside [1, max_batch]");
  ck(cudaSetDevice(device_), "cudaSetDevice");
  const size_t bytes = static_cast<size_t>(B) * model_.tap_dim(layer) * sizeof(float);
  float* d = nullptr;
  ck(cudaMallocAsync(reinterpret_cast<void**>(&d), bytes, stream_), "lookup: alloc");
  const cudaError_t e = cudaMemcpyAsync(d, taps_host, bytes, cudaMemcpyHostToDevice, stream_);
  if (e != cudaSuccess) {
    cudaFreeAsync(d, stream_);
    ck(e, "lookup: h2d");
  }
  try {
    lookup(layer, d, B, hit, label, prob, pr, logits);
  } catch (...) {
    cudaFreeAsync(d, stream_);
    throw;
  }
  ck(cudaFreeAsync(d, stream_), "lookup: free");
}

void Engine::set_delta(int layer, double delta) {
  std::lock_guard<std::recursive_mutex> dev_lock(dev_stream(device_).mu);
  require(layer >= 1 && layer <= model_.num_blocks, "set_delta: layer out of range");
  const int ci = cache_of_layer_[static_cast<size_t>(layer)];
  require(ci >= 0, "set_delta: no cache attached at layer " + std::to_string(layer));
  caches_[static_cast<size_t>(ci)]->delta = delta;
  variants_[static_cast<size_t>(ci)].delta = delta;
  // Graphs bake kernel parameters: re-capture on next serve.
  for (int m = 0; m < kModes; ++m) drop_graph(m);
}

namespace {
bool same_shape(const Network& a, const Network& b) {
  if (a.layers.size() != b.layers.size()) return false;
  for (size_t i = 0; i < a.layers.size(); ++i) {
    const LayerSpec &x = a.layers[i], &y = b.layers[i];
    if (x.kind != y.kind || x.in_dim != y.in_dim || x.out_dim != y.out_dim || x.pool_window != y.pool_window ||
        x.kernel != y.kernel || x.stride != y.stride)
      return false;
  }
  return true;
}
void put_f32(float* dst, const std::vector<double>& v, cudaStream_t s) {
  const std::vector<float> f = to_f32(v);
  ck(cudaMemcpyAsync(dst, f.data(), f.size() * sizeof(float), cudaMemcpyHostToDevice, s), "variant upload");
}
}  // namespace

void Engine::update_variant(const CacheVariant& nv) {
  require(nv.layer >= 1 && nv.layer <= model_.num_blocks, "update_variant: layer out of range");
  const int ci = cache_of_layer_[static_cast<size_t>(nv.layer)];
  require(ci >= 0, "update_variant: no cache attached at layer " + std::to_string(nv.layer));
  CacheVariant& cur = variants_[static_cast<size_t>(ci)];
  require(same_shape(cur.predictor, nv.predictor) && same_shape(cur.selector, nv.selector),
          "update_variant: architecture differs from the attached variant");
  std::lock_guard<std::recursive_mutex> dev_lock(dev_stream(device_).mu);
  ck(cudaSetDevice(device_), "cudaSetDevice");
  // Swap between batches: everything already enqueued finishes with the old networks.
  ck(cudaStreamSynchronize(stream_), "update_variant: sync");
  DevCache& c = *caches_[static_cast<size_t>(ci)];
  const auto& PW = nv.predictor.weights;
  if (c.family == 0) {
    const TapInfo ti = model_.taps[static_cast<size_t>(nv.layer - 1)];
    const std::vector<float> w = fc_w1_layout(PW[0].w, c, ti, model_.family == "mlp");
    std::vector<__nv_bfloat16> hi, lo;
    split_planes(w, hi, lo);
    h2d(c.W1.hi, hi.data(), w.size() * 2);
    if (c.W1.lo) h2d(c.W1.lo, lo.data(), w.size() * 2);
    if (c.fused) {  // the concatenated copy the serve GEMM reads
      const size_t e1 = static_cast<size_t>(c.fn1) * c.Dk;
      ck(cudaMemcpyAsync(c.fw.hi + e1, c.W1.hi, w.size() * 2, cudaMemcpyDeviceToDevice, stream_), "fused W");
      if (c.fw.lo) ck(cudaMemcpyAsync(c.fw.lo + e1, c.W1.lo, w.size() * 2, cudaMemcpyDeviceToDevice, stream_), "fused W");
    }
    put_f32(c.b1, PW[0].b, stream_);
    put_f32(c.W2, PW[2].w, stream_);
    put_f32(c.b2, PW[2].b, stream_);
  } else if (c.family == 1) {
    put_f32(c.W2, PW[1].w, stream_);
    put_f32(c.b2, PW[1].b, stream_);
  } else {
    put_f32(c.w1, PW[0].w, stream_);
    c.b1c = static_cast<float>(PW[0].b[0]);
    put_f32(c.W2, PW[2].w, stream_);
    put_f32(c.b2, PW[2].b, stream_);
  }
  put_f32(c.Ws1, nv.selector.weights[0].w, stream_);
  put_f32(c.bs1, nv.selector.weights[0].b, stream_);
  put_f32(c.ws2, nv.selector.weights[2].w, stream_);
  c.bs2 = static_cast<float>(nv.selector.weights[2].b[0]);
  c.delta = nv.delta;
  cur = nv;
  ck(cudaStreamSynchronize(stream_), "update_variant: upload");
  for (int m = 0; m < kModes; ++m) drop_graph(m);
}

void Engine::read_taps(int layer, int B, double* host_out) {
  std::lock_guard<std::recursive_mutex> dev_lock(dev_stream(device_).mu);
  ck(cudaSetDevice(device_), "cudaSetDevice");
  require(model_.family == "mlp", "read_taps: retraining records come from the MLP base family");
  require(layer >= 1 && layer <= model_.num_blocks && B >= 0 && B <= max_batch_, "read_taps: bad layer or batch");
  const DevFC& f = mlp_fc_[static_cast<size_t>(layer - 1)];
  const Planes act = mlp_act_[static_cast<size_t>(layer - 1)];
  if (B == 0) return;
  double* d = nullptr;
  ck(cudaMallocAsync(&d, static_cast<size_t>(B) * f.out * sizeof(double), stream_), "read_taps alloc");
  launch_planes_to_f64(act.hi, act.lo, f.outp, f.out, B, d, stream_);
  const cudaError_t e = cudaMemcpyAsync(host_out, d, static_cast<size_t>(B) * f.out * sizeof(double),
                                        cudaMemcpyDeviceToHost, stream_);
  cudaFreeAsync(d, stream_);
  ck(e, "read_taps copy");
  ck(cudaStreamSynchronize(stream_), "read_taps");
}

void Engine::read_base_probs(int B, double* host_out) {
  std::lock_guard<std::recursive_mutex> dev_lock(dev_stream(device_).mu);
  ck(cudaSetDevice(device_), "cudaSetDevice");
  require(model_.family == "mlp", "read_base_probs: retraining records come from the MLP base family");
  require(B >= 0 && B <= max_batch_, "read_base_probs: bad batch");
  if (B == 0) return;
  const DevFC& f = mlp_fc_.back();
  const Planes act = mlp_act_.back();
  const int C = model_.num_classes;
  double* d = nullptr;
  ck(cudaMallocAsync(&d, 2 * static_cast<size_t>(B) * C * sizeof(double), stream_), "read_base_probs alloc");
  launch_head_probs_f64(act.hi, act.lo, f.outp, f.out, head_w_, head_b_, C, B, d, d + static_cast<size_t>(B) * C,
                        stream_);
  const cudaError_t e = cudaMemcpyAsync(host_out, d + static_cast<size_t>(B) * C, static_cast<size_t>(B) * C * sizeof(double),
                                        cudaMemcpyDeviceToHost, stream_);
  cudaFreeAsync(d, stream_);
  ck(e, "read_base_probs copy");
  ck(cudaStreamSynchronize(stream_), "read_base_probs");
}

double Engine::delta(int layer) const {
  const int ci = cache_of_layer_.at(static_cast<size_t>(layer));
  if (ci < 0) throw std::invalid_argument("delta: no cache attached at layer " + std::to_string(layer));
  return caches_[static_cast<size_t>(ci)]->delta;
}

// Rescale the selector's output layer (FC(16,1)) and set its bias; used to
// calibrate synthetic deployments to a target exit profile (the analogue of
// the reference tests' force_selector, test_serving.cpp:123-129).
void Engine::set_selector_out(int layer, double gain, double bias) {
  std::lock_guard<std::recursive_mutex> dev_lock(dev_stream(device_).mu);
  const int ci = cache_of_layer_.at(static_cast<size_t>(layer));
  require(ci >= 0, "set_selector_out: no cache attached at layer " + std::to_string(layer));
  CacheVariant& v = variants_[static_cast<size_t>(ci)];
  for (double& w : v.selector.weights[2].w) w *= gain;
  v.selector.weights[2].b[0] = bias;
  DevCache& c = *caches_[static_cast<size_t>(ci)];
  const std::vector<float> w = to_f32(v.selector.weights[2].w);
  ck(cudaSetDevice(device_), "cudaSetDevice");
  h2d(c.ws2, w.data(), w.size() * sizeof(float));
  ck(cudaStreamSynchronize(stream_), "selector upload");
  c.bs2 = static_cast<float>(bias);
  for (int m = 0; m < kModes; ++m) drop_graph(m);
  c.lookup_steps.clear();
}

std::vector<StepProfile> Engine::profile(int B, bool shadow) {
  std::lock_guard<std::recursive_mutex> dev_lock(dev_stream(device_).mu);
  require(B > 0 && B <= max_batch_, "profile: batch outside [1, max_batch]");
  ck(cudaSetDevice(device_), "cudaSetDevice");
  cur_batch_ = B;
  std::vector<Step>& st = steps_for(shadow);
  std::vector<cudaEvent_t> ev(st.size() + 1);
  for (auto& e : ev) ck(cudaEventCreate(&e), "event");
  ck(cudaEventRecord(ev[0], stream_), "event");
  for (size_t i = 0; i < st.size(); ++i) {
    st[i].run(stream_);
    ck(cudaEventRecord(ev[i + 1], stream_), "event");
  }
  ck(cudaStreamSynchronize(stream_), "profile sync");
  std::vector<int> counts(static_cast<size_t>(model_.num_blocks) + 2);
  ck(cudaMemcpy(counts.data(), d_counts_, counts.size() * sizeof(int), cudaMemcpyDeviceToHost), "counts");
  std::vector<StepProfile> out;
  for (size_t i = 0; i < st.size(); ++i) {
    float ms = 0.0f;
    ck(cudaEventElapsedTime(&ms, ev[i], ev[i + 1]), "elapsed");
    const double units = st[i].count_idx >= 0 ? counts[static_cast<size_t>(st[i].count_idx)] : 0.0;
    out.push_back({st[i].kind, ms, st[i].flops_per_unit * units, st[i].bytes_per_unit * units});
  }
  for (auto& e : ev) cudaEventDestroy(e);
  return out;
}

double Engine::serve_timed(int B, bool shadow) {
  std::lock_guard<std::recursive_mutex> dev_lock(dev_stream(device_).mu);
  steps_for(shadow);
  ck(cudaEventRecord(ev0_, stream_), "event");
  serve(B, shadow, true);
  ck(cudaEventRecord(ev1_, stream_), "event");
  ck(cudaEventSynchronize(ev1_), "event sync");
  float ms = 0.0f;
  ck(cudaEventElapsedTime(&ms, ev0_, ev1_), "elapsed");
  return ms;
}

double Engine::time_serve_ms(int B, bool shadow, int iters) {
  std::lock_guard<std::recursive_mutex> dev_lock(dev_stream(device_).mu);
  serve(B, shadow, true);  // capture outside the timed region
  ck(cudaStreamSynchronize(stream_), "sync");
  ck(cudaEventRecord(ev0_, stream_), "event");
  for (int i = 0; i < iters; ++i) serve(B, shadow, true);
  ck(cudaEventRecord(ev1_, stream_), "event");
  ck(cudaEventSynchronize(ev1_), "event sync");
  float ms = 0.0f;
  ck(cudaEventElapsedTime(&ms, ev0_, ev1_), "elapsed");
  return ms / iters;
}

}  // namespace lcb
