// CNN base-model families named by BASELINE.json (ResNet-18 CIFAR, ResNet-50 /
// ResNet-152 ImageNet, VGG-16 CIFAR). The reference only implements the block
// MLP (base_model.cpp:30-54), so these layer definitions are the build's own;
// their CPU restatement lives in oracle/lc_oracle.c (lco_cnn_forward).
//
// Every op's output gets its own slot (SSA); the engine maps slots to device
// buffers with liveness-based reuse. Taps are the outputs of residual blocks
// (ResNets) or of the pooling stages (VGG), exactly where GATI attaches its
// per-layer caches.
#include <cmath>

#include "lcb_host.hpp"

namespace lcb {

namespace {

struct Builder {
  BaseModel& m;
  Rng rng;
  int next_slot = 0;
  int op_index = 0;

  Builder(BaseModel& model, uint64_t seed) : m(model), rng(mix_seed(seed, 0xc0de)) {}

  // He-normal conv weights; folded batch-norm scale/shift.
  int conv(int in, int C, int H, int W, int Cout, int k, int stride, int pad, bool relu, int res, double bn_gain,
           CnnOpKind kind = CnnOpKind::Conv) {
    CnnOp o;
    o.kind = kind;
    o.in = in;
    o.out = next_slot++;
    o.res = res;
    o.C = C;
    o.H = H;
    o.W = W;
    o.Cout = Cout;
    o.k = k;
    o.stride = stride;
    o.pad = pad;
    o.relu = relu;
    const double std = std::sqrt(2.0 / (static_cast<double>(C) * k * k));
    o.w.resize(static_cast<size_t>(Cout) * C * k * k);
    for (double& v : o.w) v = rng.normal() * std;
    o.scale.resize(static_cast<size_t>(Cout));
    o.shift.resize(static_cast<size_t>(Cout));
    for (int c = 0; c < Cout; ++c) {
      o.scale[static_cast<size_t>(c)] = bn_gain * rng.uniform(0.8, 1.2);
      o.shift[static_cast<size_t>(c)] = rng.uniform(-0.1, 0.1);
    }
    m.ops.push_back(std::move(o));
    ++op_index;
    return m.ops.back().out;
  }

  int maxpool(int in, int C, int H, int W, int k, int stride, int pad) {
    CnnOp o;
    o.kind = CnnOpKind::MaxPool;
    o.in = in;
    o.out = next_slot++;
    o.C = C;
    o.H = H;
    o.W = W;
    o.Cout = C;
    o.k = k;
    o.stride = stride;
    o.pad = pad;
    m.ops.push_back(std::move(o));
    return m.ops.back().out;
  }

  void head(int in, int C, int H, int W, int classes) {
    CnnOp o;
    o.kind = CnnOpKind::Head;
    o.in = in;
    o.out = next_slot++;
    o.C = C;
    o.H = H;
    o.W = W;
    o.Cout = classes;
    const double limit = std::sqrt(6.0 / (C + classes));
    o.w.resize(static_cast<size_t>(classes) * C);
    for (double& v : o.w) v = rng.uniform(-limit, limit);
    o.shift.assign(static_cast<size_t>(classes), 0.0);
    m.ops.push_back(std::move(o));
  }

  void mark_tap(int C, int H, int W) {
    m.ops.back().tap = static_cast<int>(m.taps.size());
    TapInfo t;
    t.C = C;
    t.H = H;
    t.W = W;
    m.taps.push_back(t);
  }
};

void resnet(BaseModel& m, Builder& b, bool imagenet, bool bottleneck, const int* blocks_per_stage) {
  int H = m.in_H, W = m.in_W, C = 64;
  int x;
  if (imagenet) {
    x = b.conv(-1, 3, H, W, 64, 7, 2, 3, true, -1, 1.0, CnnOpKind::Stem);
    H = (H + 6 - 7) / 2 + 1;
    W = (W + 6 - 7) / 2 + 1;
    x = b.maxpool(x, 64, H, W, 3, 2, 1);
    H = (H + 2 - 3) / 2 + 1;
    W = (W + 2 - 3) / 2 + 1;
  } else {
    x = b.conv(-1, 3, H, W, 64, 3, 1, 1, true, -1, 1.0, CnnOpKind::Stem);
  }
  const int widths[4] = {64, 128, 256, 512};
  // Residual-branch gain keeps activations O(1) as blocks accumulate.
  const double branch_gain = bottleneck ? 0.2 : 0.5;
  for (int s = 0; s < 4; ++s) {
    for (int i = 0; i < blocks_per_stage[s]; ++i) {
      const int stride = (i == 0 && s > 0) ? 2 : 1;
      const int Ho = (H - 1) / stride + 1, Wo = (W - 1) / stride + 1;
      if (!bottleneck) {
        const int Cout = widths[s];
        const int t1 = b.conv(x, C, H, W, Cout, 3, stride, 1, true, -1, 1.0);
        int res = x;
        if (stride != 1 || C != Cout) res = b.conv(x, C, H, W, Cout, 1, stride, 0, false, -1, 1.0);
        x = b.conv(t1, Cout, Ho, Wo, Cout, 3, 1, 1, true, res, branch_gain);
        C = Cout;
      } else {
        const int w = widths[s], Cout = 4 * w;
        const int t1 = b.conv(x, C, H, W, w, 1, 1, 0, true, -1, 1.0);
        const int t2 = b.conv(t1, w, H, W, w, 3, stride, 1, true, -1, 1.0);
        int res = x;
        if (stride != 1 || C != Cout) res = b.conv(x, C, H, W, Cout, 1, stride, 0, false, -1, 1.0);
        x = b.conv(t2, w, Ho, Wo, Cout, 1, 1, 0, true, res, branch_gain);
        C = Cout;
      }
      H = Ho;
      W = Wo;
      b.mark_tap(C, H, W);
    }
  }
  b.head(x, C, H, W, m.num_classes);
}

void vgg16(BaseModel& m, Builder& b) {
  static const int cfg[] = {64, 64, -1, 128, 128, -1, 256, 256, 256, -1, 512, 512, 512, -1, 512, 512, 512, -1};
  int H = m.in_H, W = m.in_W, C = 3, x = -1;
  bool first = true;
  for (int v : cfg) {
    if (v < 0) {
      x = b.maxpool(x, C, H, W, 2, 2, 0);
      H /= 2;
      W /= 2;
      b.mark_tap(C, H, W);
    } else {
      x = b.conv(x, C, H, W, v, 3, 1, 1, true, -1, 1.0, first ? CnnOpKind::Stem : CnnOpKind::Conv);
      first = false;
      C = v;
    }
  }
  b.head(x, C, H, W, m.num_classes);
}

}  // namespace

BaseModel make_cnn_model(const std::string& arch, int num_classes, uint64_t seed) {
  if (num_classes < 2) throw std::invalid_argument("base model: need at least two classes");
  BaseModel m;
  m.family = "cnn";
  m.arch = arch;
  m.num_classes = num_classes;
  m.in_C = 3;
  Builder b(m, seed);
  if (arch == "resnet18_cifar") {
    m.in_H = m.in_W = 32;
    const int blocks[4] = {2, 2, 2, 2};
    resnet(m, b, false, false, blocks);
  } else if (arch == "resnet50") {
    m.in_H = m.in_W = 224;
    const int blocks[4] = {3, 4, 6, 3};
    resnet(m, b, true, true, blocks);
  } else if (arch == "resnet152") {
    m.in_H = m.in_W = 224;
    const int blocks[4] = {3, 8, 36, 3};
    resnet(m, b, true, true, blocks);
  } else if (arch == "vgg16_cifar") {
    m.in_H = m.in_W = 32;
    vgg16(m, b);
  } else {
    throw std::invalid_argument("base model: unknown CNN architecture '" + arch + "'");
  }
  m.num_blocks = static_cast<int>(m.taps.size());
  m.nslots = b.next_slot;
  return m;
}

}  // namespace lcb
