// Host restatement of the reference's non-kernel path pieces (see lcb_host.hpp).
#include <algorithm>
#include <charconv>
#include <cmath>
#include <sstream>

#include "lcb_host.hpp"

namespace lcb {

namespace {
void require(bool ok, const std::string& msg) {
  if (!ok) throw std::invalid_argument(msg);
}

// Whitespace tokenizer over an artifact string (the reference reads with
// operator>> on an istream).
struct Tok {
  const std::string& s;
  size_t pos;
  Tok(const std::string& str, size_t p = 0) : s(str), pos(p) {}
  void skip_ws() {
    while (pos < s.size() && std::isspace(static_cast<unsigned char>(s[pos]))) ++pos;
  }
  bool eof() {
    skip_ws();
    return pos >= s.size();
  }
  std::string word() {
    skip_ws();
    const size_t b = pos;
    while (pos < s.size() && !std::isspace(static_cast<unsigned char>(s[pos]))) ++pos;
    return s.substr(b, pos - b);
  }
  std::string line() {
    const size_t b = pos;
    while (pos < s.size() && s[pos] != '\n') ++pos;
    std::string out = s.substr(b, pos - b);
    if (pos < s.size()) ++pos;
    return out;
  }
  // After a magic line: skip "# ..." comment lines (base_model.cpp:132).
  void skip_comments() {
    for (;;) {
      skip_ws();
      if (pos < s.size() && s[pos] == '#') {
        line();
      } else {
        return;
      }
    }
  }
  long long integer(const char* what) {
    const std::string w = word();
    long long v = 0;
    auto r = std::from_chars(w.data(), w.data() + w.size(), v);
    if (w.empty() || r.ec != std::errc() || r.ptr != w.data() + w.size())
      throw std::runtime_error(std::string(what) + ": bad integer '" + w + "'");
    return v;
  }
};
}  // namespace

// ================================================================= RNG
uint64_t mix_seed(uint64_t seed, uint64_t tag) {
  uint64_t s = seed + 0x9e3779b97f4a7c15ULL * (tag + 0x632be59bd9b4e019ULL);
  const uint64_t a = splitmix64(s);
  const uint64_t b = splitmix64(s);
  return a ^ (b << 1);
}

Rng::Rng(uint64_t seed) {
  uint64_t sm = seed;
  for (auto& w : s_) w = splitmix64(sm);
}

uint64_t Rng::next_u64() {
  auto rotl = [](uint64_t x, int k) { return (x << k) | (x >> (64 - k)); };
  const uint64_t result = rotl(s_[1] * 5, 7) * 9;
  const uint64_t t = s_[1] << 17;
  s_[2] ^= s_[0];
  s_[3] ^= s_[1];
  s_[1] ^= s_[2];
  s_[0] ^= s_[3];
  s_[2] ^= t;
  s_[3] = rotl(s_[3], 45);
  return result;
}

int Rng::next_int(int n) {
  const uint64_t bound = static_cast<uint64_t>(n);
  const uint64_t limit = UINT64_MAX - UINT64_MAX % bound;
  uint64_t r;
  do {
    r = next_u64();
  } while (r >= limit);
  return static_cast<int>(r % bound);
}

double Rng::normal() {
  if (has_spare_) {
    has_spare_ = false;
    return spare_;
  }
  const double u1 = 1.0 - next_double();
  const double u2 = next_double();
  const double r = std::sqrt(-2.0 * std::log(u1));
  const double theta = 2.0 * 3.14159265358979323846 * u2;
  spare_ = r * std::sin(theta);
  has_spare_ = true;
  return r * std::cos(theta);
}

// ================================================================= text
std::string fmt_double(double v) {
  char buf[64];
  auto r = std::to_chars(buf, buf + sizeof(buf), v);
  if (r.ec != std::errc()) throw std::runtime_error("fmt_double: conversion failed");
  return std::string(buf, r.ptr);
}
double parse_double(const std::string& s) {
  double v = 0.0;
  auto r = std::from_chars(s.data(), s.data() + s.size(), v);
  if (r.ec != std::errc() || r.ptr != s.data() + s.size())
    throw std::runtime_error("parse_double: bad value '" + s + "'");
  return v;
}
long long parse_int(const std::string& s) {
  long long v = 0;
  auto r = std::from_chars(s.data(), s.data() + s.size(), v);
  if (r.ec != std::errc() || r.ptr != s.data() + s.size()) throw std::runtime_error("parse_int: bad value '" + s + "'");
  return v;
}

// ================================================================= networks
LayerSpec LayerSpec::fc(int in, int out) {
  require(in > 0 && out > 0, "fully_connected: dimensions must be positive");
  LayerSpec s;
  s.kind = LayerKind::FC;
  s.in_dim = in;
  s.out_dim = out;
  return s;
}
LayerSpec LayerSpec::relu(int dim) {
  require(dim > 0, "relu: dimension must be positive");
  LayerSpec s;
  s.kind = LayerKind::ReLU;
  s.in_dim = s.out_dim = dim;
  return s;
}
LayerSpec LayerSpec::pool(int in, int window) {
  require(in > 0 && window > 0, "average_pool: dimensions must be positive");
  require(in % window == 0, "average_pool: window must divide the input dimension");
  LayerSpec s;
  s.kind = LayerKind::Pool;
  s.in_dim = in;
  s.out_dim = in / window;
  s.pool_window = window;
  return s;
}
LayerSpec LayerSpec::conv1d(int in, int kernel, int stride) {
  require(in > 0 && kernel > 0 && stride > 0, "conv1d: dimensions must be positive");
  require(kernel <= in, "conv1d: kernel larger than input");
  LayerSpec s;
  s.kind = LayerKind::Conv1d;
  s.in_dim = in;
  s.out_dim = (in - kernel) / stride + 1;
  s.kernel = kernel;
  s.stride = stride;
  return s;
}
LayerSpec LayerSpec::softmax(int dim) {
  require(dim > 0, "softmax: dimension must be positive");
  LayerSpec s;
  s.kind = LayerKind::Softmax;
  s.in_dim = s.out_dim = dim;
  return s;
}

// network.cpp:75-102: Glorot-uniform weights, zero biases, one Rng stream.
Network make_network(std::vector<LayerSpec> layers, uint64_t seed) {
  require(!layers.empty(), "make_network: at least one layer required");
  for (size_t i = 1; i < layers.size(); ++i) {
    require(layers[i].in_dim == layers[i - 1].out_dim,
            "make_network: layer " + std::to_string(i) + " input dim " + std::to_string(layers[i].in_dim) +
                " does not match previous output dim " + std::to_string(layers[i - 1].out_dim));
  }
  Network net;
  net.layers = std::move(layers);
  net.weights.resize(net.layers.size());
  Rng rng(seed);
  for (size_t i = 0; i < net.layers.size(); ++i) {
    const LayerSpec& s = net.layers[i];
    LayerWeights& lw = net.weights[i];
    if (s.kind == LayerKind::FC) {
      const double limit = std::sqrt(6.0 / (s.in_dim + s.out_dim));
      lw.w.resize(static_cast<size_t>(s.out_dim) * s.in_dim);
      for (double& v : lw.w) v = rng.uniform(-limit, limit);
      lw.b.assign(static_cast<size_t>(s.out_dim), 0.0);
    } else if (s.kind == LayerKind::Conv1d) {
      const double limit = std::sqrt(6.0 / (s.kernel + 1));
      lw.w.resize(static_cast<size_t>(s.kernel));
      for (double& v : lw.w) v = rng.uniform(-limit, limit);
      lw.b.assign(1, 0.0);
    }
  }
  return net;
}

long long mac_count(const Network& net) {
  long long n = 0;
  for (const LayerSpec& s : net.layers) {
    if (s.kind == LayerKind::FC) n += static_cast<long long>(s.in_dim) * s.out_dim;
    else if (s.kind == LayerKind::Conv1d) n += static_cast<long long>(s.out_dim) * s.kernel;
  }
  return n;
}
long long parameter_count(const Network& net) {
  long long n = 0;
  for (const LayerWeights& lw : net.weights) n += static_cast<long long>(lw.w.size() + lw.b.size());
  return n;
}

// network.cpp:330-359
std::string save_network(const Network& net) {
  std::ostringstream out;
  out << "latecache-network v1\n";
  out << "layers " << net.layers.size() << '\n';
  for (const LayerSpec& s : net.layers) {
    switch (s.kind) {
      case LayerKind::FC:
        out << "fc " << s.in_dim << ' ' << s.out_dim << '\n';
        break;
      case LayerKind::ReLU:
        out << "relu " << s.in_dim << '\n';
        break;
      case LayerKind::Pool:
        out << "pool " << s.in_dim << ' ' << s.pool_window << '\n';
        break;
      case LayerKind::Conv1d:
        out << "conv1d " << s.in_dim << ' ' << s.kernel << ' ' << s.stride << '\n';
        break;
      case LayerKind::Softmax:
        out << "softmax " << s.in_dim << '\n';
        break;
    }
  }
  auto tensor = [&](const char* tag, const std::vector<double>& t) {
    out << tag << ' ' << t.size();
    for (double v : t) out << ' ' << fmt_double(v);
    out << '\n';
  };
  for (size_t i = 0; i < net.weights.size(); ++i) {
    if (net.weights[i].w.empty()) continue;
    out << "param " << i << '\n';
    tensor("w", net.weights[i].w);
    tensor("b", net.weights[i].b);
  }
  out << "end\n";
  return out.str();
}

// network.cpp:361-409
Network load_network(const std::string& text, size_t& pos) {
  Tok t(text, pos);
  std::string w = t.word();
  if (w != "latecache-network") throw std::runtime_error("network checkpoint: bad magic '" + w + "'");
  w = t.word();
  if (w != "v1") throw std::runtime_error("network checkpoint: unsupported version '" + w + "'");
  if (t.word() != "layers") throw std::runtime_error("network checkpoint: expected 'layers'");
  const long long count = t.integer("network checkpoint");
  std::vector<LayerSpec> layers;
  for (long long i = 0; i < count; ++i) {
    w = t.word();
    if (w == "fc") {
      const int a = static_cast<int>(t.integer("network checkpoint")), b = static_cast<int>(t.integer("network checkpoint"));
      layers.push_back(LayerSpec::fc(a, b));
    } else if (w == "relu") {
      layers.push_back(LayerSpec::relu(static_cast<int>(t.integer("network checkpoint"))));
    } else if (w == "pool") {
      const int a = static_cast<int>(t.integer("network checkpoint")), b = static_cast<int>(t.integer("network checkpoint"));
      layers.push_back(LayerSpec::pool(a, b));
    } else if (w == "conv1d") {
      const int a = static_cast<int>(t.integer("network checkpoint"));
      const int b = static_cast<int>(t.integer("network checkpoint"));
      const int c = static_cast<int>(t.integer("network checkpoint"));
      layers.push_back(LayerSpec::conv1d(a, b, c));
    } else if (w == "softmax") {
      layers.push_back(LayerSpec::softmax(static_cast<int>(t.integer("network checkpoint"))));
    } else {
      throw std::runtime_error("network checkpoint: unknown layer '" + w + "'");
    }
  }
  // Validates the dimension chain and seeds every parameter like the
  // reference (make_network(layers, 0)); the params below overwrite them.
  Network net = make_network(std::move(layers), /*seed=*/0);
  for (;;) {
    if (t.eof()) throw std::runtime_error("network checkpoint: missing 'end'");
    w = t.word();
    if (w == "end") break;
    if (w != "param") throw std::runtime_error("network checkpoint: expected 'param' got '" + w + "'");
    const long long idx = t.integer("network checkpoint");
    if (idx < 0 || idx >= static_cast<long long>(net.layers.size()) ||
        (net.layers[static_cast<size_t>(idx)].kind != LayerKind::FC &&
         net.layers[static_cast<size_t>(idx)].kind != LayerKind::Conv1d)) {
      throw std::runtime_error("network checkpoint: parameters for a parameterless layer");
    }
    const LayerSpec& s = net.layers[static_cast<size_t>(idx)];
    const size_t wn = s.kind == LayerKind::FC ? static_cast<size_t>(s.out_dim) * s.in_dim : static_cast<size_t>(s.kernel);
    const size_t bn = s.kind == LayerKind::FC ? static_cast<size_t>(s.out_dim) : 1;
    auto read = [&](const char* tag, size_t n) {
      const std::string tw = t.word();
      if (tw != tag)
        throw std::runtime_error("network checkpoint: expected '" + std::string(tag) + "' got '" + tw + "'");
      const long long cnt = t.integer("network checkpoint");
      if (cnt != static_cast<long long>(n)) throw std::runtime_error("network checkpoint: tensor size mismatch");
      std::vector<double> v(n);
      for (size_t k = 0; k < n; ++k) {
        if (t.eof()) throw std::runtime_error("network checkpoint: truncated tensor data");
        v[k] = parse_double(t.word());
      }
      return v;
    };
    net.weights[static_cast<size_t>(idx)].w = read("w", wn);
    net.weights[static_cast<size_t>(idx)].b = read("b", bn);
  }
  pos = t.pos;
  return net;
}

// ================================================================= base model
long long BaseModel::macs_to_block(int block) const {
  long long n = 0;
  if (family == "mlp") {
    const int upto = block <= 0 ? -1 : tap_layer.at(static_cast<size_t>(block - 1));
    for (int i = 0; i <= upto; ++i) {
      const LayerSpec& s = net.layers[static_cast<size_t>(i)];
      if (s.kind == LayerKind::FC) n += static_cast<long long>(s.in_dim) * s.out_dim;
    }
    if (block >= num_blocks) n = mac_count(net);
    return n;
  }
  for (const CnnOp& o : ops) {
    if (o.kind == CnnOpKind::Stem || o.kind == CnnOpKind::Conv)
      n += static_cast<long long>(o.Ho()) * o.Wo() * o.Cout * o.C * o.k * o.k;
    else if (o.kind == CnnOpKind::Head)
      n += static_cast<long long>(o.Cout) * o.C;
    if (o.tap >= 0 && o.tap + 1 == block && block < num_blocks) return n;
  }
  return n;
}

// base_model.cpp:30-54
BaseModel make_base_model(int input_dim, int num_classes, std::vector<int> widths, int blocks, uint64_t seed) {
  require(blocks > 0, "base model: need at least one block");
  require(num_classes >= 2, "base model: need at least two classes");
  if (widths.size() == 1) widths.assign(static_cast<size_t>(blocks), widths[0]);
  require(static_cast<int>(widths.size()) == blocks,
          "base model: widths must have one entry per block (or a single entry)");
  std::vector<LayerSpec> layers;
  BaseModel m;
  int dim = input_dim;
  for (int b = 0; b < blocks; ++b) {
    const int w = widths[static_cast<size_t>(b)];
    layers.push_back(LayerSpec::fc(dim, w));
    layers.push_back(LayerSpec::relu(w));
    m.tap_layer.push_back(static_cast<int>(layers.size()) - 1);
    TapInfo ti;
    ti.C = w;
    ti.H = ti.W = 1;
    m.taps.push_back(ti);
    dim = w;
  }
  layers.push_back(LayerSpec::fc(dim, num_classes));
  layers.push_back(LayerSpec::softmax(num_classes));
  m.net = make_network(std::move(layers), mix_seed(seed, 0xba5e));
  m.num_blocks = blocks;
  m.num_classes = num_classes;
  m.family = "mlp";
  m.arch = "mlp";
  return m;
}

// base_model.cpp:143-154
std::string save_base_model(const BaseModel& m) {
  if (m.family != "mlp") throw std::invalid_argument("save_base_model: only the reference MLP family has a text format");
  std::ostringstream out;
  out << "latecache-model v1\n";
  out << "blocks " << m.num_blocks << " classes " << m.num_classes << '\n';
  out << "tap_layers";
  for (int t : m.tap_layer) out << ' ' << t;
  out << "\ntap_dims";
  for (const TapInfo& t : m.taps) out << ' ' << t.C;
  out << '\n';
  out << save_network(m.net);
  return out.str();
}

// base_model.cpp:156-175
BaseModel load_base_model(const std::string& text) {
  Tok t(text);
  if (t.line() != "latecache-model v1") throw std::runtime_error("model checkpoint: bad or missing header");
  t.skip_comments();
  BaseModel m;
  if (t.word() != "blocks") throw std::runtime_error("model checkpoint: expected 'blocks'");
  m.num_blocks = static_cast<int>(t.integer("model checkpoint"));
  if (t.word() != "classes") throw std::runtime_error("model checkpoint: expected 'classes'");
  m.num_classes = static_cast<int>(t.integer("model checkpoint"));
  if (m.num_blocks <= 0 || m.num_classes < 2) throw std::runtime_error("model checkpoint: malformed shape line");
  if (t.word() != "tap_layers") throw std::runtime_error("model checkpoint: expected 'tap_layers'");
  for (int i = 0; i < m.num_blocks; ++i) m.tap_layer.push_back(static_cast<int>(t.integer("model checkpoint")));
  if (t.word() != "tap_dims") throw std::runtime_error("model checkpoint: expected 'tap_dims'");
  for (int i = 0; i < m.num_blocks; ++i) {
    TapInfo ti;
    ti.C = static_cast<int>(t.integer("model checkpoint"));
    ti.H = ti.W = 1;
    m.taps.push_back(ti);
  }
  size_t pos = t.pos;
  m.net = load_network(text, pos);
  // The serve path relies on the make_base_model shape (FC+ReLU blocks, taps
  // after each ReLU, FC+Softmax head); validate it up front.
  const auto& L = m.net.layers;
  require(L.size() == static_cast<size_t>(2 * m.num_blocks + 2) && L.back().kind == LayerKind::Softmax &&
              L[L.size() - 2].kind == LayerKind::FC,
          "model checkpoint: not a block-MLP base model");
  for (int b = 0; b < m.num_blocks; ++b) {
    require(L[static_cast<size_t>(2 * b)].kind == LayerKind::FC && L[static_cast<size_t>(2 * b + 1)].kind == LayerKind::ReLU &&
                m.tap_layer[static_cast<size_t>(b)] == 2 * b + 1,
            "model checkpoint: not a block-MLP base model");
  }
  m.family = "mlp";
  m.arch = "mlp";
  return m;
}

// ================================================================= caches
ArchSpec ArchSpec::parse(const std::string& text) {
  const auto open = text.find('('), close = text.rfind(')');
  if (open == std::string::npos || close == std::string::npos || close != text.size() - 1 || open == 0)
    throw std::invalid_argument("arch: cannot parse '" + text + "'");
  const std::string name = text.substr(0, open), args = text.substr(open + 1, close - open - 1);
  ArchSpec a;
  if (name == "FC" || name == "Pool") {
    a.family = name == "FC" ? ArchFamily::FC : ArchFamily::Pool;
    a.hidden = static_cast<int>(parse_int(args));
    require(a.hidden > 0, name == "FC" ? "arch: fc width must be positive" : "arch: pool width must be positive");
    return a;
  }
  if (name == "Conv") {
    const auto comma = args.find(',');
    if (comma == std::string::npos) throw std::invalid_argument("arch: conv needs kernel,stride in '" + text + "'");
    a.family = ArchFamily::Conv;
    a.kernel = static_cast<int>(parse_int(args.substr(0, comma)));
    a.stride = static_cast<int>(parse_int(args.substr(comma + 1)));
    require(a.kernel > 0 && a.stride > 0, "arch: conv kernel and stride must be positive");
    return a;
  }
  throw std::invalid_argument("arch: unknown family in '" + text + "'");
}

std::string ArchSpec::to_string() const {
  switch (family) {
    case ArchFamily::FC:
      return "FC(" + std::to_string(hidden) + ")";
    case ArchFamily::Pool:
      return "Pool(" + std::to_string(hidden) + ")";
    case ArchFamily::Conv:
      return "Conv(" + std::to_string(kernel) + "," + std::to_string(stride) + ")";
  }
  return "?";
}

// cache.cpp:29-33
int clamp_pool_width(int want, long long dim) {
  long long w = std::min<long long>(want, dim);
  while (dim % w != 0) --w;
  return static_cast<int>(w);
}

// cache.cpp:104-140
CacheVariant build_variant(int layer, int variant_idx, const ArchSpec& arch, long long tap_dim, int num_classes,
                           uint64_t global_seed) {
  require(layer >= 1, "build_variant: layers are 1-based");
  require(tap_dim > 0 && num_classes >= 2, "build_variant: bad dimensions");
  require(tap_dim < (1LL << 31), "build_variant: tap dimension too large");
  const int D = static_cast<int>(tap_dim);
  CacheVariant v;
  v.layer = layer;
  v.variant = variant_idx;
  v.arch = arch;
  const uint64_t seed = mix_seed(mix_seed(global_seed, static_cast<uint64_t>(layer)), static_cast<uint64_t>(variant_idx));
  std::vector<LayerSpec> pred;
  switch (arch.family) {
    case ArchFamily::FC:
      pred = {LayerSpec::fc(D, arch.hidden), LayerSpec::relu(arch.hidden), LayerSpec::fc(arch.hidden, num_classes)};
      break;
    case ArchFamily::Pool: {
      const int width = clamp_pool_width(arch.hidden, D);
      pred = {LayerSpec::pool(D, D / width), LayerSpec::fc(width, num_classes)};
      break;
    }
    case ArchFamily::Conv: {
      require(arch.kernel <= D, "build_variant: conv kernel " + std::to_string(arch.kernel) +
                                    " wider than tap dimension " + std::to_string(D));
      const LayerSpec c = LayerSpec::conv1d(D, arch.kernel, arch.stride);
      pred = {c, LayerSpec::relu(c.out_dim), LayerSpec::fc(c.out_dim, num_classes)};
      break;
    }
  }
  v.predictor = make_network(std::move(pred), mix_seed(seed, 0x9ced));
  v.selector = make_network({LayerSpec::fc(num_classes, 16), LayerSpec::relu(16), LayerSpec::fc(16, 1)},
                            mix_seed(seed, 0x5e1e));
  v.delta = 0.5;
  return v;
}

// cache.cpp:452-462
std::string save_variant(const CacheVariant& v) {
  std::ostringstream out;
  out << "latecache-variant v1\n";
  out << "layer " << v.layer << " variant " << v.variant << " arch " << v.arch.to_string() << " delta "
      << fmt_double(v.delta) << '\n';
  out << "predictor\n" << save_network(v.predictor);
  out << "selector\n" << save_network(v.selector);
  return out.str();
}

// cache.cpp:464-489
CacheVariant load_variant(const std::string& text) {
  Tok t(text);
  if (t.line() != "latecache-variant v1") throw std::runtime_error("variant checkpoint: bad or missing header");
  t.skip_comments();
  CacheVariant v;
  if (t.word() != "layer") throw std::runtime_error("variant checkpoint: expected 'layer'");
  v.layer = static_cast<int>(t.integer("variant checkpoint"));
  if (t.word() != "variant") throw std::runtime_error("variant checkpoint: expected 'variant'");
  v.variant = static_cast<int>(t.integer("variant checkpoint"));
  if (t.word() != "arch") throw std::runtime_error("variant checkpoint: expected 'arch'");
  v.arch = ArchSpec::parse(t.word());
  if (t.word() != "delta") throw std::runtime_error("variant checkpoint: expected 'delta'");
  v.delta = parse_double(t.word());
  if (t.word() != "predictor") throw std::runtime_error("variant checkpoint: expected 'predictor'");
  size_t pos = t.pos;
  v.predictor = load_network(text, pos);
  t.pos = pos;
  if (t.word() != "selector") throw std::runtime_error("variant checkpoint: expected 'selector'");
  pos = t.pos;
  v.selector = load_network(text, pos);
  return v;
}

// ================================================================= plan
double LayerProfile::prefix(int k) const {
  if (k < 0 || k > blocks()) throw std::invalid_argument("layer profile: prefix index out of range");
  double acc = 0.0;
  for (int i = 0; i < k; ++i) acc += latency_ms[static_cast<size_t>(i)];
  return acc;
}

// cache.cpp:424-450
std::vector<VariantMetrics> load_metrics(const std::string& text) {
  std::istringstream in(text);
  std::string line;
  if (!std::getline(in, line) || line != "latecache-metrics v1")
    throw std::runtime_error("metrics file: bad or missing header");
  std::vector<VariantMetrics> rows;
  while (std::getline(in, line)) {
    if (line.empty() || line[0] == '#') continue;
    std::istringstream ls(line);
    VariantMetrics m;
    std::string arch, w;
    ls >> m.layer >> m.variant >> arch;
    m.arch = ArchSpec::parse(arch);
    ls >> w;
    m.hit_rate = parse_double(w);
    ls >> w;
    m.accuracy = parse_double(w);
    ls >> w;
    m.lookup_ms = parse_double(w);
    ls >> w;
    m.memory_mb = parse_double(w);
    ls >> m.tp >> m.fp >> m.tn >> m.fn;
    if (!ls) throw std::runtime_error("metrics file: malformed row '" + line + "'");
    rows.push_back(m);
  }
  return rows;
}

// composer.cpp:65-89
SelectionPlan make_plan(std::vector<size_t> chosen, const std::vector<VariantMetrics>& metrics) {
  for (size_t idx : chosen) require(idx < metrics.size(), "plan: variant index out of range");
  std::sort(chosen.begin(), chosen.end(), [&](size_t a, size_t b) {
    return metrics[a].layer != metrics[b].layer ? metrics[a].layer < metrics[b].layer : a < b;
  });
  for (size_t k = 1; k < chosen.size(); ++k)
    require(metrics[chosen[k - 1]].layer != metrics[chosen[k]].layer,
            "plan: more than one variant at layer " + std::to_string(metrics[chosen[k]].layer));
  SelectionPlan plan;
  plan.chosen = std::move(chosen);
  double absorbed = 0.0;
  for (size_t idx : plan.chosen) {
    const double raw = metrics[idx].hit_rate - absorbed;
    const double eh = std::max(0.0, raw);
    if (raw < 0.0) plan.notes.push_back("clamped negative effective hit rate at layer " + std::to_string(metrics[idx].layer));
    plan.eh.push_back(eh);
    absorbed += eh;
  }
  return plan;
}

// composer.cpp:330-365
SelectionPlan load_plan(const std::string& text, const std::vector<VariantMetrics>& metrics) {
  std::istringstream in(text);
  std::string line;
  if (!std::getline(in, line) || line != "latecache-plan v1") throw std::runtime_error("plan file: bad or missing header");
  while (in >> std::ws && in.peek() == '#') std::getline(in, line);
  std::string word;
  size_t count = 0;
  in >> word >> count;
  if (!in || word != "choices") throw std::runtime_error("plan file: missing choice count");
  std::vector<size_t> chosen;
  for (size_t i = 0; i < count; ++i) {
    int layer = 0, variant = 0;
    std::string arch;
    in >> word >> layer >> variant >> arch;
    if (!in || word != "choice") throw std::runtime_error("plan file: malformed choice row");
    std::getline(in, line);
    bool found = false;
    for (size_t row = 0; row < metrics.size(); ++row) {
      if (metrics[row].layer != layer || metrics[row].variant != variant) continue;
      if (metrics[row].arch.to_string() != arch)
        throw std::runtime_error("plan file: choice at layer " + std::to_string(layer) + " names architecture " + arch +
                                 " but the metrics table has " + metrics[row].arch.to_string());
      chosen.push_back(row);
      found = true;
      break;
    }
    if (!found)
      throw std::runtime_error("plan file: no metrics row for layer " + std::to_string(layer) + " variant " +
                               std::to_string(variant));
  }
  return make_plan(std::move(chosen), metrics);
}

// composer.cpp:106-126
double expected_latency(const SelectionPlan& plan, const std::vector<VariantMetrics>& metrics,
                        const LayerProfile& profile) {
  require(plan.chosen.size() == plan.eh.size(), "expected_latency: plan missing effective hit rates");
  double served = 0.0, sum = 0.0;
  for (size_t k = 0; k < plan.chosen.size(); ++k) {
    const VariantMetrics& m = metrics[plan.chosen[k]];
    sum += plan.eh[k] * (profile.prefix(m.layer) + m.lookup_ms);
    served += plan.eh[k];
  }
  return sum + (1.0 - served) * profile.total();
}
double plan_accuracy(const SelectionPlan& plan, const std::vector<VariantMetrics>& metrics) {
  require(plan.chosen.size() == plan.eh.size(), "plan_accuracy: plan missing effective hit rates");
  double served = 0.0, sum = 0.0;
  for (size_t k = 0; k < plan.chosen.size(); ++k) {
    sum += plan.eh[k] * metrics[plan.chosen[k]].accuracy;
    served += plan.eh[k];
  }
  return sum + (1.0 - served);
}

// composer.cpp:128-160
ConstraintReport check_constraints(const SelectionPlan& plan, const std::vector<VariantMetrics>& metrics,
                                   const LayerProfile& profile, const ComposerConfig& cfg) {
  ConstraintReport r;
  auto violate = [&](std::string why) {
    r.feasible = false;
    r.violations.push_back(std::move(why));
  };
  double total_mem = 0.0;
  for (size_t k = 0; k < plan.chosen.size(); ++k) {
    const VariantMetrics& m = metrics[plan.chosen[k]];
    total_mem += m.memory_mb;
    if (k > 0 && metrics[plan.chosen[k - 1]].layer == m.layer) violate("more than one variant at layer " + std::to_string(m.layer));
    const int next_layer = k + 1 < plan.chosen.size() ? metrics[plan.chosen[k + 1]].layer : profile.blocks();
    const double slack = profile.prefix(next_layer) - profile.prefix(m.layer);
    if (m.lookup_ms > slack)
      violate("lookup at layer " + std::to_string(m.layer) + " (" + fmt_double(m.lookup_ms) + " ms) exceeds the " +
              fmt_double(slack) + " ms available before the next serve point");
  }
  if (total_mem > cfg.memory_budget_mb)
    violate("memory " + fmt_double(total_mem) + " MB exceeds budget " + fmt_double(cfg.memory_budget_mb) + " MB");
  const double acc = plan_accuracy(plan, metrics);
  if (acc < cfg.accuracy_threshold)
    violate("plan accuracy " + fmt_double(acc) + " below floor " + fmt_double(cfg.accuracy_threshold));
  return r;
}

// ================================================================= workload
// serving.cpp:61-91
std::vector<Request> gen_workload(const WorkloadSpec& spec, const std::vector<int>& labels, int dataset_classes) {
  require(spec.num_classes >= 1 && spec.num_classes <= dataset_classes, "workload: class count must fit the dataset");
  require(spec.zipf_alpha > 0.0, "workload: zipf skew must be positive");
  require(spec.rotation_period_min > 0.0, "workload: rotation period must be positive");
  require(spec.requests_per_sec > 0.0 && spec.duration_min > 0.0, "workload: rate and duration must be positive");
  std::vector<std::vector<int>> pools(static_cast<size_t>(dataset_classes));
  for (size_t i = 0; i < labels.size(); ++i) pools[static_cast<size_t>(labels[i])].push_back(static_cast<int>(i));
  for (int c = 0; c < spec.num_classes; ++c)
    require(!pools[static_cast<size_t>(c)].empty(), "workload: no test samples for class " + std::to_string(c));
  const long long n = std::llround(spec.requests_per_sec * spec.duration_min * 60.0);
  std::vector<double> cdf;
  double acc = 0.0;
  for (int r = 1; r <= spec.num_classes; ++r) {
    acc += std::pow(static_cast<double>(r), -spec.zipf_alpha);
    cdf.push_back(acc);
  }
  for (double& c : cdf) c /= acc;
  Rng rng(mix_seed(spec.seed, 0x3f10));
  std::vector<Request> stream;
  stream.reserve(static_cast<size_t>(n));
  for (long long i = 0; i < n; ++i) {
    Request q;
    q.id = i;
    q.time_min = static_cast<double>(i) / (spec.requests_per_sec * 60.0);
    const long long period = static_cast<long long>(q.time_min / spec.rotation_period_min);
    const double u = rng.next_double();
    const int rank = static_cast<int>(std::lower_bound(cdf.begin(), cdf.end(), u) - cdf.begin()) + 1;
    q.true_class = static_cast<int>((rank - 1 + period) % spec.num_classes);
    const auto& pool = pools[static_cast<size_t>(q.true_class)];
    q.sample_idx = pool[static_cast<size_t>(rng.next_int(static_cast<int>(pool.size())))];
    stream.push_back(q);
  }
  return stream;
}

double nearest_rank(std::vector<double> v, double q) {
  require(!v.empty(), "nearest_rank: empty sample");
  std::sort(v.begin(), v.end());
  const size_t idx = static_cast<size_t>(
      std::max<long long>(0, std::llround(std::ceil(q * static_cast<double>(v.size()))) - 1));
  return v[std::min(idx, v.size() - 1)];
}

// serving.cpp:342-376
SimSummary summarize(const std::vector<RequestTrace>& traces, const LayerProfile& profile) {
  require(!traces.empty(), "summarize: no traces");
  SimSummary s;
  s.requests = static_cast<long long>(traces.size());
  std::vector<double> lat;
  long long agree = 0, correct = 0, hits = 0;
  double sum = 0.0;
  for (const RequestTrace& t : traces) {
    lat.push_back(t.latency_ms);
    sum += t.latency_ms;
    agree += t.served_pred == t.base_pred;
    correct += t.served_pred == t.true_class;
    if (t.hit_layer > 0) {
      ++hits;
      ++s.hits_by_layer[t.hit_layer];
    }
  }
  const double n = static_cast<double>(traces.size());
  s.avg_latency_ms = sum / n;
  s.p50_latency_ms = nearest_rank(lat, 0.50);
  s.p99_latency_ms = nearest_rank(lat, 0.99);
  s.max_latency_ms = *std::max_element(lat.begin(), lat.end());
  s.agreement = static_cast<double>(agree) / n;
  s.accuracy = static_cast<double>(correct) / n;
  s.hit_rate = static_cast<double>(hits) / n;
  s.speedup = profile.total() / s.avg_latency_ms;
  return s;
}

}  // namespace lcb
