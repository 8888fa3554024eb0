// Binary weight format: a little-endian mirror of the
// reference's text checkpoints latecache-network/model/variant v1
// (network.cpp:301-409, base_model.cpp:143-175, cache.cpp:452-489) that
// stores every double as its 8 raw bytes — the same content, no decimal
// formatting or parsing (multi-GB CNN / FC(h) cache weights), plus the CNN op
// list the text format has no section for. Layout:
//   "LCBBIN1\0" | u32 kind (1 model, 2 variant) | payload
// Network: u32 layers, per layer {u32 kind, i32 in, out, window, kernel,
// stride, vec<f64> w, vec<f64> b}; vec<T> = u64 count + count * sizeof(T) bytes;
// str = vec<char>.
#include <cstring>

#include "lcb_host.hpp"

namespace lcb {

namespace {

constexpr char kMagic[8] = {'L', 'C', 'B', 'B', 'I', 'N', '1', '\0'};

struct Writer {
  std::string out;
  template <typename T>
  void put(T v) {
    const char* p = reinterpret_cast<const char*>(&v);
    out.append(p, sizeof(T));
  }
  template <typename T>
  void vec(const std::vector<T>& v) {
    put<uint64_t>(v.size());
    if (!v.empty()) out.append(reinterpret_cast<const char*>(v.data()), v.size() * sizeof(T));
  }
  void str(const std::string& s) {
    put<uint64_t>(s.size());
    out.append(s);
  }
};

struct Reader {
  const char* p;
  size_t n, pos = 0;
  std::string what;
  void need(size_t k) {
    if (k > n - pos) throw std::runtime_error(what + ": truncated binary checkpoint");
  }
  template <typename T>
  T get() {
    need(sizeof(T));
    T v;
    std::memcpy(&v, p + pos, sizeof(T));
    pos += sizeof(T);
    return v;
  }
  template <typename T>
  std::vector<T> vec() {
    const uint64_t c = get<uint64_t>();
    if (c > (n - pos) / sizeof(T)) throw std::runtime_error(what + ": truncated binary checkpoint");
    std::vector<T> v(static_cast<size_t>(c));
    if (c) std::memcpy(v.data(), p + pos, static_cast<size_t>(c) * sizeof(T));
    pos += static_cast<size_t>(c) * sizeof(T);
    return v;
  }
  std::string str() {
    const std::vector<char> c = vec<char>();
    return std::string(c.begin(), c.end());
  }
};

void put_network(Writer& w, const Network& net) {
  w.put<uint32_t>(static_cast<uint32_t>(net.layers.size()));
  for (size_t i = 0; i < net.layers.size(); ++i) {
    const LayerSpec& l = net.layers[i];
    w.put<uint32_t>(static_cast<uint32_t>(l.kind));
    w.put<int32_t>(l.in_dim);
    w.put<int32_t>(l.out_dim);
    w.put<int32_t>(l.pool_window);
    w.put<int32_t>(l.kernel);
    w.put<int32_t>(l.stride);
    w.vec(net.weights[i].w);
    w.vec(net.weights[i].b);
  }
}

Network get_network(Reader& r) {
  Network net;
  const uint32_t n = r.get<uint32_t>();
  if (n == 0 || n > 4096) throw std::runtime_error(r.what + ": bad layer count in binary checkpoint");
  for (uint32_t i = 0; i < n; ++i) {
    LayerSpec l;
    const uint32_t k = r.get<uint32_t>();
    if (k > static_cast<uint32_t>(LayerKind::Softmax)) throw std::runtime_error(r.what + ": unknown layer kind");
    l.kind = static_cast<LayerKind>(k);
    l.in_dim = r.get<int32_t>();
    l.out_dim = r.get<int32_t>();
    l.pool_window = r.get<int32_t>();
    l.kernel = r.get<int32_t>();
    l.stride = r.get<int32_t>();
    LayerWeights wt;
    wt.w = r.vec<double>();
    wt.b = r.vec<double>();
    const size_t want_w = l.kind == LayerKind::FC ? static_cast<size_t>(l.in_dim) * l.out_dim
                          : l.kind == LayerKind::Conv1d ? static_cast<size_t>(l.kernel) : 0;
    const size_t want_b = l.kind == LayerKind::FC ? static_cast<size_t>(l.out_dim) : l.kind == LayerKind::Conv1d ? 1 : 0;
    if (wt.w.size() != want_w || wt.b.size() != want_b)
      throw std::runtime_error(r.what + ": weight shape mismatch in binary checkpoint");
    if (!net.layers.empty() && net.layers.back().out_dim != l.in_dim)
      throw std::runtime_error(r.what + ": layer dims do not chain");
    net.layers.push_back(l);
    net.weights.push_back(std::move(wt));
  }
  return net;
}

void header(Writer& w, uint32_t kind) {
  w.out.append(kMagic, sizeof(kMagic));
  w.put<uint32_t>(kind);
}

void check_header(Reader& r, uint32_t kind) {
  r.need(sizeof(kMagic));
  if (std::memcmp(r.p, kMagic, sizeof(kMagic)) != 0) throw std::runtime_error(r.what + ": not a latecache-b200 binary checkpoint");
  r.pos = sizeof(kMagic);
  if (r.get<uint32_t>() != kind) throw std::runtime_error(r.what + ": wrong checkpoint kind");
}

}  // namespace

std::string save_base_model_binary(const BaseModel& m) {
  Writer w;
  header(w, 1);
  w.str(m.family);
  w.str(m.arch);
  w.put<int32_t>(m.num_blocks);
  w.put<int32_t>(m.num_classes);
  w.vec(m.tap_layer);
  w.put<uint64_t>(m.taps.size());
  for (const TapInfo& t : m.taps) {
    w.put<int32_t>(t.C);
    w.put<int32_t>(t.H);
    w.put<int32_t>(t.W);
  }
  w.put<uint8_t>(m.family == "mlp" ? 1 : 0);
  if (m.family == "mlp") put_network(w, m.net);
  w.put<int32_t>(m.in_C);
  w.put<int32_t>(m.in_H);
  w.put<int32_t>(m.in_W);
  w.put<int32_t>(m.nslots);
  w.put<uint64_t>(m.ops.size());
  for (const CnnOp& o : m.ops) {
    for (int v : {static_cast<int>(o.kind), o.in, o.out, o.res, o.C, o.H, o.W, o.Cout, o.k, o.stride, o.pad, o.tap})
      w.put<int32_t>(v);
    w.put<uint8_t>(o.relu ? 1 : 0);
    w.vec(o.w);
    w.vec(o.scale);
    w.vec(o.shift);
  }
  return w.out;
}

BaseModel load_base_model_binary(const std::string& data) {
  Reader r{data.data(), data.size(), 0, "load_base_model_binary"};
  check_header(r, 1);
  BaseModel m;
  m.family = r.str();
  m.arch = r.str();
  if (m.family != "mlp" && m.family != "cnn") throw std::runtime_error(r.what + ": unknown model family");
  m.num_blocks = r.get<int32_t>();
  m.num_classes = r.get<int32_t>();
  if (m.num_blocks <= 0 || m.num_classes <= 0) throw std::runtime_error(r.what + ": bad model header");
  m.tap_layer = r.vec<int>();
  const uint64_t nt = r.get<uint64_t>();
  if (nt != static_cast<uint64_t>(m.num_blocks)) throw std::runtime_error(r.what + ": tap count != blocks");
  for (uint64_t i = 0; i < nt; ++i) {
    TapInfo t;
    t.C = r.get<int32_t>();
    t.H = r.get<int32_t>();
    t.W = r.get<int32_t>();
    m.taps.push_back(t);
  }
  if (r.get<uint8_t>()) m.net = get_network(r);
  m.in_C = r.get<int32_t>();
  m.in_H = r.get<int32_t>();
  m.in_W = r.get<int32_t>();
  m.nslots = r.get<int32_t>();
  const uint64_t nops = r.get<uint64_t>();
  if (nops > 100000) throw std::runtime_error(r.what + ": bad op count");
  for (uint64_t i = 0; i < nops; ++i) {
    CnnOp o;
    int v[12];
    for (int& x : v) x = r.get<int32_t>();
    if (v[0] < 0 || v[0] > static_cast<int>(CnnOpKind::Head)) throw std::runtime_error(r.what + ": unknown op kind");
    o.kind = static_cast<CnnOpKind>(v[0]);
    o.in = v[1], o.out = v[2], o.res = v[3], o.C = v[4], o.H = v[5], o.W = v[6], o.Cout = v[7], o.k = v[8];
    o.stride = v[9], o.pad = v[10], o.tap = v[11];
    o.relu = r.get<uint8_t>() != 0;
    o.w = r.vec<double>();
    o.scale = r.vec<double>();
    o.shift = r.vec<double>();
    m.ops.push_back(std::move(o));
  }
  if (r.pos != r.n) throw std::runtime_error(r.what + ": trailing bytes in binary checkpoint");
  return m;
}

std::string save_variant_binary(const CacheVariant& v) {
  Writer w;
  header(w, 2);
  w.put<int32_t>(v.layer);
  w.put<int32_t>(v.variant);
  w.put<uint32_t>(static_cast<uint32_t>(v.arch.family));
  w.put<int32_t>(v.arch.hidden);
  w.put<int32_t>(v.arch.kernel);
  w.put<int32_t>(v.arch.stride);
  put_network(w, v.predictor);
  put_network(w, v.selector);
  w.put<double>(v.delta);
  return w.out;
}

CacheVariant load_variant_binary(const std::string& data) {
  Reader r{data.data(), data.size(), 0, "load_variant_binary"};
  check_header(r, 2);
  CacheVariant v;
  v.layer = r.get<int32_t>();
  v.variant = r.get<int32_t>();
  const uint32_t fam = r.get<uint32_t>();
  if (fam > static_cast<uint32_t>(ArchFamily::Conv)) throw std::runtime_error(r.what + ": unknown predictor family");
  v.arch.family = static_cast<ArchFamily>(fam);
  v.arch.hidden = r.get<int32_t>();
  v.arch.kernel = r.get<int32_t>();
  v.arch.stride = r.get<int32_t>();
  v.predictor = get_network(r);
  v.selector = get_network(r);
  v.delta = r.get<double>();
  if (v.layer < 1) throw std::runtime_error(r.what + ": bad layer");
  if (r.pos != r.n) throw std::runtime_error(r.what + ": trailing bytes in binary checkpoint");
  return v;
}

}  // namespace lcb
