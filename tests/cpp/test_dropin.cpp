// Drop-in test in the reference's own style (doctest-free; exits non-zero on
// failure): the same artifacts go through the UNMODIFIED reference library
// (namespace latecache, oracle/_ref) and through the B200 façade
// (namespace latecache_b200), and the serve traces must agree
// (cf. same_traces, test_serving.cpp:100-111).
//   argv[1] = tests/golden/trained directory
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "latecache/base_model.hpp"
#include "latecache/cache.hpp"
#include "latecache/dataset.hpp"
#include "latecache/serving.hpp"
#include "latecache_b200.hpp"

static int g_fail = 0;
#define CHECK(c)                                                     \
  do {                                                               \
    if (!(c)) {                                                      \
      std::fprintf(stderr, "CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #c); \
      ++g_fail;                                                      \
    }                                                                \
  } while (0)

int main(int argc, char** argv) {
  const std::string dir = argc > 1 ? argv[1] : "tests/golden/trained";
  auto open = [&](const std::string& name) { return std::ifstream(dir + "/" + name); };

  // reference side
  std::ifstream mf = open("model.txt");
  const latecache::BaseModel ref_model = latecache::load_base_model(mf);
  std::ifstream df = open("dataset.txt");
  const latecache::Dataset data = latecache::load_dataset(df);
  std::vector<latecache::CacheVariant> ref_vars;
  std::vector<latecache_b200::CacheVariant> b200_vars;
  for (int k = 0;; ++k) {
    std::ifstream vf = open("variant_" + std::to_string(k) + ".txt");
    if (!vf) break;
    std::stringstream buf;
    buf << vf.rdbuf();
    std::istringstream a(buf.str()), b(buf.str());
    ref_vars.push_back(latecache::load_variant(a));
    b200_vars.push_back(latecache_b200::load_variant(b));
  }
  for (auto& v : ref_vars) v.delta = 0.99;  // spread exits over the layers
  for (auto& v : b200_vars) v.set_delta(0.99);

  // B200 side: same model file through the façade
  std::ifstream mf2 = open("model.txt");
  const latecache_b200::BaseModel model = latecache_b200::load_base_model(mf2);
  CHECK(model.num_blocks == ref_model.num_blocks && model.num_classes == ref_model.num_classes);
  std::vector<const latecache_b200::CacheVariant*> chosen;
  for (auto& v : b200_vars) chosen.push_back(&v);
  latecache_b200::Deployment dep(model, chosen, 512);

  // reference simulate_model over the test split
  std::vector<latecache::VariantMetrics> rows;
  std::vector<size_t> idx;
  for (size_t k = 0; k < ref_vars.size(); ++k) {
    latecache::VariantMetrics m;
    m.layer = ref_vars[k].layer;
    m.variant = ref_vars[k].variant;
    m.arch = ref_vars[k].arch;
    rows.push_back(m);
    idx.push_back(k);
  }
  latecache::Deployment rdep;
  rdep.model = &ref_model;
  rdep.variants = &ref_vars;
  rdep.plan = latecache::make_plan(idx, rows);
  rdep.metrics = rows;
  rdep.profile = latecache::LayerProfile::uniform(ref_model.num_blocks, 4.0);
  rdep.composer.accuracy_threshold = 0.5;
  std::vector<latecache::Request> stream;
  std::vector<std::vector<double>> inputs;
  for (size_t i = 0; i < data.test.size(); ++i) {
    latecache::Request r;
    r.id = static_cast<long long>(i);
    r.sample_idx = i;
    stream.push_back(r);
    inputs.push_back(data.test[i].x.data);
  }
  const auto ref_traces = latecache::simulate_model(rdep, data, stream);
  const auto traces = dep.simulate_model(inputs, /*shadow=*/true);
  CHECK(ref_traces.size() == traces.size());
  // probabilities near delta may legitimately flip (fp32 vs fp64): count, don't fail
  int mismatch = 0, near = 0;
  for (size_t i = 0; i < traces.size(); ++i) {
    const bool same = traces[i].hit_layer == ref_traces[i].hit_layer &&
                      traces[i].served_pred == ref_traces[i].served_pred &&
                      traces[i].base_pred == ref_traces[i].base_pred;
    if (!same) {
      bool in_band = false;
      const auto tf = latecache::forward_with_taps(ref_model, data.test[i].x);
      for (const auto& v : ref_vars) {
        const auto res = latecache::lookup(v, tf.taps[static_cast<size_t>(v.layer - 1)]);
        if (std::fabs(res.selector_prob - v.delta) < 1e-4) in_band = true;
        if (res.hit) break;
      }
      near += in_band;
      mismatch += !in_band;
    }
  }
  std::printf("drop-in traces: %zu requests, %d outside-band mismatches, %d in-band\n", traces.size(), mismatch, near);
  CHECK(mismatch == 0);
  int hist[16] = {0};
  for (const auto& t : traces) hist[t.hit_layer < 16 ? t.hit_layer : 15]++;
  std::printf("exit histogram:");
  for (int l = 0; l <= ref_model.num_blocks; ++l) std::printf(" %d", hist[l]);
  std::printf("\n");

  // lookup parity per chosen layer on the reference's own taps
  for (size_t k = 0; k < ref_vars.size(); ++k) {
    const int layer = ref_vars[k].layer;
    std::vector<std::vector<double>> taps;
    for (size_t i = 0; i < 64 && i < data.test.size(); ++i)
      taps.push_back(latecache::forward_with_taps(ref_model, data.test[i].x).taps[static_cast<size_t>(layer - 1)].data);
    const auto got = dep.lookup(layer, taps);
    for (size_t i = 0; i < taps.size(); ++i) {
      const auto want = latecache::lookup(ref_vars[k], latecache::Tensor::vec(taps[i]));
      const double scale = std::max({1.0, std::fabs(want.selector_prob), std::fabs(got[i].selector_prob)});
      CHECK(std::fabs(want.selector_prob - got[i].selector_prob) <= 1e-3 * scale);
      if (std::fabs(want.selector_prob - ref_vars[k].delta) >= 1e-4) CHECK(want.hit == got[i].hit);
    }
  }
  // retraining (cache.cpp:179-257): the reference's train_predictor /
  // train_selector and the façade's GPU versions on the same records, then
  // the swap into the running deployment
  {
    const int k = 0;
    const int layer = ref_vars[k].layer;
    std::vector<latecache::Sample> samples(data.test.begin(), data.test.begin() + 120);
    const std::vector<latecache::TapRecord> recs = latecache::collect_taps(ref_model, samples);
    std::vector<std::vector<double>> taps, ys;
    for (const auto& r : recs) {
      taps.push_back(r.taps[static_cast<size_t>(layer - 1)].data);
      ys.push_back(r.y.data);
    }
    latecache::TrainConfig rc;
    rc.learning_rate = 0.01;
    rc.epochs = 3;
    rc.seed = 41;
    latecache::CacheVariant ref_v = ref_vars[k];
    latecache::train_predictor(ref_v, recs, rc, 2.0, 0.5, {});
    latecache::train_selector(ref_v, recs, rc, 5.0, 1.0, {});
    latecache_b200::TrainConfig bc;
    bc.learning_rate = 0.01;
    bc.epochs = 3;
    bc.seed = 41;
    latecache_b200::CacheVariant& v = b200_vars[k];
    latecache_b200::train_predictor(v, taps, ys, bc, 2.0, 0.5);
    latecache_b200::train_selector(v, taps, ys, bc, 5.0, 1.0);
    std::ostringstream a, b;
    latecache::save_variant(a, ref_v);
    latecache_b200::save_variant(b, v);
    std::istringstream ai(a.str()), bi(b.str());
    const latecache::CacheVariant back = latecache::load_variant(bi);  // parse ours with the reference
    double err = 0.0;
    for (size_t i = 0; i < back.predictor.weights.size(); ++i)
      for (size_t j = 0; j < back.predictor.weights[i].w.data.size(); ++j)
        err = std::max(err, std::fabs(back.predictor.weights[i].w.data[j] - ref_v.predictor.weights[i].w.data[j]));
    for (size_t i = 0; i < back.selector.weights.size(); ++i)
      for (size_t j = 0; j < back.selector.weights[i].w.data.size(); ++j)
        err = std::max(err, std::fabs(back.selector.weights[i].w.data[j] - ref_v.selector.weights[i].w.data[j]));
    CHECK(err <= 1e-9);
    dep.swap_in(v);
    const auto got = dep.lookup(layer, {taps[0]});
    const latecache::LookupResult want = latecache::lookup(ref_v, recs[0].taps[static_cast<size_t>(layer - 1)]);
    CHECK(std::fabs(want.selector_prob - got[0].selector_prob) <= 1e-3);
  }
  // reference error types survive the boundary
  bool threw = false;
  try {
    std::istringstream bad("latecache-variant v2\n");
    latecache_b200::load_variant(bad);
  } catch (const std::runtime_error&) {
    threw = true;
  }
  CHECK(threw);
  threw = false;
  try {
    dep.lookup(1, {std::vector<double>(3, 0.0)});
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  CHECK(threw);
  std::printf("%s (%d failures)\n", g_fail ? "DROPIN FAILED" : "DROPIN OK", g_fail);
  return g_fail ? 1 : 0;
}
