// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// extern "C" driver over the UNMODIFIED reference library (latecache, compiled
// from /root/reference/proj/src by oracle/Makefile into oracle/_ref/). It lets
// pytest, the golden-fixture generator and bench.py's reference arm call the
// reference's own code path:
//   make_base_model / load_base_model   base_model.cpp:30 / :156
//   build_variant / load_variant        cache.cpp:104 / :464
//   forward / forward_with_taps         network.cpp:104 / base_model.cpp:56
//   lookup                              cache.cpp:259
//   simulate_model (-> serve_one)       serving.cpp:147 (-> :97)
// and the offline pipeline (train_base, explore_variants, compose_relaxed,
// gen_workload) that produces trained deployments for golden fixtures.
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "latecache/base_model.hpp"
#include "latecache/cache.hpp"
#include "latecache/composer.hpp"
#include "latecache/dataset.hpp"
#include "latecache/losses.hpp"
#include "latecache/network.hpp"
#include "latecache/rng.hpp"
#include "latecache/serving.hpp"

using namespace latecache;

namespace {
thread_local std::string g_err;

char* dup_string(const std::string& s) {
  char* out = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(out, s.data(), s.size());
  out[s.size()] = '\0';
  return out;
}

// 0 ok, 1 invalid_argument, 2 runtime_error, 3 other
template <typename F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::runtime_error& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 3;
  }
}

Tensor vec_of(const double* x, int n) { return Tensor::vec(std::vector<double>(x, x + n)); }

// A Deployment whose plan chooses every given variant and always passes
// check_constraints (composer.cpp:128): zero memory, unit accuracy and the
// minimal lookup cost; the per-variant metrics rows only carry layer ids.
struct PassThroughDeployment {
  std::vector<CacheVariant> variants;
  std::vector<VariantMetrics> metrics;
  Deployment dep;
};

void make_passthrough(PassThroughDeployment& pd, const BaseModel& model, void** vars, int nv) {
  for (int i = 0; i < nv; ++i) {
    const CacheVariant& v = *static_cast<CacheVariant*>(vars[i]);
    pd.variants.push_back(v);
    VariantMetrics m;
    m.layer = v.layer;
    m.variant = v.variant;
    m.arch = v.arch;
    m.hit_rate = 0.0;
    m.accuracy = 1.0;
    m.lookup_ms = 0.0;
    m.memory_mb = 0.0;
    pd.metrics.push_back(m);
  }
  std::vector<std::size_t> chosen;
  for (int i = 0; i < nv; ++i) chosen.push_back(static_cast<std::size_t>(i));
  pd.dep.model = &model;
  pd.dep.variants = &pd.variants;
  pd.dep.plan = make_plan(chosen, pd.metrics);
  pd.dep.metrics = pd.metrics;
  pd.dep.profile = LayerProfile::uniform(model.num_blocks, 4.0);
  pd.dep.composer.accuracy_threshold = 0.5;
  pd.dep.composer.memory_budget_mb = 0.0;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
void ref_free(void* p) { std::free(p); }

// ------------------------------------------------------------------ models
void* ref_model_make(int input_dim, int classes, const int* widths, int nw, int blocks, uint64_t seed) {
  BaseModel* out = nullptr;
  guard([&] {
    out = new BaseModel(make_base_model(input_dim, classes, std::vector<int>(widths, widths + nw), blocks, seed));
  });
  return out;
}

void* ref_model_load(const char* text) {
  BaseModel* out = nullptr;
  guard([&] {
    std::istringstream in(text);
    out = new BaseModel(load_base_model(in));
  });
  return out;
}

char* ref_model_save(void* m) {
  std::ostringstream out;
  save_base_model(out, *static_cast<BaseModel*>(m));
  return dup_string(out.str());
}

void ref_model_free(void* m) { delete static_cast<BaseModel*>(m); }

int ref_model_info(void* mp, int* blocks, int* classes, int* input_dim, int* tap_dims) {
  const BaseModel& m = *static_cast<BaseModel*>(mp);
  *blocks = m.num_blocks;
  *classes = m.num_classes;
  *input_dim = m.input_dim();
  if (tap_dims)
    for (int i = 0; i < m.num_blocks; ++i) tap_dims[i] = m.tap_dims[static_cast<std::size_t>(i)];
  return 0;
}

// ------------------------------------------------------------------ variants
void* ref_variant_build(int layer, int vidx, const char* arch, int tap_dim, int classes, uint64_t seed) {
  CacheVariant* out = nullptr;
  guard([&] { out = new CacheVariant(build_variant(layer, vidx, ArchSpec::parse(arch), tap_dim, classes, seed)); });
  return out;
}

void* ref_variant_load(const char* text) {
  CacheVariant* out = nullptr;
  guard([&] {
    std::istringstream in(text);
    out = new CacheVariant(load_variant(in));
  });
  return out;
}

char* ref_variant_save(void* v) {
  std::ostringstream out;
  save_variant(out, *static_cast<CacheVariant*>(v));
  return dup_string(out.str());
}

void ref_variant_free(void* v) { delete static_cast<CacheVariant*>(v); }

int ref_variant_set_delta(void* v, double delta) {
  static_cast<CacheVariant*>(v)->delta = delta;
  return 0;
}

// test_serving.cpp:123-129 force_selector: zero the selector, plant a final bias.
int ref_variant_force_selector(void* vp, double bias) {
  CacheVariant& v = *static_cast<CacheVariant*>(vp);
  for (LayerWeights& lw : v.selector.weights) {
    std::fill(lw.w.data.begin(), lw.w.data.end(), 0.0);
    std::fill(lw.b.data.begin(), lw.b.data.end(), 0.0);
  }
  v.selector.weights.back().b.data.back() = bias;
  return 0;
}

// Selector output layer *= gain, final bias = bias (calibrated synthetic
// deployments; mirrors lc_variant_set_selector_out in the product).
int ref_variant_set_selector_out(void* vp, double gain, double bias) {
  CacheVariant& v = *static_cast<CacheVariant*>(vp);
  LayerWeights& lw = v.selector.weights.back();
  for (double& w : lw.w.data) w *= gain;
  lw.b.data.back() = bias;
  return 0;
}

// Selector logit, the input to sigmoid in lookup (cache.cpp:262).
int ref_selector_logit(void* vp, const double* tap, int D, double* logit) {
  return guard([&] {
    const CacheVariant& v = *static_cast<CacheVariant*>(vp);
    const Tensor pr = softmax(forward(v.predictor, vec_of(tap, D)).output());
    *logit = forward(v.selector, pr).output()[0];
  });
}

// ------------------------------------------------------------------ compute
int ref_forward_taps(void* mp, const double* x, double* taps_concat, double* y) {
  return guard([&] {
    const BaseModel& m = *static_cast<BaseModel*>(mp);
    const TapForward tf = forward_with_taps(m, vec_of(x, m.input_dim()));
    std::size_t off = 0;
    for (const Tensor& t : tf.taps) {
      std::memcpy(taps_concat + off, t.data.data(), t.data.size() * sizeof(double));
      off += t.data.size();
    }
    std::memcpy(y, tf.y.data.data(), tf.y.data.size() * sizeof(double));
  });
}

// Base logits = input of the final Softmax layer (network.hpp:57-60).
int ref_forward_logits(void* mp, const double* x, double* logits) {
  return guard([&] {
    const BaseModel& m = *static_cast<BaseModel*>(mp);
    const ForwardTrace tr = forward(m.net, vec_of(x, m.input_dim()));
    const Tensor& l = tr.activations[tr.activations.size() - 2];
    std::memcpy(logits, l.data.data(), l.data.size() * sizeof(double));
  });
}

int ref_lookup(void* vp, const double* tap, int D, int* hit, double* prob, double* pr, double* logits) {
  return guard([&] {
    const CacheVariant& v = *static_cast<CacheVariant*>(vp);
    const Tensor t = vec_of(tap, D);
    const LookupResult r = lookup(v, t);
    *hit = r.hit ? 1 : 0;
    *prob = r.selector_prob;
    if (pr) std::memcpy(pr, r.pr.data.data(), r.pr.data.size() * sizeof(double));
    if (logits) {
      const Tensor l = forward(v.predictor, t).output();
      std::memcpy(logits, l.data.data(), l.data.size() * sizeof(double));
    }
  });
}

// The reference serve path end to end: simulate_model over B requests whose
// inputs are the rows of `inputs` (request i -> test sample i). Runs on
// `threads` host threads over contiguous request shards (each shard is an
// independent simulate_model call on the shared const deployment).
int ref_simulate(void* mp, void** vars, int nv, const double* inputs, int B, int* hit_layer, int* served, int* base,
                 int threads, double* elapsed_s) {
  return guard([&] {
    const BaseModel& m = *static_cast<BaseModel*>(mp);
    PassThroughDeployment pd;
    make_passthrough(pd, m, vars, nv);
    Dataset data;
    data.num_classes = m.num_classes;
    data.input_dim = m.input_dim();
    data.test.resize(static_cast<std::size_t>(B));
    for (int i = 0; i < B; ++i) {
      data.test[static_cast<std::size_t>(i)].x = vec_of(inputs + static_cast<std::size_t>(i) * m.input_dim(), m.input_dim());
      data.test[static_cast<std::size_t>(i)].label = 0;
    }
    std::vector<Request> stream(static_cast<std::size_t>(B));
    for (int i = 0; i < B; ++i) {
      stream[static_cast<std::size_t>(i)].id = i;
      stream[static_cast<std::size_t>(i)].sample_idx = static_cast<std::size_t>(i);
    }
    const int T = std::max(1, std::min(threads, B));
    std::vector<std::vector<RequestTrace>> parts(static_cast<std::size_t>(T));
    std::vector<std::string> errs(static_cast<std::size_t>(T));
    const auto t0 = std::chrono::steady_clock::now();
    auto work = [&](int k) {
      const int lo = static_cast<int>(static_cast<long long>(B) * k / T);
      const int hi = static_cast<int>(static_cast<long long>(B) * (k + 1) / T);
      std::vector<Request> shard(stream.begin() + lo, stream.begin() + hi);
      try {
        parts[static_cast<std::size_t>(k)] = simulate_model(pd.dep, data, shard);
      } catch (const std::exception& e) {
        errs[static_cast<std::size_t>(k)] = e.what();
      }
    };
    if (T == 1) {
      work(0);
    } else {
      std::vector<std::thread> pool;
      for (int k = 0; k < T; ++k) pool.emplace_back(work, k);
      for (auto& th : pool) th.join();
    }
    const auto t1 = std::chrono::steady_clock::now();
    if (elapsed_s) *elapsed_s = std::chrono::duration<double>(t1 - t0).count();
    for (const auto& e : errs)
      if (!e.empty()) throw std::invalid_argument(e);
    int i = 0;
    for (const auto& part : parts)
      for (const RequestTrace& t : part) {
        hit_layer[i] = t.hit_layer;
        served[i] = t.served_pred;
        base[i] = t.base_pred;
        ++i;
      }
  });
}

// ------------------------------------------------------------------ explore measurement
// measure_metrics (cache.cpp:316-335) and tune_delta (cache.cpp:267-307) of one
// variant over the records collect_taps (cache.cpp:142-154) makes from the rows
// of `inputs` (labels unused by both). counts = {tp, fp, tn, fn}.
int ref_measure_metrics(void* mp, void* vp, const double* inputs, int B, long long* counts, double* hit_rate,
                        double* accuracy) {
  return guard([&] {
    const BaseModel& m = *static_cast<BaseModel*>(mp);
    const CacheVariant& v = *static_cast<CacheVariant*>(vp);
    std::vector<Sample> samples(static_cast<std::size_t>(B));
    for (int i = 0; i < B; ++i)
      samples[static_cast<std::size_t>(i)].x = vec_of(inputs + static_cast<std::size_t>(i) * m.input_dim(), m.input_dim());
    const std::vector<TapRecord> recs = collect_taps(m, samples);
    const VariantMetrics r = measure_metrics(v, recs, CostModel{});
    counts[0] = r.tp;
    counts[1] = r.fp;
    counts[2] = r.tn;
    counts[3] = r.fn;
    *hit_rate = r.hit_rate;
    *accuracy = r.accuracy;
  });
}

int ref_tune_delta(void* mp, void* vp, const double* inputs, int B, double target, const double* grid, int ng,
                   double* delta) {
  return guard([&] {
    const BaseModel& m = *static_cast<BaseModel*>(mp);
    CacheVariant v = *static_cast<CacheVariant*>(vp);
    std::vector<Sample> samples(static_cast<std::size_t>(B));
    for (int i = 0; i < B; ++i)
      samples[static_cast<std::size_t>(i)].x = vec_of(inputs + static_cast<std::size_t>(i) * m.input_dim(), m.input_dim());
    const std::vector<TapRecord> recs = collect_taps(m, samples);
    *delta = tune_delta(v, recs, target, std::vector<double>(grid, grid + ng));
  });
}

// ------------------------------------------------------------------ retraining
// train_predictor / train_selector (cache.cpp:179-257) on a COPY of the
// variant, records built from taps at the variant's layer ([N][D]) and the
// base distributions y ([N][C]); weights may be null (1.0 each). The trained
// copy is returned as a new handle.
std::vector<TapRecord> records_at(const CacheVariant& v, const double* taps, int D, const double* y, int C, int N) {
  std::vector<TapRecord> recs(static_cast<std::size_t>(N));
  for (int n = 0; n < N; ++n) {
    TapRecord& r = recs[static_cast<std::size_t>(n)];
    r.taps.resize(static_cast<std::size_t>(v.layer));
    r.taps.back() = vec_of(taps + static_cast<std::size_t>(n) * D, D);
    r.y = vec_of(y + static_cast<std::size_t>(n) * C, C);
  }
  return recs;
}

void* ref_train(void* vp, int which, const double* taps, int D, const double* y, int C, int N, const double* weights,
                double lr, double momentum, int epochs, int batch, uint64_t seed, double a, double b) {
  void* out = nullptr;
  const int st = guard([&] {
    auto v = std::make_unique<CacheVariant>(*static_cast<CacheVariant*>(vp));
    const std::vector<TapRecord> recs = records_at(*v, taps, D, y, C, N);
    TrainConfig cfg;
    cfg.learning_rate = lr;
    cfg.momentum = momentum;
    cfg.epochs = epochs;
    cfg.batch_size = batch;
    cfg.seed = seed;
    const std::vector<double> w = weights ? std::vector<double>(weights, weights + N) : std::vector<double>();
    if (which == 0)
      train_predictor(*v, recs, cfg, a, b, w);
    else
      train_selector(*v, recs, cfg, a, b, w);
    out = v.release();
  });
  return st == 0 ? out : nullptr;
}

// run_adaptation (serving.cpp:213-340) over a pass-through deployment of the
// given variants; original_train = collect_taps of orig_inputs. cfg8 =
// {sample_rate, window_min, retrain_interval_min, recency_decay,
// mixin_fraction, epochs, learning_rate, retrain_pause_ms}; train4 = {tau,
// beta, w_fp, w_fn}. ev [cap][5] = {interval, time_min, window_size,
// mixin_size, applied}; final_vars receives nv new variant handles.
int ref_run_adaptation(void* mp, void** vars, int nv, const double* inputs, const int* labels, int n_samples,
                       const double* times, const int* sample_idx, int R, const double* cfg8, const double* train4,
                       const double* orig_inputs, int N0, uint64_t seed, int adapt_on, int* hit_layer, int* served,
                       int* base, int* ev_n, double* ev, int ev_cap, void** final_vars) {
  return guard([&] {
    const BaseModel& m = *static_cast<BaseModel*>(mp);
    PassThroughDeployment pd;
    make_passthrough(pd, m, vars, nv);
    Dataset data;
    data.num_classes = m.num_classes;
    data.input_dim = m.input_dim();
    for (int i = 0; i < n_samples; ++i) {
      Sample smp;
      smp.x = vec_of(inputs + static_cast<std::size_t>(i) * m.input_dim(), m.input_dim());
      smp.label = labels[i];
      data.test.push_back(smp);
    }
    std::vector<Request> stream(static_cast<std::size_t>(R));
    for (int i = 0; i < R; ++i) {
      stream[static_cast<std::size_t>(i)].id = i;
      stream[static_cast<std::size_t>(i)].time_min = times[i];
      stream[static_cast<std::size_t>(i)].sample_idx = static_cast<std::size_t>(sample_idx[i]);
      stream[static_cast<std::size_t>(i)].true_class = labels[sample_idx[i]];
    }
    AdaptationConfig cfg;
    cfg.sample_rate = cfg8[0];
    cfg.window_min = cfg8[1];
    cfg.retrain_interval_min = cfg8[2];
    cfg.recency_decay = cfg8[3];
    cfg.mixin_fraction = cfg8[4];
    cfg.epochs = static_cast<int>(cfg8[5]);
    cfg.learning_rate = cfg8[6];
    cfg.retrain_pause_ms = cfg8[7];
    CacheTrainConfig tc;
    tc.tau = train4[0];
    tc.beta = train4[1];
    tc.w_fp = train4[2];
    tc.w_fn = train4[3];
    std::vector<Sample> orig(static_cast<std::size_t>(N0));
    for (int i = 0; i < N0; ++i) orig[static_cast<std::size_t>(i)].x = vec_of(orig_inputs + static_cast<std::size_t>(i) * m.input_dim(), m.input_dim());
    const std::vector<TapRecord> original = collect_taps(m, orig);
    const AdaptationResult res = run_adaptation(pd.dep, data, stream, cfg, tc, original, seed, adapt_on != 0);
    for (int i = 0; i < R; ++i) {
      hit_layer[i] = res.traces[static_cast<std::size_t>(i)].hit_layer;
      served[i] = res.traces[static_cast<std::size_t>(i)].served_pred;
      base[i] = res.traces[static_cast<std::size_t>(i)].base_pred;
    }
    *ev_n = static_cast<int>(res.retrains.size());
    for (int i = 0; i < std::min(ev_cap, *ev_n); ++i) {
      const RetrainEvent& e = res.retrains[static_cast<std::size_t>(i)];
      double* o = ev + static_cast<std::size_t>(i) * 5;
      o[0] = e.interval;
      o[1] = e.time_min;
      o[2] = static_cast<double>(e.window_size);
      o[3] = static_cast<double>(e.mixin_size);
      o[4] = e.applied ? 1.0 : 0.0;
    }
    for (int k = 0; k < nv; ++k) final_vars[k] = new CacheVariant(res.final_variants[static_cast<std::size_t>(k)]);
  });
}

// ------------------------------------------------------------------ pipeline
// Trained deployment in the style of test_acceptance.cpp:69-137: dataset ->
// train_base -> collect_taps -> explore_variants -> compose_relaxed ->
// gen_workload -> simulate_model. Writes the reference's own artifact formats
// into `dir` (model.txt, variant_<k>.txt for the plan's chosen rows in plan
// order, metrics.txt, plan.txt, dataset.txt, traces.txt).
int ref_pipeline(const char* dir, uint64_t seed, int classes, int input_dim, int width, int blocks,
                 const char* menu_csv, int base_epochs, int cache_epochs, double minutes) {
  return guard([&] {
    DatasetSpec ds;
    ds.num_classes = classes;
    ds.input_dim = input_dim;
    ds.samples_per_class = 60;
    ds.separation = 5.0;
    ds.noise_stddev = 1.1;
    ds.seed = mix_seed(seed, 1);
    const Dataset data = gen_dataset(ds);
    BaseModel model = make_base_model(input_dim, classes, {width}, blocks, mix_seed(seed, 2));
    TrainConfig bc;
    bc.learning_rate = 0.02;
    bc.epochs = base_epochs;
    bc.seed = mix_seed(seed, 3);
    train_base(model, data, bc);
    const LayerProfile profile = LayerProfile::uniform(blocks, 4.0);
    const CacheData split = split_cache_data(collect_taps(model, data.val), 0.7, mix_seed(seed, 4));
    std::vector<ArchSpec> menu;
    {
      std::string s(menu_csv), tok;
      std::istringstream ss(s);
      while (std::getline(ss, tok, ';'))
        if (!tok.empty()) menu.push_back(ArchSpec::parse(tok));
    }
    CacheTrainConfig cc;
    cc.predictor.epochs = cache_epochs;
    cc.selector.epochs = cache_epochs;
    const CostModel cost;
    const ExploreResult ex = explore_variants(model, split, menu, cc, cost, mix_seed(seed, 5), 1);
    ComposerConfig comp;
    comp.accuracy_threshold = 0.97;
    comp.memory_budget_mb = 64.0;
    comp.alpha = 0.2;
    const SelectionPlan plan = compose_relaxed(ex.metrics, profile, comp);
    WorkloadSpec w;
    w.num_classes = classes;
    w.duration_min = minutes;
    w.seed = mix_seed(seed, 6);
    const std::vector<Request> stream = gen_workload(w, data);
    const Deployment dep{&model, &ex.variants, plan, ex.metrics, profile, cost, comp};
    const std::vector<RequestTrace> traces = simulate_model(dep, data, stream);

    const std::string d(dir);
    auto write = [&](const std::string& name, const std::string& body) {
      std::ofstream f(d + "/" + name);
      if (!f) throw std::runtime_error("cannot write " + d + "/" + name);
      f << body;
    };
    {
      std::ostringstream o;
      save_base_model(o, model);
      write("model.txt", o.str());
    }
    for (std::size_t k = 0; k < plan.chosen.size(); ++k) {
      std::ostringstream o;
      save_variant(o, ex.variants[plan.chosen[k]]);
      write("variant_" + std::to_string(k) + ".txt", o.str());
    }
    {
      std::ostringstream o;
      save_metrics(o, ex.metrics);
      write("metrics.txt", o.str());
    }
    {
      std::ostringstream o;
      save_plan(o, plan, ex.metrics);
      write("plan.txt", o.str());
    }
    {
      std::ostringstream o;
      save_dataset(o, data);
      write("dataset.txt", o.str());
    }
    {
      std::ostringstream o;
      save_traces(o, traces);
      write("traces.txt", o.str());
      std::ostringstream r;
      for (const Request& q : stream) r << q.id << ' ' << q.sample_idx << '\n';
      write("requests.txt", r.str());
    }
    {
      std::ostringstream o;
      save_summary(o, summarize(traces, profile));
      write("summary.txt", o.str());
    }
  });
}

// gen_workload (serving.cpp:61) over a dataset file: writes sample indices and
// true classes so the product's restatement can be pinned.
int ref_gen_workload(const char* dataset_text, int classes, double alpha, double period, double rps, double minutes,
                     uint64_t seed, long long* n_out, long long* sample_idx, int* true_class, long long cap) {
  return guard([&] {
    std::istringstream in(dataset_text);
    const Dataset data = load_dataset(in);
    WorkloadSpec w;
    w.num_classes = classes;
    w.zipf_alpha = alpha;
    w.rotation_period_min = period;
    w.requests_per_sec = rps;
    w.duration_min = minutes;
    w.seed = seed;
    const std::vector<Request> s = gen_workload(w, data);
    *n_out = static_cast<long long>(s.size());
    for (long long i = 0; i < static_cast<long long>(s.size()) && i < cap; ++i) {
      sample_idx[i] = static_cast<long long>(s[static_cast<std::size_t>(i)].sample_idx);
      true_class[i] = s[static_cast<std::size_t>(i)].true_class;
    }
  });
}

// Raw RNG streams (rng.hpp) for pinning the product's restatement.
int ref_rng_stream(uint64_t seed, int kind, int n, double* out_d, uint64_t* out_u) {
  Rng r(seed);
  for (int i = 0; i < n; ++i) {
    if (kind == 0) out_u[i] = r.next_u64();
    else if (kind == 1) out_d[i] = r.next_double();
    else out_d[i] = r.normal();
  }
  return 0;
}
uint64_t ref_mix_seed(uint64_t seed, uint64_t tag) { return mix_seed(seed, tag); }

}  // extern "C"
