"""Online adaptation (§8f rank 3) measurement: retrain parity/latency and the
run_adaptation loop, GPU vs the compiled reference (oracle/_ref) on this host.

  python tools/adapt_bench.py > gpurun_out/adapt_bench.json
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2101_07344_b200 as lcb  # noqa: E402
from oracle import oracle as O  # noqa: E402
from tests.helpers import GOLDEN  # noqa: E402


def load_trained():
    d = os.path.join(GOLDEN, "trained")
    model_txt = open(os.path.join(d, "model.txt")).read()
    vtxt = []
    k = 0
    while os.path.exists(os.path.join(d, f"variant_{k}.txt")):
        vtxt.append(open(os.path.join(d, f"variant_{k}.txt")).read())
        k += 1
    test = [l.split() for l in open(os.path.join(d, "dataset.txt")).read().split("\n") if l.startswith("test ")]
    X = np.array([[float(v) for v in t[2:]] for t in test])
    labels = np.array([int(t[1]) for t in test], np.int32)
    reqs = [tuple(map(int, l.split())) for l in open(os.path.join(d, "requests.txt")).read().split("\n") if l]
    return model_txt, vtxt, X, labels, reqs


def net_err(a_txt, b_txt):
    out = {}
    for which in ("predictor", "selector"):
        e = 0.0
        for a, b in zip(O.parse_variant(a_txt)[which], O.parse_variant(b_txt)[which]):
            if a["w"] is None:
                continue
            for k in ("w", "b"):
                e = max(e, float(np.max(np.abs(a[k] - b[k]))) / max(1.0, float(np.max(np.abs(b[k])))))
        out[which] = e
    return out


def records(rm, X, layer):
    taps, ys = [], []
    for x in X:
        t, y = rm.forward_taps(x)
        taps.append(t[layer - 1])
        ys.append(y)
    return np.array(taps), np.array(ys)


def main():
    model_txt, vtxt, X, labels, reqs = load_trained()
    rm = O.RefModel.load(model_txt)
    out = {"retrain": [], "adaptation": {}}
    # ---- retrain parity + latency per family on window-sized record sets
    for k in (0, 1):
        for N in (150, 2000):
            xs = X[np.arange(N) % len(X)]
            v = lcb.load_variant(vtxt[k])
            rv = O.RefVariant.load(vtxt[k])
            taps, y = records(rm, xs, v.layer)
            cfg = lcb.TrainConfig(learning_rate=0.002, epochs=5, batch_size=16, seed=9)
            lcb.train_predictor(v, taps[:16], y[:16], cfg)  # warm-up (context, module load)
            v = lcb.load_variant(vtxt[k])
            t0 = time.perf_counter()
            lcb.train_predictor(v, taps, y, cfg)
            lcb.train_selector(v, taps, y, cfg)
            gpu_s = time.perf_counter() - t0
            t0 = time.perf_counter()
            rp = O.ref_train(rv, "predictor", taps, y, lr=0.002, epochs=5, batch=16, seed=9, a=2.0, b=0.5)
            rs = O.ref_train(rp, "selector", taps, y, lr=0.002, epochs=5, batch=16, seed=9, a=5.0, b=1.0)
            ref_s = time.perf_counter() - t0
            out["retrain"].append({"variant": vtxt[k].split("\n")[1], "records": N, "epochs": 5,
                                   "gpu_ms": gpu_s * 1e3, "reference_cpu_ms": ref_s * 1e3,
                                   "max_rel_err": net_err(v.save(), rs.save())})
    # ---- a CNN-sized cache retrain (GPU only; the tap dim of a ResNet-18 layer-2 tap)
    D, C, N = 32768, 10, 2000
    v = lcb.build_variant(3, 0, "FC(1024)", D, C, 7)
    rng = np.random.default_rng(1)
    taps = rng.standard_normal((N, D)).astype(np.float64)
    y = rng.dirichlet(np.ones(C), N)
    cfg = lcb.TrainConfig(learning_rate=0.002, epochs=5, batch_size=16, seed=9)
    lcb.train_predictor(v, taps[:16], y[:16], cfg)
    t0 = time.perf_counter()
    lcb.train_predictor(v, taps, y, cfg)
    lcb.train_selector(v, taps, y, cfg)
    out["retrain_fc1024_d32768"] = {"records": N, "epochs": 5, "gpu_ms": (time.perf_counter() - t0) * 1e3,
                                    "params": 1024 * D + 1024 + 1024 * C + C}
    # ---- run_adaptation vs the reference loop
    n_req, minutes = 3000, 60.0
    times = np.sort(np.random.default_rng(11).uniform(0.0, minutes, n_req))
    samp = np.array([reqs[i % len(reqs)][1] for i in range(n_req)], np.int32)
    sel = list(range(len(vtxt)))
    m = lcb.load_base_model(model_txt)
    DELTA = 0.995  # a strict threshold so the stream mixes hits and misses

    def ours(k):
        v = lcb.load_variant(vtxt[k])
        v.delta = DELTA
        return v

    vs = [ours(k) for k in sel]
    dep = lcb.Deployment(m, vs, precision="bf16x3", max_batch=256)
    rvs = [O.RefVariant.load(vtxt[k]) for k in sel]
    for rv in rvs:
        rv.set_delta(DELTA)
    orig_x = X[-200:]
    otaps = []
    for v in vs:
        t, oy = records(rm, orig_x, v.layer)
        otaps.append(t)
    cfg = lcb.AdaptationConfig(sample_rate=0.2, window_min=60.0, retrain_interval_min=15.0, epochs=5,
                               learning_rate=0.002)
    stream = [lcb.Request(i, float(times[i]), int(labels[samp[i]]), int(samp[i])) for i in range(n_req)]
    lcb.run_adaptation(dep, X, labels, stream, cfg, otaps, oy, seed=5, adapt_on=True)  # warm-up (all paths)
    dep.close()
    dep = lcb.Deployment(m, [ours(k) for k in sel], precision="bf16x3", max_batch=256)
    t0 = time.perf_counter()
    res = lcb.run_adaptation(dep, X, labels, stream, cfg, otaps, oy, seed=5, adapt_on=True)
    gpu_s = time.perf_counter() - t0
    cfg8 = [cfg.sample_rate, cfg.window_min, cfg.retrain_interval_min, cfg.recency_decay, cfg.mixin_fraction,
            cfg.epochs, cfg.learning_rate, cfg.retrain_pause_ms]
    t0 = time.perf_counter()
    hl, sv, bp, ev, finals = O.ref_run_adaptation(rm, rvs, X, labels, times, samp, cfg8,
                                                   [cfg.tau, cfg.beta, cfg.w_fp, cfg.w_fn], orig_x, 5, True)
    ref_s = time.perf_counter() - t0
    ohl = np.array([t.hit_layer for t in res.traces])
    osv = np.array([t.served_pred for t in res.traces])
    out["adaptation"] = {
        "requests": n_req, "caches": len(sel), "retrains": len(res.retrains),
        "schedule_identical": all((e.interval, e.window_size, e.mixin_size, int(e.applied)) ==
                                  (int(r[0]), int(r[2]), int(r[3]), int(r[4])) for e, r in zip(res.retrains, ev))
        and len(ev) == len(res.retrains),
        "hit_layer_agreement": float(np.mean(ohl == hl)), "served_agreement": float(np.mean(osv == sv)),
        "hit_rate": float(np.mean(ohl > 0)), "reference_hit_rate": float(np.mean(hl > 0)),
        "final_max_rel_err": max(max(net_err(a.save(), b.save()).values()) for a, b in zip(res.final_variants,
                                                                                          finals)),
        "gpu_wall_ms": gpu_s * 1e3, "reference_cpu_wall_ms": ref_s * 1e3,
        "timeline": [(s.interval, s.requests, s.hits) for s in res.timeline],
    }
    print(json.dumps(out))


if __name__ == "__main__":
    main()
