"""Parity tests proper (need a B200): the CUDA serve path through the C-ABI
against the CPU oracle, which tests/test_oracle.py pins bit-exactly to the
compiled reference and its golden fixtures.

Contract (north_star / SURVEY §8c), written here as code:
  * selector probabilities / logits / pr within 1e-3 relative
    (close_rel: |a-b| <= tol * max(1, |a|, |b|), test_util.hpp:19-22);
  * exit layer and served label bit-exact, except requests whose oracle
    selector probability lies within BAND = 1e-4 of delta at any probed layer
    (reported separately) and label near-ties (top-2 gap < 1e-4);
  * base prediction bit-exact where computed (shadow mode: all requests).
Precision tier under test: bf16x3 (fp32-class). The bf16 tier is reported
as an agreement rate with its own, looser bound.
"""
import json
import os

import numpy as np
import pytest

from tests.helpers import GOLDEN, have_gpu, requires_ref

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not have_gpu(), reason="needs a B200")]

import paper_2101_07344_b200 as lcb  # noqa: E402
from paper_2101_07344_b200.synthetic import (C1_MENU, C1_WIDTHS, calibrate_variants, image_inputs,  # noqa: E402
                                             mlp_inputs)

O = pytest.importorskip("oracle.oracle")

TOL = 1e-3
BAND = 1e-4
GAP = 1e-4


def close_rel(a, b, tol=TOL):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return np.abs(a - b) <= tol * np.maximum(1.0, np.maximum(np.abs(a), np.abs(b)))


def in_band(probs_o, exit_o, deltas):
    """probs_o [B][L] oracle probs (NaN = unprobed); a request is in band if any
    probed layer up to its oracle exit has |p - delta| < BAND."""
    B, L = probs_o.shape
    band = np.zeros(B, bool)
    for i in range(B):
        last = exit_o[i] if exit_o[i] > 0 else L
        for l in range(1, last + 1):
            p = probs_o[i, l - 1]
            if not np.isnan(p) and abs(p - deltas.get(l, 0.5)) < BAND:
                band[i] = True
    return band


def compare_serve(res, exit_o, served_o, base_o, probs_o, deltas, shadow, label_gap=None):
    band = in_band(probs_o, exit_o, deltas)
    ok = ~band
    if label_gap is not None:
        ok &= ~label_gap
    assert np.array_equal(res.exit_layer[ok], exit_o[ok]), (
        f"exit mismatch on {np.sum(res.exit_layer[ok] != exit_o[ok])} of {ok.sum()} requests")
    assert np.array_equal(res.served[ok], served_o[ok])
    if shadow:
        assert np.array_equal(res.base_pred[ok], base_o[ok])
    else:
        miss = ok & (exit_o == 0)
        assert np.array_equal(res.base_pred[miss], base_o[miss])
    # probabilities at every layer the reference probes (ascending, up to the exit)
    L = probs_o.shape[1]
    last = np.where(exit_o > 0, exit_o, L)
    probed = ~np.isnan(probs_o) & (np.arange(1, L + 1)[None, :] <= last[:, None])
    gp = res.probs.T  # [B][L]
    assert np.all(close_rel(gp[probed & ok[:, None]], probs_o[probed & ok[:, None]]))
    return int(band.sum())


# ------------------------------------------------------------------ MLP tier (reference family)
def _load_trained():
    d = os.path.join(GOLDEN, "trained")
    model_txt = open(os.path.join(d, "model.txt")).read()
    vtxt = []
    k = 0
    while os.path.exists(os.path.join(d, f"variant_{k}.txt")):
        vtxt.append(open(os.path.join(d, f"variant_{k}.txt")).read())
        k += 1
    test = [l.split() for l in open(os.path.join(d, "dataset.txt")).read().split("\n") if l.startswith("test ")]
    X = np.array([[float(v) for v in t[2:]] for t in test])
    reqs = [tuple(map(int, l.split())) for l in open(os.path.join(d, "requests.txt")).read().split("\n") if l]
    traces = [l.split() for l in open(os.path.join(d, "traces.txt")).read().split("\n")[1:]
              if l and not l.startswith("#")]
    return model_txt, vtxt, X, reqs, traces


@pytest.mark.parametrize("shadow", [True, False])
def test_golden_trained_deployment(shadow):
    """The reference's own trained deployment + traces (tests/golden/trained)."""
    model_txt, vtxt, X, reqs, traces = _load_trained()
    m = lcb.load_base_model(model_txt)
    vs = [lcb.load_variant(t) for t in vtxt]
    dep = lcb.Deployment(m, vs, precision="bf16x3", max_batch=4096)
    idx = np.array([s for _, s in reqs])
    res = dep.serve(X[idx], shadow=shadow)
    exit_ref = np.array([int(t[5]) for t in traces])
    served_ref = np.array([int(t[4]) for t in traces])
    base_ref = np.array([int(t[3]) for t in traces])
    model = O.parse_model(model_txt)
    caches = []
    for t in vtxt:
        meta = O.parse_variant(t)
        caches.append((meta["layer"], meta["predictor"], meta["selector"], meta["delta"]))
    el, sv, bp, probs = O.oracle_serve_mlp(model, caches, X[idx])
    assert np.array_equal(el, exit_ref) and np.array_equal(sv, served_ref)
    deltas = {c[0]: c[3] for c in caches}
    nb = compare_serve(res, exit_ref, served_ref, base_ref, probs, deltas, shadow)
    assert nb <= 0.01 * len(idx)


@pytest.mark.parametrize("delta", [0.9, 0.99, 0.999])
def test_trained_deployment_threshold_sweep(delta):
    """Same deployment with raised thresholds so requests exit at every layer
    (the C4 confidence-threshold sweep on the reference family)."""
    model_txt, vtxt, X, reqs, _ = _load_trained()
    m = lcb.load_base_model(model_txt)
    vs = [lcb.load_variant(t) for t in vtxt]
    for v in vs:
        v.delta = delta
    dep = lcb.Deployment(m, vs, precision="bf16x3", max_batch=1024)
    x = X[:1024] if len(X) >= 1024 else X
    res = dep.serve(x, shadow=False)
    model = O.parse_model(model_txt)
    caches = []
    for t in vtxt:
        meta = O.parse_variant(t)
        caches.append((meta["layer"], meta["predictor"], meta["selector"], delta))
    el, sv, bp, probs = O.oracle_serve_mlp(model, caches, x)
    compare_serve(res, el, sv, bp, probs, {c[0]: delta for c in caches}, shadow=False)
    # the compacted run agrees with the shadow run on every decision
    sh = dep.serve(x, shadow=True)
    assert np.array_equal(sh.exit_layer, res.exit_layer) and np.array_equal(sh.served, res.served)


def test_golden_c1_config():
    """C1 reference config (3072-input block MLP, ResNet-18 stage widths, a
    cache after every block from all three families)."""
    spec = json.load(open(os.path.join(GOLDEN, "c1", "c1.json")))
    m = lcb.make_base_model(spec["input_dim"], spec["classes"], spec["widths"], spec["blocks"], spec["model_seed"])
    vs = []
    for l in range(spec["blocks"]):
        v = lcb.build_variant(l + 1, l, spec["menu"][l], m.tap_dim(l + 1), spec["classes"], spec["cache_seed"])
        v.set_selector_out(spec["gains"][str(l + 1)], spec["biases"][str(l + 1)])
        v.delta = spec["delta"]
        vs.append(v)
    x = mlp_inputs(spec["n"], spec["input_dim"], spec["input_seed"])
    probs_o = np.array(spec["probs"])
    exit_o, served_o, base_o = (np.array(spec[k]) for k in ("exit_layer", "served", "base"))
    deltas = {l + 1: spec["delta"] for l in range(spec["blocks"])}
    for shadow in (True, False):
        dep = lcb.Deployment(m, vs, precision="bf16x3", max_batch=128)
        res = dep.serve(x, shadow=shadow)
        compare_serve(res, exit_o, served_o, base_o, probs_o, deltas, shadow)
        dep.close()


@pytest.mark.parametrize("arch", ["FC(1024)", "FC(32)", "Pool(16)", "Pool(8192)", "Conv(3,1)", "Conv(5,2)"])
def test_lookup_mlp_taps(arch):
    m = lcb.make_base_model(64, 10, [96], 2, 5)
    v = lcb.build_variant(2, 0, arch, 96, 10, 11)
    v.set_selector_out(30.0, 0.0)
    dep = lcb.Deployment(m, [v], max_batch=64)
    taps = np.random.default_rng(1).uniform(-1.5, 1.5, (64, 96))
    got = dep.lookup(2, taps)
    pred, sel, d = O.variant_layers_from_product(v)
    pn, sn = O.OracleNet(pred), O.OracleNet(sel)
    for i in range(64):
        hit, p, pr, lg = O.oracle_lookup(pn, sn, d, taps[i])
        assert close_rel(got["prob"][i], p)
        assert np.all(close_rel(got["pr"][i], pr)) and np.all(close_rel(got["logits"][i], lg))
        if abs(p - d) >= BAND:
            assert bool(got["hit"][i]) == hit
        top = np.sort(pr)[::-1]
        if top[0] - top[1] >= GAP:
            assert got["label"][i] == O.argmax(pr)


@pytest.mark.parametrize("heads", ["auto", "warp"])
@pytest.mark.parametrize("classes,widths", [(10, [64, 128, 64]), (100, [96, 100, 64])])
def test_mlp_direct_heads_vs_oracle(classes, widths, heads, monkeypatch):
    """Block-MLP serving where the heads read the request's row themselves
    (Pool(w) / Conv(k,s) predictor inside the head, static weights staged
    before the programmatic-launch wait, the row held in registers for the
    compacted copy) and the FC(h) head, against the oracle's serve_one, in
    shadow and compact mode: 10 classes (direct Pool head, 16-byte row
    vectors), and 100 classes with a 100-wide tap (Pool(w) through the
    batched logits GEMM, Conv(k,s) direct with the scalar row path). heads =
    "warp" forces the warp-per-row head kernel (LCB_BLOCK_HEADS=2), which the
    engine otherwise picks only for batch capacities >= 512."""
    if heads == "warp":
        monkeypatch.setenv("LCB_BLOCK_HEADS", "2")
    m = lcb.make_base_model(48, classes, widths, 3, 13)
    archs = ["Pool(32)", "Conv(3,1)", "FC(64)"]
    vs = [lcb.build_variant(l + 1, 0, a, m.tap_dim(l + 1), classes, 17 + l) for l, a in enumerate(archs)]
    for v in vs:
        v.set_selector_out(25.0, 0.0)
    x = mlp_inputs(96, 48, 29)
    model = O.parse_model(m.save())
    metas = [O.parse_variant(v.save()) for v in vs]

    def oracle(ds):
        return O.oracle_serve_mlp(model, [(mt["layer"], mt["predictor"], mt["selector"], d) for mt, d in zip(metas, ds)], x)

    # thresholds at quantiles of the oracle's selector probabilities (no exits
    # at delta 2): about a quarter of the requests exit at each cache
    probs_all = oracle([2.0] * 3)[3]
    ds = [float(np.quantile(probs_all[:, l], q)) for l, q in enumerate((0.75, 0.7, 0.6))]
    for v, d in zip(vs, ds):
        v.delta = d
    el, sv, bp, probs = oracle(ds)
    assert np.all(np.bincount(el, minlength=4) >= 10)  # requests exit at every cache and at the end
    deltas = {mt["layer"]: d for mt, d in zip(metas, ds)}
    dep = lcb.Deployment(m, vs, precision="bf16x3", max_batch=128)
    for shadow in (True, False):
        res = dep.serve(x, shadow=shadow)
        compare_serve(res, el, sv, bp, probs, deltas, shadow)
    dep.close()


def test_inclusive_threshold_on_gpu():
    # test_cache.cpp:218-227 on the device: zeroed selector -> prob exactly 0.5
    m = lcb.make_base_model(4, 3, [4], 1, 1)
    v = lcb.build_variant(1, 0, "FC(8)", 4, 3, 9)
    v.set_selector_out(0.0, 0.0)
    dep = lcb.Deployment(m, [v], max_batch=4)
    tap = np.array([[0.3, -0.1, 0.2, 0.0]])
    r = dep.lookup(1, tap)
    assert r["prob"][0] == 0.5 and r["hit"][0] == 1
    dep.set_delta(1, 0.5000000001)
    assert dep.lookup(1, tap)["hit"][0] == 0


def test_errors_are_reference_typed():
    m = lcb.make_base_model(16, 10, [64], 3, 1)
    v1 = lcb.build_variant(2, 0, "Pool(16)", 64, 10, 1)
    v2 = lcb.build_variant(2, 1, "FC(32)", 64, 10, 1)
    with pytest.raises(ValueError, match="more than one variant at layer 2"):
        lcb.Deployment(m, [v1, v2], max_batch=8)
    bad = lcb.build_variant(2, 0, "Pool(16)", 32, 10, 1)  # wrong tap dim
    with pytest.raises(ValueError):
        lcb.Deployment(m, [bad], max_batch=8)
    dep = lcb.Deployment(m, [v1], max_batch=8)
    with pytest.raises(ValueError):
        dep.serve(np.zeros((9, 16), np.float32))
    with pytest.raises(ValueError):
        dep.lookup(1, np.zeros((2, 64)))  # no cache at layer 1


def test_graph_and_direct_launch_identical():
    spec = json.load(open(os.path.join(GOLDEN, "c1", "c1.json")))
    m = lcb.make_base_model(3072, 10, C1_WIDTHS, 8, spec["model_seed"])
    vs = []
    for l in range(8):
        v = lcb.build_variant(l + 1, l, C1_MENU[l], m.tap_dim(l + 1), 10, spec["cache_seed"])
        v.set_selector_out(spec["gains"][str(l + 1)], spec["biases"][str(l + 1)])
        vs.append(v)
    dep = lcb.Deployment(m, vs, max_batch=128)
    x = mlp_inputs(128, 3072, 3)
    a = dep.serve(x, graph=True)
    b = dep.serve(x, graph=False)
    c = dep.serve(x, graph=True)
    for r in (b, c):
        assert np.array_equal(a.exit_layer, r.exit_layer) and np.array_equal(a.served, r.served)
        assert np.array_equal(a.probs, r.probs, equal_nan=True)


# ------------------------------------------------------------------ CNN tier
def _cnn_deployment(arch, classes, seed, B, precision="bf16x3", cache="Pool", full_fraction=0.2):
    m = lcb.make_cnn_model(arch, classes, seed)
    vs = []
    for l in range(1, m.num_blocks + 1):
        C, H, W = m.tap(l)
        if cache == "FC+Pool":  # BASELINE C4: FC and pool cache models on alternate taps
            a = f"Pool({C})" if l % 2 else "FC(256)"
        else:
            a = f"Pool({C})" if cache == "Pool" else cache
        vs.append(lcb.build_variant(l, 0, a, m.tap_dim(l), classes, seed + l))
    side = 32 if arch.endswith("cifar") else 224
    calib = image_inputs(B, 3, side, side, seed=seed + 100)
    calibrate_variants(m, vs, calib, full_fraction, precision=precision)
    return m, vs


def _oracle_cnn(m, vs, x, threads=8):
    ops = m.cnn_ops()
    taps, logits = O.oracle_cnn_forward(ops, m.nslots, x, m.num_blocks, m.tap_dims, m.num_classes, threads=threads)
    B = x.shape[0]
    L = m.num_blocks
    nets = {}
    for v in vs:
        pred, sel, d = O.variant_layers_from_product(v)
        nets[v.layer] = (O.OracleNet(pred), O.OracleNet(sel), d)
    exit_o = np.zeros(B, int)
    served = np.zeros(B, int)
    base = np.array([O.argmax(O.softmax(logits[i])) for i in range(B)])
    probs = np.full((B, L), np.nan)
    gaps = np.zeros(B, bool)
    for i in range(B):
        top = np.sort(O.softmax(logits[i]))[::-1]
        gaps[i] |= top[0] - top[1] < GAP
        served[i] = base[i]
        for l in sorted(nets):
            pn, sn, d = nets[l]
            hit, p, pr, _ = O.oracle_lookup(pn, sn, d, taps[l - 1][i])
            probs[i, l - 1] = p
            if hit:
                exit_o[i] = l
                served[i] = O.argmax(pr)
                t2 = np.sort(pr)[::-1]
                gaps[i] |= t2[0] - t2[1] < GAP
                break
    return exit_o, served, base, probs, gaps, taps, logits


@pytest.mark.parametrize("shadow", [True, False])
def test_resnet18_cifar_serve_vs_oracle(shadow):
    m, vs = _cnn_deployment("resnet18_cifar", 10, 21, 64)
    x = image_inputs(24, 3, 32, 32, seed=5)
    dep = lcb.Deployment(m, vs, precision="bf16x3", max_batch=32)
    res = dep.serve(x, shadow=shadow)
    exit_o, served_o, base_o, probs_o, gaps, _, _ = _oracle_cnn(m, vs, x)
    deltas = {v.layer: v.delta for v in vs}
    compare_serve(res, exit_o, served_o, base_o, probs_o, deltas, shadow, label_gap=gaps)
    assert len(set(exit_o.tolist())) >= 3  # exits spread over several layers


def test_ragged_batches_vs_oracle():
    """One engine (max_batch 256) serving ragged batch sizes — 1, 7, 129 (one
    past a 128-row tile), 256 (the maximum) — in compact and shadow mode
    against the oracle; a request's decisions do not depend on the batch it
    rides in (the captured graph is batch-size agnostic: every size lives in
    device memory; only the split-K degree of the deep layers follows the
    survivor count, so probabilities agree within the parity tolerance, not
    bit for bit: measured ~1e-4 between a batch of 1 and of 256); sizes 0
    and max_batch + 1 are rejected like the reference's invalid_argument."""
    m, vs = _cnn_deployment("resnet18_cifar", 10, 21, 64)
    dep = lcb.Deployment(m, vs, precision="bf16x3", max_batch=256)
    deltas = {v.layer: v.delta for v in vs}
    x = image_inputs(256, 3, 32, 32, seed=77)
    exit_o, served_o, base_o, probs_o, gaps, _, _ = _oracle_cnn(m, vs, x, threads=os.cpu_count() or 8)
    full = {sh: dep.serve(x, shadow=sh) for sh in (True, False)}
    for B in (1, 7, 129, 256):
        for shadow in (True, False):
            res = dep.serve(x[:B], shadow=shadow)
            compare_serve(res, exit_o[:B], served_o[:B], base_o[:B], probs_o[:B], deltas, shadow, label_gap=gaps[:B])
            f = full[shadow]
            ok = ~(in_band(probs_o[:B], exit_o[:B], deltas) | gaps[:B])
            assert np.array_equal(res.exit_layer[ok], f.exit_layer[:B][ok])
            assert np.array_equal(res.served[ok], f.served[:B][ok])
            both = ~np.isnan(res.probs) & ~np.isnan(f.probs[:, :B])
            assert np.array_equal(both, ~np.isnan(res.probs))
            assert np.all(close_rel(res.probs[both], f.probs[:, :B][both]))
    for bad in (0, 257):
        with pytest.raises(ValueError):
            dep.serve(np.zeros((bad, 3 * 32 * 32), np.float32), shadow=False)
    dep.close()


@pytest.mark.parametrize("shadow", [True, False])
@pytest.mark.parametrize("mode", ["post", "tile"])
def test_conv_head_opt_in_vs_oracle(shadow, mode, monkeypatch):
    """Opt-in variant (LCB_NO_CONV_HEAD=0): the tap conv finishes each row's
    lookup (GAP sum, head, selector, threshold) — after a grid barrier that
    follows its last tile (post) or from the CTA finishing the row's last tile
    (tile) — and the last head runs the first-hit exit + compaction. Slower
    than the separate head launch today (profiles/r02_fused_head_ab.txt) but
    kept correct."""
    monkeypatch.setenv("LCB_NO_CONV_HEAD", "0")
    monkeypatch.setenv("LCB_CONV_HEAD_TILE", "1" if mode == "tile" else "0")
    m, vs = _cnn_deployment("resnet18_cifar", 10, 21, 64)
    x = image_inputs(24, 3, 32, 32, seed=5)
    dep = lcb.Deployment(m, vs, precision="bf16x3", max_batch=32)
    res = dep.serve(x, shadow=shadow)
    exit_o, served_o, base_o, probs_o, gaps, _, _ = _oracle_cnn(m, vs, x)
    deltas = {v.layer: v.delta for v in vs}
    compare_serve(res, exit_o, served_o, base_o, probs_o, deltas, shadow, label_gap=gaps)
    dep.close()


def test_fused_gap_matches_unfused_pool(monkeypatch):
    """Pool(C) caches read GAP partials written by the tap conv's epilogue;
    the unfused path (LCB_NO_GAP_FUSION=1) pools the stored tap instead. Both
    must agree on every decision and to fp32 rounding on the probabilities."""
    m, vs = _cnn_deployment("resnet18_cifar", 10, 21, 64)
    x = image_inputs(32, 3, 32, 32, seed=8)
    fused = lcb.Deployment(m, vs, precision="bf16x3", max_batch=32)
    monkeypatch.setenv("LCB_NO_GAP_FUSION", "1")
    plain = lcb.Deployment(m, vs, precision="bf16x3", max_batch=32)
    for shadow in (True, False):
        a, b = fused.serve(x, shadow=shadow), plain.serve(x, shadow=shadow)
        assert np.array_equal(a.exit_layer, b.exit_layer) and np.array_equal(a.served, b.served)
        both = ~np.isnan(a.probs) & ~np.isnan(b.probs)
        assert np.array_equal(np.isnan(a.probs), np.isnan(b.probs))
        # the fused partials sum the fp32 epilogue values, the unfused pool the
        # stored hi+lo planes (~2^-17 apart); calibrated selector gains amplify it
        assert np.all(np.abs(a.probs[both] - b.probs[both]) <= 1e-4)
    fused.close()
    plain.close()


@pytest.mark.parametrize("fusions", ["default", "unfused"])
def test_resnet50_serve_vs_oracle(fusions, monkeypatch):
    """ImageNet shape (224x224, 1000 classes, 16 bottleneck blocks): stem,
    max-pool, 1x1/3x3/strided convs, fused GAP partials, split-K deep layers
    and the 1000-class lookups, against the fp64 restatement. Both with the
    graph-level fusions (downsample projection as residual K-steps, max-pool
    halves in the stem epilogue) and with them off."""
    if fusions == "unfused":
        monkeypatch.setenv("LCB_NO_PROJ_FUSION", "1")
        monkeypatch.setenv("LCB_NO_STEM_POOL", "1")
    m, vs = _cnn_deployment("resnet50", 1000, 31, 8, full_fraction=0.3)
    x = image_inputs(6, 3, 224, 224, seed=12)
    dep = lcb.Deployment(m, vs, precision="bf16x3", max_batch=8)
    exit_o, served_o, base_o, probs_o, gaps, _, _ = _oracle_cnn(m, vs, x, threads=os.cpu_count() or 8)
    deltas = {v.layer: v.delta for v in vs}
    for shadow in (True, False):
        res = dep.serve(x, shadow=shadow)
        compare_serve(res, exit_o, served_o, base_o, probs_o, deltas, shadow, label_gap=gaps)
    dep.close()


@pytest.mark.parametrize("delta", [0.5, 0.9])
def test_vgg16_fc_pool_caches_vs_oracle(delta):
    """BASELINE C4: VGG-16 CIFAR with FC(256) and Pool(C) cache models on
    alternate pool-stage taps, at two points of the confidence-threshold sweep."""
    m, vs = _cnn_deployment("vgg16_cifar", 10, 41, 64, cache="FC+Pool", full_fraction=0.2)
    for v in vs:
        v.delta = delta
    x = image_inputs(24, 3, 32, 32, seed=14)
    dep = lcb.Deployment(m, vs, precision="bf16x3", max_batch=32)
    exit_o, served_o, base_o, probs_o, gaps, _, _ = _oracle_cnn(m, vs, x)
    deltas = {v.layer: v.delta for v in vs}
    for shadow in (True, False):
        res = dep.serve(x, shadow=shadow)
        compare_serve(res, exit_o, served_o, base_o, probs_o, deltas, shadow, label_gap=gaps)
    dep.close()


def test_resnet152_serve_vs_oracle():
    """BASELINE C5 shape (ResNet-152, 50 bottleneck blocks, 1000 classes) on a
    small batch against the fp64 restatement."""
    m, vs = _cnn_deployment("resnet152", 1000, 51, 4, full_fraction=0.3)
    x = image_inputs(3, 3, 224, 224, seed=15)
    dep = lcb.Deployment(m, vs, precision="bf16x3", max_batch=4)
    exit_o, served_o, base_o, probs_o, gaps, _, _ = _oracle_cnn(m, vs, x, threads=os.cpu_count() or 8)
    deltas = {v.layer: v.delta for v in vs}
    for shadow in (True, False):
        res = dep.serve(x, shadow=shadow)
        compare_serve(res, exit_o, served_o, base_o, probs_o, deltas, shadow, label_gap=gaps)
    dep.close()


def test_resnet18_cnn_lookups_on_oracle_taps():
    """Cache heads of every family on real CNN taps (NCHW-flat from the fp64
    oracle), through the engine's lookup entry point."""
    m = lcb.make_cnn_model("resnet18_cifar", 10, 4)
    x = image_inputs(4, 3, 32, 32, seed=9)
    taps, _ = O.oracle_cnn_forward(m.cnn_ops(), m.nslots, x, m.num_blocks, m.tap_dims, 10, threads=4)
    for layer, arch in [(1, "Pool(64)"), (1, "Pool(8192)"), (2, "Pool(4096)"), (5, "Pool(256)"), (7, "Conv(3,1)"),
                        (8, "Conv(5,2)"), (8, "FC(256)"), (8, "Pool(8192)")]:
        v = lcb.build_variant(layer, 0, arch, m.tap_dim(layer), 10, 17)
        v.set_selector_out(20.0, 0.0)
        dep = lcb.Deployment(m, [v], max_batch=4)
        got = dep.lookup(layer, taps[layer - 1])
        pred, sel, d = O.variant_layers_from_product(v)
        pn, sn = O.OracleNet(pred), O.OracleNet(sel)
        for i in range(4):
            _, p, pr, lg = O.oracle_lookup(pn, sn, d, taps[layer - 1][i])
            assert close_rel(got["prob"][i], p), (layer, arch)
            assert np.all(close_rel(got["logits"][i], lg)), (layer, arch)
        dep.close()


def test_resnet18_bf16_tier_agreement():
    m, vs = _cnn_deployment("resnet18_cifar", 10, 21, 64, precision="bf16")
    x = image_inputs(32, 3, 32, 32, seed=6)
    d3 = lcb.Deployment(m, vs, precision="bf16x3", max_batch=32)
    d1 = lcb.Deployment(m, vs, precision="bf16", max_batch=32)
    a, b = d3.serve(x, shadow=True), d1.serve(x, shadow=True)
    agree = np.mean((a.exit_layer == b.exit_layer) & (a.served == b.served))
    assert agree >= 0.8, (agree, a.exit_layer, b.exit_layer, a.served, b.served)


def test_repeated_serves_bit_identical():
    """Deterministic reductions everywhere (fixed-order split-K, no float
    atomics): repeated serves of the same batch are bit-identical."""
    m, vs = _cnn_deployment("resnet18_cifar", 10, 21, 64)
    x = image_inputs(32, 3, 32, 32, seed=6)
    dep = lcb.Deployment(m, vs, precision="bf16x3", max_batch=32)
    ref = dep.serve(x, shadow=True)
    for _ in range(10):
        for shadow in (True, False):
            r = dep.serve(x, shadow=shadow)
            assert np.array_equal(r.exit_layer, ref.exit_layer) and np.array_equal(r.served, ref.served)
            if shadow:
                assert np.array_equal(r.probs, ref.probs, equal_nan=True)
                assert np.array_equal(r.base_pred, ref.base_pred)


def test_cpp_dropin_against_reference_library():
    """tests/cpp/test_dropin.cpp: the unmodified reference library and the
    B200 façade (include/latecache_b200.hpp) in one C++ binary."""
    import subprocess
    from tests.helpers import ROOT
    exe = os.path.join(ROOT, "oracle", "_ref", "test_dropin")
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref/test_dropin not built (make -C oracle dropin)")
    r = subprocess.run([exe, os.path.join(GOLDEN, "trained")], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "DROPIN OK" in r.stdout, r.stdout + r.stderr


# ------------------------------------------------------------------ explore measurement (§8f rank 1)
@requires_ref
def test_measure_metrics_and_tune_delta_vs_reference():
    """Batched measure_metrics / tune_delta (one shadow serve + confusion counts
    on the GPU) against the reference's per-record loops (cache.cpp:267-335)
    run by oracle/_ref on the same trained deployment and records."""
    model_txt, vtxt, X, _, _ = _load_trained()
    x = X[:512]
    m = lcb.load_base_model(model_txt)
    vs = [lcb.load_variant(t) for t in vtxt]
    dep = lcb.Deployment(m, vs, precision="bf16x3", max_batch=len(x))
    rm = O.RefModel.load(model_txt)
    rvs = [O.RefVariant.load(t) for t in vtxt]
    grid = [0.5, 0.55, 0.6, 0.65, 0.7, 0.75, 0.8, 0.85, 0.9, 0.95]  # cache.hpp:99
    ours = dep.measure_metrics(x, grid)
    sh = dep.serve(x, shadow=True)  # GPU probabilities at every layer: in-band accounting
    for v, rv in zip(vs, rvs):
        for row in ours[v.layer]:
            rv.set_delta(row["delta"])
            ref_c, ref_hr, ref_acc = O.ref_measure_metrics(rm, rv, x)
            p = sh.probs[v.layer - 1]
            band = int(np.sum(np.abs(p.astype(np.float64) - row["delta"]) < BAND))
            diff = sum(abs(row[k] - ref_c[k]) for k in ("tp", "fp", "tn", "fn"))
            assert diff <= 2 * band, (v.layer, row, ref_c, band)
            if diff == 0:
                assert abs(row["hit_rate"] - ref_hr) < 1e-12 and abs(row["accuracy"] - ref_acc) < 1e-12
    for target in (0.8, 0.95, 0.999):
        tuned = dep.tune_delta(x, target, grid, apply=False)
        for v, rv in zip(vs, rvs):
            assert tuned[v.layer] == O.ref_tune_delta(rm, rv, x, target, grid), (v.layer, target)
    # applied thresholds drive the serve path
    tuned = dep.tune_delta(x, 0.95, grid, apply=True)
    res = dep.serve(x)
    for v in vs:
        assert v.delta == tuned[v.layer]
        hit_here = res.exit_layer == v.layer
        assert np.all(sh.probs[v.layer - 1][hit_here] >= tuned[v.layer] - BAND)
    dep.close()


def test_pipelined_submit_collect_matches_serve():
    """The pipelined e2e entry point (two slots in flight, uploads on a copy
    stream) returns exactly what the synchronous serve returns per batch."""
    import torch
    m, vs = _cnn_deployment("resnet18_cifar", 10, 21, 64)
    dep = lcb.Deployment(m, vs, precision="bf16x3", max_batch=32)
    xs = [torch.from_numpy(image_inputs(32, 3, 32, 32, seed=40 + k).astype(np.float32)).pin_memory() for k in range(5)]
    ref = [dep.serve(x.numpy()) for x in xs]
    pending, got = [], []
    for x in xs:
        pending.append(dep.submit(x.numpy()))
        if len(pending) == 2:
            got.append(dep.collect(pending.pop(0)))
    while pending:
        got.append(dep.collect(pending.pop(0)))
    for a, b in zip(ref, got):
        assert np.array_equal(a.exit_layer, b.exit_layer) and np.array_equal(a.served, b.served)
        assert np.array_equal(a.base_pred, b.base_pred)
        assert np.array_equal(a.probs, b.probs, equal_nan=True)
        assert np.all(b.latency_ms >= 0)
    dep.close()


def test_layer_times_hardware_profile():
    """Device-measured LayerProfile + lookup costs (§8f rank 2) on the trained
    deployment and a CNN: positive per-block times, a lookup time at every
    cache layer, and their sum close to the shadow batch's device time."""
    model_txt, vtxt, X, _, _ = _load_trained()
    m = lcb.load_base_model(model_txt)
    vs = [lcb.load_variant(t) for t in vtxt]
    dep = lcb.Deployment(m, vs, precision="bf16x3", max_batch=256)
    block_ms, lookup_ms = dep.layer_times(X[:256])
    assert np.all(block_ms > 0)
    assert set(lookup_ms) == {v.layer for v in vs} and all(t > 0 for t in lookup_ms.values())
    metrics = open(os.path.join(GOLDEN, "trained", "metrics.txt")).read()
    plan = open(os.path.join(GOLDEN, "trained", "plan.txt")).read()
    measured = lcb.with_measured_lookup_ms(metrics, lookup_ms)
    ok, viol, _ = lcb.plan_check(measured, plan, list(block_ms), 0.97, 64.0)
    assert isinstance(ok, bool)
    dep.close()
    cm, cvs = _cnn_deployment("resnet18_cifar", 10, 21, 64)
    cdep = lcb.Deployment(cm, cvs, precision="bf16x3", max_batch=64)
    x = image_inputs(64, 3, 32, 32, seed=3)
    bm, lm = cdep.layer_times(x)
    assert np.all(bm > 0) and all(t > 0 for t in lm.values())
    import torch
    cdep.stage_input_device(torch.from_numpy(x.astype(np.float32)).cuda().data_ptr(), 64)
    total = np.median([cdep.serve_timed(64, shadow=True) for _ in range(5)])
    assert 0.5 * total < bm.sum() + sum(lm.values()) < 1.5 * total, (bm.sum(), sum(lm.values()), total)
    cdep.close()


@pytest.mark.parametrize("cfg", ["resnet18_cifar", "resnet50"])
def test_full_size_invariants(cfg):
    """BASELINE sizes (R18 b256, R50 b128, bench-calibrated selectors), through
    size-independent properties: the compacted serve makes exactly the shadow
    serve's decisions (exit layer, label, probabilities where probed), the
    no-cache engine's base prediction equals the shadow pass's, serves are
    bit-identical run to run, and the pipelined submit/collect path returns the
    synchronous results."""
    import torch
    from bench import CONFIGS, build_deployment
    B = CONFIGS[cfg][3]
    m, vs, dep, base, gen, _ = build_deployment(cfg, B, "bf16x3", 0)
    x = gen(B, 99).astype(np.float32)
    sh = dep.serve(x, shadow=True)
    cp = dep.serve(x)
    assert np.array_equal(cp.exit_layer, sh.exit_layer) and np.array_equal(cp.served, sh.served)
    probed = ~np.isnan(cp.probs)
    # compaction changes the tile grouping / split-K factor of the deeper convs
    # (fp32 summation order), so probabilities agree within the contract's
    # close_rel(1e-3), not bit for bit (calibrated selector gains amplify it)
    assert np.all(close_rel(cp.probs[probed], sh.probs[probed]))
    miss = cp.exit_layer == 0
    assert np.array_equal(cp.base_pred[miss], sh.base_pred[miss])
    nc = base.serve(x)
    assert np.array_equal(nc.base_pred, sh.base_pred) and np.all(nc.exit_layer == 0)
    again = dep.serve(x)
    assert np.array_equal(again.exit_layer, cp.exit_layer) and np.array_equal(again.probs, cp.probs, equal_nan=True)
    pinned = torch.from_numpy(x).pin_memory()
    t = dep.submit(pinned.numpy())
    pr = dep.collect(t)
    assert np.array_equal(pr.exit_layer, cp.exit_layer) and np.array_equal(pr.served, cp.served)
    assert 0.5 < np.mean(cp.exit_layer > 0) <= 1.0  # calibrated selectors: most requests exit early
    dep.close()
    base.close()


# ---------------------------------------------------------------- retraining / online adaptation (§8f rank 3)
def _net_params(text, which):
    return [l for l in O.parse_variant(text)[which] if l["w"] is not None]


def _assert_nets_close(ours_txt, ref_txt, rtol):
    for which in ("predictor", "selector"):
        for a, b in zip(_net_params(ours_txt, which), _net_params(ref_txt, which)):
            for k in ("w", "b"):
                scale = max(1.0, float(np.max(np.abs(b[k]))))
                err = float(np.max(np.abs(a[k] - b[k])))
                assert err <= rtol * scale, (which, k, err, scale)


def _ref_records(rm, X, layer):
    taps, ys = [], []
    for x in X:
        t, y = rm.forward_taps(x)
        taps.append(t[layer - 1])
        ys.append(y)
    return np.array(taps), np.array(ys)


@pytest.mark.parametrize("unfused", [False, True])  # one-block schedule / per-phase kernels in a graph
@pytest.mark.parametrize("k", [0, 1])  # FC(32) at layer 1, Conv(3,1) at layer 2
@requires_ref
def test_train_predictor_selector_vs_reference(k, unfused, monkeypatch):
    """GPU fp64 SGD (train_predictor / train_selector, cache.cpp:179-257)
    against the reference's own functions on the same double records:
    identical schedule (Rng shuffles, batches, weights), weights within
    rounding (tree-ordered forward dots, CUDA exp/log)."""
    if unfused:
        monkeypatch.setenv("LCB_TRAIN_UNFUSED", "1")
    model_txt, vtxt, X, _, _ = _load_trained()
    rm = O.RefModel.load(model_txt)
    v = lcb.load_variant(vtxt[k])
    rv = O.RefVariant.load(vtxt[k])
    taps, y = _ref_records(rm, X[:150], v.layer)
    w = np.random.default_rng(3).uniform(0.2, 1.0, len(taps))
    cfg = lcb.TrainConfig(learning_rate=0.01, epochs=4, batch_size=16, seed=77)
    lcb.train_predictor(v, taps, y, cfg, tau=2.0, beta=0.5, sample_weights=w)
    rp = O.ref_train(rv, "predictor", taps, y, weights=w, lr=0.01, epochs=4, batch=16, seed=77, a=2.0, b=0.5)
    _assert_nets_close(v.save(), rp.save(), 1e-9)
    cfg2 = lcb.TrainConfig(learning_rate=0.02, epochs=3, batch_size=16, seed=78)
    lcb.train_selector(v, taps, y, cfg2, w_fp=5.0, w_fn=1.0)
    rs = O.ref_train(rp, "selector", taps, y, lr=0.02, epochs=3, batch=16, seed=78, a=5.0, b=1.0)
    _assert_nets_close(v.save(), rs.save(), 1e-9)


@requires_ref
def test_train_wide_tap_cache_vs_reference():
    """A CNN-sized tap (4096 features) into FC(64): the split-input forward
    and the 4x2 weight-gradient kernels (not the one-block schedule)."""
    D, C, N = 4096, 10, 48
    v = lcb.build_variant(2, 0, "FC(64)", D, C, 21)
    rv = O.RefVariant.build(2, 0, "FC(64)", D, C, 21)
    rng = np.random.default_rng(5)
    taps = np.maximum(rng.standard_normal((N, D)), 0.0)
    y = rng.dirichlet(np.ones(C), N)
    lcb.train_predictor(v, taps, y, lcb.TrainConfig(learning_rate=0.01, epochs=2, batch_size=16, seed=3))
    rp = O.ref_train(rv, "predictor", taps, y, lr=0.01, epochs=2, batch=16, seed=3, a=2.0, b=0.5)
    _assert_nets_close(v.save(), rp.save(), 1e-9)
    lcb.train_selector(v, taps, y, lcb.TrainConfig(learning_rate=0.02, epochs=2, batch_size=16, seed=4))
    rs = O.ref_train(rp, "selector", taps, y, lr=0.02, epochs=2, batch=16, seed=4, a=5.0, b=1.0)
    _assert_nets_close(v.save(), rs.save(), 1e-9)


def test_train_errors_are_reference_typed():
    """Bad records are invalid_argument (ValueError); a diverging loss is the
    reference's runtime_error (RuntimeError) and leaves the variant as it was."""
    model_txt, vtxt, X, _, _ = _load_trained()
    rm = O.RefModel.load(model_txt)
    v = lcb.load_variant(vtxt[0])
    before = v.save()
    taps, y = _ref_records(rm, X[:32], v.layer)
    with pytest.raises(ValueError):  # tap dimension mismatch
        lcb.train_predictor(v, taps[:, :3], y)
    with pytest.raises(ValueError):  # sample weight count mismatch
        lcb.train_predictor(v, taps, y, sample_weights=[1.0])
    with pytest.raises(RuntimeError, match="diverged"):
        lcb.train_predictor(v, taps * 1e200, y, lcb.TrainConfig(learning_rate=1e200, epochs=2))
    assert v.save() == before


def _adapt_setup(n_req=900, minutes=60.0):
    model_txt, vtxt, X, reqs, _ = _load_trained()
    test = [l.split() for l in open(os.path.join(GOLDEN, "trained", "dataset.txt")).read().split("\n")
            if l.startswith("test ")]
    labels = np.array([int(t[1]) for t in test], np.int32)
    rng = np.random.default_rng(11)
    times = np.sort(rng.uniform(0.0, minutes, n_req))
    samp = np.array([reqs[i % len(reqs)][1] for i in range(n_req)], np.int32)
    return model_txt, vtxt, X, labels, times, samp


@pytest.mark.parametrize("pause_ms", [0.0, 90000.0])
@requires_ref
def test_run_adaptation_vs_reference(pause_ms):
    """run_adaptation (serving.cpp:213-340) on the GPU against the reference
    loop on the same deployment, stream and original records: identical
    retrain schedule (window sizes, mix-in draws, applied flags), traces
    equal up to bf16x3 tap rounding, final caches within 1e-3."""
    model_txt, vtxt, X, labels, times, samp = _adapt_setup()
    sel = [0, 1, 3]  # FC(32) L1, Conv(3,1) L2, FC(32) L4
    m = lcb.load_base_model(model_txt)
    vs = [lcb.load_variant(vtxt[k]) for k in sel]
    rm = O.RefModel.load(model_txt)
    rvs = [O.RefVariant.load(vtxt[k]) for k in sel]
    for v, rv in zip(vs, rvs):  # strict thresholds: the stream mixes hits and misses
        v.delta = 0.995
        rv.set_delta(0.995)
    dep = lcb.Deployment(m, vs, precision="bf16x3", max_batch=256)
    orig_x = X[-120:]
    otaps, oy = [], []
    for v in vs:
        t, y = _ref_records(rm, orig_x, v.layer)
        otaps.append(t)
        oy = y
    cfg = lcb.AdaptationConfig(sample_rate=0.3, window_min=30.0, retrain_interval_min=15.0, epochs=3,
                               learning_rate=0.005, retrain_pause_ms=pause_ms)
    stream = [lcb.Request(i, float(times[i]), int(labels[samp[i]]), int(samp[i])) for i in range(len(times))]
    res = lcb.run_adaptation(dep, X, labels, stream, cfg, otaps, oy, seed=5, adapt_on=True)
    cfg8 = [cfg.sample_rate, cfg.window_min, cfg.retrain_interval_min, cfg.recency_decay, cfg.mixin_fraction,
            cfg.epochs, cfg.learning_rate, cfg.retrain_pause_ms]
    hl, sv, bp, ev, finals = O.ref_run_adaptation(rm, rvs, X, labels, times, samp, cfg8,
                                                   [cfg.tau, cfg.beta, cfg.w_fp, cfg.w_fn], orig_x, 5, True)
    assert len(res.retrains) == len(ev) >= 3
    for e, r in zip(res.retrains, ev):
        assert (e.interval, e.window_size, e.mixin_size, int(e.applied)) == (int(r[0]), int(r[2]), int(r[3]),
                                                                             int(r[4]))
        assert e.time_min == r[1]
    ours_hl = np.array([t.hit_layer for t in res.traces])
    ours_sv = np.array([t.served_pred for t in res.traces])
    ours_bp = np.array([t.base_pred for t in res.traces])
    assert np.mean(ours_bp == bp) >= 0.995
    assert np.mean(ours_hl == hl) >= 0.98, np.mean(ours_hl == hl)
    assert np.mean(ours_sv == sv) >= 0.98
    assert 0.05 < np.mean(hl > 0) < 0.95  # both hits and misses exercised
    for v, rv in zip(res.final_variants, finals):
        _assert_nets_close(v.save(), rv.save(), 1e-3)
    # the adapted caches changed (the loop really retrained and swapped)
    assert any(f.save() != lcb.load_variant(vtxt[k]).save() for f, k in zip(res.final_variants, sel))
    assert sum(s.requests for s in res.timeline) == len(times)
    dep.close()


def test_run_adaptation_frozen_matches_serve():
    """adapt_on=False: no retrains, caches frozen, traces equal the plain
    shadow serve of the same requests (serving.hpp:125-128)."""
    model_txt, vtxt, X, labels, times, samp = _adapt_setup(n_req=300)
    m = lcb.load_base_model(model_txt)
    vs = [lcb.load_variant(t) for t in vtxt]
    dep = lcb.Deployment(m, vs, precision="bf16x3", max_batch=128)
    stream = [lcb.Request(i, float(times[i]), int(labels[samp[i]]), int(samp[i])) for i in range(len(times))]
    res = lcb.run_adaptation(dep, X, labels, stream, lcb.AdaptationConfig(), [np.zeros((0, 1))] * len(vs),
                             np.zeros((0, m.num_classes)), seed=1, adapt_on=False)
    assert res.retrains == []
    sh = dep.serve(X[samp[:128]], shadow=True)
    assert np.array_equal(np.array([t.hit_layer for t in res.traces[:128]]), sh.exit_layer)
    assert np.array_equal(np.array([t.served_pred for t in res.traces[:128]]), sh.served)
    for f, t in zip(res.final_variants, vtxt):
        assert f.save() == lcb.load_variant(t).save()
    with pytest.raises(ValueError):  # original records must cover every attached cache
        lcb.run_adaptation(dep, X, labels, stream, lcb.AdaptationConfig(), [np.zeros((4, 3))],
                           np.zeros((4, m.num_classes)), seed=1)
    with pytest.raises(ValueError):  # invalid config -> the reference's invalid_argument
        lcb.run_adaptation(dep, X, labels, stream, lcb.AdaptationConfig(sample_rate=1.5), [np.zeros((0, 1))] * len(vs),
                           np.zeros((0, m.num_classes)), seed=1)
    dep.close()


def _adapt_pair(cfg, sel=(0,), n_req=720, minutes=6.0, selector_out=None, seed=31, adapt_on=True, delta=None):
    model_txt, vtxt, X, labels, times, samp = _adapt_setup(n_req=n_req, minutes=minutes)
    m = lcb.load_base_model(model_txt)
    rm = O.RefModel.load(model_txt)
    vs = [lcb.load_variant(vtxt[k]) for k in sel]
    rvs = [O.RefVariant.load(vtxt[k]) for k in sel]
    for v, rv in zip(vs, rvs):
        if selector_out is not None:
            v.set_selector_out(*selector_out)
            rv.set_selector_out(*selector_out)
        if delta is not None:
            v.delta = delta
            rv.set_delta(delta)
    orig_x = X[-100:]
    otaps = []
    oy = None
    for v in vs:
        t, oy = _ref_records(rm, orig_x, v.layer)
        otaps.append(t)
    dep = lcb.Deployment(m, vs, precision="bf16x3", max_batch=256)
    stream = [lcb.Request(i, float(times[i]), int(labels[samp[i]]), int(samp[i])) for i in range(len(times))]
    res = lcb.run_adaptation(dep, X, labels, stream, cfg, otaps, oy, seed=seed, adapt_on=adapt_on)
    cfg8 = [cfg.sample_rate, cfg.window_min, cfg.retrain_interval_min, cfg.recency_decay, cfg.mixin_fraction,
            cfg.epochs, cfg.learning_rate, cfg.retrain_pause_ms]
    ref = O.ref_run_adaptation(rm, rvs, X, labels, times, samp, cfg8, [cfg.tau, cfg.beta, cfg.w_fp, cfg.w_fn],
                               orig_x, seed, adapt_on)
    before = [lcb.load_variant(vtxt[k]).save() for k in sel]
    dep.close()
    return res, ref, before


@requires_ref
def test_adaptation_schedule_window_and_mixin():
    """test_serving.cpp:563-595 on the GPU loop: retrains at every interval
    boundary with the declared window and mix-in sizes, deterministic reruns."""
    cfg = lcb.AdaptationConfig(sample_rate=1.0, retrain_interval_min=2.0, window_min=2.0, epochs=2)
    res, (hl, sv, bp, ev, finals), _ = _adapt_pair(cfg)
    assert [(e.interval, e.time_min) for e in res.retrains] == [(1, 2.0), (2, 4.0)]
    assert all(e.applied for e in res.retrains)
    for e, r in zip(res.retrains, ev):
        assert (e.window_size, e.mixin_size) == (int(r[2]), int(r[3]))
        assert e.mixin_size == min(100, e.window_size)  # fraction 0.5 -> one per window sample, capped
    again, _, _ = _adapt_pair(cfg)
    assert [(t.hit_layer, t.served_pred) for t in again.traces] == [(t.hit_layer, t.served_pred) for t in res.traces]
    assert again.final_variants[0].save() == res.final_variants[0].save()  # bit-deterministic on the GPU
    assert np.mean(np.array([t.hit_layer for t in res.traces]) == hl) >= 0.98


@requires_ref
def test_adaptation_diverging_retrains_are_discarded():
    """test_serving.cpp:597-620: an infinite learning rate diverges; every
    retrain notes it, the old caches keep serving, traces equal the static run."""
    cfg = lcb.AdaptationConfig(sample_rate=1.0, retrain_interval_min=2.0, window_min=2.0, epochs=3,
                               learning_rate=float("inf"))
    res, (hl, sv, bp, ev, finals), before = _adapt_pair(cfg)
    assert len(res.retrains) == 2 and all("diverged" in e.note for e in res.retrains), [e.note for e in res.retrains]
    static, _, _ = _adapt_pair(lcb.AdaptationConfig(), adapt_on=False)
    assert [t.hit_layer for t in res.traces] == [t.hit_layer for t in static.traces]
    assert res.final_variants[0].save() == before[0]
    assert np.array_equal(np.array([t.hit_layer for t in res.traces]), hl)


@requires_ref
def test_adaptation_wakes_a_dead_cache_after_the_pause():
    """test_serving.cpp:622-667: a silenced selector cannot hit before the first
    retrain; retraining wakes it, and a swap pause delays the wake-up."""
    cfg = lcb.AdaptationConfig(sample_rate=1.0, retrain_interval_min=2.0, window_min=4.0, mixin_fraction=0.0,
                               epochs=25, learning_rate=0.01)
    res, (hl, sv, bp, ev, finals), _ = _adapt_pair(cfg, n_req=960, minutes=8.0, selector_out=(0.0, -3.0))
    t = np.array([r.time_min for r in res.traces])
    h = np.array([r.hit_layer for r in res.traces])
    assert np.all(h[t < 2.0] == 0) and np.sum(h[t >= 2.0] > 0) > 0
    assert np.mean(h == hl) >= 0.98
    paused = lcb.AdaptationConfig(sample_rate=1.0, retrain_interval_min=2.0, window_min=4.0, mixin_fraction=0.0,
                                  epochs=25, learning_rate=0.01, retrain_pause_ms=2.0 * 60000.0)
    res2, (hl2, _, _, _, _), _ = _adapt_pair(paused, n_req=960, minutes=8.0, selector_out=(0.0, -3.0))
    h2 = np.array([r.hit_layer for r in res2.traces])
    assert np.all(h2[t < 4.0] == 0) and np.sum(h2[t >= 4.0] > 0) > 0
    assert np.mean(h2 == hl2) >= 0.98


@pytest.mark.parametrize("pause_ms", [0.0, 90000.0])
def test_adaptation_swaps_replay_on_a_second_replica(pause_ms):
    """Cross-replica adaptation (§8f rank 3, serving.cpp:303-315): the swap hook
    captures every swap run_adaptation lands, the payload goes through the
    fleet broadcast encoding (pack/unpack, shard.py), and a second replica
    (fresh Deployment) serving the same stream with serve_with_swaps matches
    the trainer's traces (up to split-K rounding of differently composed
    batches) and ends on byte-identical caches."""
    from paper_2101_07344_b200.shard import (apply_swap_to_deployment, capture_swaps, pack_swaps, serve_with_swaps,
                                             unpack_swaps)
    model_txt, vtxt, X, labels, times, samp = _adapt_setup()
    sel = [0, 1, 3]
    m = lcb.load_base_model(model_txt)

    def fresh():
        vs = [lcb.load_variant(vtxt[k]) for k in sel]
        for v in vs:
            v.delta = 0.995
        return lcb.Deployment(m, vs, precision="bf16x3", max_batch=256), vs

    dep, vs = fresh()
    rm = O.RefModel.load(model_txt) if os.path.exists(O.REF_SO) else None
    orig_x = X[-120:]
    if rm is not None:
        otaps, oy = [], None
        for v in vs:
            t, oy = _ref_records(rm, orig_x, v.layer)
            otaps.append(t)
    else:  # records from the GPU's own shadow taps
        pytest.skip("needs oracle/_ref for the original records")
    cfg = lcb.AdaptationConfig(sample_rate=0.3, window_min=30.0, retrain_interval_min=15.0, epochs=3,
                               learning_rate=0.005, retrain_pause_ms=pause_ms)
    stream = [lcb.Request(i, float(times[i]), int(labels[samp[i]]), int(samp[i])) for i in range(len(times))]
    swaps = capture_swaps(dep)
    res = lcb.run_adaptation(dep, X, labels, stream, cfg, otaps, oy, seed=5, adapt_on=True)
    dep.set_swap_hook(None)
    assert len(swaps) >= 2 and all(len(s.blobs) == len(sel) for s in swaps)
    assert all(a.time_min <= b.time_min for a, b in zip(swaps, swaps[1:]))
    swaps = unpack_swaps(pack_swaps(swaps))  # the broadcast payload
    rep, _ = fresh()

    def chunks(d, xs):  # batches of at most max_batch requests
        rs = [d.serve(xs[i:i + d.max_batch], shadow=True) for i in range(0, xs.shape[0], d.max_batch)]
        return {"exit_layer": np.concatenate([r.exit_layer for r in rs]),
                "served": np.concatenate([r.served for r in rs]),
                "base_pred": np.concatenate([r.base_pred for r in rs])}

    def serve(xs):
        return chunks(rep, xs)

    out = serve_with_swaps(serve, lambda s: apply_swap_to_deployment(rep, s), X[samp], times, swaps)
    hl = np.array([t.hit_layer for t in res.traces])
    sv = np.array([t.served_pred for t in res.traces])
    bp = np.array([t.base_pred for t in res.traces])
    assert np.mean(out["exit_layer"] == hl) >= 0.99, np.mean(out["exit_layer"] == hl)
    assert np.mean(out["served"] == sv) >= 0.99
    assert np.mean(out["base_pred"] == bp) >= 0.995
    for k in range(len(sel)):
        assert rep.variant(k).save() == dep.variant(k).save()
    # the swaps matter: a frozen replica's traces differ
    frozen, _ = fresh()
    fz = chunks(frozen, X[samp])
    assert np.mean(fz["exit_layer"] == hl) < np.mean(out["exit_layer"] == hl)
    for d in (dep, rep, frozen):
        d.close()
