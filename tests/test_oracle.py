"""Pins the CPU oracle (oracle/lc_oracle.c) before anything is compared to it:
bit-exact against the compiled reference (oracle/_ref) on random networks,
the reference tests' known-answer values, and the golden fixtures generated
from the reference (tests/golden/). CNN-tier restatement: cross-checked with
torch fp64 (no reference counterpart exists)."""
import json
import os

import numpy as np
import pytest

from tests.helpers import GOLDEN, requires_ref

O = pytest.importorskip("oracle.oracle")


def fc(i, o, w, b):
    return dict(kind=0, in_dim=i, out_dim=o, pool_window=0, kernel=0, stride=0, w=np.array(w, float),
                b=np.array(b, float))


def run(layers, x):
    net = O.OracleNet(layers)
    out = np.zeros(layers[-1]["out_dim"])
    O.orc().lco_forward(net.ptr, net.n, O._dp(np.array(x, float)), O._dp(out), None)
    return out


def test_kats_from_reference_tests():
    # test_nn.cpp:36-44 FC 3.5 / 6.5
    assert list(run([fc(2, 2, [1, 2, 3, 4], [0.5, -0.5])], [1, 1])) == [3.5, 6.5]
    # :46-58 pool 1.5 / 3.5
    pool = dict(kind=2, in_dim=4, out_dim=2, pool_window=2, kernel=0, stride=0, w=None, b=None)
    assert list(run([pool], [1, 2, 3, 4])) == [1.5, 3.5]
    # :72-79 conv1d 3.25 / 5.25
    conv = dict(kind=3, in_dim=3, out_dim=2, pool_window=0, kernel=2, stride=1, w=np.array([1.0, 1.0]),
                b=np.array([0.25]))
    assert list(run([conv], [1, 2, 3])) == [3.25, 5.25]
    # :81-92 relu
    relu = dict(kind=1, in_dim=3, out_dim=3, pool_window=0, kernel=0, stride=0, w=None, b=None)
    assert list(run([relu], [-1, 0, 2])) == [0, 0, 2]
    # :94-114 softmax
    assert np.all(O.softmax(np.array([3.0] * 4)) == 0.25)
    # :30-34 argmax ties -> lowest index
    assert O.argmax(np.array([0.1, 0.9, 0.9])) == 1
    assert O.argmax(np.array([-3.0, -1.0, -2.0])) == 1


@requires_ref
def test_inclusive_threshold_like_reference():
    # test_cache.cpp:218-227: zeroed selector -> prob exactly 0.5; hits at 0.5, misses at 0.5000000001
    v = O.RefVariant.build(1, 0, "FC(8)", 4, 3, 9)
    v.force_selector(0.0)
    meta = O.parse_variant(v.save())
    pred, sel = O.OracleNet(meta["predictor"]), O.OracleNet(meta["selector"])
    tap = np.array([0.3, -0.1, 0.2, 0.0])
    hit, p, _, _ = O.oracle_lookup(pred, sel, 0.5, tap)
    assert hit and p == 0.5
    hit, _, _, _ = O.oracle_lookup(pred, sel, 0.5000000001, tap)
    assert not hit
    v.set_delta(0.5000000001)
    assert v.lookup(tap, 3)[0] is False


@requires_ref
@pytest.mark.parametrize("arch", ["FC(32)", "Pool(16)", "Pool(8192)", "Conv(3,1)", "Conv(5,2)"])
def test_oracle_lookup_bit_exact_vs_reference(arch):
    rng = np.random.default_rng(5)
    for seed in range(4):
        v = O.RefVariant.build(2, seed, arch, 48, 7, 100 + seed)
        meta = O.parse_variant(v.save())
        pred, sel = O.OracleNet(meta["predictor"]), O.OracleNet(meta["selector"])
        for _ in range(8):
            tap = rng.uniform(-1.5, 1.5, 48)
            rh, rp, rpr, rlg = v.lookup(tap, 7)
            oh, op, opr, olg = O.oracle_lookup(pred, sel, 0.5, tap)
            assert rh == oh and rp == op
            assert np.array_equal(rpr, opr) and np.array_equal(rlg, olg)


@requires_ref
def test_oracle_serve_bit_exact_vs_reference_simulate():
    rng = np.random.default_rng(7)
    m = O.RefModel.make(24, 5, [16, 12, 16, 8], 4, 31)
    variants = [O.RefVariant.build(1, 0, "FC(8)", 16, 5, 3), O.RefVariant.build(3, 1, "Conv(3,1)", 16, 5, 3),
                O.RefVariant.build(4, 2, "Pool(4)", 8, 5, 3)]
    for v, d in zip(variants, [0.55, 0.5, 0.45]):
        v.set_delta(d)
    x = rng.uniform(-1.5, 1.5, (64, 24))
    hl, sv, bp, _ = O.ref_simulate(m, variants, x)
    model = O.parse_model(m.save())
    caches = []
    for v in variants:
        meta = O.parse_variant(v.save())
        caches.append((meta["layer"], meta["predictor"], meta["selector"], meta["delta"]))
    el, s2, b2, _ = O.oracle_serve_mlp(model, caches, x)
    assert np.array_equal(hl, el) and np.array_equal(sv, s2) and np.array_equal(bp, b2)
    # multi-threaded request sharding reproduces the single-thread traces
    hl4, sv4, bp4, _ = O.ref_simulate(m, variants, x, threads=4)
    assert np.array_equal(hl, hl4) and np.array_equal(sv, sv4) and np.array_equal(bp, bp4)


def _trained():
    d = os.path.join(GOLDEN, "trained")
    model = O.parse_model(open(os.path.join(d, "model.txt")).read())
    caches = []
    k = 0
    while os.path.exists(os.path.join(d, f"variant_{k}.txt")):
        meta = O.parse_variant(open(os.path.join(d, f"variant_{k}.txt")).read())
        caches.append((meta["layer"], meta["predictor"], meta["selector"], meta["delta"]))
        k += 1
    test = [l.split() for l in open(os.path.join(d, "dataset.txt")).read().split("\n") if l.startswith("test ")]
    X = np.array([[float(v) for v in t[2:]] for t in test])
    reqs = [tuple(map(int, l.split())) for l in open(os.path.join(d, "requests.txt")).read().split("\n") if l]
    traces = [l.split() for l in open(os.path.join(d, "traces.txt")).read().split("\n")[1:]
              if l and not l.startswith("#")]
    return model, caches, X, reqs, traces


def test_oracle_reproduces_golden_trained_traces():
    """The reference's own pipeline traces (tests/golden/trained/traces.txt)."""
    model, caches, X, reqs, traces = _trained()
    idx = [s for _, s in reqs]
    el, sv, bp, _ = O.oracle_serve_mlp(model, caches, X[idx])
    assert [int(t[5]) for t in traces] == el.tolist()   # hit_layer
    assert [int(t[4]) for t in traces] == sv.tolist()   # served_pred
    assert [int(t[3]) for t in traces] == bp.tolist()   # base_pred


def test_oracle_reproduces_golden_c1():
    import paper_2101_07344_b200 as lcb
    from paper_2101_07344_b200.synthetic import mlp_inputs
    spec = json.load(open(os.path.join(GOLDEN, "c1", "c1.json")))
    m = lcb.make_base_model(spec["input_dim"], spec["classes"], spec["widths"], spec["blocks"], spec["model_seed"])
    model = O.parse_model(m.save())
    caches = []
    for l in range(spec["blocks"]):
        v = lcb.build_variant(l + 1, l, spec["menu"][l], m.tap_dim(l + 1), spec["classes"], spec["cache_seed"])
        v.set_selector_out(spec["gains"][str(l + 1)], spec["biases"][str(l + 1)])
        v.delta = spec["delta"]
        pred, sel, d = O.variant_layers_from_product(v)
        caches.append((l + 1, pred, sel, d))
    x = mlp_inputs(spec["n"], spec["input_dim"], spec["input_seed"])
    el, sv, bp, probs = O.oracle_serve_mlp(model, caches, x)
    assert el.tolist() == spec["exit_layer"]
    assert sv.tolist() == spec["served"]
    assert bp.tolist() == spec["base"]
    exp = np.array(spec["probs"])
    probed = ~np.isnan(probs)
    assert np.array_equal(probs[probed], exp[probed])


def test_cnn_oracle_vs_torch_fp64():
    torch = pytest.importorskip("torch")
    import torch.nn.functional as F
    import paper_2101_07344_b200 as lcb
    m = lcb.make_cnn_model("resnet18_cifar", 10, 3)
    ops = m.cnn_ops()
    x = np.random.default_rng(0).standard_normal((2, 3 * 32 * 32))
    taps, logits = O.oracle_cnn_forward(ops, m.nslots, x, m.num_blocks, m.tap_dims, 10, threads=2)
    # independent torch fp64 restatement of the same op list
    slots = {}
    X = torch.tensor(x.reshape(2, 3, 32, 32), dtype=torch.float64)
    ttaps = {}
    for o in ops:
        inp = X if o["in"] < 0 else slots[o["in"]]
        if o["kind"] in (0, 1):
            w = torch.tensor(o["w"]).reshape(o["Cout"], o["C"], o["k"], o["k"])
            y = F.conv2d(inp, w, stride=o["stride"], padding=o["pad"])
            y = y * torch.tensor(o["scale"]).view(1, -1, 1, 1) + torch.tensor(o["shift"]).view(1, -1, 1, 1)
            if o["res"] >= 0:
                y = y + slots[o["res"]]
            if o["relu"]:
                y = torch.relu(y)
            slots[o["out"]] = y
        elif o["kind"] == 2:
            slots[o["out"]] = F.max_pool2d(inp, o["k"], o["stride"], o["pad"])
        else:
            g = inp.mean(dim=(2, 3))
            lg = g @ torch.tensor(o["w"]).reshape(o["Cout"], o["C"]).T + torch.tensor(o["shift"])
        if o["tap"] >= 0:
            ttaps[o["tap"]] = slots[o["out"]].reshape(2, -1).numpy()
    for t in range(m.num_blocks):
        np.testing.assert_allclose(taps[t], ttaps[t], rtol=1e-10, atol=1e-10)
    np.testing.assert_allclose(logits, lg.numpy(), rtol=1e-10, atol=1e-10)
    # activations stay O(1) through depth (synthetic weights are usable)
    assert 0.05 < np.abs(taps[-1]).mean() < 20


@requires_ref
def test_oracle_mlp_taps_and_logits_bit_exact_vs_reference():
    """oracle_mlp_forward (taps after every block's ReLU and the base logits,
    activations[size-2]) against the reference's forward_with_taps and forward
    (oracle/_ref) on the golden trained model: the serve-path logits/taps
    parity tests compare the GPU with exactly these values."""
    d = os.path.join(GOLDEN, "trained")
    txt = open(os.path.join(d, "model.txt")).read()
    model = O.parse_model(txt)
    rm = O.RefModel.load(txt)
    x = np.random.default_rng(3).uniform(-1.5, 1.5, (16, model["layers"][0]["in_dim"]))
    taps, logits = O.oracle_mlp_forward(model, x)
    for i in range(16):
        rt, _ = rm.forward_taps(x[i])
        for k in range(model["blocks"]):
            assert np.array_equal(taps[k][i], rt[k])
        assert np.array_equal(logits[i], rm.logits(x[i]))


@pytest.mark.parametrize("arch,classes", [("resnet18_cifar", 10), ("resnet50", 1000), ("vgg16_cifar", 10)])
def test_oracle_cnn_builder_matches_product(arch, classes):
    """oracle/cnn_models.py rebuilds the product's synthetic CNN (host/cnn.cpp)
    from the reference RNG without the product library: same ops, geometry,
    taps and weights bit for bit. bench.py's reference arm relies on it."""
    import paper_2101_07344_b200 as lcb
    from oracle.cnn_models import CnnModel
    ours = CnnModel(arch, classes, 2101)
    m = lcb.make_cnn_model(arch, classes, 2101)
    prod = m.cnn_ops()
    assert ours.nslots == m.nslots and ours.tap_dims == m.tap_dims and len(ours.ops) == len(prod)
    for a, b in zip(ours.ops, prod):
        for k in ("kind", "in", "out", "res", "C", "H", "W", "Cout", "k", "stride", "pad", "relu", "tap"):
            assert a[k] == b[k], (k, a[k], b[k])
        for k in ("w", "scale", "shift"):
            if b[k] is None or len(b[k]) == 0:
                assert a[k] is None or len(a[k]) == 0 or not np.any(a[k]), k
            else:
                assert np.array_equal(a[k], b[k]), k
