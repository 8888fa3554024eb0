"""TEST INFRASTRUCTURE ONLY — ctypes face of the CPU checkers.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline/reference
legs may import this module; the product (paper_2101_07344_b200) never does.

  ref()  : oracle/_ref/liblatecache_ref.so — the UNMODIFIED reference sources
           (/root/reference/proj/src) + oracle/ref_driver.cpp, built by
           oracle/Makefile. Runs the reference's own code path.
  orc()  : oracle/liblc_oracle.so — the plain-C restatement (lc_oracle.c),
           pinned bit-exactly against ref() in tests/test_oracle.py.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import List, Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "liblatecache_ref.so")
ORC_SO = os.path.join(HERE, "liblc_oracle.so")

P, I, D, U64, LL = C.c_void_p, C.c_int, C.c_double, C.c_uint64, C.c_longlong
pI, pD = C.POINTER(C.c_int), C.POINTER(C.c_double)


def build() -> None:
    """Compile the checkers (needs /root/reference for the _ref part)."""
    targets = ["ref"] if os.path.isdir("/root/reference/proj") else []
    subprocess.run(["make", "-C", HERE, os.path.join(HERE, "liblc_oracle.so")] + targets, check=True,
                   stdout=subprocess.DEVNULL)


_ref = None
_orc = None


def ref() -> C.CDLL:
    global _ref
    if _ref is None:
        lib = C.CDLL(REF_SO)
        sig = {
            "ref_last_error": (C.c_char_p, []),
            "ref_free": (None, [P]),
            "ref_model_make": (P, [I, I, pI, I, I, U64]),
            "ref_model_load": (P, [C.c_char_p]),
            "ref_model_save": (P, [P]),
            "ref_model_free": (None, [P]),
            "ref_model_info": (I, [P, pI, pI, pI, pI]),
            "ref_variant_build": (P, [I, I, C.c_char_p, I, I, U64]),
            "ref_variant_load": (P, [C.c_char_p]),
            "ref_variant_save": (P, [P]),
            "ref_variant_free": (None, [P]),
            "ref_variant_set_delta": (I, [P, D]),
            "ref_variant_force_selector": (I, [P, D]),
            "ref_variant_set_selector_out": (I, [P, D, D]),
            "ref_selector_logit": (I, [P, pD, I, pD]),
            "ref_forward_taps": (I, [P, pD, pD, pD]),
            "ref_forward_logits": (I, [P, pD, pD]),
            "ref_lookup": (I, [P, pD, I, pI, pD, pD, pD]),
            "ref_simulate": (I, [P, C.POINTER(P), I, pD, I, pI, pI, pI, I, pD]),
            "ref_measure_metrics": (I, [P, P, pD, I, C.POINTER(LL), pD, pD]),
            "ref_tune_delta": (I, [P, P, pD, I, D, pD, I, pD]),
            "ref_pipeline": (I, [C.c_char_p, U64, I, I, I, I, C.c_char_p, I, I, D]),
            "ref_gen_workload": (I, [C.c_char_p, I, D, D, D, D, U64, C.POINTER(LL), C.POINTER(LL), pI, LL]),
            "ref_rng_stream": (I, [U64, I, I, pD, C.POINTER(U64)]),
            "ref_mix_seed": (U64, [U64, U64]),
            "ref_train": (P, [P, I, pD, I, pD, I, I, pD, D, D, I, I, U64, D, D]),
            "ref_run_adaptation": (I, [P, C.POINTER(P), I, pD, pI, I, pD, pI, I, pD, pD, pD, I, U64, I, pI, pI, pI,
                                       pI, pD, I, C.POINTER(P)]),
        }
        for k, (r, a) in sig.items():
            f = getattr(lib, k)
            f.restype = r
            f.argtypes = a
        _ref = lib
    return _ref


def orc() -> C.CDLL:
    global _orc
    if _orc is None:
        lib = C.CDLL(ORC_SO)
        lib.lco_forward.restype = I
        lib.lco_forward.argtypes = [P, I, pD, pD, pD]
        lib.lco_sigmoid.restype = D
        lib.lco_sigmoid.argtypes = [D]
        lib.lco_softmax.restype = None
        lib.lco_softmax.argtypes = [pD, I, pD]
        lib.lco_argmax.restype = I
        lib.lco_argmax.argtypes = [pD, I]
        lib.lco_lookup.restype = I
        lib.lco_lookup.argtypes = [P, I, P, I, D, pD, pD, pD, pD]
        lib.lco_serve_mlp.restype = I
        lib.lco_serve_mlp.argtypes = [P, I, pI, I, P, I, pD, pI, pI, pI, pD]
        lib.lco_cnn_forward_batch.restype = I
        lib.lco_cnn_forward_batch.argtypes = [P, I, I, C.c_size_t, pD, C.c_size_t, I, I, C.POINTER(pD),
                                              C.POINTER(C.c_size_t), pD, I, I]
        _orc = lib
    return _orc


def _dp(a: np.ndarray):
    return a.ctypes.data_as(pD)


def _ip(a: np.ndarray):
    return a.ctypes.data_as(pI)


def _check(st: int) -> None:
    if st != 0:
        msg = ref().ref_last_error().decode()
        if st == 1:
            raise ValueError(msg)
        raise RuntimeError(msg)


def _take(p) -> str:
    s = C.string_at(p).decode()
    ref().ref_free(p)
    return s


# ------------------------------------------------------------------ reference objects
class RefModel:
    def __init__(self, handle):
        if not handle:
            _check(1)
        self.h = handle
        b, c, d = C.c_int(), C.c_int(), C.c_int()
        ref().ref_model_info(self.h, C.byref(b), C.byref(c), C.byref(d), None)
        self.blocks, self.classes, self.input_dim = b.value, c.value, d.value
        td = (C.c_int * self.blocks)()
        ref().ref_model_info(self.h, C.byref(b), C.byref(c), C.byref(d), td)
        self.tap_dims = list(td)

    @staticmethod
    def make(input_dim, classes, widths, blocks, seed) -> "RefModel":
        w = np.ascontiguousarray(widths, np.int32)
        return RefModel(ref().ref_model_make(input_dim, classes, _ip(w), len(w), blocks, seed))

    @staticmethod
    def load(text: str) -> "RefModel":
        return RefModel(ref().ref_model_load(text.encode()))

    def save(self) -> str:
        return _take(ref().ref_model_save(self.h))

    def __del__(self):
        if getattr(self, "h", None):
            ref().ref_model_free(self.h)
            self.h = None

    def forward_taps(self, x: np.ndarray):
        x = np.ascontiguousarray(x, np.float64)
        taps = np.zeros(sum(self.tap_dims), np.float64)
        y = np.zeros(self.classes, np.float64)
        _check(ref().ref_forward_taps(self.h, _dp(x), _dp(taps), _dp(y)))
        out, off = [], 0
        for d in self.tap_dims:
            out.append(taps[off:off + d])
            off += d
        return out, y

    def logits(self, x: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float64)
        out = np.zeros(self.classes, np.float64)
        _check(ref().ref_forward_logits(self.h, _dp(x), _dp(out)))
        return out


class RefVariant:
    def __init__(self, handle):
        if not handle:
            _check(1)
        self.h = handle

    @staticmethod
    def build(layer, vidx, arch, tap_dim, classes, seed) -> "RefVariant":
        return RefVariant(ref().ref_variant_build(layer, vidx, arch.encode(), tap_dim, classes, seed))

    @staticmethod
    def load(text: str) -> "RefVariant":
        return RefVariant(ref().ref_variant_load(text.encode()))

    def save(self) -> str:
        return _take(ref().ref_variant_save(self.h))

    def set_delta(self, d: float) -> None:
        ref().ref_variant_set_delta(self.h, d)

    def force_selector(self, bias: float) -> None:
        ref().ref_variant_force_selector(self.h, bias)

    def set_selector_out(self, gain: float, bias: float) -> None:
        ref().ref_variant_set_selector_out(self.h, gain, bias)

    def __del__(self):
        if getattr(self, "h", None):
            ref().ref_variant_free(self.h)
            self.h = None

    def lookup(self, tap: np.ndarray, classes: int):
        t = np.ascontiguousarray(tap, np.float64)
        hit, prob = C.c_int(), C.c_double()
        pr = np.zeros(classes, np.float64)
        lg = np.zeros(classes, np.float64)
        _check(ref().ref_lookup(self.h, _dp(t), len(t), C.byref(hit), C.byref(prob), _dp(pr), _dp(lg)))
        return bool(hit.value), prob.value, pr, lg

    def selector_logit(self, tap: np.ndarray) -> float:
        t = np.ascontiguousarray(tap, np.float64)
        z = C.c_double()
        _check(ref().ref_selector_logit(self.h, _dp(t), len(t), C.byref(z)))
        return z.value


def ref_simulate(model: RefModel, variants: Sequence[RefVariant], inputs: np.ndarray, threads: int = 1):
    """The reference's simulate_model over rows of `inputs` (request i = row i)."""
    x = np.ascontiguousarray(inputs, np.float64)
    B = x.shape[0]
    arr = (P * max(1, len(variants)))(*[v.h for v in variants])
    hl = np.zeros(B, np.int32)
    sv = np.zeros(B, np.int32)
    bp = np.zeros(B, np.int32)
    el = C.c_double()
    _check(ref().ref_simulate(model.h, arr, len(variants), _dp(x), B, _ip(hl), _ip(sv), _ip(bp), threads,
                              C.byref(el)))
    return hl, sv, bp, el.value


def ref_measure_metrics(model: RefModel, variant: RefVariant, inputs: np.ndarray):
    """The reference's measure_metrics (cache.cpp:316-335) over collect_taps of
    the rows of `inputs`: ({tp, fp, tn, fn}, hit_rate, accuracy)."""
    x = np.ascontiguousarray(inputs, np.float64)
    cnt = (LL * 4)()
    hr, acc = C.c_double(), C.c_double()
    _check(ref().ref_measure_metrics(model.h, variant.h, _dp(x), x.shape[0], cnt, C.byref(hr), C.byref(acc)))
    return {"tp": cnt[0], "fp": cnt[1], "tn": cnt[2], "fn": cnt[3]}, hr.value, acc.value


def ref_tune_delta(model: RefModel, variant: RefVariant, inputs: np.ndarray, target: float, grid) -> float:
    """The reference's tune_delta (cache.cpp:267-307) on a copy of the variant."""
    x = np.ascontiguousarray(inputs, np.float64)
    g = np.ascontiguousarray(grid, np.float64)
    d = C.c_double()
    _check(ref().ref_tune_delta(model.h, variant.h, _dp(x), x.shape[0], target, _dp(g), len(g), C.byref(d)))
    return d.value


# ------------------------------------------------------------------ text format -> numpy
def ref_train(variant: "RefVariant", which: str, taps: np.ndarray, y: np.ndarray, weights=None, lr=0.01,
              momentum=0.9, epochs=20, batch=16, seed=1, a=2.0, b=0.5) -> "RefVariant":
    """The reference's train_predictor (which="predictor", a=tau, b=beta) or
    train_selector (which="selector", a=w_fp, b=w_fn) (cache.cpp:179-257) on a
    copy of the variant; returns the trained copy."""
    t = np.ascontiguousarray(taps, np.float64)
    yy = np.ascontiguousarray(y, np.float64)
    w = None if weights is None else np.ascontiguousarray(weights, np.float64)
    h = ref().ref_train(variant.h, 0 if which == "predictor" else 1, _dp(t), t.shape[1], _dp(yy), yy.shape[1],
                        t.shape[0], None if w is None else _dp(w), lr, momentum, epochs, batch, seed, a, b)
    if not h:
        raise RuntimeError(ref().ref_last_error().decode())
    return RefVariant(h)


def ref_run_adaptation(model: "RefModel", variants, inputs: np.ndarray, labels: np.ndarray, times: np.ndarray,
                       sample_idx: np.ndarray, cfg8, train4, orig_inputs: np.ndarray, seed: int, adapt_on: bool):
    """The reference's run_adaptation (serving.cpp:213-340) over a pass-through
    deployment: (hit_layer, served, base, events [n][5], final RefVariants)."""
    x = np.ascontiguousarray(inputs, np.float64)
    lab = np.ascontiguousarray(labels, np.int32)
    t = np.ascontiguousarray(times, np.float64)
    si = np.ascontiguousarray(sample_idx, np.int32)
    c8 = np.ascontiguousarray(cfg8, np.float64)
    t4 = np.ascontiguousarray(train4, np.float64)
    oi = np.ascontiguousarray(orig_inputs, np.float64)
    R = t.shape[0]
    hl, sv, bp = np.zeros(R, np.int32), np.zeros(R, np.int32), np.zeros(R, np.int32)
    cap = 4096
    ev = np.zeros((cap, 5), np.float64)
    n = C.c_int()
    arr = (C.c_void_p * len(variants))(*[v.h for v in variants])
    out = (C.c_void_p * len(variants))()
    _check(ref().ref_run_adaptation(model.h, arr, len(variants), _dp(x), _ip(lab), x.shape[0], _dp(t), _ip(si), R,
                                    _dp(c8), _dp(t4), _dp(oi), oi.shape[0], seed, 1 if adapt_on else 0, _ip(hl),
                                    _ip(sv), _ip(bp), C.byref(n), _dp(ev), cap, out))
    return hl, sv, bp, ev[:min(n.value, cap)], [RefVariant(out[k]) for k in range(len(variants))]


def parse_network(text: str, pos: int = 0):
    """latecache-network v1 (network.cpp:330-409) -> (layers, end_pos)."""
    toks = text[pos:].split()
    i = 0

    def nxt():
        nonlocal i
        i += 1
        return toks[i - 1]

    assert nxt() == "latecache-network" and nxt() == "v1" and nxt() == "layers"
    n = int(nxt())
    layers = []
    for _ in range(n):
        k = nxt()
        if k == "fc":
            a, b = int(nxt()), int(nxt())
            layers.append(dict(kind=0, in_dim=a, out_dim=b, pool_window=0, kernel=0, stride=0, w=None, b=None))
        elif k == "relu":
            a = int(nxt())
            layers.append(dict(kind=1, in_dim=a, out_dim=a, pool_window=0, kernel=0, stride=0, w=None, b=None))
        elif k == "pool":
            a, w = int(nxt()), int(nxt())
            layers.append(dict(kind=2, in_dim=a, out_dim=a // w, pool_window=w, kernel=0, stride=0, w=None, b=None))
        elif k == "conv1d":
            a, kk, s = int(nxt()), int(nxt()), int(nxt())
            layers.append(dict(kind=3, in_dim=a, out_dim=(a - kk) // s + 1, pool_window=0, kernel=kk, stride=s,
                               w=None, b=None))
        elif k == "softmax":
            a = int(nxt())
            layers.append(dict(kind=4, in_dim=a, out_dim=a, pool_window=0, kernel=0, stride=0, w=None, b=None))
    while True:
        w = nxt()
        if w == "end":
            break
        idx = int(nxt())
        assert nxt() == "w"
        cnt = int(nxt())
        layers[idx]["w"] = np.array([float(nxt()) for _ in range(cnt)], np.float64)
        assert nxt() == "b"
        cnt = int(nxt())
        layers[idx]["b"] = np.array([float(nxt()) for _ in range(cnt)], np.float64)
    # end position in the original text
    consumed = " ".join(toks[:i])
    return layers, consumed


def parse_variant(text: str):
    lines = text.split("\n")
    assert lines[0] == "latecache-variant v1"
    body = "\n".join(l for l in lines[1:] if not l.startswith("#"))
    toks = body.split()
    meta = dict(layer=int(toks[1]), variant=int(toks[3]), arch=toks[5], delta=float(toks[7]))
    rest = body.split("predictor", 1)[1]
    pred_txt, sel_txt = rest.split("\nselector\n", 1)
    meta["predictor"], _ = parse_network(pred_txt)
    meta["selector"], _ = parse_network(sel_txt)
    return meta


def parse_model(text: str):
    lines = text.split("\n")
    assert lines[0] == "latecache-model v1"
    body = [l for l in lines[1:] if not l.startswith("#")]
    head = body[0].split()
    blocks, classes = int(head[1]), int(head[3])
    tap_layers = [int(v) for v in body[1].split()[1:]]
    tap_dims = [int(v) for v in body[2].split()[1:]]
    layers, _ = parse_network("\n".join(body[3:]))
    return dict(blocks=blocks, classes=classes, tap_layers=tap_layers, tap_dims=tap_dims, layers=layers)


# ------------------------------------------------------------------ C restatement
class LcoLayer(C.Structure):
    _fields_ = [("kind", I), ("in_dim", I), ("out_dim", I), ("pool_window", I), ("kernel", I), ("stride", I),
                ("w", pD), ("b", pD)]


class LcoCache(C.Structure):
    _fields_ = [("layer", I), ("pred", P), ("np", I), ("sel", P), ("ns", I), ("delta", D)]


class LcoCnnOp(C.Structure):
    _fields_ = [("op", I), ("in_buf", I), ("out_buf", I), ("res_buf", I), ("C", I), ("H", I), ("W", I),
                ("Cout", I), ("kh", I), ("kw", I), ("stride", I), ("pad", I), ("relu", I), ("w", pD),
                ("scale", pD), ("shift", pD), ("tap", I)]


class OracleNet:
    """Layer list (dicts with numpy weights) -> lco_layer array (keeps refs)."""

    def __init__(self, layers: List[dict]):
        self.keep = []
        self.arr = (LcoLayer * len(layers))()
        for i, l in enumerate(layers):
            e = self.arr[i]
            e.kind, e.in_dim, e.out_dim = l["kind"], l["in_dim"], l["out_dim"]
            e.pool_window, e.kernel, e.stride = l["pool_window"], l["kernel"], l["stride"]
            for name in ("w", "b"):
                a = l.get(name)
                if a is not None:
                    a = np.ascontiguousarray(a, np.float64)
                    self.keep.append(a)
                    setattr(e, name, _dp(a))
        self.n = len(layers)
        self.out_dim = layers[-1]["out_dim"]

    @property
    def ptr(self):
        return C.cast(self.arr, P)


def variant_layers_from_product(v) -> tuple:
    """Product CacheVariant -> (pred layer dicts, sel layer dicts, delta)."""
    def conv(ls):
        return [dict(kind=l.kind, in_dim=l.in_dim, out_dim=l.out_dim, pool_window=l.pool_window, kernel=l.kernel,
                     stride=l.stride, w=l.w, b=l.b) for l in ls]
    return conv(v.layers(0)), conv(v.layers(1)), v.delta


def oracle_lookup(pred: OracleNet, sel: OracleNet, delta: float, tap: np.ndarray):
    t = np.ascontiguousarray(tap, np.float64)
    C_ = pred.out_dim
    prob = C.c_double()
    pr = np.zeros(C_, np.float64)
    lg = np.zeros(C_, np.float64)
    hit = orc().lco_lookup(pred.ptr, pred.n, sel.ptr, sel.n, delta, _dp(t), C.byref(prob), _dp(pr), _dp(lg))
    return bool(hit), prob.value, pr, lg


def oracle_serve_mlp(model: dict, caches: Sequence[tuple], x: np.ndarray):
    """serve_one over a parsed make_base_model network. caches: (layer, pred_layers, sel_layers, delta)."""
    base = OracleNet(model["layers"])
    tl = np.ascontiguousarray(model["tap_layers"], np.int32)
    cs = sorted(caches, key=lambda c: c[0])
    nets = [(OracleNet(p), OracleNet(s)) for _, p, s, _ in cs]
    carr = (LcoCache * max(1, len(cs)))()
    for k, (layer, _, _, delta) in enumerate(cs):
        carr[k].layer = layer
        carr[k].pred = nets[k][0].ptr
        carr[k].np = nets[k][0].n
        carr[k].sel = nets[k][1].ptr
        carr[k].ns = nets[k][1].n
        carr[k].delta = delta
    X = np.ascontiguousarray(x, np.float64)
    B = X.shape[0]
    L = model["blocks"]
    exit_l = np.zeros(B, np.int32)
    served = np.zeros(B, np.int32)
    base_p = np.zeros(B, np.int32)
    probs = np.zeros((B, L), np.float64)
    for i in range(B):
        e, s, b = C.c_int(), C.c_int(), C.c_int()
        row = np.ascontiguousarray(X[i])
        pr = np.zeros(L, np.float64)
        st = orc().lco_serve_mlp(base.ptr, base.n, _ip(tl), L, C.cast(carr, P), len(cs), _dp(row), C.byref(e),
                                 C.byref(s), C.byref(b), _dp(pr))
        assert st == 0
        exit_l[i], served[i], base_p[i] = e.value, s.value, b.value
        probs[i] = pr
    return exit_l, served, base_p, probs


def oracle_mlp_forward(model: dict, x: np.ndarray):
    """forward() over a parsed make_base_model network (network.cpp:104-164) with
    every activation kept: per block the post-ReLU tap (base_model.cpp:56-63,
    tap_layers) and the base logits = activations[size-2] (network.hpp:57-60).
    Returns (taps [blocks] -> [B][width], logits [B][classes])."""
    net = OracleNet(model["layers"])
    layers = model["layers"]
    offs = [layers[0]["in_dim"]]
    for l in layers:
        offs.append(offs[-1] + l["out_dim"])
    X = np.ascontiguousarray(x, np.float64)
    B = X.shape[0]
    taps = [np.zeros((B, model["tap_dims"][k]), np.float64) for k in range(model["blocks"])]
    logits = np.zeros((B, model["classes"]), np.float64)
    acts = np.zeros(offs[-1], np.float64)
    out = np.zeros(layers[-1]["out_dim"], np.float64)
    n = len(layers)
    for i in range(B):
        row = np.ascontiguousarray(X[i])
        assert orc().lco_forward(net.ptr, net.n, _dp(row), _dp(out), _dp(acts)) == 0
        for k, t in enumerate(model["tap_layers"]):
            taps[k][i] = acts[offs[t]:offs[t] + layers[t]["out_dim"]]
        logits[i] = acts[offs[n - 2]:offs[n - 2] + layers[n - 2]["out_dim"]]
    return taps, logits


def oracle_cnn_forward(ops: List[dict], nslots: int, x: np.ndarray, ntaps: int, tap_dims: Sequence[int],
                       classes: int, threads: int = 1):
    """lco_cnn_forward over the product's CNN op list (fp64, NCHW).
    Returns (taps [t] -> [B][dim], logits [B][classes])."""
    keep = []
    arr = (LcoCnnOp * len(ops))()
    buf_len = 0
    for i, o in enumerate(ops):
        e = arr[i]
        e.op = {0: 0, 1: 0, 2: 1, 3: 2}[o["kind"]]
        e.in_buf, e.out_buf, e.res_buf = o["in"], (o["out"] if o["kind"] != 3 else -1), o["res"]
        e.C, e.H, e.W, e.Cout = o["C"], o["H"], o["W"], o["Cout"]
        e.kh = e.kw = o["k"]
        e.stride, e.pad, e.relu, e.tap = o["stride"], o["pad"], o["relu"], o["tap"]
        for name in ("w", "scale", "shift"):
            a = o.get(name)
            if a is not None:
                a = np.ascontiguousarray(a, np.float64)
                keep.append(a)
                setattr(e, name, _dp(a))
        if o["kind"] in (0, 1):
            Ho = (o["H"] + 2 * o["pad"] - o["k"]) // o["stride"] + 1
            Wo = (o["W"] + 2 * o["pad"] - o["k"]) // o["stride"] + 1
            buf_len = max(buf_len, o["Cout"] * Ho * Wo)
        elif o["kind"] == 2:
            Ho = (o["H"] + 2 * o["pad"] - o["k"]) // o["stride"] + 1
            Wo = (o["W"] + 2 * o["pad"] - o["k"]) // o["stride"] + 1
            buf_len = max(buf_len, o["C"] * Ho * Wo)
    X = np.ascontiguousarray(x, np.float64)
    B = X.shape[0]
    taps = [np.zeros((B, d), np.float64) for d in tap_dims]
    tptr = (pD * max(1, ntaps))(*[_dp(t) for t in taps])
    tdims = (C.c_size_t * max(1, ntaps))(*tap_dims)
    logits = np.zeros((B, classes), np.float64)
    st = orc().lco_cnn_forward_batch(C.cast(arr, P), len(ops), nslots, buf_len, _dp(X), X.shape[1], B, ntaps, tptr,
                                     tdims, _dp(logits), classes, threads)
    assert st == 0
    return taps, logits


def softmax(x: np.ndarray) -> np.ndarray:
    out = np.zeros_like(x)
    orc().lco_softmax(_dp(np.ascontiguousarray(x, np.float64)), len(x), _dp(out))
    return out


def argmax(x: np.ndarray) -> int:
    return int(orc().lco_argmax(_dp(np.ascontiguousarray(x, np.float64)), len(x)))
