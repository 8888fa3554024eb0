"""Python face of the B200 learned-cache serve path, mirroring the reference's
C++ API (namespace latecache) over the C-ABI in include/latecache_b200.h.

Reference name            -> here
  make_base_model          base_model.cpp:30      make_base_model()
  load_base_model          base_model.cpp:156     load_base_model()
  save_base_model          base_model.cpp:143     BaseModel.save()
  build_variant            cache.cpp:104          build_variant()
  load_variant/save_variant cache.cpp:464/452     load_variant() / CacheVariant.save()
  CacheVariant::delta      cache.hpp:63           CacheVariant.delta
  lookup                   cache.cpp:259          Deployment.lookup()  (batched, on the GPU)
  Deployment               serving.hpp:61         Deployment (device-resident)
  simulate_model/serve_one serving.cpp:147/97     Deployment.serve() / simulate_model()
  gen_workload             serving.cpp:61         gen_workload()
  summarize (nearest-rank) serving.cpp:342        summarize()
Exceptions: std::invalid_argument -> ValueError, std::runtime_error ->
RuntimeError (same messages as the reference where it has them).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence

import numpy as np

from ._lib import (AdaptConfig, RetrainEventC, LC_PREC_BF16, LC_PREC_BF16X3, LC_SERVE_NO_GRAPH, LC_SERVE_SHADOW, CnnOpDesc, check, lib,
                   take_bytes, take_string)

_PREC = {"bf16x3": LC_PREC_BF16X3, "bf16": LC_PREC_BF16}


def _iptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_int))


def _fptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_float))


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


# ---------------------------------------------------------------- base model
class BaseModel:
    """latecache::BaseModel (base_model.hpp:31-39); also the CNN families."""

    def __init__(self, handle: C.c_void_p):
        self._h = handle
        blocks, classes, dim = C.c_int(), C.c_int(), C.c_longlong()
        check(lib.lc_model_info(self._h, C.byref(blocks), C.byref(classes), C.byref(dim)))
        self.num_blocks = blocks.value
        self.num_classes = classes.value
        self.input_dim = dim.value

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib.lc_model_free(h)
            self._h = None

    def save(self) -> str:
        p, n = C.c_void_p(), C.c_size_t()
        check(lib.lc_model_save(self._h, C.byref(p), C.byref(n)))
        return take_string(p, n)

    def save_binary(self) -> bytes:
        """Binary checkpoint (raw doubles; CNN op lists included)."""
        p, n = C.c_void_p(), C.c_size_t()
        check(lib.lc_model_save_binary(self._h, C.byref(p), C.byref(n)))
        return take_bytes(p, n)

    def tap(self, layer: int):
        c, h, w = C.c_int(), C.c_int(), C.c_int()
        check(lib.lc_model_tap(self._h, layer, C.byref(c), C.byref(h), C.byref(w)))
        return c.value, h.value, w.value

    def tap_dim(self, layer: int) -> int:
        c, h, w = self.tap(layer)
        return c * h * w

    @property
    def tap_dims(self) -> List[int]:
        return [self.tap_dim(i + 1) for i in range(self.num_blocks)]

    def macs(self, block: int) -> int:
        return int(lib.lc_model_macs(self._h, block))

    def cnn_ops(self) -> List[dict]:
        n, s = C.c_int(), C.c_int()
        check(lib.lc_model_cnn_ops(self._h, C.byref(n), C.byref(s)))
        out = []
        for i in range(n.value):
            d = CnnOpDesc()
            check(lib.lc_model_cnn_op(self._h, i, C.byref(d)))
            op = {k: getattr(d, k) for k in ("kind", "out", "res", "C", "H", "W", "Cout", "k", "stride", "pad",
                                               "relu", "tap")}
            op["in"] = d.in_
            op["w"] = np.ctypeslib.as_array(d.w, shape=(d.w_len,)).copy() if d.w else None
            cnt = d.Cout if op["kind"] in (0, 1, 3) else 0
            op["scale"] = np.ctypeslib.as_array(d.scale, shape=(cnt,)).copy() if d.scale else None
            op["shift"] = np.ctypeslib.as_array(d.shift, shape=(cnt,)).copy() if d.shift else None
            out.append(op)
        self.nslots = s.value
        return out


def make_base_model(input_dim: int, num_classes: int, widths: Sequence[int], blocks: int, seed: int) -> BaseModel:
    w = np.ascontiguousarray(widths, dtype=np.int32)
    h = C.c_void_p()
    check(lib.lc_model_make_mlp(input_dim, num_classes, _iptr(w), len(w), blocks, C.c_uint64(seed), C.byref(h)))
    return BaseModel(h)


def load_base_model(text: str) -> BaseModel:
    b = text.encode()
    h = C.c_void_p()
    check(lib.lc_model_load(b, len(b), C.byref(h)))
    return BaseModel(h)


def load_base_model_binary(data: bytes) -> BaseModel:
    h = C.c_void_p()
    check(lib.lc_model_load_binary(data, len(data), C.byref(h)))
    return BaseModel(h)


def make_cnn_model(arch: str, num_classes: int, seed: int) -> BaseModel:
    h = C.c_void_p()
    check(lib.lc_model_make_cnn(arch.encode(), num_classes, C.c_uint64(seed), C.byref(h)))
    return BaseModel(h)


# ---------------------------------------------------------------- variants
@dataclass
class NetLayer:
    kind: int
    in_dim: int
    out_dim: int
    pool_window: int
    kernel: int
    stride: int
    w: Optional[np.ndarray]
    b: Optional[np.ndarray]


class CacheVariant:
    """latecache::CacheVariant (cache.hpp:57-64)."""

    def __init__(self, handle: C.c_void_p):
        self._h = handle

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib.lc_variant_free(h)
            self._h = None

    def _info(self):
        layer, vi, delta = C.c_int(), C.c_int(), C.c_double()
        buf = C.create_string_buffer(64)
        check(lib.lc_variant_info(self._h, C.byref(layer), C.byref(vi), C.byref(delta), buf, 64))
        return layer.value, vi.value, delta.value, buf.value.decode()

    @property
    def layer(self) -> int:
        return self._info()[0]

    @property
    def variant(self) -> int:
        return self._info()[1]

    @property
    def arch(self) -> str:
        return self._info()[3]

    @property
    def delta(self) -> float:
        return self._info()[2]

    @delta.setter
    def delta(self, value: float) -> None:
        check(lib.lc_variant_set_delta(self._h, float(value)))

    def macs(self) -> int:
        return int(lib.lc_variant_macs(self._h))

    def save(self) -> str:
        p, n = C.c_void_p(), C.c_size_t()
        check(lib.lc_variant_save(self._h, C.byref(p), C.byref(n)))
        return take_string(p, n)

    def save_binary(self) -> bytes:
        p, n = C.c_void_p(), C.c_size_t()
        check(lib.lc_variant_save_binary(self._h, C.byref(p), C.byref(n)))
        return take_bytes(p, n)

    def layers(self, which: int) -> List[NetLayer]:
        """which = 0: predictor, 1: selector; weights copied out as fp64 arrays."""
        out = []
        i = 0
        while True:
            vals = [C.c_int() for _ in range(6)]
            w, b = C.POINTER(C.c_double)(), C.POINTER(C.c_double)()
            wl, bl = C.c_longlong(), C.c_longlong()
            st = lib.lc_variant_layer(self._h, which, i, *[C.byref(v) for v in vals], C.byref(w), C.byref(wl),
                                      C.byref(b), C.byref(bl))
            if st != 0:
                break
            wa = np.ctypeslib.as_array(w, shape=(wl.value,)).copy() if wl.value else None
            ba = np.ctypeslib.as_array(b, shape=(bl.value,)).copy() if bl.value else None
            out.append(NetLayer(*[v.value for v in vals], wa, ba))
            i += 1
        return out

    def set_selector_out(self, gain: float, bias: float) -> None:
        check(lib.lc_variant_set_selector_out(self._h, float(gain), float(bias)))


def build_variant(layer: int, variant_idx: int, arch: str, tap_dim: int, num_classes: int, seed: int) -> CacheVariant:
    h = C.c_void_p()
    check(lib.lc_variant_build(layer, variant_idx, arch.encode(), tap_dim, num_classes, C.c_uint64(seed), C.byref(h)))
    return CacheVariant(h)


def load_variant(text: str) -> CacheVariant:
    b = text.encode()
    h = C.c_void_p()
    check(lib.lc_variant_load(b, len(b), C.byref(h)))
    return CacheVariant(h)


def load_variant_binary(data: bytes) -> CacheVariant:
    h = C.c_void_p()
    check(lib.lc_variant_load_binary(data, len(data), C.byref(h)))
    return CacheVariant(h)


# ---------------------------------------------------------------- plan / workload
def with_measured_lookup_ms(metrics_text: str, lookup_ms: Dict[int, float]) -> str:
    """The reference metrics file (cache.cpp:412-450; columns layer variant arch
    hit_rate accuracy lookup_ms memory_mb tp fp tn fn) with the modeled
    lookup_ms of every row at a measured layer replaced by the device time."""
    out = []
    for line in metrics_text.split("\n"):
        f = line.split()
        if len(f) >= 11 and not line.startswith("#") and f[0].lstrip("-").isdigit() and int(f[0]) in lookup_ms:
            f[5] = repr(float(lookup_ms[int(f[0])]))
            line = " ".join(f)
        out.append(line)
    return "\n".join(out)


def plan_check(metrics_text: str, plan_text: str, profile_ms: Sequence[float], accuracy_threshold: float,
               memory_budget_mb: float):
    """load_metrics + load_plan + check_constraints; returns (feasible, violations, [(layer, variant)])."""
    prof = np.ascontiguousarray(profile_ms, dtype=np.float64)
    feas, n = C.c_int(), C.c_int()
    layers = np.zeros(256, np.int32)
    variants = np.zeros(256, np.int32)
    rep = C.c_void_p()
    check(lib.lc_plan_check(metrics_text.encode(), plan_text.encode(), _dptr(prof), len(prof), accuracy_threshold,
                            memory_budget_mb, C.byref(feas), _iptr(layers), _iptr(variants), 256, C.byref(n),
                            C.byref(rep)))
    report = C.string_at(rep).decode()
    lib.lc_free(rep)
    viol = [v for v in report.split("\n") if v]
    return bool(feas.value), viol, list(zip(layers[:n.value].tolist(), variants[:n.value].tolist()))


@dataclass
class Request:
    id: int
    time_min: float
    true_class: int
    sample_idx: int


def gen_workload(labels: Sequence[int], dataset_classes: int, num_classes: int = 10, zipf_alpha: float = 1.5,
                 rotation_period_min: float = 15.0, requests_per_sec: float = 2.0, duration_min: float = 60.0,
                 seed: int = 1) -> List[Request]:
    lab = np.ascontiguousarray(labels, dtype=np.int32)
    n = C.c_longlong()
    cap = int(round(requests_per_sec * duration_min * 60.0)) + 1
    si = np.zeros(cap, np.int64)
    tc = np.zeros(cap, np.int32)
    tm = np.zeros(cap, np.float64)
    check(lib.lc_gen_workload(num_classes, zipf_alpha, rotation_period_min, requests_per_sec, duration_min,
                              C.c_uint64(seed), _iptr(lab), len(lab), dataset_classes, C.byref(n),
                              si.ctypes.data_as(C.POINTER(C.c_longlong)), _iptr(tc), _dptr(tm), cap))
    return [Request(i, float(tm[i]), int(tc[i]), int(si[i])) for i in range(n.value)]


def nearest_rank(values: Sequence[float], q: float) -> float:
    v = np.ascontiguousarray(values, dtype=np.float64)
    return float(lib.lc_nearest_rank(_dptr(v), len(v), q))


# ---------------------------------------------------------------- deployment
@dataclass
class ServeResult:
    exit_layer: np.ndarray  # 0 = miss (served by the base model)
    served: np.ndarray
    base_pred: np.ndarray   # -1 where compaction skipped the full pass
    probs: np.ndarray       # [blocks][B] selector probability per probed layer (NaN = not probed)
    latency_ms: np.ndarray  # device time from batch start to the request's exit
    logits: np.ndarray = None  # [B][classes] base logits (NaN rows where compaction skipped the full pass)


class Deployment:
    """A latecache::Deployment resident on one B200 (serving.hpp:61-69)."""

    def __init__(self, model: BaseModel, variants: Sequence[CacheVariant], precision: str = "bf16x3",
                 max_batch: int = 256, device: int = 0):
        arr = (C.c_void_p * max(1, len(variants)))(*[v._h for v in variants])
        h = C.c_void_p()
        check(lib.lc_engine_create(device, model._h, arr, len(variants), _PREC[precision], max_batch, C.byref(h)))
        self._h = h
        self.model = model
        # the engine probes (and indexes) its caches in ascending layer order
        # (make_plan, composer.cpp:65-89); keep the same order here so every
        # per-cache array (run_adaptation's original_taps, variant(k)) lines up
        self.variants = sorted(variants, key=lambda v: v.layer)
        self.precision = precision
        self.max_batch = max_batch
        self.blocks = model.num_blocks
        self.classes = model.num_classes

    def close(self):
        h = getattr(self, "_h", None)
        if h:
            check(lib.lc_engine_destroy(h))
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_delta(self, layer: int, delta: float) -> None:
        check(lib.lc_engine_set_delta(self._h, layer, float(delta)))

    def set_selector_out(self, layer: int, gain: float, bias: float) -> None:
        check(lib.lc_engine_set_selector_out(self._h, layer, float(gain), float(bias)))

    def update_variant(self, variant: CacheVariant) -> None:
        """Swap a retrained variant in for the cache at its layer (after every
        batch already enqueued; serving.cpp:301-315)."""
        check(lib.lc_engine_update_variant(self._h, variant._h))

    def set_swap_hook(self, fn) -> None:
        """fn(swap_time_min) after each swap run_adaptation lands (serving.cpp:303-315):
        requests at time >= swap_time_min are served by the caches variant(k)
        returns at that moment. None clears. (lc_engine_set_swap_hook)"""
        from ._lib import SWAP_HOOK
        if fn is None:
            self._swap_cb = None
            check(lib.lc_engine_set_swap_hook(self._h, SWAP_HOOK(), None))
            return
        self._swap_cb = SWAP_HOOK(lambda _ctx, t: fn(float(t)))  # kept alive with the deployment
        check(lib.lc_engine_set_swap_hook(self._h, self._swap_cb, None))

    def variant(self, k: int) -> CacheVariant:
        """Copy of the k-th attached variant (probe order: ascending layer) as the engine holds it."""
        h = C.c_void_p()
        check(lib.lc_engine_variant(self._h, k, C.byref(h)))
        return CacheVariant(h)

    def input_ptr(self) -> int:
        p = C.c_void_p()
        check(lib.lc_engine_input(self._h, C.byref(p)))
        return int(p.value)

    def serve(self, inputs: np.ndarray, shadow: bool = False, graph: bool = True) -> ServeResult:
        x = np.ascontiguousarray(inputs, dtype=np.float32)
        B = x.shape[0]
        el = np.zeros(B, np.int32)
        sv = np.zeros(B, np.int32)
        bp = np.zeros(B, np.int32)
        pr = np.zeros((self.blocks, B), np.float32)
        lg = np.zeros((B, self.classes), np.float32)
        lat = np.zeros(B, np.float64)
        flags = (LC_SERVE_SHADOW if shadow else 0) | (0 if graph else LC_SERVE_NO_GRAPH)
        check(lib.lc_serve_batch(self._h, _fptr(x), B, flags, _iptr(el), _iptr(sv), _iptr(bp), _fptr(pr), _fptr(lg),
                                 _dptr(lat)))
        return ServeResult(el, sv, bp, pr, lat, lg)

    def read_tap(self, inputs: np.ndarray, layer: int) -> np.ndarray:
        """forward_with_taps (base_model.cpp:56-63): the tap of block `layer` for
        each input, [B][tap_dim] fp32 NCHW-flat, as the reference's caches see it."""
        x = np.ascontiguousarray(inputs, dtype=np.float32)
        B = x.shape[0]
        out = np.zeros((B, self.model.tap_dim(layer)), np.float32)
        check(lib.lc_engine_read_tap(self._h, _fptr(x), B, layer, _fptr(out)))
        return out

    def submit(self, inputs: np.ndarray, shadow: bool = False) -> tuple:
        """Pipelined serve: enqueue one batch (H2D on a copy stream overlapping the
        previous batch's compute) and return a ticket for collect(). `inputs`
        should live in pinned host memory (e.g. a torch pin_memory() tensor's
        numpy view) for the copy to be asynchronous; it must stay alive until collect."""
        x = np.ascontiguousarray(inputs, dtype=np.float32)
        slot = C.c_int()
        check(lib.lc_serve_submit(self._h, _fptr(x), x.shape[0], LC_SERVE_SHADOW if shadow else 0, C.byref(slot)))
        return (slot.value, x.shape[0], x)

    def collect(self, ticket: tuple) -> ServeResult:
        slot, B, _ = ticket
        el = np.zeros(B, np.int32)
        sv = np.zeros(B, np.int32)
        bp = np.zeros(B, np.int32)
        pr = np.zeros((self.blocks, B), np.float32)
        lg = np.zeros((B, self.classes), np.float32)
        lat = np.zeros(B, np.float64)
        check(lib.lc_serve_collect(self._h, slot, B, _iptr(el), _iptr(sv), _iptr(bp), _fptr(pr), _fptr(lg),
                                   _dptr(lat)))
        return ServeResult(el, sv, bp, pr, lat, lg)

    def stage_input_device(self, src_ptr: int, B: int) -> None:
        """Copy B inputs from device memory (raw pointer) into the engine's input buffer."""
        check(lib.lc_engine_stage_input(self._h, C.c_void_p(src_ptr), B, 1))

    def serve_device(self, B: int, shadow: bool = False, graph: bool = True) -> None:
        flags = (LC_SERVE_SHADOW if shadow else 0) | (0 if graph else LC_SERVE_NO_GRAPH)
        check(lib.lc_serve_device(self._h, B, flags))

    def sync(self) -> None:
        check(lib.lc_engine_sync(self._h))

    def serve_timed(self, B: int, shadow: bool = False) -> float:
        """One batch from the device input buffer; device ms (CUDA events on the engine stream)."""
        ms = C.c_double()
        check(lib.lc_serve_timed(self._h, B, LC_SERVE_SHADOW if shadow else 0, C.byref(ms)))
        return ms.value

    def results(self, B: int) -> ServeResult:
        el = np.zeros(B, np.int32)
        sv = np.zeros(B, np.int32)
        bp = np.zeros(B, np.int32)
        pr = np.zeros((self.blocks, B), np.float32)
        lg = np.zeros((B, self.classes), np.float32)
        lat = np.zeros(B, np.float64)
        check(lib.lc_engine_results(self._h, B, _iptr(el), _iptr(sv), _iptr(bp), _fptr(pr), _fptr(lg), _dptr(lat)))
        return ServeResult(el, sv, bp, pr, lat, lg)

    def counts(self) -> np.ndarray:
        c = np.zeros(self.blocks + 1, np.int32)
        check(lib.lc_engine_counts(self._h, _iptr(c)))
        return c

    def lookup(self, layer: int, taps: np.ndarray) -> Dict[str, np.ndarray]:
        """Batched reference lookup() (cache.cpp:259-265) on NCHW-flat taps [B][tap_dim]."""
        t = np.ascontiguousarray(taps, dtype=np.float32)
        B = t.shape[0]
        hit = np.zeros(B, np.int32)
        label = np.zeros(B, np.int32)
        prob = np.zeros(B, np.float32)
        pr = np.zeros((B, self.classes), np.float32)
        lg = np.zeros((B, self.classes), np.float32)
        check(lib.lc_lookup_batch(self._h, layer, _fptr(t), B, _iptr(hit), _iptr(label), _fptr(prob), _fptr(pr),
                                  _fptr(lg)))
        return {"hit": hit, "label": label, "prob": prob, "pr": pr, "logits": lg}

    def measure_metrics(self, inputs: np.ndarray, deltas: Sequence[float] = None) -> Dict[int, List[Dict]]:
        """Batched measure_metrics (cache.cpp:316-335) of every attached cache at
        every threshold in `deltas` (default: each variant's own delta) over one
        shadow serve of `inputs`: {layer: [{delta, tp, fp, tn, fn, hit_rate,
        accuracy}, ...]} with the reference's definitions (hit_rate =
        (tp+fp)/total, accuracy = tp/(tp+fp), 1 when nothing hits)."""
        x = np.ascontiguousarray(inputs, dtype=np.float32)
        B = x.shape[0]
        if deltas is None:
            grid = sorted({float(v.delta) for v in self.variants})
        else:
            grid = [float(d) for d in deltas]
        g = np.ascontiguousarray(grid, np.float64)
        cnt = np.zeros((self.blocks, len(g), 4), np.int64)
        check(lib.lc_measure_metrics(self._h, _fptr(x), B, _dptr(g), len(g),
                                     cnt.ctypes.data_as(C.POINTER(C.c_longlong))))
        out = {}
        own = {v.layer: float(v.delta) for v in self.variants}
        for v in self.variants:
            rows = []
            for j, d in enumerate(grid):
                if deltas is None and d != own[v.layer]:
                    continue
                tp, fp, tn, fn = (int(c) for c in cnt[v.layer - 1, j])
                hits = tp + fp
                total = tp + fp + tn + fn
                rows.append({"delta": d, "tp": tp, "fp": fp, "tn": tn, "fn": fn,
                             "hit_rate": hits / total if total else 0.0,
                             "accuracy": tp / hits if hits else 1.0})
            out[v.layer] = rows
        return out

    def tune_delta(self, inputs: np.ndarray, target_accuracy: float, grid: Sequence[float],
                   apply: bool = True) -> Dict[int, float]:
        """Batched tune_delta (cache.cpp:267-307) for every attached cache: the
        smallest threshold of `grid` whose hit accuracy reaches the target (else
        the most accurate). apply: set the engine's thresholds (and the variants')."""
        x = np.ascontiguousarray(inputs, dtype=np.float32)
        g = np.ascontiguousarray(list(grid), np.float64)
        d = np.zeros(self.blocks, np.float64)
        check(lib.lc_tune_delta(self._h, _fptr(x), x.shape[0], float(target_accuracy), _dptr(g), len(g), _dptr(d),
                                1 if apply else 0))
        out = {v.layer: float(d[v.layer - 1]) for v in self.variants}
        if apply:
            for v in self.variants:
                v.delta = out[v.layer]
        return out

    def layer_times(self, inputs: np.ndarray, shadow: bool = True):
        """Hardware-aware profile: device-measured base time
        per block (the LayerProfile) and lookup time per cache layer (the
        VariantMetrics::lookup_ms column) from one shadow batch of `inputs`
        (shadow=False: the compacted step, survivors only)."""
        x = np.ascontiguousarray(inputs, dtype=np.float32)
        bm = np.zeros(self.blocks, np.float64)
        lm = np.zeros(self.blocks, np.float64)
        check(lib.lc_engine_layer_times(self._h, _fptr(x), x.shape[0], LC_SERVE_SHADOW if shadow else 0, _dptr(bm),
                                        _dptr(lm)))
        return bm, {v.layer: float(lm[v.layer - 1]) for v in self.variants}

    def time_batch(self, B: int, iters: int, shadow: bool = False) -> float:
        ms = C.c_double()
        check(lib.lc_engine_time(self._h, B, LC_SERVE_SHADOW if shadow else 0, iters, C.byref(ms)))
        return ms.value

    def kernel_count(self, shadow: bool = False, kind: int = -1) -> int:
        return int(lib.lc_engine_kernel_count(self._h, LC_SERVE_SHADOW if shadow else 0, kind))

    def profile(self, B: int, shadow: bool = False) -> Dict[str, np.ndarray]:
        """Per-step device ms + algorithmic FLOPs/bytes of one batch (no graph).
        kind: 0 other, 1 tensor-core contraction, 2 lookup, 3 exit/compaction."""
        cap = 4096
        n = C.c_int()
        kinds = np.zeros(cap, np.int32)
        ms = np.zeros(cap)
        fl = np.zeros(cap)
        by = np.zeros(cap)
        check(lib.lc_engine_profile(self._h, B, LC_SERVE_SHADOW if shadow else 0, cap, C.byref(n), _iptr(kinds),
                                    _dptr(ms), _dptr(fl), _dptr(by)))
        k = n.value
        return {"kind": kinds[:k], "ms": ms[:k], "flops": fl[:k], "bytes": by[:k]}


@dataclass
class RequestTrace:
    id: int
    time_min: float
    true_class: int
    base_pred: int
    served_pred: int
    hit_layer: int
    latency_ms: float


def simulate_model(dep: Deployment, inputs: np.ndarray, stream: Sequence[Request], batch: Optional[int] = None,
                   shadow: bool = True) -> List[RequestTrace]:
    """simulate_model (serving.cpp:147-158) batched on the GPU: request i
    serves inputs[stream[i].sample_idx]. latency_ms is the measured device
    time to the request's exit within its batch (the reference models it)."""
    batch = batch or dep.max_batch
    traces: List[RequestTrace] = []
    for s in range(0, len(stream), batch):
        chunk = stream[s:s + batch]
        x = inputs[[r.sample_idx for r in chunk]]
        res = dep.serve(x, shadow=shadow)
        for j, r in enumerate(chunk):
            traces.append(RequestTrace(r.id, r.time_min, r.true_class, int(res.base_pred[j]), int(res.served[j]),
                                       int(res.exit_layer[j]), float(res.latency_ms[j])))
    return traces


@dataclass
class SimSummary:
    requests: int
    avg_latency_ms: float
    p50_latency_ms: float
    p99_latency_ms: float
    max_latency_ms: float
    agreement: float
    accuracy: float
    hit_rate: float
    hits_by_layer: Dict[int, int] = field(default_factory=dict)


def summarize(traces: Sequence[RequestTrace]) -> SimSummary:
    """summarize (serving.cpp:342-376); percentiles nearest-rank. Agreement
    counts only requests whose base prediction is known (shadow mode: all)."""
    if not traces:
        raise ValueError("summarize: no traces")
    lat = [t.latency_ms for t in traces]
    n = len(traces)
    known = [t for t in traces if t.base_pred >= 0]
    hits: Dict[int, int] = {}
    for t in traces:
        if t.hit_layer > 0:
            hits[t.hit_layer] = hits.get(t.hit_layer, 0) + 1
    return SimSummary(
        requests=n, avg_latency_ms=sum(lat) / n, p50_latency_ms=nearest_rank(lat, 0.50),
        p99_latency_ms=nearest_rank(lat, 0.99), max_latency_ms=max(lat),
        agreement=(sum(t.served_pred == t.base_pred for t in known) / len(known)) if known else float("nan"),
        accuracy=sum(t.served_pred == t.true_class for t in traces) / n,
        hit_rate=sum(t.hit_layer > 0 for t in traces) / n, hits_by_layer=hits)


# ---------------------------------------------------------------- retraining / adaptation
@dataclass
class TrainConfig:
    """latecache::TrainConfig (network.hpp:70-76)."""
    learning_rate: float = 0.01
    momentum: float = 0.9
    epochs: int = 20
    batch_size: int = 16
    seed: int = 1


def _records(taps: np.ndarray, y: np.ndarray, sample_weights):
    t = np.ascontiguousarray(taps, np.float64)
    yy = np.ascontiguousarray(y, np.float64)
    if t.ndim != 2 or yy.ndim != 2 or t.shape[0] != yy.shape[0]:
        raise ValueError("records: taps [N][D] and y [N][C] must have the same N")
    w = None if sample_weights is None else np.ascontiguousarray(sample_weights, np.float64)
    if w is not None and w.shape != (t.shape[0],):  # the C-ABI reads exactly N weights
        raise ValueError("train: sample weight count mismatch")
    return t, yy, w


def train_predictor(variant: CacheVariant, taps: np.ndarray, y: np.ndarray, cfg: TrainConfig = TrainConfig(),
                    tau: float = 2.0, beta: float = 0.5, sample_weights=None, device: int = 0) -> None:
    """train_predictor (cache.cpp:179-208) on the GPU, in place: taps [N][D] at
    the variant's layer, y [N][C] base-model distributions."""
    t, yy, w = _records(taps, y, sample_weights)
    check(lib.lc_train_predictor(device, variant._h, _dptr(t), t.shape[1], _dptr(yy), yy.shape[1], t.shape[0],
                                 None if w is None else _dptr(w), cfg.learning_rate, cfg.momentum, cfg.epochs,
                                 cfg.batch_size, C.c_uint64(cfg.seed), tau, beta))


def train_selector(variant: CacheVariant, taps: np.ndarray, y: np.ndarray, cfg: TrainConfig = TrainConfig(),
                   w_fp: float = 5.0, w_fn: float = 1.0, sample_weights=None, device: int = 0) -> None:
    """train_selector (cache.cpp:220-257) on the GPU, in place."""
    t, yy, w = _records(taps, y, sample_weights)
    check(lib.lc_train_selector(device, variant._h, _dptr(t), t.shape[1], _dptr(yy), yy.shape[1], t.shape[0],
                                None if w is None else _dptr(w), cfg.learning_rate, cfg.momentum, cfg.epochs,
                                cfg.batch_size, C.c_uint64(cfg.seed), w_fp, w_fn))


@dataclass
class AdaptationConfig:
    """AdaptationConfig (serving.hpp:85-94) plus the CacheTrainConfig fields the
    retrain uses (cache.hpp:92-100)."""
    sample_rate: float = 0.2
    window_min: float = 60.0
    retrain_interval_min: float = 15.0
    recency_decay: float = 0.7
    mixin_fraction: float = 0.5
    epochs: int = 5
    learning_rate: float = 0.002
    retrain_pause_ms: float = 0.0
    tau: float = 2.0
    beta: float = 0.5
    w_fp: float = 5.0
    w_fn: float = 1.0


@dataclass
class RetrainEvent:
    interval: int
    time_min: float
    window_size: int
    mixin_size: int
    applied: bool
    note: str


@dataclass
class IntervalStat:
    interval: int
    requests: int = 0
    hits: int = 0

    def hit_rate(self) -> float:
        return 0.0 if self.requests == 0 else self.hits / self.requests


@dataclass
class AdaptationResult:
    traces: List[RequestTrace]
    timeline: List[IntervalStat]
    retrains: List[RetrainEvent]
    final_variants: List[CacheVariant]


def run_adaptation(dep: Deployment, inputs: np.ndarray, labels: Sequence[int], stream: Sequence[Request],
                   cfg: AdaptationConfig, original_taps: Sequence[np.ndarray], original_y: np.ndarray, seed: int,
                   adapt_on: bool = True) -> AdaptationResult:
    """run_adaptation (serving.cpp:213-340) on the GPU: shadow-batched serving
    between control points, window records read back from the device, GPU
    retraining and in-place swaps. original_taps[k] = [N0][D_k] for the k-th
    attached cache in probe order (ascending layer, = dep.variants[k]),
    original_y [N0][C]. The engine ends holding the final
    variants (also returned)."""
    x = np.ascontiguousarray(inputs, np.float32)
    R = len(stream)
    times = np.ascontiguousarray([r.time_min for r in stream], np.float64)
    samp = np.ascontiguousarray([r.sample_idx for r in stream], np.int32)
    oy = np.ascontiguousarray(original_y, np.float64)
    N0 = oy.shape[0] if oy.ndim == 2 else 0
    ot = [np.ascontiguousarray(t, np.float64) for t in original_taps]
    if N0:  # the C-ABI reads N0 rows of every attached cache's tap array
        if len(ot) != len(dep.variants):
            raise ValueError("run_adaptation: one original tap array per attached cache is required")
        for t, v in zip(ot, dep.variants):
            if t.shape != (N0, dep.model.tap_dim(v.layer)):
                raise ValueError("run_adaptation: original record shape mismatch")
        if oy.shape[1] != dep.classes:
            raise ValueError("run_adaptation: original record shape mismatch")
    tp = (C.POINTER(C.c_double) * max(1, len(ot)))(*[_dptr(t) for t in ot])
    c = AdaptConfig(cfg.sample_rate, cfg.window_min, cfg.retrain_interval_min, cfg.recency_decay,
                    cfg.mixin_fraction, cfg.epochs, cfg.learning_rate, cfg.retrain_pause_ms, cfg.tau, cfg.beta,
                    cfg.w_fp, cfg.w_fn)
    hl, sv, bp = np.zeros(R, np.int32), np.zeros(R, np.int32), np.zeros(R, np.int32)
    lat = np.zeros(R, np.float64)
    cap = 4096
    evs = (RetrainEventC * cap)()
    n = C.c_int()
    check(lib.lc_run_adaptation(dep._h, _fptr(x), x.shape[0], _dptr(times), _iptr(samp), R, C.byref(c), tp,
                                _dptr(oy) if N0 else None, N0, C.c_uint64(seed), 1 if adapt_on else 0, _iptr(hl),
                                _iptr(sv), _iptr(bp), _dptr(lat), evs, cap, C.byref(n)))
    traces = [RequestTrace(r.id, r.time_min, int(labels[r.sample_idx]), int(bp[i]), int(sv[i]), int(hl[i]),
                           float(lat[i])) for i, r in enumerate(stream)]
    timeline: List[IntervalStat] = []
    for t in traces:  # serving.cpp:321-327
        iv = int(t.time_min / cfg.retrain_interval_min)
        if not timeline or timeline[-1].interval < iv:
            timeline.append(IntervalStat(iv))
        timeline[-1].requests += 1
        timeline[-1].hits += 1 if t.hit_layer > 0 else 0
    retrains = [RetrainEvent(e.interval, e.time_min, e.window_size, e.mixin_size, bool(e.applied),
                             e.note.decode()) for e in evs[:min(n.value, cap)]]
    finals = [dep.variant(k) for k in range(len(dep.variants))]
    return AdaptationResult(traces, timeline, retrains, finals)
