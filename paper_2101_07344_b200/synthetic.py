"""Synthetic deployments for configurations without trained caches.

The reference trains its caches (explore phase, cache.cpp:337-403); the
BASELINE configs are quoted on synthetic weights, where random selectors fire
all-or-nothing. Following the reference tests' force_selector
(test_serving.cpp:123-129), each chosen layer's selector output layer is
rescaled (gain) and its final bias placed so that a target fraction of a
calibration batch exits at that layer — a controlled exit profile.
"""
from __future__ import annotations

import math
from typing import Dict, List, Sequence

import numpy as np


def logit(p: float) -> float:
    return math.log(p) - math.log1p(-p)


def exit_profile(layers: Sequence[int], full_fraction: float) -> Dict[int, float]:
    """Fractions of the batch exiting at each cached layer (front-loaded,
    geometric), leaving `full_fraction` to run the whole model — e.g. the
    paper's full-DNN shares: R18 3.51 %, R50 1.53 %."""
    n = len(layers)
    w = np.array([0.8 ** i for i in range(n)])
    w = w / w.sum() * (1.0 - full_fraction)
    return {l: float(f) for l, f in zip(layers, w)}


def gains_for(z_raw: Dict[int, np.ndarray], target_std: float = 2.0) -> Dict[int, float]:
    """Gain that brings each layer's selector-logit spread to `target_std`."""
    out = {}
    for l, z in z_raw.items():
        s = float(np.std(z))
        out[l] = target_std / s if s > 1e-12 else 1.0
    return out


def calibrate_biases(z: Dict[int, np.ndarray], fractions: Dict[int, float], delta: float) -> Dict[int, float]:
    """Sequential calibration: at each layer (ascending) the top round(f*N)
    of the still-unserved requests fire. z: selector logits with bias 0
    (after gain). Thresholds sit midway between neighbouring logits so the
    calibration batch keeps a margin from delta."""
    layers = sorted(z)
    N = len(z[layers[0]])
    remaining = np.ones(N, bool)
    biases = {}
    for l in layers:
        zl = np.asarray(z[l], np.float64)
        cand = np.sort(zl[remaining])[::-1]
        k = min(int(round(fractions.get(l, 0.0) * N)), len(cand))
        if len(cand) == 0 or k == 0:
            t = (cand[0] if len(cand) else 0.0) + 1.0
        elif k == len(cand):
            t = cand[-1] - 1.0
        else:
            t = 0.5 * (cand[k - 1] + cand[k])
        biases[l] = logit(delta) - t
        remaining &= ~(zl >= t)
    return biases


def selector_logits_from_probs(p: np.ndarray) -> np.ndarray:
    q = np.clip(np.asarray(p, np.float64), 1e-7, 1 - 1e-7)
    return np.log(q) - np.log1p(-q)


def calibrate_variants(model, variants, calib_x: np.ndarray, full_fraction: float, delta: float = 0.5,
                       precision: str = "bf16x3", device: int = 0):
    """Set each variant's selector gain/bias (host objects, in place) so the
    calibration batch follows exit_profile(); returns the fractions used.
    Uses one shadow-mode pass on the GPU to read every layer's selector output."""
    from .api import Deployment
    for v in variants:
        v.delta = delta
    B = calib_x.shape[0]
    dep = Deployment(model, variants, precision=precision, max_batch=B, device=device)
    res = dep.serve(calib_x, shadow=True)
    dep.close()
    layers = sorted(v.layer for v in variants)
    z = {l: selector_logits_from_probs(res.probs[l - 1]) for l in layers}
    # selectors start with zero final bias (make_network), so z is linear in the gain
    gains = gains_for(z)
    fr = exit_profile(layers, full_fraction)
    biases = calibrate_biases({l: z[l] * gains[l] for l in layers}, fr, delta)
    for v in variants:
        v.set_selector_out(gains[v.layer], biases[v.layer])
    return fr


def mlp_inputs(B: int, dim: int, seed: int) -> np.ndarray:
    """Uniform [-1.5, 1.5) inputs (test_util.hpp:73-77 random_vec)."""
    return np.random.default_rng(seed).uniform(-1.5, 1.5, size=(B, dim))


def image_inputs(B: int, C: int, H: int, W: int, seed: int) -> np.ndarray:
    """i.i.d. N(0,1) NCHW images, flattened per request."""
    return np.random.default_rng(seed).standard_normal((B, C * H * W))


C1_WIDTHS = [64, 64, 128, 128, 256, 256, 512, 512]  # ResNet-18 CIFAR stage widths as MLP widths
C1_MENU = ["FC(1024)", "Pool(8192)", "Conv(3,1)", "FC(512)", "Pool(4096)", "Conv(5,2)", "FC(1024)", "Pool(8192)"]
