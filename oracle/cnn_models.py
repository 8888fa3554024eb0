"""TEST INFRASTRUCTURE ONLY — the synthetic CNN base models of BASELINE.json
rebuilt on the CPU without the product library.

The reference has no CNN; the build's own layer definitions live
in paper_2101_07344_b200/csrc/host/cnn.cpp. This module restates that builder
(op order, geometry, the He-normal / folded-BN / Glorot draws from the
reference RNG, rng.hpp:15-98, restated in oracle/lc_oracle.c) so that
`bench.py --impl reference` and the CPU baseline can construct the same
network as the product's `make_cnn_model(arch, classes, seed)` — identical
weights, bit for bit (tests/test_oracle.py pins it) — without importing or
loading the product. Output: op dicts in the format of
`BaseModel.cnn_ops()`, consumed by `oracle.oracle_cnn_forward`.
"""
import ctypes as C
import math
from typing import List, Tuple

import numpy as np

from oracle.oracle import _dp, orc

KIND_STEM, KIND_CONV, KIND_MAXPOOL, KIND_HEAD = 0, 1, 2, 3


class _Rng(C.Structure):
    _fields_ = [("s", C.c_ulonglong * 4), ("has_spare", C.c_int), ("spare", C.c_double)]


def _lib():
    lib = orc()
    if not getattr(lib, "_cnn_models_sigs", False):
        P = C.POINTER(_Rng)
        pD = C.POINTER(C.c_double)
        lib.lco_mix_seed.restype = C.c_ulonglong
        lib.lco_mix_seed.argtypes = [C.c_ulonglong, C.c_ulonglong]
        lib.lco_rng_init.argtypes = [P, C.c_ulonglong]
        lib.lco_rng_normal_fill.argtypes = [P, pD, C.c_size_t, C.c_double]
        lib.lco_rng_uniform_fill.argtypes = [P, pD, C.c_size_t, C.c_double, C.c_double]
        lib.lco_rng_bn_fill.argtypes = [P, C.c_int, C.c_double, pD, pD]
        lib._cnn_models_sigs = True
    return lib


class _Builder:
    """cnn.cpp Builder: one slot per op output, taps after residual blocks /
    pooling stages, weights drawn from Rng(mix_seed(seed, 0xc0de))."""

    def __init__(self, seed: int):
        self.lib = _lib()
        self.rng = _Rng()
        self.lib.lco_rng_init(C.byref(self.rng), self.lib.lco_mix_seed(seed, 0xC0DE))
        self.ops: List[dict] = []
        self.next_slot = 0
        self.taps: List[Tuple[int, int, int]] = []

    def conv(self, inp, Cin, H, W, Cout, k, stride, pad, relu, res, bn_gain, kind=KIND_CONV):
        std = math.sqrt(2.0 / (float(Cin) * k * k))
        w = np.zeros(Cout * Cin * k * k, np.float64)
        self.lib.lco_rng_normal_fill(C.byref(self.rng), _dp(w), w.size, std)
        scale = np.zeros(Cout, np.float64)
        shift = np.zeros(Cout, np.float64)
        self.lib.lco_rng_bn_fill(C.byref(self.rng), Cout, bn_gain, _dp(scale), _dp(shift))
        out = self.next_slot
        self.next_slot += 1
        self.ops.append(dict(kind=kind, out=out, res=res, C=Cin, H=H, W=W, Cout=Cout, k=k, stride=stride, pad=pad,
                             relu=int(relu), tap=-1, w=w, scale=scale, shift=shift, **{"in": inp}))
        return out

    def maxpool(self, inp, Cin, H, W, k, stride, pad):
        out = self.next_slot
        self.next_slot += 1
        self.ops.append(dict(kind=KIND_MAXPOOL, out=out, res=-1, C=Cin, H=H, W=W, Cout=Cin, k=k, stride=stride,
                             pad=pad, relu=0, tap=-1, w=None, scale=None, shift=None, **{"in": inp}))
        return out

    def head(self, inp, Cin, H, W, classes):
        limit = math.sqrt(6.0 / (Cin + classes))
        w = np.zeros(classes * Cin, np.float64)
        self.lib.lco_rng_uniform_fill(C.byref(self.rng), _dp(w), w.size, -limit, limit)
        out = self.next_slot
        self.next_slot += 1
        self.ops.append(dict(kind=KIND_HEAD, out=out, res=-1, C=Cin, H=H, W=W, Cout=classes, k=1, stride=1, pad=0,
                             relu=0, tap=-1, w=w, scale=None, shift=np.zeros(classes, np.float64), **{"in": inp}))

    def mark_tap(self, Cin, H, W):
        self.ops[-1]["tap"] = len(self.taps)
        self.taps.append((Cin, H, W))


def _resnet(b: _Builder, H: int, W: int, imagenet: bool, bottleneck: bool, blocks_per_stage, classes: int):
    C_ = 64
    if imagenet:
        x = b.conv(-1, 3, H, W, 64, 7, 2, 3, True, -1, 1.0, KIND_STEM)
        H = (H + 6 - 7) // 2 + 1
        W = (W + 6 - 7) // 2 + 1
        x = b.maxpool(x, 64, H, W, 3, 2, 1)
        H = (H + 2 - 3) // 2 + 1
        W = (W + 2 - 3) // 2 + 1
    else:
        x = b.conv(-1, 3, H, W, 64, 3, 1, 1, True, -1, 1.0, KIND_STEM)
    widths = (64, 128, 256, 512)
    branch_gain = 0.2 if bottleneck else 0.5
    for s in range(4):
        for i in range(blocks_per_stage[s]):
            stride = 2 if (i == 0 and s > 0) else 1
            Ho, Wo = (H - 1) // stride + 1, (W - 1) // stride + 1
            if not bottleneck:
                Cout = widths[s]
                t1 = b.conv(x, C_, H, W, Cout, 3, stride, 1, True, -1, 1.0)
                res = x
                if stride != 1 or C_ != Cout:
                    res = b.conv(x, C_, H, W, Cout, 1, stride, 0, False, -1, 1.0)
                x = b.conv(t1, Cout, Ho, Wo, Cout, 3, 1, 1, True, res, branch_gain)
                C_ = Cout
            else:
                w = widths[s]
                Cout = 4 * w
                t1 = b.conv(x, C_, H, W, w, 1, 1, 0, True, -1, 1.0)
                t2 = b.conv(t1, w, H, W, w, 3, stride, 1, True, -1, 1.0)
                res = x
                if stride != 1 or C_ != Cout:
                    res = b.conv(x, C_, H, W, Cout, 1, stride, 0, False, -1, 1.0)
                x = b.conv(t2, w, Ho, Wo, Cout, 1, 1, 0, True, res, branch_gain)
                C_ = Cout
            H, W = Ho, Wo
            b.mark_tap(C_, H, W)
    b.head(x, C_, H, W, classes)


def _vgg16(b: _Builder, H: int, W: int, classes: int):
    cfg = (64, 64, -1, 128, 128, -1, 256, 256, 256, -1, 512, 512, 512, -1, 512, 512, 512, -1)
    C_, x, first = 3, -1, True
    for v in cfg:
        if v < 0:
            x = b.maxpool(x, C_, H, W, 2, 2, 0)
            H //= 2
            W //= 2
            b.mark_tap(C_, H, W)
        else:
            x = b.conv(x, C_, H, W, v, 3, 1, 1, True, -1, 1.0, KIND_STEM if first else KIND_CONV)
            first = False
            C_ = v
    b.head(x, C_, H, W, classes)


class CnnModel:
    """ops (BaseModel.cnn_ops() format), nslots, taps [(C, H, W)], input geometry."""

    def __init__(self, arch: str, classes: int, seed: int):
        if classes < 2:
            raise ValueError("base model: need at least two classes")
        b = _Builder(seed)
        if arch == "resnet18_cifar":
            self.in_shape = (3, 32, 32)
            _resnet(b, 32, 32, False, False, (2, 2, 2, 2), classes)
        elif arch == "resnet50":
            self.in_shape = (3, 224, 224)
            _resnet(b, 224, 224, True, True, (3, 4, 6, 3), classes)
        elif arch == "resnet152":
            self.in_shape = (3, 224, 224)
            _resnet(b, 224, 224, True, True, (3, 8, 36, 3), classes)
        elif arch == "vgg16_cifar":
            self.in_shape = (3, 32, 32)
            _vgg16(b, 32, 32, classes)
        else:
            raise ValueError(f"base model: unknown CNN architecture '{arch}'")
        self.arch = arch
        self.num_classes = classes
        self.ops = b.ops
        self.nslots = b.next_slot
        self.taps = b.taps
        self.num_blocks = len(b.taps)
        self.tap_dims = [c * h * w for c, h, w in b.taps]
