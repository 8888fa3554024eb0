"""Per-step roofline of one serve batch (CUDA events around every step, no graph).

  python tools/step_roofline.py resnet50 bf16x3 [shadow]

Prints, for every step: kind (0 other, 1 tensor-core contraction, 2 lookup),
device us, algorithmic GFLOP and MB, the tensor-core time floor (MMA FLOPs at
the measured bf16 peak; bf16x3 issues 3 MMAs per algorithmic MAC), the HBM
time floor (algorithmic bytes at the measured copy bandwidth), the binding
floor and the fraction of it achieved. Ends with per-kind totals.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench import CONFIGS, build_deployment, load_peaks  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "resnet18_cifar"
prec = sys.argv[2] if len(sys.argv) > 2 else "bf16x3"
shadow = len(sys.argv) > 3 and sys.argv[3] == "shadow"
B = CONFIGS[cfg][3]
m, vs, dep, base, gen, _ = build_deployment(cfg, B, prec, 0)
x = gen(B, 7).astype(np.float32)
dep.stage_input_device(torch.from_numpy(x).cuda().data_ptr(), B)
for _ in range(3):
    dep.profile(B, shadow=shadow)
prof = dep.profile(B, shadow=shadow)
hbm, bf16, _, src = load_peaks()
mf = 3.0 if prec == "bf16x3" else 1.0
tot = {}
print(f"{cfg} {prec} {'shadow' if shadow else 'compact'} peaks({src}): {bf16} TFLOP/s, {hbm} GB/s")
print(f"{'i':>3} {'k':>1} {'us':>8} {'GFLOP':>8} {'MB':>8} {'t_tc':>7} {'t_hbm':>7} bound  frac")
for i, (k, ms, fl, by) in enumerate(zip(prof["kind"], prof["ms"], prof["flops"], prof["bytes"])):
    us = ms * 1e3
    ttc = fl * mf / (bf16 * 1e12) * 1e6
    thb = by / (hbm * 1e9) * 1e6
    fl_ = max(ttc, thb)
    b = "tc " if ttc >= thb else "hbm"
    print(f"{i:3d} {k:1d} {us:8.1f} {fl/1e9:8.3f} {by/1e6:8.2f} {ttc:7.1f} {thb:7.1f} {b} {fl_/us if us else 0:5.2f}")
    t = tot.setdefault(int(k), [0.0, 0.0, 0.0, 0.0])
    t[0] += us
    t[1] += ttc
    t[2] += thb
    t[3] += fl_
for k, (us, ttc, thb, fl_) in sorted(tot.items()):
    print(f"kind {k}: {us:9.1f} us  tc-floor {ttc:8.1f}  hbm-floor {thb:8.1f}  roofline frac {fl_/us:5.3f}")
print("counts", dep.counts().tolist())
