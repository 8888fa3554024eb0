"""Generates the golden fixtures in tests/golden/ from the REFERENCE itself
(oracle/_ref/liblatecache_ref.so = the unmodified /root/reference sources).
Run here (needs /root/reference to build _ref): python tests/golden/make_golden.py

trained/ : the reference's own offline pipeline (dataset -> train_base ->
           explore {FC(32), Pool(16), Conv(3,1)} -> compose -> gen_workload ->
           simulate_model), in the style of test_acceptance.cpp:69-137. The
           artifacts are the reference's text formats; traces.txt holds the
           reference's per-request hit_layer / served / base predictions.
c1/      : the C1 reference config: make_base_model(3072, 10,
           ResNet-18 stage widths, 8 blocks) with one build_variant cache per
           block from seeds, selectors calibrated to an exit profile; expected
           reference simulate_model outputs for 128 seeded requests.
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_2101_07344_b200.synthetic import (C1_MENU, C1_WIDTHS, calibrate_biases, exit_profile,  # noqa: E402
                                             gains_for, mlp_inputs)

HERE = os.path.dirname(os.path.abspath(__file__))


def trained():
    d = os.path.join(HERE, "trained")
    os.makedirs(d, exist_ok=True)
    seed, minutes = 9, 30.0
    st = O.ref().ref_pipeline(d.encode(), seed, 10, 16, 32, 8, b"FC(32);Pool(16);Conv(3,1)", 15, 20, minutes)
    O._check(st)
    with open(os.path.join(d, "meta.txt"), "w") as f:
        f.write(f"seed={seed} minutes={minutes} workload_seed={O.ref().ref_mix_seed(seed, 6)}\n")


def c1():
    d = os.path.join(HERE, "c1")
    os.makedirs(d, exist_ok=True)
    model_seed, cache_seed, input_seed, calib_seed, delta = 2101, 7344, 11, 12, 0.5
    m = O.RefModel.make(3072, 10, C1_WIDTHS, 8, model_seed)
    variants = [O.RefVariant.build(l + 1, l, C1_MENU[l], m.tap_dims[l], 10, cache_seed) for l in range(8)]
    calib = mlp_inputs(256, 3072, calib_seed)
    taps = [m.forward_taps(x)[0] for x in calib]
    z = {l + 1: np.array([variants[l].selector_logit(t[l]) for t in taps]) for l in range(8)}
    gains = gains_for(z)
    zg = {l: z[l] * gains[l] for l in z}
    biases = calibrate_biases(zg, exit_profile(list(range(1, 9)), 0.15), delta)
    for l in range(8):
        variants[l].set_selector_out(gains[l + 1], biases[l + 1])
    x = mlp_inputs(128, 3072, input_seed)
    hl, sv, bp, _ = O.ref_simulate(m, variants, x)
    probs = np.full((128, 8), np.nan)
    for i in range(128):
        t, _ = m.forward_taps(x[i])
        for l in range(8):
            _, p, _, _ = variants[l].lookup(t[l], 10)
            probs[i, l] = p
    spec = dict(input_dim=3072, classes=10, widths=C1_WIDTHS, blocks=8, model_seed=model_seed, menu=C1_MENU,
                cache_seed=cache_seed, delta=delta, gains={str(k): v for k, v in gains.items()},
                biases={str(k): v for k, v in biases.items()}, input_seed=input_seed, n=128,
                exit_layer=hl.tolist(), served=sv.tolist(), base=bp.tolist(),
                probs=[[float(v) for v in row] for row in probs])
    with open(os.path.join(d, "c1.json"), "w") as f:
        json.dump(spec, f, indent=0)
    print("c1 exit histogram:", np.bincount(hl, minlength=9).tolist())


if __name__ == "__main__":
    O.build()
    trained()
    c1()
