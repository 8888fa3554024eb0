"""Small-cache retrain (the reference's FC(32) on a 64-wide MLP tap), for ncu."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2101_07344_b200 as lcb  # noqa: E402

v = lcb.build_variant(1, 0, "FC(32)", 64, 10, 3)
rng = np.random.default_rng(1)
N = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
taps = np.maximum(rng.standard_normal((N, 64)), 0)
y = rng.dirichlet(np.ones(10), N)
cfg = lcb.TrainConfig(learning_rate=0.002, epochs=5, batch_size=16, seed=9)
lcb.train_predictor(v, taps[:32], y[:32], cfg)
for _ in range(2):
    t0 = time.perf_counter()
    lcb.train_predictor(v, taps, y, cfg)
    t1 = time.perf_counter()
    lcb.train_selector(v, taps, y, cfg)
    t2 = time.perf_counter()
    print(f"predictor {1e3 * (t1 - t0):.2f} ms selector {1e3 * (t2 - t1):.2f} ms")
