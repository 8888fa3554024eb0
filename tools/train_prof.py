"""Launch list of one large-cache retrain (FC(1024) over a 32768-wide tap) for
ncu: python tools/train_prof.py [N] [epochs]"""
import sys
import time

import os
import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2101_07344_b200 as lcb

N = int(sys.argv[1]) if len(sys.argv) > 1 else 64
E = int(sys.argv[2]) if len(sys.argv) > 2 else 1
D, C = 32768, 10
v = lcb.build_variant(3, 0, "FC(1024)", D, C, 7)
rng = np.random.default_rng(1)
taps = rng.standard_normal((N, D))
y = rng.dirichlet(np.ones(C), N)
cfg = lcb.TrainConfig(learning_rate=0.002, epochs=E, batch_size=16, seed=9)
t0 = time.perf_counter()
lcb.train_predictor(v, taps, y, cfg)
t1 = time.perf_counter()
lcb.train_selector(v, taps, y, cfg)
t2 = time.perf_counter()
print(f"predictor {1e3 * (t1 - t0):.1f} ms selector {1e3 * (t2 - t1):.1f} ms (N={N}, epochs={E})")
