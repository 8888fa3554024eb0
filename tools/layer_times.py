"""Device per-block base time and per-cache lookup time (graph, %globaltimer
stamps): python tools/layer_times.py resnet18_cifar [bf16x3] [compact]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from bench import CONFIGS, build_deployment  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "resnet18_cifar"
prec = sys.argv[2] if len(sys.argv) > 2 else "bf16x3"
B = CONFIGS[cfg][3]
m, vs, dep, base, gen, _ = build_deployment(cfg, B, prec, 0)
x = gen(B, 5).astype(np.float32)
shadow = not (len(sys.argv) > 3 and sys.argv[3] == "compact")
for _ in range(3):
    dep.layer_times(x, shadow)
runs = [dep.layer_times(x, shadow) for _ in range(5)]
cnt = dep.counts()
bm = np.median([r[0] for r in runs], axis=0)
lm = {l: float(np.median([r[1][l] for r in runs])) for l in runs[0][1]}
print(f"{cfg} {prec} B={B} " + ("(shadow: every request at every block)" if shadow else "(compact: survivors only)"))
for l in range(1, len(bm) + 1):
    print(f"  block {l:2d}: rows {cnt[l-1]:4d}  base {bm[l-1]*1e3:8.1f} us   lookup {lm.get(l, 0.0)*1e3:7.1f} us")
print(f"  total base {bm.sum()*1e3:.1f} us, lookups {sum(lm.values())*1e3:.1f} us")
