import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2101_07344_b200 as lcb
from paper_2101_07344_b200.synthetic import calibrate_variants, image_inputs
m = lcb.make_cnn_model("vgg16_cifar", 10, 41)
vs = []
for l in range(1, m.num_blocks + 1):
    C, H, W = m.tap(l)
    a = f"Pool({C})" if l % 2 else "FC(256)"
    vs.append(lcb.build_variant(l, 0, a, m.tap_dim(l), 10, 41 + l))
    print(l, (C, H, W), a, flush=True)
for op in m.cnn_ops():
    print(op["kind"], op["C"], op["H"], op["W"], op["Cout"], op["k"], op["stride"], op["tap"], flush=True)
dep = lcb.Deployment(m, vs, precision="bf16x3", max_batch=32)
x = image_inputs(24, 3, 32, 32, seed=14)
print("shadow", flush=True)
r = dep.serve(x, shadow=True, graph=False)
print("compact", flush=True)
r = dep.serve(x, shadow=False, graph=False)
print("ok", flush=True)
