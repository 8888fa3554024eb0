import sys; sys.path.insert(0, '/root/repo')
import numpy as np
import paper_2101_07344_b200 as lcb
from paper_2101_07344_b200.synthetic import image_inputs, calibrate_variants
m = lcb.make_cnn_model("resnet18_cifar", 10, 21)
vs = [lcb.build_variant(l, 0, f"Pool({m.tap(l)[0]})", m.tap_dim(l), 10, 21 + l) for l in range(1, 9)]
calib = image_inputs(64, 3, 32, 32, seed=121)
fr = calibrate_variants(m, vs, calib, 0.2, precision="bf16")
print("fractions", fr)
for v in vs:
    sel = v.layers(1)
    print(v.layer, v.delta, "w2", np.round(sel[2].w[:4], 3), "b2", sel[2].b)
x = image_inputs(32, 3, 32, 32, seed=6)
d3 = lcb.Deployment(m, vs, precision="bf16x3", max_batch=32)
d1 = lcb.Deployment(m, vs, precision="bf16", max_batch=32)
a, b = d3.serve(x, shadow=True), d1.serve(x, shadow=True)
print("x3 exit", a.exit_layer.tolist(), "served", a.served.tolist())
print("bf exit", b.exit_layer.tolist(), "served", b.served.tolist())
print("x3 probs l1", np.round(a.probs[0], 4).tolist())
print("bf probs l1", np.round(b.probs[0], 4).tolist())
