"""Determinism / race stress: repeated serves must be bit-identical."""
import sys; sys.path.insert(0, '/root/repo')
import numpy as np
import paper_2101_07344_b200 as lcb
from paper_2101_07344_b200.synthetic import image_inputs, calibrate_variants
n_iter = int(sys.argv[1]) if len(sys.argv) > 1 else 30
m = lcb.make_cnn_model("resnet18_cifar", 10, 21)
bad = 0
for it in range(3):
    vs = [lcb.build_variant(l, 0, f"Pool({m.tap(l)[0]})", m.tap_dim(l), 10, 21 + l) for l in range(1, 9)]
    calibrate_variants(m, vs, image_inputs(64, 3, 32, 32, seed=121), 0.2, precision="bf16")
    x = image_inputs(32, 3, 32, 32, seed=6)
    for prec in ["bf16x3", "bf16"]:
        d = lcb.Deployment(m, vs, precision=prec, max_batch=32)
        ref = d.serve(x, shadow=True)
        for k in range(n_iter):
            for shadow in (True, False):
                r = d.serve(x, shadow=shadow)
                same = np.array_equal(r.exit_layer, ref.exit_layer) and np.array_equal(r.served, ref.served)
                if shadow:
                    same = same and np.array_equal(r.probs, ref.probs, equal_nan=True) and np.array_equal(r.base_pred, ref.base_pred)
                if not same:
                    bad += 1
                    print("MISMATCH", prec, it, k, shadow, r.exit_layer.tolist(), ref.exit_layer.tolist())
        d.close()
print("stress done, mismatches:", bad)
