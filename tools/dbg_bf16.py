import sys; sys.path.insert(0, '/root/repo')
import numpy as np
import paper_2101_07344_b200 as lcb
from paper_2101_07344_b200.synthetic import image_inputs, mlp_inputs
for fam in ["mlp", "cnn"]:
    if fam == "mlp":
        m = lcb.make_base_model(64, 10, [64, 128], 2, 1)
        vs = [lcb.build_variant(1, 0, "Pool(16)", 64, 10, 3), lcb.build_variant(2, 0, "FC(128)", 128, 10, 3)]
        x = mlp_inputs(8, 64, 1)
    else:
        m = lcb.make_cnn_model("resnet18_cifar", 10, 3)
        vs = [lcb.build_variant(l, 0, f"Pool({m.tap(l)[0]})", m.tap_dim(l), 10, 5) for l in range(1, 9)]
        x = image_inputs(8, 3, 32, 32, 2)
    for prec in ["bf16x3", "bf16"]:
        d = lcb.Deployment(m, vs, precision=prec, max_batch=8)
        r = d.serve(x, shadow=True)
        print(fam, prec, "base", r.base_pred.tolist(), "exit", r.exit_layer.tolist())
        print("   probs[:,0..3]", np.round(r.probs[:, :3], 5).tolist())
        d.close()
