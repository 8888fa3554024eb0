"""Bisect the golden trained deployment on the GPU: which requests/layers differ."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2101_07344_b200 as lcb  # noqa: E402
from oracle import oracle as O  # noqa: E402
from tests.test_gpu_parity import _load_trained  # noqa: E402

model_txt, vtxt, X, reqs, traces = _load_trained()
m = lcb.load_base_model(model_txt)
vs = [lcb.load_variant(t) for t in vtxt]
idx = np.array([s for _, s in reqs])
served_ref = np.array([int(t[4]) for t in traces])
exit_ref = np.array([int(t[5]) for t in traces])
for mb in (4096, 512):
    dep = lcb.Deployment(m, vs, precision="bf16x3", max_batch=mb)
    el, sv = [], []
    for i in range(0, len(idx), mb):
        r = dep.serve(X[idx[i:i + mb]], shadow=True)
        el.append(r.exit_layer)
        sv.append(r.served)
    el, sv = np.concatenate(el), np.concatenate(sv)
    bad = np.nonzero(sv != served_ref)[0]
    print(f"max_batch={mb}: exit mismatches {np.sum(el != exit_ref)}, served mismatches {len(bad)}", bad[:10],
          sv[bad[:10]], served_ref[bad[:10]], el[bad[:10]])
    dep.close()
# environment toggles (engine reads them at construction)
for env in ("LCB_DIRECT_STORE", "LCB_NO_MMA_RESIDUAL"):
    os.environ[env] = "1"
    dep = lcb.Deployment(m, vs, precision="bf16x3", max_batch=4096)
    r = dep.serve(X[idx], shadow=True)
    print(env, "served mismatches", int(np.sum(r.served != served_ref)), "exit", int(np.sum(r.exit_layer != exit_ref)))
    dep.close()
    del os.environ[env]
