"""One serve step of a bench config inside cudaProfilerStart/Stop, for
`ncu --profile-from-start off` (launch list / full capture of the top kernel).

  ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
      --csv --log-file gpurun_out/launches.csv python tools/profile_step.py resnet18_cifar bf16x3
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench import CONFIGS, build_deployment  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "resnet18_cifar"
prec = sys.argv[2] if len(sys.argv) > 2 else "bf16x3"
shadow = len(sys.argv) > 3 and sys.argv[3] == "shadow"
B = int(os.environ.get("LCB_PROFILE_BATCH", CONFIGS[cfg][3]))
m, vs, dep, base, gen, _ = build_deployment(cfg, B, prec, 0)
x = gen(B, 7).astype(np.float32)
for _ in range(3):
    dep.serve(x, shadow=shadow, graph=False)
torch.cuda.synchronize()
torch.cuda.profiler.start()
dep.serve(x, shadow=shadow, graph=False)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("profiled one step:", cfg, prec, "shadow" if shadow else "compact", "counts", dep.counts().tolist())
