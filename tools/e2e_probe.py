"""e2e path probe: sync serve vs pipelined submit/collect (R18 bench config)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench import CONFIGS, build_deployment  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "resnet18_cifar"
B = CONFIGS[cfg][3]
m, vs, dep, base, gen, _ = build_deployment(cfg, B, "bf16x3", 0)
xs = [torch.from_numpy(gen(B, 100 + j).astype(np.float32)).pin_memory() for j in range(4)]
pg = [gen(B, 100 + j).astype(np.float32) for j in range(4)]
N = 50


def t_sync(bufs):
    for j in range(3):
        dep.serve(bufs[j % 4])
    t0 = time.perf_counter()
    for s in range(N):
        dep.serve(bufs[s % 4])
    return (time.perf_counter() - t0) / N * 1e3


def t_pipe(bufs, depth=2):
    t0 = time.perf_counter()
    pending = []
    for s in range(N):
        pending.append(dep.submit(bufs[s % 4]))
        if len(pending) == depth:
            dep.collect(pending.pop(0))
    while pending:
        dep.collect(pending.pop(0))
    return (time.perf_counter() - t0) / N * 1e3


def t_submit_only(bufs):
    t0 = time.perf_counter()
    tk = []
    for s in range(N):
        a = time.perf_counter()
        tk.append(dep.submit(bufs[s % 4]))
        if s < 3:
            print(f"  submit {s} host {1e3*(time.perf_counter()-a):.3f} ms")
        if len(tk) == 2:
            dep.collect(tk.pop(0))
    while tk:
        dep.collect(tk.pop(0))
    return (time.perf_counter() - t0) / N * 1e3


dev = torch.from_numpy(pg[0]).cuda()
dep.stage_input_device(dev.data_ptr(), B)
dev_ms = np.mean([dep.serve_timed(B) for _ in range(20)])
print(f"{cfg}: device {dev_ms:.3f} ms/step")
print(f"sync pinned   {t_sync([x.numpy() for x in xs]):.3f} ms/step")
print(f"sync pageable {t_sync(pg):.3f} ms/step")
print(f"pipe pinned   {t_pipe([x.numpy() for x in xs]):.3f} ms/step")
print(f"pipe pageable {t_pipe(pg):.3f} ms/step")
print(f"pipe pinned   {t_submit_only([x.numpy() for x in xs]):.3f} ms/step (timed submits)")
