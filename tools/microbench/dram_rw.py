"""DRAM bandwidth by access mix (write-only fill, copy, read-only reduce, 1:2 read:write), best of 10."""
import torch
n = 1 << 29  # 1 GiB of bf16
a = torch.empty(n, dtype=torch.bfloat16, device="cuda")
b = torch.empty(n, dtype=torch.bfloat16, device="cuda")
c = torch.empty(n // 2, dtype=torch.bfloat16, device="cuda")
def t(f, nbytes, name):
    for _ in range(3): f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(10):
        e0.record(); f(); e1.record(); torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1))
    print(f"{name:30s} {nbytes/best/1e6:8.1f} GB/s")
t(lambda: a.fill_(1.0), 2*n, "write only (fill)")
t(lambda: b.copy_(a), 4*n, "copy (read+write)")
t(lambda: torch.sum(a.view(-1, 1024).float(), dim=1), 2*n, "read only (sum)")
# 1 read : 2 write  (c -> a[:n/2], a[n/2:])
t(lambda: torch.cat([c, c]), 2*(n//2) + 2*n, "read 1 : write 2 (cat c,c)")
