"""Launch list + DRAM traffic of one serve step from an ncu CSV:

  ncu --profile-from-start off --clock-control none --csv --log-file L.csv \
      --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      python tools/profile_step.py resnet18_cifar bf16x3
  python tools/traffic.py L.csv profiles/traffic_resnet18_cifar_bf16x3.json

Writes the per-step DRAM bytes of the tensor-core contraction kernels
(tc_conv / tc_stem), which bench.py reports as roofline.traffic next to the
algorithmic bytes, and prints the per-kernel summary.
"""
import csv
import json
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
launches = defaultdict(dict)
names = {}
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    i = int(d["ID"])
    names[i] = d["Kernel Name"].split("(")[0].replace("void ", "").replace("lcb::", "").replace("<unnamed>::", "")
    v = float(d["Metric Value"].replace(",", ""))
    u = d["Metric Unit"]
    scale = {"ns": 1e-3, "us": 1.0, "ms": 1e3, "usecond": 1.0, "nsecond": 1e-3, "msecond": 1e3,
             "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(u, 1.0)
    launches[i][d["Metric Name"]] = v * scale
agg = defaultdict(lambda: [0, 0.0, 0.0])
tc_bytes, tc_n, tc_us = 0.0, 0, 0.0
for i in sorted(launches):
    m = launches[i]
    b = m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    t = m.get("gpu__time_duration.sum", 0.0)
    a = agg[names[i].split("<")[0]]
    a[0] += 1
    a[1] += t
    a[2] += b
    if "tc_conv" in names[i] or "tc_stem" in names[i]:
        tc_bytes += b
        tc_n += 1
        tc_us += t
tot = sum(a[1] for a in agg.values())
print(f"total {tot:.1f} us over {sum(a[0] for a in agg.values())} launches (ncu: serialised, caches flushed)")
for k, (n, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"  {k:32s} n={n:4d} {t:9.1f} us {100*t/tot:5.1f} %  DRAM {b/1e6:9.1f} MB")
if len(sys.argv) > 2:
    json.dump({"dram_bytes_per_step": tc_bytes, "launches": tc_n, "ncu_us_per_step": tc_us,
               "source": sys.argv[1].split("/")[-1],
               "by_kernel": {k: {"launches": n, "ncu_us": t, "dram_bytes": b} for k, (n, t, b) in agg.items()},
               "note": "sum over the step's tc_conv/tc_stem launches of dram__bytes_read.sum + dram__bytes_write.sum "
                       "(ncu, cache control all = cold L2 per launch)"}, open(sys.argv[2], "w"), indent=1)
