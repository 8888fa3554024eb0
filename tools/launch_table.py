"""Per-launch table of an ncu launch-list CSV (time, DRAM bytes, grid):
python tools/launch_table.py L.csv [L2.csv]  (two files: side by side by launch index)"""
import csv
import sys


def load(f):
    h, d = None, {}
    for r in csv.reader(open(f)):
        if not r:
            continue
        if r[0] == "ID":
            h = r
            continue
        if not h or len(r) != len(h):
            continue
        x = dict(zip(h, r))
        i = int(x["ID"])
        k = x["Kernel Name"].replace("(anonymous namespace)::", "").replace("<unnamed>::", "").replace("void ", "")
        e = d.setdefault(i, {"k": k.split("(")[0][:34], "g": x["Grid Size"]})
        v = float(x["Metric Value"].replace(",", ""))
        u = x["Metric Unit"]
        if "time" in x["Metric Name"]:
            v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(u, 1e-3)
        e[x["Metric Name"]] = v
    return [d[i] for i in sorted(d)]


A = load(sys.argv[1])
B = load(sys.argv[2]) if len(sys.argv) > 2 else None
for i, a in enumerate(A):
    mb = (a.get("dram__bytes_read.sum", 0) + a.get("dram__bytes_write.sum", 0)) / 1e6
    line = f"{i:3d} {a['k']:34s} {a['g']:>12s} {a['gpu__time_duration.sum']:8.1f} us {mb:8.1f} MB"
    if B and i < len(B):
        line += f"   | {B[i]['k'][:20]:20s} {B[i]['gpu__time_duration.sum']:8.1f} us"
    print(line)
print("total", round(sum(a["gpu__time_duration.sum"] for a in A), 1), "us",
      ("| " + str(round(sum(b["gpu__time_duration.sum"] for b in B), 1)) + " us") if B else "")
