"""Stall reasons by kernel region: per SASS instruction stall columns of an
ncu report, aggregated over source-line ranges (e.g. the epilogue).
  python tools/ncu_stalls.py <report.ncu-rep> [file:line0-line1 ...]
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
ranges = []
for a in sys.argv[2:]:
    f, lr = a.split(":")
    l0, l1 = lr.split("-")
    ranges.append((f, int(l0), int(l1)))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname, hdr = None, None
agg = defaultdict(lambda: defaultdict(float))
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif r and r[0] == "Line No":
        hdr = r
    elif hdr and r and len(r) == len(hdr) and r[0].strip().isdigit():
        ln = int(r[0])
        key = "other"
        for f, l0, l1 in ranges:
            if fname == f and l0 <= ln <= l1:
                key = f"{f}:{l0}-{l1}"
        for i, h in enumerate(hdr):
            if h.startswith("stall_") and "Not Issued" not in h:
                try:
                    agg[key][h] += float(r[i] or 0)
                except ValueError:
                    pass
        try:
            agg[key]["inst"] += float(r[hdr.index("Instructions Executed")] or 0)
        except ValueError:
            pass
for k, d in agg.items():
    tot = sum(v for h, v in d.items() if h.startswith("stall_"))
    print(f"{k}: instructions {d['inst']:.0f}, stall samples {tot:.0f}")
    for h, v in sorted(d.items(), key=lambda kv: -kv[1]):
        if h.startswith("stall_") and v > 0.02 * tot:
            print(f"    {h:24s} {v:8.0f} {100 * v / max(tot, 1):5.1f}%")
