"""Summarise an ncu launch-list CSV (gpu__time_duration.sum per launch)."""
import csv
import sys
from collections import defaultdict


def load(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    out = []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d["Metric Name"] == "gpu__time_duration.sum":
                name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("unnamed>::", "")
                v = float(d["Metric Value"].replace(",", ""))
                if d["Metric Unit"] == "us":
                    v *= 1e3
                elif d["Metric Unit"] == "ms":
                    v *= 1e6
                out.append((name, d["Grid Size"], v))
    return out


if __name__ == "__main__":
    out = load(sys.argv[1])
    verbose = len(sys.argv) > 2
    tot = sum(o[2] for o in out)
    agg = defaultdict(lambda: [0.0, 0])
    for i, o in enumerate(out):
        if verbose:
            print(f"{i:4d} {o[0][:40]:40s} {o[1]:>14s} {o[2]/1e3:9.1f} us")
        agg[o[0]][0] += o[2]
        agg[o[0]][1] += 1
    print(f"total {tot/1e3:.1f} us over {len(out)} launches")
    for k, (v, n) in sorted(agg.items(), key=lambda x: -x[1][0]):
        print(f"  {k[:48]:48s} n={n:4d} {v/1e3:9.1f} us {100*v/tot:5.1f} %")
