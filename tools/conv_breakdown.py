"""Pair the tc_conv launches of an ncu launch list with the model's conv ops
(engine step order) and print per-conv times plus totals per conv type.
  python tools/conv_breakdown.py <launches.csv> <arch> <classes>
"""
import os
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import paper_2101_07344_b200 as lcb  # noqa: E402
from launches import load  # noqa: E402

path, arch, classes = sys.argv[1], sys.argv[2], int(sys.argv[3])
m = lcb.make_cnn_model(arch, classes, 2101)
convs = [o for o in m.cnn_ops() if o["kind"] in (0, 1)]
tc = [o for o in load(path) if o[0].startswith("tc_")]
agg = defaultdict(float)
for o, l in zip(convs, tc):
    key = f"{o['k']}x{o['k']} s{o['stride']} {o['C']}->{o['Cout']} @{o['H']}x{o['W']}{' res' if o['res'] >= 0 else ''}{' tap' if o['tap'] >= 0 else ''}"
    print(f"{key:40s} {l[0][:22]:22s} {l[2]/1e3:8.1f} us")
    agg[f"{o['k']}x{o['k']} s{o['stride']}"] += l[2]
print("totals:", {k: round(v / 1e3, 1) for k, v in agg.items()})
