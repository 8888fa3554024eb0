"""Per-source-line instruction counts and stall samples of an ncu report.
  python tools/ncu_lines.py <report.ncu-rep> [top_n]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
by_stall = len(sys.argv) > 3 and sys.argv[3] == "stall"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname, hdr, data = None, None, []
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif r and r[0] == "Line No":
        hdr = r
    elif hdr and r and r[0] not in ("", "Function Name") and len(r) == len(hdr):
        ie, st = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
        f = lambda x: float(x) if x not in ("", "-") else 0.0  # noqa: E731
        data.append((f(r[ie]), f(r[st]), fname, r[0], r[1].strip()[:90]))
ti = sum(d[0] for d in data)
ts = sum(d[1] for d in data)
print(f"instructions {ti:.0f}  stall samples {ts:.0f}")
for d in sorted(data, key=lambda d: d[1] if by_stall else d[0], reverse=True)[:top]:
    print(f"{d[0]:10.0f} {100*d[0]/ti:5.1f}%  st {100*d[1]/max(ts,1):5.1f}%  {d[2]}:{d[3]:5s} {d[4]}")
