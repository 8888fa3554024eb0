"""Key metrics + top stall instructions of an ncu report (one kernel launch).
  python tools/ncu_summary.py <report.ncu-rep> [top_n]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 15
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
want = ["gpu__time_duration.sum", "sm__cycles_active.avg", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum",
        "l1tex__t_requests_pipe_lsu_mem_global_op_st.sum", "smsp__inst_executed.sum", "launch__registers_per_thread",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio"]
for r in rows[2:]:
    print("kernel:", r[hdr.index("Kernel Name")][:70])
    for w in want:
        if w in hdr:
            print(f"  {w:80s} {r[hdr.index(w)]} {units[hdr.index(w)]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
srows = list(csv.reader(io.StringIO(src)))
h = None
data = []
seen = set()
for r in srows:
    if "Warp Stall Sampling (All Samples)" in r:
        h = r
        continue
    if h and len(r) == len(h) and r[0].startswith("0x") and r[0] not in seen:
        seen.add(r[0])
        data.append(r)
if h:
    i = h.index("Warp Stall Sampling (All Samples)")
    f = lambda x: float(x) if x not in ("", "-") else 0.0  # noqa: E731
    tot = sum(f(r[i]) for r in data)
    stall_cols = [k for k, name in enumerate(h) if name.startswith("stall_") and "Not Issued" not in name]
    print(f"stall samples: {tot:.0f}")
    for r in sorted(data, key=lambda r: -f(r[i]))[:top]:
        reasons = sorted(((f(r[k]), h[k]) for k in stall_cols), reverse=True)[:2]
        print(f"  {f(r[i]):6.0f} {100*f(r[i])/tot:5.1f}%  {r[1][:60]:60s} {reasons}")
