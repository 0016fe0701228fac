"""Pipe utilisation and stall breakdown of an ncu --set full report.

usage: python tools/ncu_pipes.py report.ncu-rep
"""
import csv
import io
import subprocess
import sys

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
h = rr[0]
for row in rr[2:]:
    print(row[h.index("Kernel Name")][:60])
    for i, k in enumerate(h):
        if k.startswith("sm__inst_executed_pipe_") and k.endswith(".avg.pct_of_peak_sustained_active"):
            try:
                if float(row[i]) > 1.0:
                    print(f"  {k[23:-34]:28s} {float(row[i]):6.1f} %")
            except ValueError:
                pass
    st = []
    for i, k in enumerate(h):
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
            try:
                st.append((float(row[i]), k[34:-23]))
            except ValueError:
                pass
    print("  stalls/issue: " + ", ".join(f"{n} {v:.2f}" for v, n in sorted(st, reverse=True) if v > 0.03))
