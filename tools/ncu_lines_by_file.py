"""Per-CUDA-source-line executed warp instructions and stall samples of an
ncu report (one kernel), in report order: where the instructions go.

usage: python tools/ncu_lines_by_file.py report.ncu-rep [min_pct]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
minp = float(sys.argv[2]) if len(sys.argv) > 2 else 0.2
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr, out = None, []
for r in rows:
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr) or not r[0].isdigit() or r[2] != "-":
        continue
    try:
        inst = int(r[hdr.index("Instructions Executed")] or 0)
        samp = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
    except ValueError:
        continue
    out.append((int(r[0]), inst, samp, r[1].strip()))
toti = sum(o[1] for o in out) or 1
tots = sum(o[2] for o in out) or 1
print(f"total warp instructions {toti:.4e}")
for ln, inst, samp, src in out:
    if 100 * inst / toti >= minp or 100 * samp / tots >= minp:
        print(f"{ln:4d} {100*inst/toti:5.1f}% ins {100*samp/tots:5.1f}% smp | {src[:100]}")
