"""Summarise an ncu source page by executed instructions: per source file
and line, warp instructions per unit (tuning aid).

usage: python tools/ncu_lines_by_instr.py report.ncu-rep [top] [units]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 60
units = float(sys.argv[3]) if len(sys.argv) > 3 else 3.2e7
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
out, fname, hdr = [], "", None
for r in rows:
    if len(r) == 2 and r[0] == "File Name":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr) or not r[0].isdigit():
        continue
    try:
        inst = int(r[hdr.index("Instructions Executed")] or 0)
    except ValueError:
        continue
    out.append((inst, f"{fname}:{r[0]}", r[1].strip()[:100]))
# the page lists SASS per CUDA line twice (cuda view rows only are kept: they have source text)
tot = sum(o[0] for o in out) or 1
print(f"warp instructions {tot:.3e} ({tot / units:.1f} per unit)")
for inst, loc, src in sorted(out, key=lambda o: -o[0])[:top]:
    print(f"{inst / units:7.2f}/unit {100 * inst / tot:5.1f}%  {loc:24s} {src}")
