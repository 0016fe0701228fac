"""Summarise an ncu source page: hottest CUDA source lines by stall samples.

usage: python tools/ncu_hot_lines.py report.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
out = []
fname = ""
hdr = None
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
        samp = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        inst = int(r[hdr.index("Instructions Executed")] or 0)
    except ValueError:
        continue
    stalls = {k: int(r[i] or 0) for i, k in enumerate(hdr) if k.startswith("stall_") and "Not Issued" not in k
              and (r[i] or "0").isdigit()}
    topst = sorted(stalls.items(), key=lambda kv: -kv[1])[:3]
    out.append((samp, inst, f"{fname}:{r[0]}", r[1].strip()[:70], topst))

tot = sum(o[0] for o in out) or 1
toti = sum(o[1] for o in out) or 1
print(f"total samples {tot}, warp instructions {toti:.3e}")
for samp, inst, loc, src, st in sorted(out, key=lambda o: -o[0])[:top]:
    print(f"{100*samp/tot:5.1f}% smp {100*inst/toti:5.1f}% ins  {loc:22s} {src:70s} {st}")
