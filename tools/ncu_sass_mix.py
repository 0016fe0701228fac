"""Executed SASS instruction mix of an ncu report, split into the hottest
basic-block run (instructions executed >= hot_frac x max) and the rest.

usage: python tools/ncu_sass_mix.py report.ncu-rep [hot_frac] [per]
  per: divide counts by this number (e.g. warp-pairs) for per-unit figures
"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
hot_frac = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
per = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr, ins = None, []
for r in rows:
    if r and r[0] == "Address":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    try:
        n = int(r[hdr.index("Instructions Executed")] or 0)
    except ValueError:
        continue
    src = r[hdr.index("Source")].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    ins.append((r[0], op.split(".")[0], n))
mx = max(n for _, _, n in ins)
hot = collections.Counter()
cold = collections.Counter()
for a, op, n in ins:
    (hot if n >= hot_frac * mx else cold)[op] += n
for name, c in (("hot", hot), ("rest", cold)):
    tot = sum(c.values())
    print(f"{name}: {tot / per:.1f} per unit ({tot:.3e})")
    print("   " + ", ".join(f"{k} {v / per:.1f}" for k, v in c.most_common(24)))
