"""Executed SASS opcodes of an ncu report with their modifiers (IMAD.MOV,
MOV, CS2R, ... are register moves the allocator inserted), per unit.

usage: python tools/ncu_sass_moves.py report.ncu-rep [per] [top]
"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
per = float(sys.argv[2]) if len(sys.argv) > 2 else 3.2e7
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = None
ops = collections.Counter()
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
    parts = r[hdr.index("Source")].split()
    if not parts:
        continue
    op = parts[1] if parts[0].startswith("@") and len(parts) > 1 else parts[0]
    ops[op] += n
tot = sum(ops.values())
mv = sum(v for k, v in ops.items() if k.startswith(("MOV", "IMAD.MOV", "CS2R", "UMOV")))
print(f"instructions {tot / per:.1f} per unit, register moves {mv / per:.1f}")
print(", ".join(f"{k} {v / per:.1f}" for k, v in ops.most_common(top)))

# where the moves are: by CUDA source line (file:line of the innermost inlined frame)
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname, cur, hdr = "", "", None
by_line = collections.Counter()
text = {}
for r in csv.reader(io.StringIO(txt)):
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    if r[0].isdigit():
        cur = f"{fname}:{r[0]}"
        text[cur] = r[1].strip()[:90]
        continue
    parts = r[3].split()
    if not parts or parts[0] == "...":
        continue
    op = parts[1] if parts[0].startswith("@") and len(parts) > 1 else parts[0]
    if op.startswith(("MOV", "IMAD.MOV", "CS2R")):
        try:
            by_line[cur] += int(r[hdr.index("Instructions Executed")] or 0)
        except ValueError:
            pass
print("register moves by source line:")
for k, v in by_line.most_common(top):
    print(f"{v / per:6.2f}  {k:24s} {text.get(k, '')}")
