"""Per-kernel totals and share of an ncu launch list
(--metrics gpu__time_duration.sum --csv).

usage: python tools/launch_share.py launches.csv
"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 14 and r[0].isdigit()]
tot = collections.defaultdict(float)
cnt = collections.Counter()
for r in rows:
    name = r[4].split("(")[0][:70]
    tot[name] += float(r[14]) * (1e-3 if r[13] == "ns" else 1.0 if r[13] == "us" else 1e3)
    cnt[name] += 1
all_us = sum(tot.values())
print(f"{len(rows)} launches, {all_us / 1e3:.2f} ms total (cold-cache, serialised)")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{100 * v / all_us:6.2f}%  {v / 1e3:9.3f} ms  x{cnt[k]:<3d} {k}")
