"""Key metrics of an ncu --set full report (one line per metric).

usage: python tools/ncu_summary.py report.ncu-rep
"""
import csv
import io
import subprocess
import sys

WANT = ["Duration", "SM Frequency", "Compute (SM) Throughput", "Memory Throughput", "DRAM Throughput",
        "L1/TEX Cache Throughput", "L2 Cache Throughput", "Executed Ipc Active", "Issue Slots Busy",
        "Executed Instructions", "Registers Per Thread", "Dynamic Shared Memory Per Block", "Theoretical Occupancy",
        "Achieved Active Warps Per SM", "Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Grid Size", "Block Size", "Waves Per SM", "Branch Efficiency"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "sm__inst_executed_pipe_fma.sum",
       "sm__inst_executed_pipe_xu.sum", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_lsu.sum", "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
       "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum",
       "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"]

rep = sys.argv[1]
txt = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
h = rows[0]
ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
seen = set()
for r in rows[1:]:
    if r[mi] in WANT and (r[ki], r[mi]) not in seen:
        seen.add((r[ki], r[mi]))
        print(f"{r[ki][:40]:40s} {r[mi]:40s} {r[vi]} {r[ui]}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
if len(rr) > 2:
    hh, units = rr[0], rr[1]
    for row in rr[2:]:
        for m in RAW:
            if m in hh:
                i = hh.index(m)
                print(f"{row[hh.index('Kernel Name')][:40]:40s} {m:40s} {row[i]} {units[i]}")
