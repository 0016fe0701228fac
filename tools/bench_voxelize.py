"""Voxelisation timing: GPU ``voxelize`` on the config-2
cloud (1M balls, a0 0.05-0.2 mm) into a 128^3 grid over the 20 mm cube,
host arrays in and out (the public call), against the oracle restatement of
the reference splat on a bounded subset with the per-ball rate extrapolated.

usage: python tools/bench_voxelize.py [n_balls] [grid]
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)
import paper_2601_00551_b200 as P  # noqa: E402
from paper_2601_00551_b200 import scenes  # noqa: E402
from oracle import render as ORR  # noqa: E402  (CPU baseline leg only)

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
g = int(sys.argv[2]) if len(sys.argv) > 2 else 128
cloud = scenes.microbench_config(n_balls=n, n_det=8).init
spacing = 20e-3 / g
spec = P.RenderSpec(dims=(g, g, g), spacing=spacing, origin=(-10e-3 + spacing / 2,) * 3)
P.voxelize(cloud.subset(np.arange(1000)), spec)   # warm-up (library load, allocator)
times = []
for _ in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    vol = P.voxelize(cloud, spec)
    torch.cuda.synchronize()
    times.append(time.perf_counter() - t0)
gpu_s = min(times)
m = 2000
sub = cloud.subset(np.arange(m))
t0 = time.perf_counter()
ORR.voxelize(sub.positions, sub.p0, sub.a0, spec.dims, spec.spacing, spec.origin, spec.support_sigma)
cpu_per_ball = (time.perf_counter() - t0) / m
print(json.dumps({"workload": f"voxelize config-2 init cloud ({n} balls, a0 0.05-0.2 mm) into {g}^3 over 20 mm",
                  "gpu_s": gpu_s, "gpu_balls_per_s": n / gpu_s,
                  "cpu_oracle_balls_per_s": 1.0 / cpu_per_ball, "cpu_sample": f"{m} balls, 1 thread (numpy)",
                  "speedup_vs_oracle": (1.0 / cpu_per_ball and (n / gpu_s) * cpu_per_ball),
                  "volume_sum": float(vol.values.sum())}))
