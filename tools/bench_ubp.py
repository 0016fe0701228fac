"""UBP baseline timing: GPU ``ubp_reconstruct`` of the
config-2 recording (1024 detectors x 4096 samples, FP64 rows) onto a grid^3
volume over the 20 mm cube, host arrays in and out (the public call), kernel
time by CUDA events, against the oracle restatement on a bounded detector
subset with the per-pair rate extrapolated.

usage: python tools/bench_ubp.py [grid]
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
from oracle import baseline as OB  # noqa: E402  (CPU baseline leg only)

g = int(sys.argv[1]) if len(sys.argv) > 1 else 128
sc = scenes.microbench_config(n_balls=20000, n_det=1024, n_samples=4096)
rows = np.random.default_rng(5).standard_normal((sc.array.positions.shape[0], sc.grid.n_samples))
real = P.SignalSet(sc.grid, rows)
spacing = 20e-3 / g
spec = P.RenderSpec(dims=(g, g, g), spacing=spacing, origin=(-10e-3 + spacing / 2,) * 3)
P.ubp_reconstruct(real, sc.array, P.RenderSpec((4, 4, 4), spacing, spec.origin))   # warm-up
times = []
for _ in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    vol, cov = P.ubp_reconstruct(real, sc.array, spec)
    torch.cuda.synchronize()
    times.append(time.perf_counter() - t0)
pairs = g ** 3 * rows.shape[0]
# device-only: re-run the kernels on resident buffers under CUDA events
from paper_2601_00551_b200 import engine as E  # noqa: E402
from paper_2601_00551_b200._lib import call, ptr  # noqa: E402
dev = E.cuda_device()
sig = torch.from_numpy(rows).to(dev)
det = torch.from_numpy(np.ascontiguousarray(sc.array.positions, dtype=np.float64)).to(dev)
deriv, vol_d = torch.empty_like(sig), torch.empty(g ** 3, dtype=torch.float64, device=dev)
skip = torch.zeros(1, dtype=torch.int64, device=dev)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ks = []
for _ in range(5):
    ev[0].record()
    call("pab_ubp", ptr(sig), rows.shape[0], rows.shape[1], float(sc.grid.t0), float(sc.grid.dt), ptr(det),
         float(sc.array.sound_speed), g, g, g, spacing, *spec.origin, ptr(deriv), ptr(vol_d), ptr(skip), E._stream())
    ev[1].record()
    torch.cuda.synchronize()
    ks.append(ev[0].elapsed_time(ev[1]) * 1e-3)
sub = 4
t0 = time.perf_counter()
OB.ubp(rows[:sub], sc.grid.t0, sc.grid.dt, sc.array.positions[:sub], sc.array.sound_speed, spec.dims, spacing,
       spec.origin)
cpu_rate = g ** 3 * sub / (time.perf_counter() - t0)
print(json.dumps({"workload": f"ubp config-2 record (1024 x 4096, FP64) onto {g}^3 over 20 mm",
                  "e2e_s": min(times), "kernel_s": min(ks), "pairs": pairs,
                  "gpu_pairs_per_s": pairs / min(ks), "e2e_pairs_per_s": pairs / min(times),
                  "cpu_oracle_pairs_per_s": cpu_rate, "cpu_sample": f"{sub} detectors x {g}^3 voxels, numpy",
                  "skipped": cov.n_skipped}))
