"""Where the end-to-end backward() time goes (config 2): torch.profiler
table of host-side ops and device kernels/copies over a few public-API
calls with pinned host inputs.

usage: python tools/e2e_profile.py [n_balls] [n_det]
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_2601_00551_b200 as P  # noqa: E402
from paper_2601_00551_b200 import radiator as R  # noqa: E402
from paper_2601_00551_b200 import scenes  # noqa: E402

n_balls = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
n_det = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
sc = scenes.microbench_config(n_balls=n_balls, n_det=n_det)
ctx = P.ForwardContext(sc.array, sc.grid, directivity=P.Directivity("cos_power", power=2.0))
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
real = P.simulate_signals(sc.truth, ctx)
host_real = P.SignalSet(sc.grid, pin(real.data))
host_cloud = P.PointCloud(pin(sc.init.positions), pin(sc.init.p0), pin(sc.init.a0))
P.backward(host_cloud, ctx, host_real, stage="fine")
for _ in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    P.backward(host_cloud, ctx, host_real, stage="fine")
    torch.cuda.synchronize()
    print(f"e2e {1e3 * (time.perf_counter() - t0):.2f} ms")
from torch.profiler import ProfilerActivity, profile  # noqa: E402
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    for _ in range(2):
        P.backward(host_cloud, ctx, host_real, stage="fine")
        torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cpu_time_total", row_limit=30))
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=20))
