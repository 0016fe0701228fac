"""GPU timeline of public-API backward() calls at config 2 with pageable
inputs (tuning tool): kernels and memcpys from the torch profiler (CUPTI),
the device-idle gaps between them and the host wall time per call."""
import os
import sys
import time

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_00551_b200 as P  # noqa: E402
from paper_2601_00551_b200 import scenes  # noqa: E402

sc = scenes.microbench_config()
ctx = P.ForwardContext(sc.array, sc.grid, directivity=P.Directivity("cos_power", power=2.0))
real = P.simulate_signals(sc.truth, ctx)
real = P.SignalSet(real.grid, np.array(real.data))          # pageable, as a caller holds it
cloud = sc.init
for _ in range(3):
    P.backward(cloud, ctx, real, stage="fine")
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    walls = []
    for _ in range(2):
        t0 = time.perf_counter()
        P.backward(cloud, ctx, real, stage="fine")
        walls.append(1e3 * (time.perf_counter() - t0))
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
evs.sort(key=lambda e: e.time_range.start)
print("wall per call (ms):", [round(w, 2) for w in walls])
t_first = evs[0].time_range.start
prev_end = None
busy = 0.0
for e in evs:
    s, t = e.time_range.start, e.time_range.end
    gap = (s - prev_end) / 1e3 if prev_end is not None else 0.0
    busy += (t - s) / 1e3
    print(f"{(s - t_first) / 1e3:9.3f} ms  +{gap:7.3f} gap  {(t - s) / 1e3:8.3f} ms  {e.name[:90]}")
    prev_end = max(prev_end or t, t)
print(f"device busy {busy:.2f} ms over {(prev_end - t_first) / 1e3:.2f} ms of timeline")
cpu = sorted(prof.key_averages(), key=lambda a: -a.cpu_time_total)[:25]
for a in cpu:
    print(f"cpu {a.key[:60]:60s} total {a.cpu_time_total / 1e3:8.2f} ms  calls {a.count}")
