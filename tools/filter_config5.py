"""Config-5 zero-gradient filter (8.8M-ball grid cloud, f = 4) timed cold and
warm through the public API, with the GPU kernels of the warm call (tuning
tool)."""
import os
import sys
import time

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_2601_00551_b200 as P  # noqa: E402
from paper_2601_00551_b200 import scenes  # noqa: E402

sc = scenes.mouse_config()
ctx = P.ForwardContext(sc.array, sc.grid, directivity=P.Directivity("cos_power", power=2.0))
real = P.simulate_signals(sc.truth, ctx)
for it in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    kept, rep = P.zero_gradient_filter(sc.init, ctx, real, f=4)
    torch.cuda.synchronize()
    print(f"filter call {it}: {time.perf_counter() - t0:.3f} s, kept {rep.n_retained}")
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    kept, rep = P.zero_gradient_filter(sc.init, ctx, real, f=4)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="self_device_time_total", row_limit=12, max_name_column_width=60))
print(prof.key_averages().table(sort_by="cpu_time_total", row_limit=12, max_name_column_width=60))
