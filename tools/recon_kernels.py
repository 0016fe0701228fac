"""Config-3 reconstruction: device time per kernel over the whole run
(torch profiler, CUDA activity; tuning tool)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_00551_b200 as P  # noqa: E402
from paper_2601_00551_b200 import scenes  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

sc = scenes.schedule_config()
ctx = P.ForwardContext(sc.array, sc.grid)
real = P.simulate_signals(sc.truth, ctx)
spacing = 28e-3 / 96
th = P.DensityThresholds.from_spacing(spacing)
lr = P.LearningRates.from_spacing(spacing)
sched = P.Schedule((P.Level(4, 100, "coarse"), P.Level(2, 100, "fine"), P.Level(1, 100, "fine")),
                   duplication_period=100)
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        kept, rep_ = P.zero_gradient_filter(sc.init, ctx, real, f=4)
        final, trace = P.run_hierarchical(kept, ctx, real, sched, th, lr=lr, seed=103, filter_every=10,
                                          plateau=False)
        torch.cuda.synchronize()
    wall = time.perf_counter() - t0
ka = prof.key_averages()
tot = sum(e.self_device_time_total for e in ka) / 1e3
print(f"wall {wall:.3f} s (under the profiler), device busy {tot:.1f} ms")
for e in sorted(ka, key=lambda e: -e.self_device_time_total)[:25]:
    print(f"{e.self_device_time_total / 1e3:9.2f} ms  x{e.count:<5d} {e.key[:90]}")
