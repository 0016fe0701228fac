"""Config-3 reconstruction (filter + 4/2/1 x 100, filter every 10, density
control every 100) under the torch profiler (tuning tool): wall time, GPU
busy time per kernel name, and the device-idle share (host/launch-bound
part of the iteration driver)."""
import collections
import os
import sys
import time

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_00551_b200 as P  # noqa: E402
from paper_2601_00551_b200 import scenes  # noqa: E402

sc = scenes.schedule_config()
ctx = P.ForwardContext(sc.array, sc.grid)
real = P.simulate_signals(sc.truth, ctx)
spacing = 28e-3 / 96
th = P.DensityThresholds.from_spacing(spacing)
lr = P.LearningRates.from_spacing(spacing)
sched = P.Schedule((P.Level(4, 100, "coarse"), P.Level(2, 100, "fine"), P.Level(1, 100, "fine")),
                   duplication_period=100)


def run():
    kept, rep = P.zero_gradient_filter(sc.init, ctx, real, f=4)
    return P.run_hierarchical(kept, ctx, real, sched, th, lr=lr, seed=103, filter_every=10, plateau=False)


run()
torch.cuda.synchronize()
t0 = time.perf_counter()
run()
torch.cuda.synchronize()
print(f"warm wall {time.perf_counter() - t0:.3f} s")
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    t0 = time.perf_counter()
    run()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
evs = sorted((e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA),
             key=lambda e: e.time_range.start)
busy = collections.Counter()
cnt = collections.Counter()
union = 0.0
end = None
for e in evs:
    s, t = e.time_range.start, e.time_range.end
    busy[e.name.split("(")[0][:70]] += (t - s) / 1e3
    cnt[e.name.split("(")[0][:70]] += 1
    if end is None or s >= end:
        union += (t - s) / 1e3
        end = t
    elif t > end:
        union += (t - end) / 1e3
        end = t
span = (evs[-1].time_range.end - evs[0].time_range.start) / 1e3
print(f"profiled wall {wall * 1e3:.1f} ms, device timeline {span:.1f} ms, device busy (union) {union:.1f} ms, "
      f"idle {span - union:.1f} ms, launches {len(evs)}")
for name, ms in busy.most_common(25):
    print(f"  {ms:9.2f} ms  x{cnt[name]:5d}  {name}")
