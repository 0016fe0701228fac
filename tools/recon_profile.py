"""Config-3 reconstruction: wall time per level vs GPU kernel time (tuning
tool): how launch/host-bound the iteration driver is."""
import os
import sys
import time

import numpy as np
import torch

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
kept, rep = P.zero_gradient_filter(sc.init, ctx, real, f=4)
torch.cuda.synchronize()
t0 = time.perf_counter()
final, trace = P.run_hierarchical(kept, ctx, real, sched, th, lr=lr, seed=103, filter_every=10, plateau=False)
torch.cuda.synchronize()
wall = time.perf_counter() - t0
ts = np.array([r.time_s for r in trace.records])
lv = np.array([r.level for r in trace.records])
cnt = np.array([r.ball_count for r in trace.records])
print(f"wall {wall:.3f} s")
for L in range(3):
    m = lv == L
    d = np.diff(np.concatenate([[0.0], ts]))[m]
    print(f"level {L}: {m.sum()} iterations, median {1e3 * np.median(d):.2f} ms/it, balls {cnt[m][0]}..{cnt[m][-1]}")
from torch.profiler import ProfilerActivity, profile  # noqa: E402
for L, lvl in enumerate(sched.levels):
    state = P.create_state(final.copy() if L else kept.copy(), lr=lr, seed=1)
    real_k = P.downsample(real, lvl.f) if lvl.f > 1 else real
    for _ in range(3):
        state, _ = P.step(state, ctx, real_k, lvl.f, lvl.stage)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        t1 = time.perf_counter()
        for _ in range(10):
            state, _ = P.step(state, ctx, real_k, lvl.f, lvl.stage)
        torch.cuda.synchronize()
        w = (time.perf_counter() - t1) / 10
    gpu = sum(e.self_device_time_total for e in prof.key_averages()) / 10 / 1e3
    print(f"level {L} step() on {state.n} balls: wall {1e3 * w:.2f} ms, GPU kernels+copies {gpu:.2f} ms")
