"""BASELINE config 5 (mouse scale) reconstruction on one GPU through the
public API: zero-gradient filter of the 8.8M-ball grid cloud at f = 4, then a
shortened 4/2/1 hierarchical schedule (ITERS iterations per level, default
10) with the filter re-applied every 10 iterations and density control at
the reference cadence.  Prints wall time per phase and per level (host wall
clock around synchronised public-API calls).

usage: python tools/recon_config5.py [ITERS]
"""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_2601_00551_b200 as P  # noqa: E402
from paper_2601_00551_b200 import scenes  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 10
t0 = time.perf_counter()
sc = scenes.mouse_config()
t_scene = time.perf_counter() - t0
ctx = P.ForwardContext(sc.array, sc.grid, directivity=P.Directivity("cos_power", power=2.0))
torch.cuda.synchronize()
t0 = time.perf_counter()
real = P.simulate_signals(sc.truth, ctx)
torch.cuda.synchronize()
t_truth = time.perf_counter() - t0
spacing = 2 * 12.5e-3 / 256
th = P.DensityThresholds.from_spacing(spacing)
lr = P.LearningRates.from_spacing(spacing)
sched = P.Schedule((P.Level(4, iters, "coarse"), P.Level(2, iters, "fine"), P.Level(1, iters, "fine")),
                   duplication_period=100)
torch.cuda.synchronize()
t0 = time.perf_counter()
kept, rep = P.zero_gradient_filter(sc.init, ctx, real, f=4)
torch.cuda.synchronize()
t_filter = time.perf_counter() - t0
level_t = {}
def cb(state, step, level, loss):   # wall time at the last iteration of each level
    level_t[level] = time.perf_counter()
t1 = time.perf_counter()
final, trace = P.run_hierarchical(kept, ctx, real, sched, th, lr=lr, seed=5, filter_every=10, plateau=False,
                                  callback=cb)
torch.cuda.synchronize()
t_sched = time.perf_counter() - t1
recs = trace.records
print(json.dumps({
    "workload": f"config5: 2048 det x 8192 samples, 256^3 grid in ellipsoid ({len(sc.init)} balls), "
                f"300k-ball truth; filter at f=4, schedule 4/2/1 x {iters}",
    "scene_s": t_scene, "truth_forward_s": t_truth, "filter_s": t_filter, "n_after_filter": len(kept),
    "schedule_s": t_sched, "iterations": len(recs), "s_per_iteration": t_sched / max(len(recs), 1),
    "level_end_s": {k: v - t1 for k, v in sorted(level_t.items())},
    "n_final": len(final), "loss_first": recs[0].loss, "loss_last": recs[-1].loss}))
