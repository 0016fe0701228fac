"""Save the config-3 reconstruction's cloud after iteration 250 (f = 1 level)
to gpurun_out/level2_cloud.npz, or (with an argument) run one forward pass of
it -- a case for ncu (tuning tool)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_00551_b200 as P  # noqa: E402
from paper_2601_00551_b200 import engine as E  # noqa: E402
from paper_2601_00551_b200 import radiator as R  # noqa: E402
from paper_2601_00551_b200 import scenes  # noqa: E402

sc = scenes.schedule_config()
ctx = P.ForwardContext(sc.array, sc.grid)
out = os.path.join("gpurun_out", "level2_cloud.npz")
if len(sys.argv) == 1:
    real = P.simulate_signals(sc.truth, ctx)
    spacing = 28e-3 / 96
    snap = {}
    sched = P.Schedule((P.Level(4, 100, "coarse"), P.Level(2, 100, "fine"), P.Level(1, 100, "fine")),
                       duplication_period=100)

    def cb(state, step, li, loss):
        if step == 250:
            snap["c"] = state.cloud.copy()
    kept, _ = P.zero_gradient_filter(sc.init, ctx, real, f=4)
    P.run_hierarchical(kept, ctx, real, sched, P.DensityThresholds.from_spacing(spacing),
                       lr=P.LearningRates.from_spacing(spacing), seed=103, filter_every=10, plateau=False, callback=cb)
    c = snap["c"]
    np.savez(out, pos=c.positions, p0=c.p0, a0=c.a0)
    print("saved", len(c))
else:
    d = np.load(out)
    det = R.device_detectors(ctx)
    acq = R._acq(ctx, 1)
    cloud = E.DeviceCloud.from_host(d["pos"], d["p0"], d["a0"], det.pos.device)
    for _ in range(2):
        cnt = E.PassCounters(det.pos.device)
        cloud.invalidate()
        E.forward_rows(cloud, det, acq, cnt)
    torch.cuda.synchronize()
    print("ok")
