"""Forward / adjoint kernel times on the config-3 reconstruction's own clouds
(captured at iterations 50, 150, 250) vs their pair counts (tuning tool)."""
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
real = P.simulate_signals(sc.truth, ctx)
spacing = 28e-3 / 96
sched = P.Schedule((P.Level(4, 100, "coarse"), P.Level(2, 100, "fine"), P.Level(1, 100, "fine")),
                   duplication_period=100)
snap = {}


def cb(state, step, li, loss):
    if step in (50, 150, 250):
        snap[step] = state.cloud.copy()


kept, _ = P.zero_gradient_filter(sc.init, ctx, real, f=4)
P.run_hierarchical(kept, ctx, real, sched, P.DensityThresholds.from_spacing(spacing),
                   lr=P.LearningRates.from_spacing(spacing), seed=103, filter_every=10, plateau=False, callback=cb)
det = R.device_detectors(ctx)
dev = det.pos.device
for step, f, stage in ((50, 4, 1), (150, 2, 2), (250, 1, 2)):
    c = snap[step]
    acq = R._acq(ctx, f)
    real_k = R.device_supervision(P.downsample(real, f).data if f > 1 else real.data, det)
    cloud = E.DeviceCloud.from_host(c.positions, c.p0, c.a0, dev)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    ts = []
    for rep in range(4):
        cnt = E.PassCounters(dev)
        cloud.invalidate()
        ev[0].record()
        res, lr_ = E.forward_rows(cloud, det, acq, cnt, real_local=real_k)
        ev[1].record()
        E.adjoint_grads(cloud, det, acq, res, 1.0, stage, 1.0, cnt, loss_rows=lr_)
        ev[2].record()
        torch.cuda.synchronize()
        ts.append((ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2])))
    _, ops = cnt.result()
    fw, ad = np.median([t[0] for t in ts[1:]]), np.median([t[1] for t in ts[1:]])
    pairs = len(c) * det.n_total
    plan = E.plan_forward(cloud, det, acq)
    meta = cloud.gmeta[: cloud.n_groups * 48].view(torch.float32).view(cloud.n_groups, 12).cpu().numpy()
    rad, amax = meta[:, 6], meta[:, 7]
    span = (2 * rad + 12 * amax) / (1500.0 * sc.grid.dt * f)   # samples a group can touch at one detector
    print(f"   group radius mm quantiles 50/90/99/max {np.quantile(rad * 1e3, [0.5, 0.9, 0.99, 1.0]).round(3)}, "
          f"groups spanning > 152 samples: {100 * np.mean(span > 152):.1f} %")
    print(f"it {step} f={f} stage={stage}: {len(c)} balls, {pairs:.3g} pairs, {ops / pairs:.1f} samples/pair; "
          f"forward {fw:.2f} ms ({ops / fw / 1e9:.2f} Gsamples/s, parts {plan.partitions}), adjoint {ad:.2f} ms "
          f"({ops / ad / 1e9:.2f} Gsamples/s, chunks {E.plan_adjoint(cloud.adjoint_cloud(), det)}); "
          f"a0 median {np.median(c.a0) * 1e3:.3f} mm, min {c.a0.min() * 1e3:.3g} max {c.a0.max() * 1e3:.3g}")
