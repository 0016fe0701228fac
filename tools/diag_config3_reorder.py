"""Diagnostic (tuning tool): sensitivity of the reduced config-3 run to the
FP32 summation order -- the same GPU schedule with the forward's cloud packed
in 5 instead of 6 radius buckets (a different, equally exact summation order
of every row) -- next to its distance from the FP64 reference."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "tests", "golden")]
import paper_2601_00551_b200 as P  # noqa: E402
from make_golden_config3 import SPACING, instance  # noqa: E402
from oracle import render as ORend  # noqa: E402
from pab_helpers import golden, rel_l2  # noqa: E402

from paper_2601_00551_b200 import engine as E  # noqa: E402
from paper_2601_00551_b200 import scenes  # noqa: E402

g = golden("config3.npz")
sc, array = instance(P, scenes)
ctx = P.ForwardContext(array, sc.grid)
real = P.SignalSet(sc.grid, g["real"].astype(np.float64))
vox = lambda c: ORend.voxelize(c.positions, c.p0, c.a0, (48, 48, 48), 28e-3 / 48, (-14e-3, -14e-3, -30e-3))


def run(buckets):
    E.A0_BUCKETS = buckets
    kept, _ = P.zero_gradient_filter(sc.init, ctx, real, f=4)
    snap = {}

    def cb(state, step, li, loss):
        if step in (100, 150, 200, 250):
            snap[step] = state.cloud.copy()
    sched = P.Schedule((P.Level(4, 100, "coarse"), P.Level(2, 100, "fine"), P.Level(1, 100, "fine")),
                       duplication_period=100)
    final, trace = P.run_hierarchical(kept.copy(), ctx, real, sched, P.DensityThresholds.from_spacing(SPACING),
                                      lr=P.LearningRates.from_spacing(SPACING), seed=P.RngSeed(103),
                                      filter_every=10, plateau=False, callback=cb)
    snap[300] = final
    return snap, np.array([r.ball_count for r in trace.records])


a, ca = run(6)
b, cb_ = run(5)
for it in (100, 150, 200, 250, 300):
    ref = None
    if f"it{it}_p0" in g:
        ref = ORend.voxelize(g[f"it{it}_pos"], g[f"it{it}_p0"], g[f"it{it}_a0"], (48, 48, 48), 28e-3 / 48,
                             (-14e-3, -14e-3, -30e-3))
    if it == 300:
        ref = g["volume"]
    va, vb = vox(a[it]), vox(b[it])
    print(f"iteration {it}: GPU(6 buckets) vs GPU(5 buckets) volume rel L2 {rel_l2(va, vb):.2e}"
          + (f"; GPU(6) vs FP64 reference {rel_l2(va, ref):.2e}" if ref is not None else ""),
          f"counts {len(a[it])} / {len(b[it])}")
print("count trajectories identical:", bool(np.array_equal(ca, cb_)))
