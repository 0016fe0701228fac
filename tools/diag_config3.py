"""Diagnostic (tuning tool): where the GPU's reduced config-3 run and the
reference's (tests/golden/config3.npz) separate, ball by ball."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "tests", "golden")]
import paper_2601_00551_b200 as P  # noqa: E402
from make_golden_config3 import SPACING, instance  # noqa: E402
from pab_helpers import golden  # noqa: E402

from paper_2601_00551_b200 import scenes  # noqa: E402

g = golden("config3.npz")
sc, array = instance(P, scenes)
ctx = P.ForwardContext(array, sc.grid)
real = P.SignalSet(sc.grid, g["real"].astype(np.float64))
kept, rep = P.zero_gradient_filter(sc.init, ctx, real, f=4)
snap = {}
stop = int(sys.argv[1]) if len(sys.argv) > 1 else 200


def cb(state, step, li, loss):
    if step in (100, 110, 120, 150, 200):
        snap[step] = state.cloud.copy()


sched = P.Schedule((P.Level(4, 100, "coarse"), P.Level(2, 100, "fine"), P.Level(1, 1, "fine")), duplication_period=100)
P.run_hierarchical(kept.copy(), ctx, real, sched, P.DensityThresholds.from_spacing(SPACING),
                   lr=P.LearningRates.from_spacing(SPACING), seed=P.RngSeed(103), filter_every=10, plateau=False,
                   callback=cb)
c = snap[200]
ra0, rp0, rpos = g["it200_a0"], g["it200_p0"], g["it200_pos"]
da = np.abs(c.a0 - ra0) / np.maximum(np.abs(ra0), 1e-30)
dp = np.linalg.norm(c.positions - rpos, axis=1)
print("n", len(c), "a0 rel diff quantiles 50/90/99/99.9/max:", np.quantile(da, [0.5, 0.9, 0.99, 0.999, 1.0]))
print("pos abs diff (m) quantiles:", np.quantile(dp, [0.5, 0.9, 0.99, 0.999, 1.0]))
worst = np.argsort(-da)[:12]
print("worst a0: ref", ra0[worst], "\n          gpu", c.a0[worst], "\n p0 ref", rp0[worst])
print("balls with a0 rel diff > 1e-3:", int((da > 1e-3).sum()), " a0 at floor (<1e-6) ref/gpu:",
      int((ra0 < 1e-6).sum()), int((c.a0 < 1e-6).sum()))
