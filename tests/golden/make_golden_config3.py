"""Freeze a reduced BASELINE config-3 reconstruction from the key-fixed
reference (run HERE, where /root/reference exists; the GPU test reads the
committed tests/golden/config3.npz).

Config-3 geometry (Fibonacci-hemisphere subset, every 4th of the 512
detectors = 128), the 50k-ball branching-tube truth, a 24^3 grid init over
the interior box (p0 0.1, a0 0.15 mm), 40 MHz x 4096 samples; filter at f=4,
then the (4,100,coarse), (2,100,fine), (1,100,fine) schedule with density
control every 100 iterations (duplication_period 100), the plateau stop off,
and the zero-gradient filter re-applied every 10 iterations -- in the
reference through run_hierarchical's ``callback`` (optimizer.py:453-500),
which filters ``state`` in place with the reference predicate
(optimizer.py:230-258): survivors keep parameters, moments and last
gradients.  Saved: supervision, filter decisions, per-iteration ball counts
and losses, the cloud (and position-gradient norms) after iterations 100 and
200, the final cloud and its voxelized volume.

    python tests/golden/make_golden_config3.py
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, HERE)
sys.path.insert(0, ROOT)

from make_golden import load_reference  # noqa: E402

GRID_N = 24
DET_STRIDE = 4
SPACING = 28e-3 / 96   # config-3 thresholds and learning rates (the 96^3 spacing)


def instance(P, scenes):
    """Shared by this script and the GPU test (P: reference paball or ours)."""
    sc = scenes.schedule_config(grid_n=GRID_N)
    array = P.SensorArray(sc.array.positions[::DET_STRIDE], 1500.0, normals=sc.array.normals[::DET_STRIDE])
    return sc, array


def main() -> None:
    paball, _, rad, opt = load_reference()
    from paball.model import PointCloud, RngSeed
    from paball.radiator import ForwardContext
    from paball.render import RenderSpec, voxelize

    from paper_2601_00551_b200 import scenes

    t = time.time()
    rad.set_num_threads(os.cpu_count() or 1)
    sc, array = instance(paball, scenes)
    ctx = ForwardContext(array, paball.TimeGrid(0.0, sc.grid.dt, sc.grid.n_samples))
    truth = PointCloud(sc.truth.positions, sc.truth.p0, sc.truth.a0)
    real = rad.simulate_signals(truth, ctx)
    real = paball.SignalSet(real.grid, real.data.astype(np.float32).astype(np.float64))   # FP32-exact supervision
    print(f"supervision {time.time() - t:.1f} s", flush=True)
    init = PointCloud(sc.init.positions, sc.init.p0, sc.init.a0)
    kept, rep = opt.zero_gradient_filter(init, ctx, real, f=4)
    print(f"filter {len(init)} -> {len(kept)}  {time.time() - t:.1f} s", flush=True)
    levels = (opt.Level(4, 100, "coarse"), opt.Level(2, 100, "fine"), opt.Level(1, 100, "fine"))
    sched = opt.Schedule(levels, duplication_period=100)
    th = opt.DensityThresholds.from_spacing(SPACING)
    lr = opt.LearningRates.from_spacing(SPACING)
    filt_counts = []
    snaps = {}

    def refilter(state, step, li, loss):
        if step in (100, 200):   # the cloud after the step, before this iteration's filter / density control
            c = state.cloud
            snaps[step] = (c.positions.copy(), c.p0.copy(), c.a0.copy(),
                           np.linalg.norm(state.last_grad.d_position, axis=1))
        if step % 10:
            return
        f = levels[li].f
        _, r = opt.zero_gradient_filter(state.cloud, ctx, real, f=f)
        keep = r.g < 0.0
        filt_counts.append(int(keep.sum()))
        if keep.all():
            return
        state.cloud = state.cloud.subset(keep)
        for d in (state.m, state.v):
            for k in list(d):
                d[k] = d[k][keep]
        if state.last_grad is not None:
            g = state.last_grad
            state.last_grad = type(g)(g.d_p0[keep], g.d_a0[keep], g.d_position[keep])
        print(f"  step {step}: {len(state.cloud)} balls, loss {loss:.4e}  {time.time() - t:.0f} s", flush=True)

    saved = opt._PLATEAU_WINDOW
    opt._PLATEAU_WINDOW = 10 ** 9          # plateau stop off for parity runs
    try:
        final, trace = opt.run_hierarchical(kept.copy(), ctx, real, sched, th, lr=lr, seed=RngSeed(103),
                                            callback=refilter)
    finally:
        opt._PLATEAU_WINDOW = saved
    spec = RenderSpec(dims=(48, 48, 48), spacing=28e-3 / 48, origin=(-14e-3, -14e-3, -30e-3))
    vol = voxelize(final, spec).values
    np.savez_compressed(os.path.join(HERE, "config3.npz"), real=real.data.astype(np.float32), filter_g=rep.g,
                        counts=np.array([x.ball_count for x in trace.records]),
                        losses=np.array([x.loss for x in trace.records]), filt_counts=np.array(filt_counts),
                        final_pos=final.positions, final_p0=final.p0, final_a0=final.a0, volume=vol,
                        **{f"it{k}_{n}": v for k, t in snaps.items() for n, v in zip(("pos", "p0", "a0", "gnorm"), t)})
    print(f"config3 golden: {len(kept)} filtered -> {len(final)} final; {time.time() - t:.1f} s")


if __name__ == "__main__":
    main()
