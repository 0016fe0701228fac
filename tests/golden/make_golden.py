"""Freeze golden vectors from the reference implementation itself.

Run in the build container (needs /root/reference; never on the GPU host):

    python tests/golden/make_golden.py

It imports the reference package ``paball`` from /root/reference/pkg/src and
builds a *fixed* radiator by compiling the reference source with the
gradient-mode cache key renamed (``f"u{slab}"`` -> ``f"ucache{slab}"``,
SURVEY.md §0.2: the literal ``"u2"`` scratch buffer otherwise overwrites slab
2's cached u whenever a backward sees > 1024 balls).  ``paball.optimizer`` is
rebound to the fixed ``backward``.  Nothing of the reference is copied into the
repository: only its outputs on seeded inputs are stored.

Fixtures (``tests/golden/*.npz``):
  rng.npz          CounterRng streams (model.py:97-145)
  radiator.npz     single ball, seeded_instance (test_radiator.py:36-51):
                   forward, decimated forward, cutoff 12, backward fine/coarse
  bugfix.npz       1,100-ball backward (fixed reference) + the unfixed loss
  filter.npz       small_instance (test_optimizer.py:44-54) filter cases
  steps.npz        Adam steps (optimizer.py:266-306), fine and coarse
  density.npz      density_control with split + duplicate (optimizer.py:314-406)
  toy.npz          BASELINE config 1 (scenes.toy_config): forward of the truth,
                   32^3 grid filter at f=1, 5 fine Adam steps
  schedule.npz     filter + short hierarchical run + voxelized volume
"""

from __future__ import annotations

import os
import sys
import time
import types

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF_SRC = "/root/reference/pkg/src"


def load_reference():
    """Import paball and attach a key-fixed radiator as paball.radiator_fixed."""
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import paball  # noqa: F401
    import paball.optimizer as opt
    import paball.radiator as rad

    src = open(rad.__file__, encoding="utf-8").read()
    fixed = src.replace('f"u{slab}"', 'f"ucache{slab}"')
    if fixed == src:
        raise RuntimeError("reference radiator changed: cache key pattern not found")
    mod = types.ModuleType("paball.radiator_fixed")
    mod.__package__ = "paball"
    mod.__file__ = rad.__file__
    sys.modules["paball.radiator_fixed"] = mod
    exec(compile(fixed, rad.__file__ + " [cache key fixed]", "exec"), mod.__dict__)
    opt.backward = mod.backward
    return paball, rad, mod, opt


def main() -> None:
    sys.path.insert(0, ROOT)
    paball, rad_bug, rad, opt = load_reference()
    from paball.geometry import generate_array
    from paball.model import CounterRng, PointCloud, RngSeed, SignalSet, TimeGrid
    from paball.radiator import ForwardContext
    from paball.render import RenderSpec, voxelize

    from paper_2601_00551_b200 import scenes

    out = {}

    # ---------------- rng ----------------
    rng = {}
    for s in (0, 1, 123, 2 ** 64 - 1):
        r = CounterRng(s)
        rng[f"u_{s}"] = r.uniform(-1.0, 2.0, 17)
        rng[f"n_{s}"] = r.normal(7, 2.0)
        rng[f"v_{s}"] = r.unit_vectors(5)
        rng[f"c_{s}"] = CounterRng(s).spawn(3).uniform(0.0, 1.0, 4)
    np.savez_compressed(os.path.join(HERE, "rng.npz"), **rng)

    # ---------------- radiator ----------------
    cloud = PointCloud([[0.0, 0.0, 0.0]], [1.0], [0.5e-3])
    arr = paball.SensorArray(positions=[[0.03, 0.0, 0.0]], sound_speed=1500.0)
    ctx = ForwardContext(arr, TimeGrid(0.0, 1e-8, 4096))
    g = {"single_rows": rad.simulate_signals(cloud, ctx).data}

    def seeded_instance(seed=123, n_balls=10, n_sensors=16, n_samples=256):
        r = CounterRng(seed)
        array = generate_array("sphere", count=n_sensors, radius=0.008)
        c = ForwardContext(array, TimeGrid(0.0, 5e-8, n_samples))
        cand = PointCloud(r.uniform(-3e-3, 3e-3, 3 * n_balls).reshape(n_balls, 3),
                          r.uniform(0.5, 1.5, n_balls), r.uniform(0.4e-3, 0.8e-3, n_balls))
        tru = PointCloud(r.uniform(-3e-3, 3e-3, 3 * n_balls).reshape(n_balls, 3),
                         r.uniform(0.5, 1.5, n_balls), r.uniform(0.4e-3, 0.8e-3, n_balls))
        return c, cand, tru, rad.simulate_signals(tru, c)

    c, cand, tru, real = seeded_instance()
    g.update(si_sensors=c.array.positions, si_normals=c.array.normals,
             si_cand_pos=cand.positions, si_cand_p0=cand.p0, si_cand_a0=cand.a0,
             si_true_pos=tru.positions, si_true_p0=tru.p0, si_true_a0=tru.a0,
             si_real=real.data, si_cand_rows=rad.simulate_signals(cand, c).data)
    for f in (2, 4, 16):
        g[f"si_cand_rows_f{f}"] = rad.simulate_at_rate(cand, c, f).data
    wide = ForwardContext(c.array, c.grid, cutoff_sigma=12.0)
    g["si_cand_rows_cut12"] = rad.simulate_signals(cand, wide).data
    for stage in ("fine", "coarse"):
        L, gr = rad.backward(cand, c, real, stage=stage)
        g[f"si_{stage}_loss"] = np.array(L)
        g[f"si_{stage}_dp0"], g[f"si_{stage}_da0"], g[f"si_{stage}_dpos"] = gr.d_p0, gr.d_a0, gr.d_position
    L4, gr4 = rad.backward(cand, c, rad.downsample(real, 4), stage="fine")
    g["si_f4_loss"], g["si_f4_dp0"], g["si_f4_da0"], g["si_f4_dpos"] = np.array(L4), gr4.d_p0, gr4.d_a0, gr4.d_position
    rad.reset_op_count()
    rad.simulate_signals(cand, c)
    g["si_ops_f1"] = np.array(rad.op_count())
    rad.reset_op_count()
    rad.simulate_at_rate(cand, c, 4)
    g["si_ops_f4"] = np.array(rad.op_count())
    np.savez_compressed(os.path.join(HERE, "radiator.npz"), **g)

    # ---------------- bug-fix pin (> 1024 balls) ----------------
    r = CounterRng(77)
    n = 1100
    array = generate_array("sphere", count=24, radius=0.008)
    c = ForwardContext(array, TimeGrid(0.0, 5e-8, 512))
    cand = PointCloud(r.uniform(-3e-3, 3e-3, 3 * n).reshape(n, 3), r.uniform(0.2, 1.0, n),
                      r.uniform(0.3e-3, 0.6e-3, n))
    tru = PointCloud(r.uniform(-3e-3, 3e-3, 3 * 20).reshape(20, 3), r.uniform(0.5, 1.0, 20),
                     np.full(20, 0.5e-3))
    real = rad.simulate_signals(tru, c)
    L, gr = rad.backward(cand, c, real, stage="fine")
    Lbug, _ = rad_bug.backward(cand, c, real, stage="fine")
    np.savez_compressed(os.path.join(HERE, "bugfix.npz"), sensors=array.positions,
                        pos=cand.positions, p0=cand.p0, a0=cand.a0, real=real.data,
                        loss=np.array(L), dp0=gr.d_p0, da0=gr.d_a0, dpos=gr.d_position,
                        loss_unfixed=np.array(Lbug),
                        loss_direct=np.array(rad.loss(rad.simulate_signals(cand, c), real)))

    # ---------------- filter / steps (small_instance) ----------------
    def small_instance(seed=5, n_sensors=32, n_samples=512):
        array = generate_array("sphere", count=n_sensors, radius=0.008)
        c = ForwardContext(array, TimeGrid(0.0, 5e-8, n_samples))
        r = CounterRng(seed)
        tru = PointCloud(r.uniform(-2.5e-3, 2.5e-3, 9).reshape(3, 3), r.uniform(0.8, 1.2, 3),
                         r.uniform(4e-4, 6e-4, 3))
        return c, tru, rad.simulate_signals(tru, c)

    c, tru, real = small_instance()
    fl = {"sensors": c.array.positions, "true_pos": tru.positions, "true_p0": tru.p0,
          "true_a0": tru.a0, "real": real.data}
    r = CounterRng(3)
    cand = PointCloud(r.uniform(-3.5e-3, 3.5e-3, 450).reshape(150, 3), np.full(150, 0.1), np.full(150, 5e-4))
    kept, rep = opt.zero_gradient_filter(cand, c, real, f=4)
    fl.update(ip_pos=cand.positions, ip_g=rep.g, ip_kept=len(kept))
    r = CounterRng(4)
    near = r.uniform(-3e-3, 3e-3, 180).reshape(60, 3)
    far = 25e-3 * CounterRng(41).unit_vectors(10)
    cand = PointCloud(np.vstack([near, far]), np.full(70, 0.1), np.full(70, 4e-4))
    kept, rep = opt.zero_gradient_filter(cand, c, real, f=2)
    fl.update(nf_pos=cand.positions, nf_g=rep.g, nf_kept=len(kept))
    np.savez_compressed(os.path.join(HERE, "filter.npz"), **fl)

    st = {}
    cloud = tru.copy()
    cloud.p0 = tru.p0 * 1.10
    cloud.positions = tru.positions + 1e-4
    state = opt.create_state(cloud, seed=1)
    losses = []
    for _ in range(3):
        state, L = opt.step(state, c, real, 1, "fine")
        losses.append(L)
    st.update(fine_losses=np.array(losses), fine_pos=state.cloud.positions,
              fine_p0=state.cloud.p0, fine_a0=state.cloud.a0)
    cloud = tru.copy()
    cloud.p0 = tru.p0 * 0.5
    state = opt.create_state(cloud, seed=1)
    real4 = rad.downsample(real, 4)
    losses = []
    for _ in range(4):
        state, L = opt.step(state, c, real4, 4, "coarse")
        losses.append(L)
    st.update(coarse_losses=np.array(losses), coarse_pos=state.cloud.positions,
              coarse_p0=state.cloud.p0, coarse_a0=state.cloud.a0)
    np.savez_compressed(os.path.join(HERE, "steps.npz"), **st)

    # ---------------- density control ----------------
    r = CounterRng(9)
    n = 40
    pos = r.uniform(-3e-3, 3e-3, 3 * n).reshape(n, 3)
    p0 = r.uniform(0.0, 1.0, n)
    p0[3] = 1e-4                      # destroyed (weak)
    a0 = r.uniform(3e-4, 1.6e-3, n)   # some above split_a0 = 1e-3
    a0[5] = 6e-3                      # destroyed (too large)
    th = opt.DensityThresholds(destroy_p0_frac=0.02, split_a0=1e-3, duplicate_grad_quantile=0.9,
                               a0_min=1e-4, a0_max=5e-3)
    dens = {"pos": pos, "p0": p0, "a0": a0}
    for stage in ("coarse", "fine"):
        state = opt.create_state(PointCloud(pos, p0, a0), seed=4)
        state.cloud.generation = 2
        state.m["p0"] = np.arange(n, dtype=np.float64)
        state.v["position"] = np.arange(3 * n, dtype=np.float64).reshape(n, 3)
        gpos = r.uniform(-1.0, 1.0, 3 * n).reshape(n, 3)
        state.last_grad = rad.ParamGradients(np.zeros(n), np.zeros(n), gpos)
        dens[f"{stage}_grad"] = gpos
        out = opt.density_control(state, th, stage)
        dens.update({f"{stage}_out_pos": out.cloud.positions, f"{stage}_out_p0": out.cloud.p0,
                     f"{stage}_out_a0": out.cloud.a0, f"{stage}_m_p0": out.m["p0"],
                     f"{stage}_v_pos": out.v["position"],
                     f"{stage}_generation": np.array(out.cloud.generation)})
    np.savez_compressed(os.path.join(HERE, "density.npz"), **dens)

    # ---------------- BASELINE config 1 (toy) ----------------
    t = time.time()
    sc = scenes.toy_config()
    ctx = ForwardContext(paball.SensorArray(sc.array.positions, 1500.0, sc.array.normals), sc.grid)
    truth = PointCloud(sc.truth.positions, sc.truth.p0, sc.truth.a0)
    real = rad.simulate_signals(truth, ctx)
    init = PointCloud(sc.init.positions, sc.init.p0, sc.init.a0)
    kept, rep = opt.zero_gradient_filter(init, ctx, real, f=1)
    lr = opt.LearningRates(p0=1e-2, a0=1e-5, position=5e-6)
    state = opt.create_state(kept.copy(), lr=lr, seed=103)
    losses = []
    for _ in range(5):
        state, L = opt.step(state, ctx, real, 1, "fine")
        losses.append(L)
    np.savez_compressed(os.path.join(HERE, "toy.npz"), real=real.data, filter_g=rep.g,
                        n_kept=np.array(len(kept)), step_losses=np.array(losses),
                        final_pos=state.cloud.positions, final_p0=state.cloud.p0,
                        final_a0=state.cloud.a0, lr=np.array([lr.p0, lr.a0, lr.position]))
    print(f"toy: kept {len(kept)} of {len(init)}; {time.time() - t:.1f} s")

    # ---------------- short schedule + voxelized volume ----------------
    t = time.time()
    c, tru, real = small_instance(seed=6)
    r = CounterRng(61)
    n = 200
    init = PointCloud(r.uniform(-3e-3, 3e-3, 3 * n).reshape(n, 3), np.full(n, 0.05), np.full(n, 5e-4))
    filt, rep = opt.zero_gradient_filter(init, c, real, f=8)
    sched = opt.Schedule((opt.Level(8, 150, "coarse"), opt.Level(2, 60, "fine"), opt.Level(1, 60, "fine")),
                         duplication_period=50)
    th = opt.DensityThresholds.from_spacing(4e-4)
    lr = opt.LearningRates.from_spacing(4e-4)
    saved = opt._PLATEAU_WINDOW
    opt._PLATEAU_WINDOW = 10 ** 9          # plateau stop off for parity runs
    try:
        final, trace = opt.run_hierarchical(filt.copy(), c, real, sched, th, lr=lr, seed=RngSeed(61))
    finally:
        opt._PLATEAU_WINDOW = saved
    spec = RenderSpec(dims=(31, 31, 31), spacing=2e-4, origin=(-3e-3, -3e-3, -3e-3))
    vol = voxelize(final, spec).values
    vol_truth = voxelize(tru, spec).values
    np.savez_compressed(os.path.join(HERE, "schedule.npz"), sensors=c.array.positions,
                        true_pos=tru.positions, true_p0=tru.p0, true_a0=tru.a0, real=real.data,
                        init_pos=init.positions, filter_g=rep.g, filt_n=np.array(len(filt)),
                        losses=np.array([x.loss for x in trace.records]),
                        counts=np.array([x.ball_count for x in trace.records]),
                        final_pos=final.positions, final_p0=final.p0, final_a0=final.a0,
                        volume=vol, volume_truth=vol_truth)
    print(f"schedule: {len(filt)} filtered -> {len(final)} final; {time.time() - t:.1f} s")


if __name__ == "__main__":
    main()
