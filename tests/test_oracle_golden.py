"""Pin the CPU oracle to the reference's own outputs (tests/golden/*.npz,
produced by tests/golden/make_golden.py from the key-fixed reference)."""

import numpy as np
import pytest

from oracle import optimizer as OO
from oracle import radiator as OR
from oracle import render as ORend
from oracle.rng import CounterRng as OracleRng
from pab_helpers import golden, rel_l2


def test_rng_streams_match_reference():
    g = golden("rng.npz")
    from paper_2601_00551_b200.model import CounterRng
    for s in (0, 1, 123, 2 ** 64 - 1):
        for R in (CounterRng, OracleRng):
            r = R(s)
            assert np.array_equal(r.uniform(-1.0, 2.0, 17), g[f"u_{s}"])
            assert np.array_equal(r.normal(7, 2.0), g[f"n_{s}"])
            assert np.array_equal(r.unit_vectors(5), g[f"v_{s}"])
            assert np.array_equal(R(s).spawn(3).uniform(0.0, 1.0, 4), g[f"c_{s}"])


def _si(g, key="cand"):
    return g[f"si_{key}_pos"], g[f"si_{key}_p0"], g[f"si_{key}_a0"]


def test_single_ball_forward_bit_exact():
    g = golden("radiator.npz")
    rows, _, _, _ = OR.run_model([[0, 0, 0]], [1.0], [0.5e-3], [[0.03, 0, 0]], None,
                                 1500.0, 0.0, 1e-8, 4096, 1)
    assert np.array_equal(rows, g["single_rows"])


@pytest.mark.parametrize("f", [1, 2, 4, 16])
def test_seeded_forward_bit_exact(f):
    g = golden("radiator.npz")
    pos, p0, a0 = _si(g)
    rows, _, _, _ = OR.run_model(pos, p0, a0, g["si_sensors"], None, 1500.0, 0.0, 5e-8, 256, f)
    want = g["si_cand_rows"] if f == 1 else g[f"si_cand_rows_f{f}"]
    assert np.array_equal(rows, want)


def test_seeded_forward_cutoff12():
    g = golden("radiator.npz")
    pos, p0, a0 = _si(g)
    rows, _, _, _ = OR.run_model(pos, p0, a0, g["si_sensors"], None, 1500.0, 0.0, 5e-8, 256, 1, cutoff=12.0)
    assert np.array_equal(rows, g["si_cand_rows_cut12"])


@pytest.mark.parametrize("stage", ["fine", "coarse"])
def test_seeded_backward(stage):
    g = golden("radiator.npz")
    pos, p0, a0 = _si(g)
    _, L, (gp0, ga0, gpos), _ = OR.run_model(pos, p0, a0, g["si_sensors"], None, 1500.0, 0.0, 5e-8,
                                             256, 1, real=g["si_real"], stage=stage)
    assert abs(L - float(g[f"si_{stage}_loss"])) <= 1e-14 * abs(L)
    assert rel_l2(gp0, g[f"si_{stage}_dp0"]) < 1e-12
    assert rel_l2(ga0, g[f"si_{stage}_da0"]) < 1e-12
    if stage == "fine":
        assert rel_l2(gpos, g[f"si_{stage}_dpos"]) < 1e-12
    else:
        assert not gpos.any() and not g["si_coarse_dpos"].any()


def test_seeded_backward_decimated_supervision():
    g = golden("radiator.npz")
    pos, p0, a0 = _si(g)
    real4 = OR.downsample(g["si_real"], 4)
    _, L, (gp0, ga0, gpos), _ = OR.run_model(pos, p0, a0, g["si_sensors"], None, 1500.0, 0.0, 5e-8,
                                             256, 4, real=real4, stage="fine")
    assert abs(L - float(g["si_f4_loss"])) <= 1e-13 * abs(L)
    assert rel_l2(gp0, g["si_f4_dp0"]) < 1e-12
    assert rel_l2(gpos, g["si_f4_dpos"]) < 1e-12


def test_op_counts_match_reference():
    g = golden("radiator.npz")
    pos, p0, a0 = _si(g)
    for f, key in ((1, "si_ops_f1"), (4, "si_ops_f4")):
        _, _, _, ops = OR.run_model(pos, p0, a0, g["si_sensors"], None, 1500.0, 0.0, 5e-8, 256, f)
        assert ops == int(g[key])


def test_bugfix_case_above_1024_balls():
    """> 1024 balls: the oracle equals the key-fixed reference, and the fixed
    backward loss equals the direct loss (the unfixed one does not)."""
    g = golden("bugfix.npz")
    _, L, (gp0, ga0, gpos), _ = OR.run_model(g["pos"], g["p0"], g["a0"], g["sensors"], None, 1500.0,
                                             0.0, 5e-8, 512, 1, real=g["real"], stage="fine")
    assert abs(L - float(g["loss"])) <= 1e-13 * L
    assert abs(float(g["loss"]) - float(g["loss_direct"])) <= 1e-13 * L
    assert abs(float(g["loss_unfixed"]) - float(g["loss_direct"])) > 1e-9 * L
    assert rel_l2(gp0, g["dp0"]) < 1e-12
    assert rel_l2(ga0, g["da0"]) < 1e-12
    assert rel_l2(gpos, g["dpos"]) < 1e-12


def _small_problem(g):
    return OO.Problem(g["sensors"], None, 1500.0, 0.0, 5e-8, 512)


def test_filter_matches_reference():
    g = golden("filter.npz")
    prob = _small_problem(g)
    for key, f in (("ip", 4), ("nf", 2)):
        pos = g[f"{key}_pos"]
        n = pos.shape[0]
        a0 = np.full(n, 5e-4 if key == "ip" else 4e-4)
        keep, gg = OO.zero_gradient_filter(prob, pos, np.full(n, 0.1), a0, g["real"], f)
        assert rel_l2(gg, g[f"{key}_g"]) < 1e-12
        assert np.array_equal(gg < 0, g[f"{key}_g"] < 0)
        assert int(keep.sum()) == int(g[f"{key}_kept"])
    assert not g["nf_g"][60:].any()


def test_adam_steps_match_reference():
    g = golden("steps.npz")
    fl = golden("filter.npz")
    prob = _small_problem(fl)
    lr = (1e-2, 4e-5, 2e-5)
    st = OO.new_state(fl["true_pos"] + 1e-4, fl["true_p0"] * 1.10, fl["true_a0"], seed=1)
    losses = [OO.step(prob, st, fl["real"], 1, "fine", lr) for _ in range(3)]
    assert np.allclose(losses, g["fine_losses"], rtol=1e-12, atol=0)
    assert np.allclose(st["pos"], g["fine_pos"], rtol=1e-12, atol=1e-18)
    assert np.allclose(st["p0"], g["fine_p0"], rtol=1e-12)
    st = OO.new_state(fl["true_pos"], fl["true_p0"] * 0.5, fl["true_a0"], seed=1)
    real4 = OR.downsample(fl["real"], 4)
    losses = [OO.step(prob, st, real4, 4, "coarse", lr) for _ in range(4)]
    assert np.allclose(losses, g["coarse_losses"], rtol=1e-12, atol=0)
    assert st["pos"].tobytes() == g["coarse_pos"].tobytes()
    assert np.allclose(st["a0"], g["coarse_a0"], rtol=1e-12)


@pytest.mark.parametrize("stage", ["coarse", "fine"])
def test_density_control_matches_reference(stage):
    g = golden("density.npz")
    n = g["p0"].shape[0]
    st = OO.new_state(g["pos"], g["p0"], g["a0"], seed=4, generation=2)
    st["m"]["p0"] = np.arange(n, dtype=np.float64)
    st["v"]["position"] = np.arange(3 * n, dtype=np.float64).reshape(n, 3)
    st["last_gpos"] = g[f"{stage}_grad"]
    th = dict(destroy_p0_frac=0.02, split_a0=1e-3, duplicate_grad_quantile=0.9, a0_min=1e-4, a0_max=5e-3)
    OO.density_control(st, th, stage)
    assert np.array_equal(st["pos"], g[f"{stage}_out_pos"])
    assert np.array_equal(st["p0"], g[f"{stage}_out_p0"])
    assert np.array_equal(st["a0"], g[f"{stage}_out_a0"])
    assert np.array_equal(st["m"]["p0"], g[f"{stage}_m_p0"])
    assert np.array_equal(st["v"]["position"], g[f"{stage}_v_pos"])
    assert st["generation"] == int(g[f"{stage}_generation"])


def _toy_problem(kind=("none",)):
    from paper_2601_00551_b200 import scenes
    sc = scenes.toy_config()
    prob = OO.Problem(sc.array.positions, sc.array.normals, 1500.0, sc.grid.t0, sc.grid.dt,
                      sc.grid.n_samples, kind=kind, threads=4)
    return sc, prob


def test_toy_forward_and_steps_match_reference():
    g = golden("toy.npz")
    sc, prob = _toy_problem()
    real = prob.simulate(sc.truth.positions, sc.truth.p0, sc.truth.a0)
    assert rel_l2(real, g["real"]) < 1e-14
    # the 5 Adam steps start from the reference's filtered cloud
    keep = g["filter_g"] < 0
    st = OO.new_state(sc.init.positions[keep], sc.init.p0[keep], sc.init.a0[keep], seed=103)
    lr = tuple(g["lr"])
    losses = [OO.step(prob, st, g["real"], 1, "fine", lr) for _ in range(5)]
    assert np.allclose(losses, g["step_losses"], rtol=1e-10)
    assert rel_l2(st["pos"], g["final_pos"]) < 1e-12
    assert rel_l2(st["p0"], g["final_p0"]) < 1e-9


@pytest.mark.slow
def test_toy_filter_matches_reference():
    g = golden("toy.npz")
    sc, prob = _toy_problem()
    keep, gg = OO.zero_gradient_filter(prob, sc.init.positions, sc.init.p0, sc.init.a0, g["real"], 1)
    assert np.array_equal(keep, g["filter_g"] < 0)
    assert rel_l2(gg, g["filter_g"]) < 1e-12
    assert int(keep.sum()) == int(g["n_kept"])


def test_schedule_and_volume_match_reference():
    g = golden("schedule.npz")
    prob = OO.Problem(g["sensors"], None, 1500.0, 0.0, 5e-8, 512)
    init = g["init_pos"]
    n = init.shape[0]
    keep, gg = OO.zero_gradient_filter(prob, init, np.full(n, 0.05), np.full(n, 5e-4), g["real"], 8)
    assert rel_l2(gg, g["filter_g"]) < 1e-12
    st = OO.new_state(init[keep], np.full(int(keep.sum()), 0.05), np.full(int(keep.sum()), 5e-4), seed=61)
    sp = 4e-4
    th = dict(destroy_p0_frac=0.02, split_a0=2 * sp, duplicate_grad_quantile=0.9, a0_min=0.25 * sp,
              a0_max=8 * sp)
    st, losses, counts = OO.run_hierarchical(prob, st, g["real"], [(8, 150, "coarse"), (2, 60, "fine"),
                                                                   (1, 60, "fine")], th,
                                             (1e-2, 0.1 * sp, 0.05 * sp), duplication_period=50,
                                             plateau=False)
    assert np.array_equal(counts, g["counts"])
    assert np.allclose(losses, g["losses"], rtol=1e-8)
    vol = ORend.voxelize(st["pos"], st["p0"], st["a0"], (31, 31, 31), 2e-4, (-3e-3, -3e-3, -3e-3))
    assert rel_l2(vol, g["volume"]) < 1e-8
    vt = ORend.voxelize(g["true_pos"], g["true_p0"], g["true_a0"], (31, 31, 31), 2e-4, (-3e-3,) * 3)
    assert rel_l2(vt, g["volume_truth"]) < 1e-14


@pytest.mark.parametrize("iters", [3, 40])
def test_positivity_refine_matches_reference(iters):
    """Oracle restatement of positivity_refine (optimizer.py:536-573) against
    the reference run (tests/golden/make_golden_refine.py)."""
    g = golden("refine.npz")
    prob = OO.Problem(g["sensors"], None, 1500.0, 0.0, 5e-8, 512)
    st = OO.new_state(g["true_pos"], g["in_p0"], g["in_a0"], seed=9)
    lr = (1e-2, 0.1 * 4e-4, 0.05 * 4e-4)   # LearningRates.from_spacing(4e-4)
    pos, p0, a0, free = OO.positivity_refine(prob, st, g["real"], iters, lr)
    assert np.allclose(pos, g[f"it{iters}_pos"], rtol=1e-10, atol=1e-16)
    assert np.allclose(p0, g[f"it{iters}_p0"], rtol=1e-10)
    assert np.allclose(a0, g[f"it{iters}_a0"], rtol=1e-10)
    assert np.allclose(free, g[f"it{iters}_a0_free"], rtol=1e-9)
    assert np.all(a0 > 0.0)


def test_softplus_pair_round_trip():
    y = np.array([1e-9, 1e-4, 0.3, 0.69999, 0.7, 2.0, 40.0])
    np.testing.assert_allclose(OO.softplus(OO.inv_softplus(y)), y, rtol=1e-12)
    with pytest.raises(ValueError):
        OO.inv_softplus(np.array([0.0]))
