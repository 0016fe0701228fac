"""Driver on the CUDA path: zero-gradient filter, Adam steps, density control,
hierarchical schedule (reference pkg/tests/test_optimizer.py re-run, plus
parity against the golden vectors of the key-fixed reference)."""

import math

import numpy as np
import pytest

from oracle import optimizer as OO
from oracle import radiator as OR
from oracle import render as ORend
from pab_helpers import golden, rel_l2

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_2601_00551_b200 as P
    return P


def small_instance(P, seed=5):
    """reference test_optimizer.py:44-54 (golden sensors/truth for seed 5)."""
    g = golden("filter.npz")
    ctx = P.ForwardContext(P.SensorArray(g["sensors"]), P.TimeGrid(0.0, 5e-8, 512))
    truth = P.PointCloud(g["true_pos"], g["true_p0"], g["true_a0"])
    return ctx, truth, P.SignalSet(ctx.grid, g["real"]), g


class TestZeroGradientFilter:
    def test_zero_data_retains_nothing(self, P):
        ctx, _, real, _ = small_instance(P)
        zero = P.SignalSet(real.grid, np.zeros_like(real.data))
        rng = P.CounterRng(1)
        cand = P.PointCloud(rng.uniform(-3e-3, 3e-3, 150).reshape(50, 3), np.full(50, 0.1), np.full(50, 5e-4))
        kept, report = P.zero_gradient_filter(cand, ctx, zero, f=4)
        assert len(kept) == 0 and report.no_evidence and not report.g.any()

    def test_true_position_kept_far_removed(self, P):
        ctx, truth, real, _ = small_instance(P)
        cand = P.PointCloud([truth.positions[0], [3.5e-3, 3.5e-3, 3.5e-3]], [0.1, 0.1], [5e-4, 5e-4])
        kept, report = P.zero_gradient_filter(cand, ctx, real, f=4)
        assert report.g[0] < 0.0 and len(kept) == 1
        np.testing.assert_array_equal(kept.positions[0], truth.positions[0])

    def test_retained_pressures_are_originals(self, P):
        ctx, _, real, _ = small_instance(P)
        rng = P.CounterRng(2)
        p0 = rng.uniform(0.01, 0.2, 80)
        cand = P.PointCloud(rng.uniform(-3e-3, 3e-3, 240).reshape(80, 3), p0, np.full(80, 5e-4))
        kept, report = P.zero_gradient_filter(cand, ctx, real, f=4)
        np.testing.assert_array_equal(kept.p0, p0[report.g < 0])
        np.testing.assert_array_equal(cand.p0, p0)

    def test_decisions_match_reference_and_inner_product(self, P):
        ctx, _, real, g = small_instance(P)
        n = g["ip_pos"].shape[0]
        cand = P.PointCloud(g["ip_pos"], np.full(n, 0.1), np.full(n, 5e-4))
        kept, report = P.zero_gradient_filter(cand, ctx, real, f=4)
        np.testing.assert_array_equal(report.g < 0, g["ip_g"] < 0)
        assert len(kept) == int(g["ip_kept"])
        assert rel_l2(report.g, g["ip_g"]) < 1e-3
        # g_i = -(2/N) <y_real, K_i> (reference test_optimizer.py:94-110)
        real_k = P.downsample(real, 4)
        for i in range(0, n, 15):
            one = P.PointCloud(cand.positions[i:i + 1], [1.0], [5e-4])
            ip = float(np.sum(real_k.data * P.simulate_at_rate(one, ctx, 4).data))
            assert (report.g[i] < 0) == (ip > 0)

    def test_support_less_balls_have_exactly_zero_gradient(self, P):
        ctx, _, real, g = small_instance(P)
        cand = P.PointCloud(g["nf_pos"], np.full(70, 0.1), np.full(70, 4e-4))
        kept, report = P.zero_gradient_filter(cand, ctx, real, f=2)
        assert report.n_retained <= report.n_input and len(kept) == report.n_retained
        assert not report.g[60:].any()
        np.testing.assert_array_equal(report.g < 0, g["nf_g"] < 0)

    def test_lax_predicate_keeps_zero_gradient(self, P):
        ctx, _, real, _ = small_instance(P)
        zero = P.SignalSet(real.grid, np.zeros_like(real.data))
        cand = P.PointCloud([[0, 0, 0]], [0.1], [5e-4])
        strict, _ = P.zero_gradient_filter(cand, ctx, zero, f=1, strict=True)
        lax, _ = P.zero_gradient_filter(cand, ctx, zero, f=1, strict=False)
        assert len(strict) == 0 and len(lax) == 1

    def test_empty_cloud_rejected(self, P):
        ctx, _, real, _ = small_instance(P)
        with pytest.raises(ValueError):
            P.zero_gradient_filter(P.PointCloud.empty(), ctx, real, f=1)


class TestStep:
    def test_perfect_fit_leaves_state_unchanged(self, P):
        ctx, truth, _, _ = small_instance(P)
        real = P.simulate_signals(truth, ctx)
        state = P.create_state(truth.copy(), seed=1)
        state, L = P.step(state, ctx, real, 1, "fine")
        assert L == 0.0
        np.testing.assert_array_equal(state.cloud.positions, truth.positions)
        np.testing.assert_array_equal(state.cloud.p0, truth.p0)
        np.testing.assert_array_equal(state.cloud.a0, truth.a0)

    def test_overshooting_pressure_decreases(self, P):
        ctx, truth, real, _ = small_instance(P)
        cloud = truth.copy()
        cloud.p0 = truth.p0 * 1.10
        state = P.create_state(cloud, seed=1)
        state, L = P.step(state, ctx, real, 1, "fine")
        assert L > 0 and np.all(state.cloud.p0 < cloud.p0)

    def test_coarse_positions_bit_identical_many_steps(self, P):
        ctx, truth, real, _ = small_instance(P)
        cloud = truth.copy()
        cloud.p0 = cloud.p0 * 0.5
        state = P.create_state(cloud, seed=1)
        real_k = P.downsample(real, 4)
        for _ in range(20):
            state, _ = P.step(state, ctx, real_k, 4, "coarse")
        assert state.cloud.positions.tobytes() == truth.positions.tobytes()

    def test_wrong_decimation_rejected(self, P):
        ctx, truth, real, _ = small_instance(P)
        state = P.create_state(truth.copy(), seed=1)
        with pytest.raises(ValueError):
            P.step(state, ctx, P.downsample(real, 2), 4, "coarse")

    def test_steps_match_reference(self, P):
        ctx, truth, real, _ = small_instance(P)
        st = golden("steps.npz")
        cloud = truth.copy()
        cloud.p0 = truth.p0 * 1.10
        cloud.positions = truth.positions + 1e-4
        state = P.create_state(cloud, seed=1)
        losses = []
        for _ in range(3):
            state, L = P.step(state, ctx, real, 1, "fine")
            losses.append(L)
        assert np.allclose(losses, st["fine_losses"], rtol=1e-4)
        assert rel_l2(state.cloud.positions - truth.positions, st["fine_pos"] - truth.positions) < 1e-3
        assert rel_l2(state.cloud.p0, st["fine_p0"]) < 1e-6


class TestDensityControl:
    TH = dict(destroy_p0_frac=0.02, split_a0=1e-3, duplicate_grad_quantile=0.90, a0_min=1e-4, a0_max=5e-3)

    @pytest.mark.parametrize("stage", ["coarse", "fine"])
    def test_matches_reference_bitwise(self, P, stage):
        g = golden("density.npz")
        n = g["p0"].shape[0]
        cloud = P.PointCloud(g["pos"], g["p0"], g["a0"])
        cloud.generation = 2
        state = P.create_state(cloud, seed=4)
        state.m["p0"] = np.arange(n, dtype=np.float64)
        state.v["position"] = np.arange(3 * n, dtype=np.float64).reshape(n, 3)
        state.last_grad = P.ParamGradients(np.zeros(n), np.zeros(n), g[f"{stage}_grad"])
        out = P.density_control(state, P.DensityThresholds(**self.TH), stage)
        np.testing.assert_array_equal(out.cloud.positions, g[f"{stage}_out_pos"])
        np.testing.assert_array_equal(out.cloud.p0, g[f"{stage}_out_p0"])
        np.testing.assert_array_equal(out.cloud.a0, g[f"{stage}_out_a0"])
        np.testing.assert_array_equal(out.m["p0"], g[f"{stage}_m_p0"])
        np.testing.assert_array_equal(out.v["position"], g[f"{stage}_v_pos"])
        assert out.cloud.generation == int(g[f"{stage}_generation"])

    def test_split_arithmetic(self, P):
        th = P.DensityThresholds(**self.TH)
        a0_big = 3.0 * th.split_a0
        state = P.create_state(P.PointCloud([[0, 0, 0], [5e-3, 0, 0]], [1.0, 1.0], [a0_big, 5e-4]), seed=2)
        out = P.density_control(state, th, "coarse")
        assert len(out.cloud) == 3
        children = np.isclose(out.cloud.a0, a0_big / math.sqrt(2.0))
        assert children.sum() == 2
        np.testing.assert_allclose(out.cloud.p0[children], 0.5)
        cp = out.cloud.positions[children]
        np.testing.assert_allclose(cp.mean(axis=0), [0, 0, 0], atol=1e-15)
        np.testing.assert_allclose(np.linalg.norm(cp[0] - cp[1]), a0_big, rtol=1e-12)

    def test_moments_carried_for_survivors_reset_for_children(self, P):
        th = P.DensityThresholds(**self.TH)
        state = P.create_state(P.PointCloud([[0, 0, 0], [5e-3, 0, 0]], [1.0, 1.0], [3e-3, 5e-4]), seed=2)
        state.m["p0"] = np.array([7.0, 9.0])
        state.v["p0"] = np.array([1.0, 2.0])
        out = P.density_control(state, th, "coarse")
        np.testing.assert_array_equal(out.m["p0"], [9.0, 0.0, 0.0])
        np.testing.assert_array_equal(out.v["p0"], [2.0, 0.0, 0.0])


class TestRunHierarchical:
    def test_zero_iteration_schedule_returns_input(self, P):
        ctx, truth, real, _ = small_instance(P)
        out, trace = P.run_hierarchical(truth.copy(), ctx, real, P.Schedule((P.Level(1, 0, "fine"),)),
                                        P.DensityThresholds())
        np.testing.assert_array_equal(out.positions, truth.positions)
        assert trace.records == []

    def test_all_points_destroyed_raises(self, P):
        ctx, _, real, _ = small_instance(P)
        zero = P.SignalSet(real.grid, np.zeros_like(real.data))
        cloud = P.PointCloud([[0, 0, 0], [1e-3, 0, 0]], [0.05, 0.05], [5e-4, 5e-4])
        with pytest.raises(P.OptimizationError, match="destroyed"):
            P.run_hierarchical(cloud, ctx, zero, P.Schedule((P.Level(1, 300, "fine"),), duplication_period=50),
                               P.DensityThresholds.from_spacing(4e-4), lr=P.LearningRates.from_spacing(4e-4))

    def test_short_schedule_volume_parity(self, P):
        """Filter + 270 iterations (8x coarse, 2x/1x fine, density control)
        against the key-fixed reference: same filter set, volume rel L2."""
        g = golden("schedule.npz")
        ctx = P.ForwardContext(P.SensorArray(g["sensors"]), P.TimeGrid(0.0, 5e-8, 512))
        real = P.SignalSet(ctx.grid, g["real"])
        n = g["init_pos"].shape[0]
        init = P.PointCloud(g["init_pos"], np.full(n, 0.05), np.full(n, 5e-4))
        filt, rep = P.zero_gradient_filter(init, ctx, real, f=8)
        np.testing.assert_array_equal(rep.g < 0, g["filter_g"] < 0)
        sched = P.Schedule((P.Level(8, 150, "coarse"), P.Level(2, 60, "fine"), P.Level(1, 60, "fine")),
                           duplication_period=50)
        final, trace = P.run_hierarchical(filt.copy(), ctx, real, sched, P.DensityThresholds.from_spacing(4e-4),
                                          lr=P.LearningRates.from_spacing(4e-4), seed=P.RngSeed(61), plateau=False)
        counts = np.array([r.ball_count for r in trace.records])
        losses = np.array([r.loss for r in trace.records])
        assert np.array_equal(counts, g["counts"])
        # measured on B200: losses within 1.1e-5, volume rel L2 8.8e-7 (north star: 1e-3)
        assert np.allclose(losses, g["losses"], rtol=1e-4)
        vol = ORend.voxelize(final.positions, final.p0, final.a0, (31, 31, 31), 2e-4, (-3e-3,) * 3)
        assert rel_l2(vol, g["volume"]) < 1e-5


def test_toy_five_adam_steps_match_reference(P):
    """BASELINE config 1: reference-filtered 32^3 grid, 5 fine Adam steps."""
    from paper_2601_00551_b200 import scenes
    g = golden("toy.npz")
    sc = scenes.toy_config()
    ctx = P.ForwardContext(sc.array, sc.grid)
    real = P.SignalSet(sc.grid, g["real"])
    keep = g["filter_g"] < 0
    lr = P.LearningRates(*g["lr"])
    state = P.create_state(sc.init.subset(keep), lr=lr, seed=103)
    losses = []
    for _ in range(5):
        state, L = P.step(state, ctx, real, 1, "fine")
        losses.append(L)
    # measured on B200: losses 1.0e-7, displacements 2.7e-6, p0 1.6e-7, a0 1.9e-6 (rel)
    assert np.allclose(losses, g["step_losses"], rtol=1e-6)
    c = state.cloud
    init = sc.init.subset(keep)
    assert rel_l2(c.positions - init.positions, g["final_pos"] - init.positions) < 3e-5
    assert rel_l2(c.p0, g["final_p0"]) < 2e-6
    assert rel_l2(c.a0, g["final_a0"]) < 2e-5


class TestPositivityRefine:
    """positivity_refine (optimizer.py:536-573) on the device against the
    reference run (tests/golden/refine.npz) and the reference's own tests
    (test_optimizer.py:379-400)."""

    def _start(self, P, g):
        ctx, truth, real, _ = small_instance(P)
        np.testing.assert_array_equal(truth.positions, g["true_pos"])
        cloud = truth.copy()
        cloud.p0 = cloud.p0 * 0.8
        cloud.a0 = cloud.a0 * 1.3
        return ctx, cloud, real

    @pytest.mark.parametrize("iters", [3, 40])
    def test_matches_reference(self, P, iters):
        g = golden("refine.npz")
        ctx, cloud, real = self._start(P, g)
        np.testing.assert_allclose(real.data, g["real"], rtol=0, atol=1e-4 * np.abs(g["real"]).max())
        state = P.create_state(cloud, lr=P.LearningRates.from_spacing(4e-4), seed=9)
        out = P.positivity_refine(state, ctx, P.SignalSet(ctx.grid, g["real"]), iters)
        # FP32 per-sample gradients (rel. 1e-5) through Adam's normalised steps
        np.testing.assert_allclose(out.p0, g[f"it{iters}_p0"], rtol=2e-4)
        np.testing.assert_allclose(out.a0, g[f"it{iters}_a0"], rtol=2e-4)
        np.testing.assert_allclose(out.positions, g[f"it{iters}_pos"], rtol=0, atol=0.02 * iters * 0.05 * 4e-4)
        np.testing.assert_allclose(out.a0_free, g[f"it{iters}_a0_free"], rtol=2e-3, atol=1e-6)
        assert np.all(out.a0 > 0.0) and np.isfinite(out.a0_free).all()
        L1 = P.loss(P.simulate_signals(out, ctx), P.SignalSet(ctx.grid, g["real"]))
        assert abs(L1 - float(g[f"it{iters}_L1"])) <= 1e-3 * float(g[f"it{iters}_L1"])

    def test_refinement_outputs_positive_sizes(self, P):
        ctx, truth, real, _ = small_instance(P)
        cloud = truth.copy()
        cloud.p0 = cloud.p0 * 0.8
        cloud.a0 = cloud.a0 * 1.3
        state = P.create_state(cloud, lr=P.LearningRates.from_spacing(4e-4), seed=9)
        L0 = P.loss(P.simulate_signals(cloud, ctx), real)
        out = P.positivity_refine(state, ctx, real, 40)
        assert np.all(out.a0 > 0.0)
        assert np.isfinite(out.a0_free).all()
        assert P.loss(P.simulate_signals(out, ctx), real) < L0

    def test_nonpositive_entry_rejected(self, P):
        ctx, truth, real, _ = small_instance(P)
        bad = truth.copy()
        bad.a0 = bad.a0.copy()
        bad.a0[0] = -1e-4
        state = P.create_state(bad, seed=9)
        with pytest.raises(ValueError):
            P.positivity_refine(state, ctx, real, 1)

    def test_softplus_helpers(self, P):
        x = np.array([-50.0, -3.0, -1e-3, 0.0, 1e-3, 3.0, 50.0])
        np.testing.assert_allclose(P.inv_softplus(P.softplus(x[2:-1])), x[2:-1], rtol=1e-9, atol=1e-12)
        np.testing.assert_allclose(P.sigmoid(x), 1.0 / (1.0 + np.exp(-x)), rtol=1e-15)
