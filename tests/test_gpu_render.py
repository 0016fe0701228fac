"""GPU voxelisation (render.voxelize, reference render.py:55-93) against the
oracle restatement, plus the reference's own render tests
(reference pkg/tests/test_render.py) re-run on the CUDA path."""

import numpy as np
import pytest

from oracle import render as ORR

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_2601_00551_b200 as P
    return P


def centered_spec(P, dims=(17, 17, 17), spacing=5e-4):
    half = (np.array(dims) - 1) / 2 * spacing
    return P.RenderSpec(dims=dims, spacing=spacing, origin=tuple(-half))


def oracle_volume(cloud, spec):
    return ORR.voxelize(cloud.positions, cloud.p0, cloud.a0, spec.dims, spec.spacing, spec.origin,
                        spec.support_sigma)


class TestReferenceCases:
    def test_empty_cloud(self, P):
        assert not P.voxelize(P.PointCloud.empty(), centered_spec(P)).values.any()

    def test_peak_and_one_sigma_values(self, P):
        spec = centered_spec(P, spacing=5e-4)
        grid = P.voxelize(P.PointCloud([[0.0, 0.0, 0.0]], [1.0], [5e-4]), spec)
        c = 8
        assert grid.values[c, c, c] == 1.0
        np.testing.assert_allclose(grid.values[c + 1, c, c], np.exp(-0.5), rtol=1e-12)

    def test_colocated_balls_superpose(self, P):
        spec = centered_spec(P)
        one = P.voxelize(P.PointCloud([[0, 0, 0]], [0.7], [5e-4]), spec)
        two = P.voxelize(P.PointCloud([[0, 0, 0], [0, 0, 0]], [0.7, 0.7], [5e-4, 5e-4]), spec)
        np.testing.assert_array_equal(two.values, 2.0 * one.values)

    def test_negative_pressure_clamped(self, P):
        assert not P.voxelize(P.PointCloud([[0, 0, 0]], [-3.0], [5e-4]), centered_spec(P)).values.any()

    def test_mass_consistency(self, P):
        a0, p0 = 6e-4, 1.3
        spec = centered_spec(P, dims=(33, 33, 33), spacing=a0 / 2)
        grid = P.voxelize(P.PointCloud([[0, 0, 0]], [p0], [a0]), spec)
        total = spec.spacing ** 3 * grid.values.sum()
        expect = p0 * (2 * np.pi) ** 1.5 * a0 ** 3
        assert abs(total - expect) <= 0.01 * expect

    def test_translation_equivariance_exact(self, P):
        spacing = 2.0 ** -11
        spec = P.RenderSpec(dims=(24, 24, 24), spacing=spacing, origin=(-12 * spacing,) * 3)
        rng = P.CounterRng(13)
        n = 4
        pos = (np.floor(rng.uniform(-4, 4, 3 * n)).reshape(n, 3)) * spacing
        cloud = P.PointCloud(pos, rng.uniform(0.5, 1.5, n), np.full(n, 2 * spacing))
        g0 = P.voxelize(cloud, spec)
        shifted = cloud.copy()
        shifted.positions = shifted.positions + np.array([spacing, 0.0, 0.0])
        g1 = P.voxelize(shifted, spec)
        np.testing.assert_array_equal(g1.values[1:], g0.values[:-1])

    def test_order_independence_exact(self, P):
        rng = P.CounterRng(14)
        n = 30
        pos = rng.uniform(-3e-3, 3e-3, 3 * n).reshape(n, 3)
        cloud = P.PointCloud(pos, rng.uniform(0.1, 2.0, n), rng.uniform(3e-4, 9e-4, n))
        perm = np.argsort(rng.uniform(0, 1, n))
        spec = centered_spec(P, dims=(21, 21, 21))
        np.testing.assert_array_equal(P.voxelize(cloud, spec).values,
                                      P.voxelize(cloud.subset(perm), spec).values)

    def test_invalid_a0(self, P):
        with pytest.raises(ValueError):
            P.voxelize(P.PointCloud([[0, 0, 0]], [1.0], [0.0]), centered_spec(P))


class TestOracleParity:
    @pytest.mark.parametrize("seed,n,dims", [(21, 300, (21, 19, 23)), (22, 2500, (40, 36, 44))])
    def test_random_cloud(self, P, seed, n, dims):
        rng = np.random.default_rng(seed)
        pos = rng.uniform(-6e-3, 6e-3, (n, 3))
        p0 = rng.uniform(-0.3, 1.5, n)              # some clamped balls
        a0 = rng.uniform(1e-4, 8e-4, n)
        # coincident keys exercise the canonical tie-breaks
        pos[: n // 10] = pos[n // 10: 2 * (n // 10)]
        cloud = P.PointCloud(pos, p0, a0)
        spec = P.RenderSpec(dims=dims, spacing=3e-4, origin=(-6e-3, -5.5e-3, -6.5e-3), support_sigma=3.0)
        got = P.voxelize(cloud, spec).values
        want = oracle_volume(cloud, spec)
        scale = np.abs(want).max()
        assert np.abs(got - want).max() <= 1e-13 * scale
        assert np.array_equal(got == 0.0, want == 0.0)

    def test_support_and_partial_boxes(self, P):
        # balls straddling every face of the grid and a wide support
        rng = np.random.default_rng(23)
        n = 400
        pos = rng.uniform(-1.2e-3, 4.2e-3, (n, 3))
        cloud = P.PointCloud(pos, rng.uniform(0.1, 1.0, n), rng.uniform(2e-4, 6e-4, n))
        spec = P.RenderSpec(dims=(12, 13, 9), spacing=2.5e-4, origin=(0.0, 0.0, 0.0), support_sigma=4.5)
        got = P.voxelize(cloud, spec).values
        want = oracle_volume(cloud, spec)
        assert np.abs(got - want).max() <= 1e-13 * np.abs(want).max()
