"""GPU universal back-projection (baseline.ubp_reconstruct, reference
baseline.py:52-89) against the reference's own volumes (tests/golden/ubp.npz,
bit for bit) and the FP64 oracle, plus the reference's UBP tests
(pkg/tests/test_baseline.py TestUbp) re-run on the CUDA path."""

import math
import os

import numpy as np
import pytest

from oracle import baseline as OB

pytestmark = pytest.mark.gpu

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "ubp.npz"))
POINT_SPEC = dict(dims=(17, 17, 17), spacing=1e-3, origin=(-8e-3, -8e-3, -8e-3))


@pytest.fixture(scope="module")
def P():
    import paper_2601_00551_b200 as P
    return P


def sphere(P, count, radius=0.02):
    """Full Fibonacci sphere of sensors (any dense closed array focuses)."""
    k = np.arange(count) + 0.5
    z = 1.0 - 2.0 * k / count
    r = np.sqrt(1.0 - z * z)
    phi = math.pi * (1.0 + 5 ** 0.5) * k
    unit = np.column_stack([r * np.cos(phi), r * np.sin(phi), z])
    return P.SensorArray(radius * unit, 1500.0, normals=unit)


# The reference's focusing tests (test_baseline.py:66-96) place the ball at
# (1.5, -1.0, 0.5) mm, half a voxel off every 1 mm grid line; run here against
# the reference itself both fail (its peak lands on a back-projection arc), and
# this implementation reproduces the reference's volume bit for bit.  The
# focusing property is therefore checked with the ball on a voxel centre.
ON_GRID = [2.0e-3, -1.0e-3, 1.0e-3]


def point_case(P, sensors=None, source=(1.5e-3, -1.0e-3, 0.5e-3)):
    array = P.SensorArray(GOLD["point_sensors"], 1500.0) if sensors is None else sensors
    tg = P.TimeGrid(0.0, 5e-8, 1024)
    if sensors is None:
        real = P.SignalSet(tg, GOLD["point_rows"].copy())
    else:
        ctx = P.ForwardContext(array, tg)
        real = P.simulate_signals(P.PointCloud([list(source)], [1.0], [2e-4]), ctx)
    return real, array, P.RenderSpec(**POINT_SPEC)


class TestGolden:
    def test_point_source_bit_exact(self, P):
        real, array, spec = point_case(P)
        grid, cov = P.ubp_reconstruct(real, array, spec)
        np.testing.assert_array_equal(grid.values, GOLD["point_vol"])
        assert cov.n_skipped == 0 and cov.n_total == 17 ** 3 * 64

    def test_short_record_bit_exact_and_counted(self, P):
        real, array, spec = point_case(P)
        short = P.SignalSet(P.TimeGrid(0.0, 5e-8, 128), real.data[:, :128].copy())
        grid, cov = P.ubp_reconstruct(short, array, spec)
        np.testing.assert_array_equal(grid.values, GOLD["short_vol"])
        assert cov.n_skipped == int(GOLD["short_skipped"])
        assert 0.0 < cov.fraction_skipped <= 1.0

    def test_noise_ragged_grid_bit_exact(self, P):
        array = P.SensorArray(GOLD["noise_sensors"], 1480.0)
        real = P.SignalSet(P.TimeGrid(1.2e-5, 4e-8, 300), GOLD["noise_rows"].copy())
        spec = P.RenderSpec(dims=(9, 11, 7), spacing=7e-4, origin=(-3e-3, -4e-3, -2e-3))
        grid, cov = P.ubp_reconstruct(real, array, spec)
        np.testing.assert_array_equal(grid.values, GOLD["noise_vol"])
        assert cov.n_skipped == int(GOLD["noise_skipped"])


class TestReferenceCases:
    def test_zero_signals_zero_volume(self, P):
        real, array, spec = point_case(P)
        grid, cov = P.ubp_reconstruct(P.SignalSet(real.grid, np.zeros_like(real.data)), array, spec)
        assert not grid.values.any()
        assert cov.n_skipped == 0

    def test_dense_array_matches_oracle(self, P):
        """The reference's off-grid 512-sensor case: GPU-simulated rows, GPU
        back-projection bit-exact against the oracle on the same rows."""
        real, array, spec = point_case(P, sphere(P, 512))
        grid, _ = P.ubp_reconstruct(real, array, spec)
        want, _ = OB.ubp(real.data, 0.0, 5e-8, array.positions, 1500.0, spec.dims, spec.spacing, spec.origin)
        np.testing.assert_array_equal(grid.values, want)

    def test_dense_array_focuses_on_source(self, P):
        real, array, spec = point_case(P, sphere(P, 512), ON_GRID)
        grid, _ = P.ubp_reconstruct(real, array, spec)
        am = np.unravel_index(np.argmax(grid.values), grid.dims)
        centre = np.array([grid.origin[a] + am[a] * grid.spacing for a in range(3)])
        assert np.all(np.abs(centre - np.array(ON_GRID)) <= grid.spacing + 1e-12)

    def test_sparse_array_has_more_artifacts(self, P):
        real_d, arr_d, spec = point_case(P, sphere(P, 512), ON_GRID)
        real_s, arr_s, _ = point_case(P, sphere(P, 64), ON_GRID)
        dense, _ = P.ubp_reconstruct(real_d, arr_d, spec)
        sparse, _ = P.ubp_reconstruct(real_s, arr_s, spec)
        am = np.unravel_index(np.argmax(sparse.values), sparse.dims)
        centre = np.array([sparse.origin[a] + am[a] * sparse.spacing for a in range(3)])
        assert np.all(np.abs(centre - np.array(ON_GRID)) <= sparse.spacing + 1e-12)

        def bg_rms(grid):
            norm = P.max_normalized(grid).values
            mask = np.ones(grid.dims, dtype=bool)
            mask[tuple(slice(max(a - 2, 0), a + 3) for a in am)] = False
            return float(np.sqrt(np.mean(norm[mask] ** 2)))

        assert bg_rms(sparse) > bg_rms(dense)

    def test_linearity_power_of_two_exact(self, P):
        real, array, spec = point_case(P)
        g1, _ = P.ubp_reconstruct(real, array, spec)
        g2, _ = P.ubp_reconstruct(P.SignalSet(real.grid, 2.0 * real.data), array, spec)
        np.testing.assert_array_equal(g2.values, 2.0 * g1.values)

    def test_errors(self, P):
        real, array, spec = point_case(P)
        with pytest.raises(ValueError):
            P.ubp_reconstruct(P.SignalSet(P.TimeGrid(0.0, 5e-8, 1), real.data[:, :1].copy()), array, spec)
        with pytest.raises(ZeroDivisionError):
            P.ubp_reconstruct(P.SignalSet(real.grid, real.data[:0].copy()), P.SensorArray(np.zeros((0, 3)), 1500.0),
                              spec)


class TestLargerScale:
    def test_many_sensors_long_record_matches_oracle(self, P):
        """256 sensors x 4096 samples onto a 24 x 20 x 28 grid, random rows,
        late t0 (both ends of the record clip): bit-exact against the oracle."""
        rng = np.random.default_rng(11)
        sensors = rng.uniform(-0.04, 0.04, (256, 3))
        rows = rng.standard_normal((256, 4096))
        array = P.SensorArray(sensors, 1510.0)
        tg = P.TimeGrid(8e-6, 1 / 40e6, 4096)
        spec = P.RenderSpec(dims=(24, 20, 28), spacing=6e-4, origin=(-7e-3, -6e-3, -8e-3))
        grid, cov = P.ubp_reconstruct(P.SignalSet(tg, rows), array, spec)
        want, skipped = OB.ubp(rows, tg.t0, tg.dt, sensors, 1510.0, spec.dims, spec.spacing, spec.origin)
        np.testing.assert_array_equal(grid.values, want)
        assert cov.n_skipped == skipped > 0
