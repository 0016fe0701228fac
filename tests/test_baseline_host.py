"""UBP baseline oracle pinned to the reference's own outputs, and the host
volume metrics (reference pkg/src/paball/baseline.py:92-186, tests in
pkg/tests/test_baseline.py)."""

import itertools
import math
import os

import numpy as np
import pytest

from oracle import baseline as OB
from paper_2601_00551_b200 import baseline as B
from paper_2601_00551_b200.model import VoxelGrid

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "ubp.npz"))


def vg(values):
    values = np.asarray(values, dtype=float)
    return VoxelGrid(values.shape, 1.0, np.zeros(3), values)


class TestOracleMatchesReference:
    """The FP64 restatement reproduces the reference's volumes bit for bit."""

    def test_point_source(self):
        v, s = OB.ubp(GOLD["point_rows"], 0.0, 5e-8, GOLD["point_sensors"], 1500.0, (17, 17, 17), 1e-3,
                      (-8e-3,) * 3)
        np.testing.assert_array_equal(v, GOLD["point_vol"])
        assert s == int(GOLD["point_skipped"]) == 0

    def test_short_record_counts_skips(self):
        v, s = OB.ubp(GOLD["point_rows"][:, :128], 0.0, 5e-8, GOLD["point_sensors"], 1500.0, (17, 17, 17), 1e-3,
                      (-8e-3,) * 3)
        np.testing.assert_array_equal(v, GOLD["short_vol"])
        assert s == int(GOLD["short_skipped"]) > 0

    def test_noise_rows_ragged_grid_late_start(self):
        v, s = OB.ubp(GOLD["noise_rows"], 1.2e-5, 4e-8, GOLD["noise_sensors"], 1480.0, (9, 11, 7), 7e-4,
                      (-3e-3, -4e-3, -2e-3))
        np.testing.assert_array_equal(v, GOLD["noise_vol"])
        assert s == int(GOLD["noise_skipped"])

    def test_derivative_is_numpy_gradient(self):
        rows = GOLD["noise_rows"]
        np.testing.assert_array_equal(OB.time_derivative(rows, 4e-8), np.gradient(rows, 4e-8, axis=1))


class TestPsnrMse:
    def test_identical(self):
        g = vg(np.random.default_rng(1).random((4, 4, 4)))
        assert B.mse(g, g) == 0.0
        assert B.psnr(g, g) == math.inf

    def test_psnr_is_ten_log_inverse_mse(self):
        for m in (1.2e-3, 6.38e-3, 0.5, 1.0, 2.0):
            assert abs(B.psnr_from_mse(m) - 10.0 * math.log10(1.0 / m)) < 1e-12

    def test_known_values(self):
        a = vg(np.zeros((2, 2, 2)))
        b = vg(np.full((2, 2, 2), 0.1))
        assert abs(B.mse(a, b) - 0.01) < 1e-15
        assert abs(B.psnr(a, b) - 20.0) < 1e-12

    def test_dims_must_match(self):
        with pytest.raises(ValueError):
            B.mse(vg(np.zeros((4, 4, 4))), vg(np.zeros((4, 4, 5))))


def brute_ssim(a, b, w=7, c1=1e-4, c2=9e-4):
    vals = []
    for i, j, k in itertools.product(*(range(d - w + 1) for d in a.shape)):
        x = a[i:i + w, j:j + w, k:k + w]
        y = b[i:i + w, j:j + w, k:k + w]
        mx, my = x.mean(), y.mean()
        sx, sy, sxy = (x * x).mean() - mx * mx, (y * y).mean() - my * my, (x * y).mean() - mx * my
        vals.append((2 * mx * my + c1) * (2 * sxy + c2) / ((mx * mx + my * my + c1) * (sx + sy + c2)))
    return float(np.mean(vals))


class TestSsim:
    def test_identical_exactly_one(self):
        g = vg(np.random.default_rng(2).random((12, 12, 12)))
        assert B.ssim(g, g) == 1.0

    def test_against_zero_below_one(self):
        assert B.ssim(vg(np.random.default_rng(3).random((10, 10, 10))), vg(np.zeros((10, 10, 10)))) < 1.0

    @pytest.mark.parametrize("dims", [(12, 12, 12), (7, 9, 8)])
    def test_matches_brute_force_windows(self, dims):
        rng = np.random.default_rng(4)
        a, b = rng.random(dims), rng.random(dims)
        assert abs(B.ssim(vg(a), vg(b)) - brute_ssim(a, b)) <= 1e-10

    def test_window_larger_than_volume(self):
        with pytest.raises(ValueError):
            B.ssim(vg(np.zeros((5, 8, 8))), vg(np.zeros((5, 8, 8))))


class TestCnr:
    def test_equal_constants_zero(self):
        roi = np.zeros((4, 4, 4), bool)
        roi[:2] = True
        assert B.cnr(vg(np.full((4, 4, 4), 0.7)), roi, ~roi) == 0.0

    def test_hand_arithmetic(self):
        v = np.array([[[1.0, 1.0, 0.0, 0.2]]])
        roi = np.array([[[True, True, False, False]]])
        assert abs(B.cnr(vg(v), roi, ~roi) - 9.0) < 1e-12  # (1 - 0.1) / 0.1

    def test_flat_background_sentinel(self):
        v = np.array([[[1.0, 1.0, 0.0, 0.0]]])
        roi = np.array([[[True, True, False, False]]])
        assert B.cnr(vg(v), roi, ~roi) == math.inf

    def test_mask_validation(self):
        g = vg(np.zeros((2, 2, 2)))
        full = np.ones((2, 2, 2), bool)
        with pytest.raises(ValueError):
            B.cnr(g, full, full)
        with pytest.raises(ValueError):
            B.cnr(g, np.zeros((2, 2, 2), bool), full)
        with pytest.raises(ValueError):
            B.cnr(g, np.ones((2, 2), bool), full)


class TestMaxNormalizedAndReport:
    def test_clamp_and_scale(self):
        g = B.max_normalized(vg([[[-1.0, 0.5, 2.0]]]))
        np.testing.assert_array_equal(g.values, [[[0.0, 0.25, 1.0]]])

    def test_all_zero_stays_zero(self):
        assert not B.max_normalized(vg(np.zeros((2, 2, 2)))).values.any()

    def test_report_formats(self):
        r = B.MetricReport(1e-3, 30.0, 0.9)
        assert r.to_text() == "mse=0.001\npsnr=30\nssim=0.9\n"
        assert "cnr" not in r.to_json()
        assert '"cnr": 2.5' in B.MetricReport(1e-3, 30.0, 0.9, 2.5).to_json()
