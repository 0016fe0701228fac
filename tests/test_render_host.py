"""Host-side render API (no GPU): RenderSpec validation, projections and
slices (reference pkg/tests/test_render.py, host cases)."""

import numpy as np
import pytest

import paper_2601_00551_b200 as P


def random_grid(seed=15, dims=(9, 11, 7)):
    vals = P.CounterRng(seed).uniform(0, 1, int(np.prod(dims))).reshape(dims)
    return P.VoxelGrid(dims, 1e-3, np.zeros(3), vals)


def test_invalid_specs():
    with pytest.raises(ValueError):
        P.RenderSpec(dims=(0, 4, 4), spacing=1e-3, origin=(0, 0, 0))
    with pytest.raises(ValueError):
        P.RenderSpec(dims=(4, 4, 4), spacing=0.0, origin=(0, 0, 0))
    with pytest.raises(ValueError):
        P.RenderSpec(dims=(4, 4, 4), spacing=1e-3, origin=(0, 0, 0), support_sigma=1.0)


def test_projection_matches_brute_force():
    g = random_grid()
    got = P.max_amplitude_projection(g, "y")
    want = np.zeros((9, 7))
    for i in range(9):
        for k in range(7):
            want[i, k] = max(g.values[i, j, k] for j in range(11))
    np.testing.assert_array_equal(got, want)


def test_slices_and_bad_axis():
    g = random_grid()
    np.testing.assert_array_equal(P.slice_plane(g, "z", 3), g.values[:, :, 3])
    with pytest.raises(ValueError):
        P.slice_plane(g, "w", 0)
    with pytest.raises(ValueError):
        P.slice_plane(g, "x", 9)
    with pytest.raises(ValueError):
        P.max_amplitude_projection(g, "q")


def test_voxelgrid_shape_checked():
    with pytest.raises(ValueError):
        P.VoxelGrid((2, 2, 2), 1e-3, np.zeros(3), np.zeros((2, 2, 3)))
