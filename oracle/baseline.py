"""Universal back-projection (reference baseline.py:52-89), FP64 numpy.
TEST INFRASTRUCTURE ONLY: the checker for csrc/pab_ubp.cu, never on the
product path.

b(x) = (1/J) sum_j [2 p_j(t) - 2 t dp_j/dt], t = |x - r_j| / v.  The
derivative is numpy's first-order-edge central difference (np.gradient);
p and dp/dt are sampled by linear interpolation at (t - t0)/dt with the index
clamped to [0, n-2] and the fraction to [0, 1]; pairs with (t - t0)/dt
outside [0, n-1] contribute nothing and are counted.  Detectors are summed in
index order, so the CUDA kernel (same order, same expression tree, no FMA)
agrees to the last bit.
"""

from __future__ import annotations

import numpy as np


def time_derivative(rows: np.ndarray, dt: float) -> np.ndarray:
    """np.gradient(rows, dt, axis=1) written out (edge_order=1)."""
    rows = np.asarray(rows, dtype=np.float64)
    out = np.empty_like(rows)
    out[:, 1:-1] = (rows[:, 2:] - rows[:, :-2]) / (2.0 * dt)
    out[:, 0] = (rows[:, 1] - rows[:, 0]) / dt
    out[:, -1] = (rows[:, -1] - rows[:, -2]) / dt
    return out


def voxel_centres(dims, spacing, origin) -> np.ndarray:
    """[nx*ny*nz, 3] centres, x slowest (model.py:399-400 axis_centers, ij order)."""
    axes = [origin[a] + np.arange(dims[a], dtype=np.float64) * spacing for a in range(3)]
    gx, gy, gz = np.meshgrid(*axes, indexing="ij")
    return np.column_stack([gx.ravel(), gy.ravel(), gz.ravel()])


def ubp(rows, t0, dt, sensors, sound_speed, dims, spacing, origin):
    """Returns (volume[nx,ny,nz], n_skipped)."""
    rows = np.asarray(rows, dtype=np.float64)
    sensors = np.asarray(sensors, dtype=np.float64).reshape(-1, 3)
    n_det, n = rows.shape
    x = voxel_centres(dims, spacing, origin)
    acc = np.zeros(x.shape[0])
    if n_det == 0:
        return acc.reshape(dims), 0
    if n < 2:
        raise ValueError("back-projection needs at least two samples per row")
    drows = time_derivative(rows, dt)
    weight = 1.0 / n_det
    skipped = 0
    for j in range(n_det):
        e = x - sensors[j]
        t = np.sqrt((e[:, 0] * e[:, 0] + e[:, 1] * e[:, 1]) + e[:, 2] * e[:, 2]) / sound_speed
        u = (t - t0) / dt
        inside = (u >= 0.0) & (u <= n - 1)
        skipped += int(inside.size - np.count_nonzero(inside))
        k = np.minimum(np.maximum(np.floor(u), 0.0), n - 2).astype(np.int64)
        f = np.minimum(np.maximum(u - k, 0.0), 1.0)
        g = 1.0 - f
        p_t = rows[j, k] * g + rows[j, k + 1] * f
        d_t = drows[j, k] * g + drows[j, k + 1] * f
        acc += np.where(inside, weight * (2.0 * p_t - (2.0 * t) * d_t), 0.0)
    return acc.reshape(dims), skipped
