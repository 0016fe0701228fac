"""Gaussian splat voxelisation (reference render.py:55-93), for the volume
parity check of the fixed schedule.  TEST INFRASTRUCTURE ONLY.

Each ball adds max(p0, 0)-gated p0 * exp(-r^2 / 2 a0^2) to voxel centres in a
+-support*a0 box; balls are visited in lexicographic (x, y, z, p0, a0) order so
the volume does not depend on cloud order.
"""

from __future__ import annotations

import numpy as np


def voxelize(pos, p0, a0, dims, spacing, origin, support=3.0):
    pos = np.asarray(pos, dtype=np.float64).reshape(-1, 3)
    vol = np.zeros(tuple(dims))
    if pos.shape[0] == 0:
        return vol
    origin = np.asarray(origin, dtype=np.float64)
    hi_idx = np.asarray(dims) - 1
    for i in np.lexsort((a0, p0, pos[:, 2], pos[:, 1], pos[:, 0])):
        if p0[i] <= 0.0:
            continue
        c, s = pos[i], a0[i]
        lo = np.maximum(np.ceil((c - support * s - origin) / spacing).astype(np.int64), 0)
        hi = np.minimum(np.floor((c + support * s - origin) / spacing).astype(np.int64), hi_idx)
        if np.any(lo > hi):
            continue
        d = [origin[a] + np.arange(lo[a], hi[a] + 1, dtype=np.float64) * spacing - c[a] for a in range(3)]
        r2 = (d[0] ** 2)[:, None, None] + (d[1] ** 2)[None, :, None] + (d[2] ** 2)[None, None, :]
        vol[lo[0]:hi[0] + 1, lo[1]:hi[1] + 1, lo[2]:hi[2] + 1] += p0[i] * np.exp((-0.5 / (s * s)) * r2)
    return vol
