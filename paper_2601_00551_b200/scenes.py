"""Seeded synthetic inputs for the BASELINE.json configurations.

The reference measures on its own seeded generators (reference
``geometry.py:340-408``, ``phantom.py:120-196``); BASELINE.json's configs name
shapes the reference does not generate (Bezier tubes, ellipsoid caps, grid
initialisations).  Everything here draws from ``CounterRng`` (SplitMix64,
reference model.py:97-145) so a seed pins the inputs on every host.

Seeds: 101 geometry, 102 truth, 103 init, 104 noise/jitter,
105 supervision p0 resample.  Units are SI (m, s).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .model import CounterRng, PointCloud, SensorArray, TimeGrid

SEED_GEOMETRY = 101
SEED_TRUTH = 102
SEED_INIT = 103
SEED_JITTER = 104
SEED_RESAMPLE = 105

MM = 1e-3


def hemisphere_random(count: int, radius: float, seed: int = SEED_GEOMETRY) -> SensorArray:
    """Area-uniform random points on the z <= 0 half sphere; outward normals
    (the receive direction -normal points at the centre)."""
    rng = CounterRng(seed)
    z = -rng.uniform(0.0, 1.0, count)
    phi = rng.uniform(0.0, 2.0 * math.pi, count)
    rxy = np.sqrt(np.maximum(0.0, 1.0 - z * z))
    unit = np.column_stack([rxy * np.cos(phi), rxy * np.sin(phi), z])
    return SensorArray(radius * unit, 1500.0, normals=unit)


def fibonacci_hemisphere(count: int, radius: float) -> SensorArray:
    """Deterministic spiral on z <= 0 (same layout rule as reference
    geometry.py:351-358), outward normals."""
    k = np.arange(count, dtype=np.float64)
    z = -(k + 0.5) / count
    r = np.sqrt(np.maximum(0.0, 1.0 - z * z))
    th = math.pi * (3.0 - math.sqrt(5.0)) * k
    unit = np.column_stack([r * np.cos(th), r * np.sin(th), z])
    return SensorArray(radius * unit, 1500.0, normals=unit)


def ellipsoid_cap(count: int, semi_axes=(30 * MM, 30 * MM, 26 * MM), z_top_frac: float = 0.3,
                  jitter_sigma: float = 2 * MM, seed: int = SEED_GEOMETRY,
                  jitter_seed: int = SEED_JITTER) -> SensorArray:
    """Area-uniform points on the ellipsoid cap z <= z_top_frac * c, jittered
    N(0, sigma) along the outward normal; normals are the unjittered surface
    normals (config 2)."""
    a, b, c = semi_axes
    rng = CounterRng(seed)
    pts = []
    need = count
    # area element of the ellipsoid relative to the unit sphere, bounded by max
    bound = max(b * c, a * c, a * b)
    while need > 0:
        m = 4 * need + 64
        zs = rng.uniform(-1.0, z_top_frac, m)
        ph = rng.uniform(0.0, 2.0 * math.pi, m)
        acc = rng.uniform(0.0, 1.0, m)
        rs = np.sqrt(np.maximum(0.0, 1.0 - zs * zs))
        xs, ys = rs * np.cos(ph), rs * np.sin(ph)
        scale = np.sqrt((b * c * xs) ** 2 + (a * c * ys) ** 2 + (a * b * zs) ** 2) / bound
        ok = acc < scale
        sel = np.column_stack([a * xs, b * ys, c * zs])[ok][:need]
        pts.append(sel)
        need -= sel.shape[0]
    p = np.concatenate(pts)[:count]
    n = p / np.array([a * a, b * b, c * c])
    n /= np.linalg.norm(n, axis=1, keepdims=True)
    jit = CounterRng(jitter_seed).normal(count, jitter_sigma)
    return SensorArray(p + jit[:, None] * n, 1500.0, normals=n)


def _bezier(ctrl: np.ndarray, t: np.ndarray) -> np.ndarray:
    s = 1.0 - t
    return ((s ** 3)[:, None] * ctrl[0] + (3 * s * s * t)[:, None] * ctrl[1]
            + (3 * s * t * t)[:, None] * ctrl[2] + (t ** 3)[:, None] * ctrl[3])


def bezier_tubes(n_balls: int, n_tubes: int = 3, tube_radius: float = 0.3 * MM,
                 half_box: float = 4.5 * MM, p0_range=(0.5, 1.0), a0: float = 0.1 * MM,
                 seed: int = SEED_TRUTH) -> PointCloud:
    """Balls along random cubic Bezier centre lines, uniform inside a tube of
    the given radius (config 1 ground truth)."""
    rng = CounterRng(seed)
    ctrl = rng.uniform(-half_box, half_box, n_tubes * 12).reshape(n_tubes, 4, 3)
    tube = np.minimum((rng.uniform(0.0, 1.0, n_balls) * n_tubes).astype(np.int64), n_tubes - 1)
    t = rng.uniform(0.0, 1.0, n_balls)
    centre = np.empty((n_balls, 3))
    for k in range(n_tubes):
        sel = tube == k
        centre[sel] = _bezier(ctrl[k], t[sel])
    direc = rng.unit_vectors(n_balls)
    rad = tube_radius * np.cbrt(rng.uniform(0.0, 1.0, n_balls))
    pos = centre + rad[:, None] * direc
    p0 = rng.uniform(p0_range[0], p0_range[1], n_balls)
    return PointCloud(pos, p0, np.full(n_balls, a0))


def grid_cloud(n_per_axis: int, lo: float, hi: float, p0: float, a0: float) -> PointCloud:
    """Cell-centred n^3 grid over [lo, hi]^3, x-major order."""
    step = (hi - lo) / n_per_axis
    ax = lo + (np.arange(n_per_axis) + 0.5) * step
    gx, gy, gz = np.meshgrid(ax, ax, ax, indexing="ij")
    pos = np.column_stack([gx.ravel(), gy.ravel(), gz.ravel()])
    n = pos.shape[0]
    return PointCloud(pos, np.full(n, p0), np.full(n, a0))


def uniform_cube(n_balls: int, half: float, p0_range, a0_range, seed: int = SEED_TRUTH) -> PointCloud:
    rng = CounterRng(seed)
    pos = rng.uniform(-half, half, 3 * n_balls).reshape(n_balls, 3)
    p0 = rng.uniform(p0_range[0], p0_range[1], n_balls)
    a0 = rng.uniform(a0_range[0], a0_range[1], n_balls)
    return PointCloud(pos, p0, a0)


@dataclass
class Scene:
    """One configuration: detectors, time grid, ground truth / candidate
    clouds and the directivity mode."""

    name: str
    array: SensorArray
    grid: TimeGrid
    truth: PointCloud | None
    init: PointCloud | None
    directivity: tuple


def toy_config(directivity=("none",)) -> Scene:
    """BASELINE config 1: 256 detectors on a random r = 20 mm hemisphere,
    2,000 balls on 3 Bezier tubes (radius 0.3 mm) in a 10 mm cube, a0 = 0.1 mm,
    20 MHz x 1024 samples; 32^3 cell-centred init grid over [-5, 5] mm with
    p0 = 0.1, a0 = 0.1 mm."""
    array = hemisphere_random(256, 20 * MM)
    grid = TimeGrid(0.0, 1.0 / 20e6, 1024)
    truth = bezier_tubes(2000)
    init = grid_cloud(32, -5 * MM, 5 * MM, 0.1, 0.1 * MM)
    return Scene("toy", array, grid, truth, init, tuple(directivity))


def microbench_config(n_balls: int = 1_000_000, n_det: int = 1024, n_samples: int = 4096,
                      directivity=("cos_power", 2.0)) -> Scene:
    """BASELINE config 2: uniform balls in a 20 mm cube, p0 ~ U[0, 1],
    a0 ~ U[0.05, 0.2] mm; 1024 detectors on a jittered ellipsoid cap with
    cos^2 directivity; 40 MHz x 4096 samples.  ``init`` holds the cloud that
    is simulated/differentiated; ``truth`` has the same positions and a0 with
    p0 resampled (seed 105) and defines the supervision."""
    array = ellipsoid_cap(n_det)
    grid = TimeGrid(0.0, 1.0 / 40e6, n_samples)
    cloud = uniform_cube(n_balls, 10 * MM, (0.0, 1.0), (0.05 * MM, 0.2 * MM))
    p0_true = CounterRng(SEED_RESAMPLE).uniform(0.0, 1.0, n_balls)
    truth = PointCloud(cloud.positions, p0_true, cloud.a0)
    return Scene("microbench", array, grid, truth, cloud, tuple(directivity))
