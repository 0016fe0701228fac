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


def branching_tubes(n_balls: int, n_tubes: int, radius_range, box_lo, box_hi, p0_range=(0.5, 1.0),
                    a0: float = 0.1 * MM, seed: int = SEED_TRUTH, segment: float = 1.0 * MM,
                    steps: int = 12) -> PointCloud:
    """Random vessel trees: a few roots inside the box, each tube a smooth
    random walk of `steps` segments; later tubes branch off random points of
    earlier ones.  Balls are spread over tubes by length, uniform in the tube
    cross-section (radius drawn per tube from `radius_range`)."""
    rng = CounterRng(seed)
    lo, hi = np.asarray(box_lo, dtype=float), np.asarray(box_hi, dtype=float)
    n_roots = max(1, n_tubes // 5)
    tubes = []
    for t in range(n_tubes):
        if t < n_roots or not tubes:
            start = lo + (hi - lo) * rng.uniform(0.2, 0.8, 3)
        else:
            parent = tubes[int(rng.uniform(0.0, len(tubes), 1)[0]) % len(tubes)]
            start = parent[int(rng.uniform(0.0, len(parent), 1)[0]) % len(parent)]
        d = rng.unit_vectors(1)[0]
        pts = [start]
        for _ in range(steps):
            d = d + 0.5 * rng.unit_vectors(1)[0]
            d /= np.linalg.norm(d)
            nxt = np.clip(pts[-1] + segment * d, lo, hi)
            pts.append(nxt)
        tubes.append(np.array(pts))
    radii = rng.uniform(radius_range[0], radius_range[1], n_tubes)
    seg_len = [np.linalg.norm(np.diff(tb, axis=0), axis=1) for tb in tubes]
    total = np.array([s.sum() for s in seg_len])
    counts = np.floor(n_balls * total / total.sum()).astype(np.int64)
    counts[: n_balls - counts.sum()] += 1
    out = []
    for tb, sl, cnt, rad in zip(tubes, seg_len, counts, radii):
        if cnt == 0:
            continue
        cum = np.concatenate([[0.0], np.cumsum(sl)])
        s = rng.uniform(0.0, max(cum[-1], 1e-12), int(cnt))
        k = np.clip(np.searchsorted(cum, s, side="right") - 1, 0, len(sl) - 1)
        frac = (s - cum[k]) / np.maximum(sl[k], 1e-12)
        centre = tb[k] + frac[:, None] * (tb[k + 1] - tb[k])
        off = rng.unit_vectors(int(cnt)) * (rad * np.cbrt(rng.uniform(0.0, 1.0, int(cnt))))[:, None]
        out.append(centre + off)
    pos = np.concatenate(out)[:n_balls]
    p0 = rng.uniform(p0_range[0], p0_range[1], pos.shape[0])
    return PointCloud(pos, p0, np.full(pos.shape[0], a0))


def schedule_config(directivity=("none",), grid_n: int = 96) -> Scene:
    """BASELINE config 3: 512 detectors = seeded random subset of a
    2,048-point Fibonacci hemisphere (r = 40 mm); 50k truth balls on 40
    branching tubes; 96^3 init grid over the interior box [-14, 14]^2 x
    [-30, -2] mm (p0 = 0.1, a0 = 0.15 mm); 40 MHz x 4096 samples."""
    full = fibonacci_hemisphere(2048, 40 * MM)
    pick = np.sort(np.argsort(CounterRng(SEED_GEOMETRY).uniform(0.0, 1.0, 2048))[:512])
    array = SensorArray(full.positions[pick], 1500.0, normals=full.normals[pick])
    grid = TimeGrid(0.0, 1.0 / 40e6, 4096)
    lo, hi = np.array([-14, -14, -30]) * MM, np.array([14, 14, -2]) * MM
    truth = branching_tubes(50_000, 40, (0.1 * MM, 0.3 * MM), lo + 2 * MM, hi - 2 * MM)
    step = (hi - lo) / grid_n
    axes = [lo[a] + (np.arange(grid_n) + 0.5) * step[a] for a in range(3)]
    gx, gy, gz = np.meshgrid(*axes, indexing="ij")
    pos = np.column_stack([gx.ravel(), gy.ravel(), gz.ravel()])
    init = PointCloud(pos, np.full(pos.shape[0], 0.1), np.full(pos.shape[0], 0.15 * MM))
    return Scene("schedule", array, grid, truth, init, tuple(directivity))


def planar_config(n_balls: int = 4_000_000, directivity=("element", 0.5 * MM)) -> Scene:
    """BASELINE config 4: 32 x 32 planar detectors at 1.5 mm pitch on z = 0,
    each outward normal (+z) tilted by theta <= 30 deg (cos theta uniform)
    about a random azimuth; 4M balls in a 30 x 30 x 15 mm slab at
    z in [-20, -5] mm, p0 = exp(N(-1, 0.5)), a0 ~ U[0.05, 0.2] mm;
    40 MHz x 6144 samples; 0.5 mm square element directivity."""
    rng = CounterRng(SEED_GEOMETRY)
    ax = (np.arange(32) - 15.5) * 1.5 * MM
    gx, gy = np.meshgrid(ax, ax, indexing="ij")
    pos = np.column_stack([gx.ravel(), gy.ravel(), np.zeros(1024)])
    cth = rng.uniform(math.cos(math.radians(30.0)), 1.0, 1024)
    az = rng.uniform(0.0, 2.0 * math.pi, 1024)
    sth = np.sqrt(1.0 - cth * cth)
    normals = np.column_stack([sth * np.cos(az), sth * np.sin(az), cth])
    array = SensorArray(pos, 1500.0, normals=normals)
    grid = TimeGrid(0.0, 1.0 / 40e6, 6144)
    r = CounterRng(SEED_TRUTH)
    bp = np.column_stack([r.uniform(-15 * MM, 15 * MM, n_balls), r.uniform(-15 * MM, 15 * MM, n_balls),
                          r.uniform(-20 * MM, -5 * MM, n_balls)])
    p0 = np.exp(-1.0 + 0.5 * r.normal(n_balls))
    a0 = r.uniform(0.05 * MM, 0.2 * MM, n_balls)
    cloud = PointCloud(bp, p0, a0)
    p0_true = np.exp(-1.0 + 0.5 * CounterRng(SEED_RESAMPLE).normal(n_balls))
    return Scene("planar", array, grid, PointCloud(bp, p0_true, a0), cloud, tuple(directivity))


def mouse_config(grid_n: int = 256, n_truth: int = 300_000, n_det: int = 2048,
                 directivity=("cos_power", 2.0)) -> Scene:
    """BASELINE config 5: 256^3 grid cropped to the ellipsoid with full axes
    25 x 20 x 40 mm (about 8.8M balls survive; BASELINE's '16M' is the
    uncropped 256^3 = 16.8M); 300k truth balls on 500 tubes of radius
    0.05-0.4 mm; 2048 detectors on a seeded ring cylinder (radius 30 mm,
    z in [-25, 25] mm) with normals tilted randomly by <= 30 deg from the
    inward radial direction; 40 MHz x 8192 samples."""
    semi = np.array([12.5, 10.0, 20.0]) * MM
    ax = [(-1.0 + (np.arange(grid_n) + 0.5) * 2.0 / grid_n) * semi[a] for a in range(3)]
    gx, gy, gz = np.meshgrid(*ax, indexing="ij")
    inside = (gx / semi[0]) ** 2 + (gy / semi[1]) ** 2 + (gz / semi[2]) ** 2 <= 1.0
    pos = np.column_stack([gx[inside], gy[inside], gz[inside]])
    init = PointCloud(pos, np.full(pos.shape[0], 0.1), np.full(pos.shape[0], 0.1 * MM))
    truth = branching_tubes(n_truth, 500, (0.05 * MM, 0.4 * MM), -0.7 * semi, 0.7 * semi,
                            a0=0.1 * MM, steps=16)
    rng = CounterRng(SEED_GEOMETRY)
    phi = rng.uniform(0.0, 2.0 * math.pi, n_det)
    z = rng.uniform(-25 * MM, 25 * MM, n_det)
    R = 30 * MM
    dpos = np.column_stack([R * np.cos(phi), R * np.sin(phi), z])
    radial = np.column_stack([np.cos(phi), np.sin(phi), np.zeros(n_det)])   # outward
    tilt = rng.unit_vectors(n_det) * np.tan(math.radians(30.0)) * np.cbrt(rng.uniform(0, 1, n_det))[:, None]
    nrm = radial + tilt - np.sum(tilt * radial, axis=1, keepdims=True) * radial
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    array = SensorArray(dpos, 1500.0, normals=nrm)
    grid = TimeGrid(0.0, 1.0 / 40e6, 8192)
    return Scene("mouse", array, grid, truth, init, tuple(directivity))


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
