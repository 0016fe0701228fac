"""Universal back-projection baseline and volume metrics (reference
``paball/baseline.py``), the back-projection on the GPU.

``ubp_reconstruct`` (baseline.py:52-89) is the §8f rank-4 kernel
(``csrc/pab_ubp.cu``): one thread per voxel, detectors in index order, the
reference's FP64 expression tree.  The metrics (MSE, PSNR, SSIM, CNR,
max-normalisation) are host array reductions of finished volumes, as in the
reference.
"""

from __future__ import annotations

import json
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import engine as E
from ._lib import call, load, ptr
from .model import VoxelGrid

__all__ = ["CoverageReport", "MetricReport", "ubp_reconstruct", "max_normalized", "mse", "psnr", "psnr_from_mse",
           "ssim", "cnr"]


@dataclass
class CoverageReport:
    """Voxel-sensor pairs whose travel time fell outside the time grid (baseline.py:41-49)."""

    n_total: int
    n_skipped: int

    @property
    def fraction_skipped(self) -> float:
        return self.n_skipped / self.n_total if self.n_total else 0.0


def ubp_reconstruct(real, array, spec) -> tuple[VoxelGrid, CoverageReport]:
    """Delay-and-sum back-projection with the temporal-derivative term
    (baseline.py:52-89): b(x) = (1/J) sum_j [2 p_j(t) - 2 t dp_j/dt],
    t = |x - r_j| / v, linear interpolation, np.gradient derivative."""
    grid = spec.empty_grid()
    nx, ny, nz = spec.dims
    n_det = int(array.positions.shape[0])
    tg = real.grid
    n = int(tg.n_samples)
    if n_det == 0:
        raise ZeroDivisionError("ubp_reconstruct: the sensor array is empty (weight 1/J)")
    load()
    dev = E.cuda_device()
    sig = torch.from_numpy(np.ascontiguousarray(real.data, dtype=np.float64)).to(dev)
    det = torch.from_numpy(np.ascontiguousarray(array.positions, dtype=np.float64).reshape(-1, 3)).to(dev)
    deriv = torch.empty_like(sig)
    vol = torch.empty(nx * ny * nz, dtype=torch.float64, device=dev)
    skipped = torch.zeros(1, dtype=torch.int64, device=dev)
    ox, oy, oz = (float(x) for x in spec.origin)
    call("pab_ubp", ptr(sig), n_det, n, float(tg.t0), float(tg.dt), ptr(det), float(array.sound_speed), nx, ny, nz,
         float(spec.spacing), ox, oy, oz, ptr(deriv), ptr(vol), ptr(skipped), E._stream())
    grid.values = vol.view(nx, ny, nz).cpu().numpy()
    return grid, CoverageReport(n_total=nx * ny * nz * n_det, n_skipped=int(skipped.item()))


def max_normalized(grid: VoxelGrid) -> VoxelGrid:
    """Negatives clamped to 0, peak scaled to 1; an all-zero volume stays
    all-zero (baseline.py:92-98)."""
    v = np.maximum(grid.values, 0.0)
    top = float(v.max()) if v.size else 0.0
    return VoxelGrid(grid.dims, grid.spacing, np.array(grid.origin, dtype=np.float64),
                     v / top if top > 0.0 else v)


def _same_shape(*grids: VoxelGrid) -> None:
    dims = {tuple(g.dims) for g in grids}
    if len(dims) != 1:
        raise ValueError(f"volume dims disagree: {sorted(dims)}")


def mse(a: VoxelGrid, b: VoxelGrid) -> float:
    """Mean squared voxel difference (baseline.py:107-110)."""
    _same_shape(a, b)
    return float(np.mean(np.square(a.values - b.values)))


def psnr_from_mse(m: float) -> float:
    """PSNR in dB at unit dynamic range, +inf for a zero error (baseline.py:113-117)."""
    return math.inf if m == 0.0 else -10.0 * math.log10(m)


def psnr(a: VoxelGrid, b: VoxelGrid) -> float:
    return psnr_from_mse(mse(a, b))


def _window_means(x: np.ndarray, w: int) -> np.ndarray:
    """Mean over every fully interior w^3 window: three separable running sums
    (prefix sum, then difference at lag w) instead of materialising windows."""
    for axis in range(3):
        c = np.cumsum(x, axis=axis)
        pad = [(0, 0)] * 3
        pad[axis] = (1, 0)
        c = np.pad(c, pad)
        hi = [slice(None)] * 3
        lo = [slice(None)] * 3
        hi[axis] = slice(w, None)
        lo[axis] = slice(0, -w)
        x = c[tuple(hi)] - c[tuple(lo)]
    return x / float(w ** 3)


def ssim(a: VoxelGrid, b: VoxelGrid, window: int = 7, k1: float = 0.01, k2: float = 0.03) -> float:
    """Mean local SSIM, uniform cubic window, unit dynamic range, population
    moments over every fully interior window (baseline.py:120-144)."""
    _same_shape(a, b)
    if min(a.dims) < window:
        raise ValueError(f"volume dims {a.dims} smaller than SSIM window {window}")
    x = np.asarray(a.values, dtype=np.float64)
    y = np.asarray(b.values, dtype=np.float64)
    mx, my = _window_means(x, window), _window_means(y, window)
    sxx = _window_means(x * x, window) - mx * mx
    syy = _window_means(y * y, window) - my * my
    sxy = _window_means(x * y, window) - mx * my
    c1, c2 = k1 ** 2, k2 ** 2
    ratio = ((2.0 * mx * my + c1) * (2.0 * sxy + c2)) / ((mx * mx + my * my + c1) * (sxx + syy + c2))
    return float(ratio.mean())


def cnr(grid: VoxelGrid, roi_mask: np.ndarray, bg_mask: np.ndarray) -> float:
    """Contrast-to-noise: (ROI mean - background mean) / background population
    std; +inf (or 0 when the means agree) for a flat background (baseline.py:147-162)."""
    roi = np.asarray(roi_mask, dtype=bool)
    bg = np.asarray(bg_mask, dtype=bool)
    shape = np.shape(grid.values)
    if roi.shape != shape or bg.shape != shape:
        raise ValueError("mask shapes must match the volume")
    if (roi & bg).any():
        raise ValueError("ROI and background masks overlap")
    if not (roi.any() and bg.any()):
        raise ValueError("ROI and background masks must both be non-empty")
    back = grid.values[bg]
    contrast = float(grid.values[roi].mean() - back.mean())
    noise = float(back.std())
    if noise == 0.0:
        return 0.0 if contrast == 0.0 else math.inf
    return contrast / noise


@dataclass
class MetricReport:
    """Volume-comparison metrics; ``cnr`` only when masks were given (baseline.py:165-186)."""

    mse: float
    psnr: float
    ssim: float
    cnr: float | None = None

    def _fields(self) -> dict:
        out = {"mse": self.mse, "psnr": self.psnr, "ssim": self.ssim}
        if self.cnr is not None:
            out["cnr"] = self.cnr
        return out

    def to_text(self) -> str:
        return "".join(f"{k}={v:.10g}\n" for k, v in self._fields().items())

    def to_json(self) -> str:
        return json.dumps(self._fields(), indent=2, allow_nan=True)
