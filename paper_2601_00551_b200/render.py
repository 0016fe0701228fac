"""Ball cloud -> voxel grid (reference ``paball/render.py``), the splat on
the GPU.

``voxelize`` (render.py:55-93) is the §8f "next" row: the canonical
lexicographic ball order (x, y, z, p0, a0) is computed on the device with
stable sorts, every ball's clipped +-support*a0 box is cut into 8^3 voxel
bricks, the (brick, rank) pairs are sorted, and one CTA per brick gathers its
balls' terms per voxel in canonical order (``csrc/pab_render.cu``).  Each
voxel sees the reference's sequence of FP64 additions and expression tree;
only ``exp`` itself may differ from numpy's in the last ulp.
``max_amplitude_projection`` and ``slice_plane`` are host array reductions
of the result, as in the reference.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import engine as E
from ._lib import call, load, ptr
from .model import VoxelGrid

__all__ = ["RenderSpec", "voxelize", "max_amplitude_projection", "slice_plane"]

_AXES = {"x": 0, "y": 1, "z": 2}


@dataclass(frozen=True)
class RenderSpec:
    """Output grid layout (render.py:24-52); origin is the centre of voxel
    (0, 0, 0); support_sigma is the per-axis splat truncation."""

    dims: tuple
    spacing: float
    origin: tuple
    support_sigma: float = 3.0

    def __post_init__(self) -> None:
        dims = tuple(int(d) for d in self.dims)
        if len(dims) != 3 or any(d <= 0 for d in dims):
            raise ValueError(f"dims must be three positive counts, got {self.dims}")
        if self.spacing <= 0.0:
            raise ValueError(f"spacing must be > 0, got {self.spacing}")
        if self.support_sigma < 2.0:
            raise ValueError(f"support_sigma must be >= 2, got {self.support_sigma}")
        object.__setattr__(self, "dims", dims)
        object.__setattr__(self, "origin", tuple(float(x) for x in self.origin))

    def empty_grid(self) -> VoxelGrid:
        return VoxelGrid(self.dims, self.spacing, np.array(self.origin), np.zeros(self.dims))


def _canonical_order(pos: torch.Tensor, p0: torch.Tensor, a0: torch.Tensor) -> torch.Tensor:
    """np.lexsort((a0, p0, z, y, x)) on the device: stable sorts from the
    least significant key up."""
    idx = torch.sort(a0, stable=True).indices
    for key in (p0, pos[:, 2], pos[:, 1], pos[:, 0]):
        idx = idx[torch.sort(key[idx], stable=True).indices]
    return idx.contiguous()


def voxelize(cloud, spec: RenderSpec) -> VoxelGrid:
    """Sum every ball's truncated Gaussian splat into the grid
    (render.py:55-93; p0 <= 0 contributes nothing)."""
    a0_h = np.asarray(cloud.a0, dtype=np.float64)
    if np.any(a0_h <= 0.0):
        raise ValueError("all a0 must be > 0 for voxelization")
    grid = spec.empty_grid()
    n = len(cloud)
    if n == 0:
        return grid
    load()
    dev = E.cuda_device()
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(dev)
    pos = t(np.asarray(cloud.positions).reshape(-1, 3))
    p0 = t(cloud.p0)
    a0 = t(a0_h)
    order = _canonical_order(pos, p0, a0)
    nx, ny, nz = spec.dims
    ox, oy, oz = spec.origin
    sp, sup = float(spec.spacing), float(spec.support_sigma)
    box = torch.empty((n, 6), dtype=torch.int32, device=dev)
    count = torch.empty(n, dtype=torch.int64, device=dev)
    stream = E._stream()
    call("pab_vox_count", ptr(pos), ptr(p0), ptr(a0), ptr(order), n, nx, ny, nz, sp, ox, oy, oz, sup, ptr(box),
         ptr(count), stream)
    offset = torch.cumsum(count, 0) - count
    total = int((offset[-1] + count[-1]).item())
    keys = torch.empty(max(total, 1), dtype=torch.int64, device=dev)
    if total:
        call("pab_vox_emit", ptr(box), ptr(offset), n, nx, ny, nz, ptr(keys), stream)
        keys = torch.sort(keys[:total]).values
    nb = int(load().pab_vox_brick_count(nx, ny, nz))
    start = torch.empty(nb, dtype=torch.int64, device=dev)
    end = torch.empty(nb, dtype=torch.int64, device=dev)
    vol = torch.empty(nx * ny * nz, dtype=torch.float64, device=dev)
    call("pab_vox_gather", ptr(pos), ptr(p0), ptr(a0), ptr(order), ptr(box), ptr(keys), total, nx, ny, nz, sp, ox,
         oy, oz, sup, ptr(start), ptr(end), ptr(vol), stream)
    grid.values = vol.view(nx, ny, nz).cpu().numpy()
    return grid


def max_amplitude_projection(grid: VoxelGrid, axis: str) -> np.ndarray:
    """Per-pixel maximum of the volume along one axis (render.py:96-100)."""
    if axis not in _AXES:
        raise ValueError(f"axis must be one of x, y, z; got {axis!r}")
    return grid.values.max(axis=_AXES[axis])


def slice_plane(grid: VoxelGrid, axis: str, index: int) -> np.ndarray:
    """Exact plane extraction at the given index along an axis (render.py:103-112)."""
    if axis not in _AXES:
        raise ValueError(f"axis must be one of x, y, z; got {axis!r}")
    a = _AXES[axis]
    if not 0 <= index < grid.dims[a]:
        raise ValueError(f"slice index {index} out of range for axis {axis} with {grid.dims[a]} planes")
    return np.take(grid.values, index, axis=a).copy()
