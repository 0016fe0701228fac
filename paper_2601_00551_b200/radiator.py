"""Reference-compatible radiator API on the B200 kernels.

Mirrors ``paball.radiator`` (/root/reference/pkg/src/paball/radiator.py):
``ForwardContext`` (:98-114), ``ParamGradients`` (:117-132), op counter and
thread knobs (:53-95), ``simulate_signals`` (:362), ``simulate_at_rate``
(:368), ``downsample`` (:382), ``loss`` (:393), ``backward`` (:419) and the
shared seam ``_run_model`` (:290).  Same argument meaning, same error
classes; arrays cross the API as float64 numpy like the reference, the
arithmetic runs in ``libpaball_b200.so`` (FP32 per-sample math, FP64 per-ball
accumulation — tolerances in DESIGN.md §3).

Additions: ``ForwardContext.directivity`` (default ``Directivity("none")`` =
reference semantics).
"""

from __future__ import annotations

import hashlib
import os
import threading
from dataclasses import dataclass, field

import numpy as np
import torch

from . import engine as E
from . import hostio
from .model import SignalSet, TimeGrid

__all__ = [
    "Directivity",
    "ForwardContext",
    "ParamGradients",
    "simulate_signals",
    "simulate_at_rate",
    "downsample",
    "loss",
    "backward",
    "op_count",
    "reset_op_count",
    "ops_paused",
    "set_num_threads",
    "get_num_threads",
]

# ---------------------------------------------------------------------------
# Op counter (reference radiator.py:53-80): kernel-window samples evaluated.
# ---------------------------------------------------------------------------

_op_lock = threading.Lock()
_op_total = 0
_threads: int | None = None


def op_count() -> int:
    return _op_total


def reset_op_count(value: int = 0) -> None:
    global _op_total
    with _op_lock:
        _op_total = int(value)


def _add_ops(n: int) -> None:
    global _op_total
    with _op_lock:
        _op_total += int(n)


class ops_paused:
    """Work done inside does not advance the op counter."""

    def __enter__(self):
        self._saved = op_count()
        return self

    def __exit__(self, *exc):
        reset_op_count(self._saved)
        return False


def set_num_threads(n: int) -> None:
    """Accepted for API compatibility (radiator.py:82-86); the GPU path does
    not use host threads."""
    global _threads
    if n < 1:
        raise ValueError(f"thread count must be >= 1, got {n}")
    _threads = int(n)


def get_num_threads() -> int:
    if _threads is not None:
        return _threads
    try:
        return max(1, int(os.environ.get("PABALL_THREADS", "1")))
    except ValueError:
        return 1


# ---------------------------------------------------------------------------
# Context and gradients
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class Directivity:
    """Detector sensitivity vs. arrival direction (not in the reference).

    kind "none": D = 1 (reference semantics);
    "cos_power": D = max(cos theta, 0)^power, cos theta between the receive
    direction (-outward normal) and the detector-to-ball direction;
    "element": square element of side ``width`` (m), far-field weight
    D = sinc(w s1 / 2 a0) sinc(w s2 / 2 a0) at the pulse's spectral peak,
    s_k = direction . e_k with in-plane axes e1 (x projected), e2 = n x e1.
    """

    kind: str = "none"
    power: float = 2.0
    width: float = 5e-4

    def __post_init__(self) -> None:
        if self.kind not in E.DIR_CODES:
            raise ValueError(f"unknown directivity kind {self.kind!r}")
        if self.kind == "cos_power" and self.power < 0.0:
            raise ValueError("cos_power directivity needs power >= 0")
        if self.kind == "element" and not self.width > 0.0:
            raise ValueError("element directivity needs width > 0")

    @property
    def code(self) -> int:
        return E.DIR_CODES[self.kind]

    @property
    def param(self) -> float:
        return self.power if self.kind == "cos_power" else (self.width if self.kind == "element" else 0.0)

    def as_tuple(self) -> tuple:
        if self.kind == "none":
            return ("none",)
        return (self.kind, self.param)


@dataclass(frozen=True)
class ForwardContext:
    """Sensor layout plus the full-rate acquisition grid (radiator.py:98-114)."""

    array: object
    grid: TimeGrid
    cutoff_sigma: float = 6.0
    directivity: Directivity = field(default_factory=Directivity)

    def __post_init__(self) -> None:
        if self.cutoff_sigma < 4.0:
            raise ValueError(f"cutoff_sigma must be >= 4, got {self.cutoff_sigma}")


@dataclass
class ParamGradients:
    d_p0: np.ndarray
    d_a0: np.ndarray
    d_position: np.ndarray

    def __post_init__(self) -> None:
        n = self.d_p0.shape[0]
        if self.d_a0.shape != (n,) or self.d_position.shape != (n, 3):
            raise ValueError("gradient field shapes disagree")

    @classmethod
    def zeros(cls, n: int) -> "ParamGradients":
        return cls(np.zeros(n), np.zeros(n), np.zeros((n, 3)))


def _directivity(ctx) -> Directivity:
    d = getattr(ctx, "directivity", None)
    return d if isinstance(d, Directivity) else Directivity()


# ---------------------------------------------------------------------------
# Device caches: detector shards per context, supervision per array
# ---------------------------------------------------------------------------

_det_cache: dict = {}


def _detector_key(arr, d, dev, shard) -> tuple:
    """Content key of a sensor layout: the reference recomputes from the
    arrays on every call (radiator.py:316-332), so an in-place edit of
    ``positions`` / ``normals`` must reach the device; the digest of ~50 KB
    costs microseconds."""
    h = hashlib.blake2b(digest_size=16)
    pos = np.ascontiguousarray(arr.positions, dtype=np.float64)
    h.update(pos.tobytes())
    nrm = getattr(arr, "normals", None)
    if nrm is not None:
        h.update(np.ascontiguousarray(nrm, dtype=np.float64).tobytes())
    return (h.digest(), pos.shape, float(arr.sound_speed), dev.index, shard, d)


def device_detectors(ctx) -> E.DeviceDetectors:
    dev = E.cuda_device()
    shard = E.current_shard_for(dev)
    d = _directivity(ctx)
    arr = ctx.array
    key = _detector_key(arr, d, dev, shard)
    hit = _det_cache.get(key)
    if hit is not None:
        return hit
    det = E.DeviceDetectors(arr.positions, getattr(arr, "normals", None), d, arr.sound_speed, dev, shard)
    if len(_det_cache) > 16:
        _det_cache.clear()
    _det_cache[key] = det
    return det


_side_streams: dict = {}


def _side_stream(dev) -> torch.cuda.Stream:
    s = _side_streams.get(dev.index)
    if s is None:
        s = _side_streams[dev.index] = torch.cuda.Stream(dev)
    return s


def device_supervision(data: np.ndarray, det: E.DeviceDetectors, defer: bool = False):
    """This rank's supervision rows as FP32 on device, uploaded on every
    call: the reference reads ``real.data`` on every call, so an in-place
    edit between calls must be seen (no content cache; the iteration
    driver ``run_hierarchical`` keeps its own device copy of the array it
    was given).

    The rows are narrowed to FP32 while they are staged into page-locked
    memory (hostio: chunked, threaded, DMA queued per chunk) on a side
    stream.  ``defer=True`` returns (tensor, event) without making the
    current stream wait, so the copy overlaps whatever is enqueued before
    the caller waits on the event."""
    dev = det.pos.device
    main = torch.cuda.current_stream(dev)
    side = _side_stream(dev)
    # no side.wait_stream(main): the copy writes a fresh buffer of the side
    # stream's pool (freed only after main's uses, record_stream below) from
    # a staging slot whose previous DMA the stager waits for, so nothing
    # orders it after the work already queued on main -- the forward kernel
    # queued just before this call (round-2 profile: waiting for it left the
    # 0.3 ms DMA unhidden after the forward)
    (t,), ev = hostio.stager("supervision").upload([(data[det.lo:det.hi], torch.float32)], dev, stream=side)
    t.record_stream(main)
    if defer:
        return t, ev
    main.wait_event(ev)
    return t


def _acq(ctx, f: int) -> E.Acq:
    d = _directivity(ctx)
    return E.Acq(float(ctx.array.sound_speed), float(ctx.grid.t0), float(ctx.grid.dt),
                 int(ctx.grid.n_samples), int(f), float(ctx.cutoff_sigma), d.code, float(d.param))


# ---------------------------------------------------------------------------
# The seam (radiator.py:290-359)
# ---------------------------------------------------------------------------


def _run_model(cloud, ctx, f, real=None, stage="fine"):
    a0 = np.asarray(cloud.a0, dtype=np.float64)
    if a0.size and np.fmin.reduce(a0) <= 0.0:   # = np.any(a0 <= 0) of radiator.py:293 (NaNs ignored), one pass
        raise ValueError("all a0 must be > 0 for forward simulation")
    grid = ctx.grid
    n_out = grid.decimated(f).n_samples if f > 1 else grid.n_samples
    need_grad = real is not None
    if need_grad and real.data.shape[1] != n_out:
        raise ValueError(f"supervision has {real.data.shape[1]} samples, expected {n_out} at factor {f}")
    n_sensors = ctx.array.positions.shape[0]
    n = len(cloud)
    if n == 0:
        rows = np.zeros((n_sensors, n_out))
        if need_grad:
            return rows, float(np.sum(real.data * real.data) / real.data.size), ParamGradients.zeros(0), 0
        return rows, None, None, 0
    det = device_detectors(ctx)
    dev = det.pos.device
    acq = _acq(ctx, f)
    # the cloud first (sorting and packing wait for it); the supervision is
    # staged and uploaded only once the forward kernel is queued, so the host
    # copy and its DMA overlap the simulation (the residual waits for it)
    dc = E.DeviceCloud.from_host(cloud.positions, cloud.p0, a0, dev)
    adj_ready = None
    if need_grad:
        real_local = lambda: device_supervision(real.data, det, defer=True)   # noqa: E731
        # the adjoint's own packing (its radius buckets: a second sort) on a
        # side stream, overlapping the forward's sort, packing, coincidence
        # test and pairing table instead of following the forward
        adj = dc.adjoint_cloud()
        if adj is not dc and n > 0:
            adj_ready = adj.pack_async(_side_stream(dev))
    counters = E.PassCounters(dev)
    if not need_grad:
        local, _ = E.forward_rows(dc, det, acq, counters)
        rows = E.full_rows(local, det).double().cpu().numpy()
        ops = counters.read()
        _add_ops(ops)
        return rows, None, None, ops
    res, loss_rows = E.forward_rows(dc, det, acq, counters, real_local=real_local)
    stage_code = 2 if stage == "fine" else 1
    n_total = det.n_total * n_out
    flat = torch.empty(5 * n + E.TAIL, dtype=torch.float64, device=dev)
    if adj_ready is not None:
        torch.cuda.current_stream(dev).wait_event(adj_ready)
    # gradients, loss, error flags and op count in one buffer: one
    # all-reduce over detector shards, one copy into page-locked host memory
    # (the returned arrays are views that keep it alive)
    E.adjoint_grads(dc, det, acq, res, 1.0, stage_code, 2.0 / n_total, counters, flat=flat, loss_rows=loss_rows)
    host = torch.empty(5 * n + E.TAIL, dtype=torch.float64, pin_memory=True)
    host.copy_(flat, non_blocking=True)
    torch.cuda.current_stream(dev).synchronize()
    h = host.numpy()
    loss_sum, ops = counters.result(host_tail=h[5 * n:], check_nonfinite=False)
    _add_ops(ops)
    grads = ParamGradients(h[:n], h[n:2 * n], h[2 * n:5 * n].reshape(n, 3))
    return None, loss_sum / n_total, grads, ops


def simulate_signals(cloud, ctx) -> SignalSet:
    """Full-rate sensor signals (radiator.py:362-365)."""
    rows, _, _, _ = _run_model(cloud, ctx, 1)
    return SignalSet(ctx.grid, rows)


def simulate_at_rate(cloud, ctx, f: int) -> SignalSet:
    """Simulate directly on the f-times coarser grid (radiator.py:368-379)."""
    f = int(f)
    if f < 1:
        raise ValueError(f"decimation factor must be >= 1, got {f}")
    rows, _, _, _ = _run_model(cloud, ctx, f)
    return SignalSet(ctx.grid.decimated(f), rows)


def downsample(real, f: int) -> SignalSet:
    """Keep samples 0, f, 2f, ... (radiator.py:382-390): pure decimation, no
    arithmetic, done where the data lives (host arrays here)."""
    f = int(f)
    if f < 1:
        raise ValueError(f"decimation factor must be >= 1, got {f}")
    if f == 1:
        return SignalSet(real.grid, real.data.copy())
    return SignalSet(real.grid.decimated(f), real.data[:, ::f].copy())


def loss(sim, real) -> float:
    """Mean squared sample difference (radiator.py:393-402), reduced on the GPU."""
    if sim.data.shape != real.data.shape or sim.grid != real.grid:
        raise ValueError(f"signal sets disagree: {sim.data.shape}/{sim.grid} vs "
                         f"{real.data.shape}/{real.grid}")
    return E.mse_device(np.asarray(sim.data, dtype=np.float64), np.asarray(real.data, dtype=np.float64))


def _infer_factor(ctx_grid, real_grid) -> int:
    ratio = real_grid.dt / ctx_grid.dt
    f = int(round(ratio))
    if f < 1 or abs(ratio - f) > 1e-9 * f or real_grid.t0 != ctx_grid.t0:
        raise ValueError("supervision grid is not an integer decimation of the context grid")
    if ctx_grid.decimated(f).n_samples != real_grid.n_samples:
        raise ValueError("supervision grid is not an integer decimation of the context grid")
    return f


def backward(cloud, ctx, real, stage: str = "fine"):
    """Loss plus analytic gradients for every ball parameter (radiator.py:419-435)."""
    if stage not in ("coarse", "fine"):
        raise ValueError(f"stage must be 'coarse' or 'fine', got {stage!r}")
    f = _infer_factor(ctx.grid, real.grid)
    _, loss_value, grads, _ = _run_model(cloud, ctx, f, real=real, stage=stage)
    return loss_value, grads
