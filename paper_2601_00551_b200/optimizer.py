"""Reference-compatible iteration driver with device-resident state.

Mirrors ``paball.optimizer`` (/root/reference/pkg/src/paball/optimizer.py):
``Level``/``Schedule``/``SCHEDULE_PRESETS`` (:62-111), ``DensityThresholds``
(:114-154), ``LearningRates`` (:157-165), ``OptimState``/``create_state``
(:173-200), ``FilterReport``/``zero_gradient_filter`` (:217-258), ``step``
(:266-306), ``density_control`` (:314-406), ``IterationTrace``/
``run_hierarchical`` (:414-500).

The cloud, Adam moments and last gradients live on the GPU between calls
(FP64 master values; the kernels read packed FP32-offset records).  Host
``PointCloud`` views are materialised only when ``state.cloud`` / ``state.m``
/ ``state.v`` are read.  Per iteration the host sees one scalar (the loss).
"""

from __future__ import annotations

import math
import time
from collections.abc import MutableMapping
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from . import engine as E
from . import radiator as R
from ._lib import call, ptr
from .model import CounterRng, OptimizationError, PointCloud, RngSeed, SimulationError

__all__ = [
    "Level", "Schedule", "SCHEDULE_PRESETS", "DensityThresholds", "LearningRates", "OptimState",
    "FilterReport", "IterationTrace", "TraceRecord", "zero_gradient_filter", "create_state", "step",
    "density_control", "run_hierarchical",
]

_PLATEAU_REL = 1e-5
_PLATEAU_WINDOW = 50
_COARSE_DENSITY_EVERY = 100
_ADAM_BETA1 = 0.9
_ADAM_BETA2 = 0.999
_A0_RUNTIME_FLOOR = 1e-9


# ---------------------------------------------------------------------------
# Schedules, thresholds, learning rates (host-side configuration)
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class Level:
    f: int
    max_iters: int
    stage: str

    def __post_init__(self) -> None:
        if self.f < 1:
            raise ValueError(f"decimation factor must be >= 1, got {self.f}")
        if self.max_iters < 0:
            raise ValueError(f"max_iters must be >= 0, got {self.max_iters}")
        if self.stage not in ("coarse", "fine"):
            raise ValueError(f"stage must be 'coarse' or 'fine', got {self.stage!r}")


@dataclass(frozen=True)
class Schedule:
    levels: tuple
    duplication_period: int = 200

    def __post_init__(self) -> None:
        levels = tuple(self.levels)
        if not levels:
            raise ValueError("schedule needs at least one level")
        fs = [lv.f for lv in levels]
        if any(b > a for a, b in zip(fs, fs[1:])):
            raise ValueError(f"decimation factors must be non-increasing, got {fs}")
        if levels[-1].f != 1 or levels[-1].stage != "fine":
            raise ValueError("final level must be fine at the native rate (f=1)")
        if self.duplication_period < 1:
            raise ValueError(f"duplication_period must be >= 1, got {self.duplication_period}")
        object.__setattr__(self, "levels", levels)


def _preset(factors, iters):
    stages = ["coarse"] + ["fine"] * (len(factors) - 1)
    return Schedule(tuple(Level(f, it, st) for f, it, st in zip(factors, iters, stages)))


SCHEDULE_PRESETS = {
    "sim-16-4-1": _preset((16, 4, 1), (2000, 1000, 1000)),
    "invivo-4-2-1": _preset((4, 2, 1), (1000, 500, 500)),
}


@dataclass(frozen=True)
class DensityThresholds:
    destroy_p0_frac: float = 0.02
    split_a0: float = 2e-3
    duplicate_grad_quantile: float = 0.90
    a0_min: float = 1e-4
    a0_max: float = 8e-3

    def __post_init__(self) -> None:
        vals = (self.destroy_p0_frac, self.split_a0, self.duplicate_grad_quantile, self.a0_min, self.a0_max)
        if any(v <= 0.0 for v in vals):
            raise ValueError("density thresholds must all be positive")
        if not (self.a0_min < self.split_a0 < self.a0_max):
            raise ValueError(f"need a0_min < split_a0 < a0_max, got "
                             f"{self.a0_min} / {self.split_a0} / {self.a0_max}")

    @classmethod
    def from_spacing(cls, spacing: float, **overrides) -> "DensityThresholds":
        kw = dict(destroy_p0_frac=0.02, split_a0=2.0 * spacing, duplicate_grad_quantile=0.90,
                  a0_min=0.25 * spacing, a0_max=8.0 * spacing)
        kw.update(overrides)
        return cls(**kw)


@dataclass(frozen=True)
class LearningRates:
    p0: float = 1e-2
    a0: float = 4e-5
    position: float = 2e-5

    @classmethod
    def from_spacing(cls, spacing: float, p0: float = 1e-2) -> "LearningRates":
        return cls(p0=p0, a0=0.1 * spacing, position=0.05 * spacing)


# ---------------------------------------------------------------------------
# Device-resident optimiser state
# ---------------------------------------------------------------------------

_KEYS = ("p0", "a0", "position")


class _DeviceMoments(MutableMapping):
    """Host view of one moment dict; item assignment uploads to the device."""

    def __init__(self, owner: "OptimState", which: str):
        self._owner, self._which = owner, which

    def _store(self) -> dict:
        return self._owner._m if self._which == "m" else self._owner._v

    def __getitem__(self, key):
        return self._store()[key].cpu().numpy().copy()

    def __setitem__(self, key, value):
        ref = self._store()[key]
        arr = np.asarray(value, dtype=np.float64).reshape(ref.shape)
        self._store()[key] = torch.from_numpy(np.ascontiguousarray(arr)).to(ref.device)

    def __delitem__(self, key):
        raise TypeError("moment keys are fixed")

    def __iter__(self):
        return iter(self._store())

    def __len__(self):
        return len(self._store())


class _DeviceGrads:
    """last_grad on device; host ParamGradients on demand."""

    def __init__(self, d_p0, d_a0, d_pos):
        self.d_p0_t, self.d_a0_t, self.d_pos_t = d_p0, d_a0, d_pos

    def host(self) -> R.ParamGradients:
        return R.ParamGradients(self.d_p0_t.cpu().numpy(), self.d_a0_t.cpu().numpy(), self.d_pos_t.cpu().numpy())


class OptimState:
    """Cloud plus adaptive-moment accumulators (optimizer.py:173-193), on the GPU."""

    def __init__(self, cloud: PointCloud, lr: LearningRates, seed: RngSeed, step_count: int = 0,
                 m: dict | None = None, v: dict | None = None, last_grad=None):
        self.lr = lr
        self.seed = seed
        self.step_count = int(step_count)
        self._dev = E.cuda_device()
        self._set_cloud(cloud)
        n = len(cloud)
        z = lambda shape: torch.zeros(shape, dtype=torch.float64, device=self._dev)
        self._m = {"p0": z(n), "a0": z(n), "position": z((n, 3))}
        self._v = {"p0": z(n), "a0": z(n), "position": z((n, 3))}
        for src, dst in ((m, self._m), (v, self._v)):
            for k, arr in (src or {}).items():
                dst[k] = torch.from_numpy(np.ascontiguousarray(arr, dtype=np.float64)).to(self._dev)
        self._last = None
        if last_grad is not None:
            self.last_grad = last_grad

    # -- cloud ------------------------------------------------------------
    def _set_cloud(self, cloud: PointCloud) -> None:
        self._dc = E.DeviceCloud.from_host(cloud.positions, cloud.p0, cloud.a0, self._dev)
        self._free = torch.from_numpy(np.ascontiguousarray(cloud.a0_free, dtype=np.float64)).to(self._dev)
        self._generation = int(cloud.generation)
        self._host_cache = None

    @property
    def cloud(self) -> PointCloud:
        if self._host_cache is None:
            dc = self._dc
            self._host_cache = PointCloud(dc.pos.cpu().numpy(), dc.p0.cpu().numpy(), dc.a0.cpu().numpy(),
                                          self._free.cpu().numpy(), self._generation)
        return self._host_cache

    @cloud.setter
    def cloud(self, value: PointCloud) -> None:
        self._set_cloud(value)

    @property
    def n(self) -> int:
        return self._dc.n

    @property
    def m(self):
        return _DeviceMoments(self, "m")

    @property
    def v(self):
        return _DeviceMoments(self, "v")

    @property
    def last_grad(self):
        return None if self._last is None else self._last.host()

    @last_grad.setter
    def last_grad(self, g) -> None:
        if g is None:
            self._last = None
            return
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(self._dev)
        self._last = _DeviceGrads(t(g.d_p0), t(g.d_a0), t(g.d_position))

    def _touched(self, resort: bool = False) -> None:
        self._host_cache = None
        self._dc.invalidate(resort=resort)


def create_state(cloud: PointCloud, lr: LearningRates | None = None, seed=0) -> OptimState:
    if not isinstance(seed, RngSeed):
        seed = RngSeed(seed)
    return OptimState(cloud=cloud, lr=lr or LearningRates(), seed=seed)


# ---------------------------------------------------------------------------
# Zero-gradient filtering (optimizer.py:217-258)
# ---------------------------------------------------------------------------


@dataclass
class FilterReport:
    g: np.ndarray
    n_input: int
    n_retained: int

    @property
    def no_evidence(self) -> bool:
        return self.n_retained == 0


def _compact_indices(key: torch.Tensor, mode: int) -> torch.Tensor:
    """Ascending indices i with key[i] < 0 (mode 0) / <= 0 (1) / != 0 (2) /
    > 0 (3) / == 0 (4)."""
    n = key.numel()
    dev = key.device
    if n == 0:
        return torch.empty(0, dtype=torch.int32, device=dev)
    ws = E.workspace(dev)
    idx = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    count = ws.get("compact_count", 1, torch.int32)
    scratch = ws.get("compact_ws", int(_lib.load().pab_compact_workspace_bytes(n)) // 4 + 1, torch.int32)
    call("pab_compact", ptr(key), n, mode, ptr(idx), ptr(count), ptr(scratch), E._stream())
    return idx[: int(count.item())]


def filter_gradient(dc: E.DeviceCloud, det: E.DeviceDetectors, acq: E.Acq, real_local: torch.Tensor,
                    counters: E.PassCounters) -> torch.Tensor:
    """g_i = dL/dp0 at p0 = 0: forward rows vanish, res = -real exactly."""
    n_total = det.n_total * acq.n_out
    d_p0, _, _ = E.adjoint_grads(dc, det, acq, real_local, -1.0, 0, 2.0 / n_total, counters, count_ops=True)
    return d_p0


def zero_gradient_filter(cloud, ctx, real, f: int, strict: bool = True):
    """Keep only balls whose pressure wants to grow away from zero."""
    if len(cloud) == 0:
        raise ValueError("cannot filter an empty cloud")
    if f < 1:
        raise ValueError(f"decimation factor must be >= 1, got {f}")
    if np.any(np.asarray(cloud.a0) <= 0.0):
        raise ValueError("all a0 must be > 0 for forward simulation")
    real_k = R.downsample(real, f) if f > 1 else real
    det = R.device_detectors(ctx)
    dev = det.pos.device
    acq = R._acq(ctx, f)
    if real_k.data.shape[1] != acq.n_out:
        raise ValueError(f"supervision has {real_k.data.shape[1]} samples, expected {acq.n_out} at factor {f}")
    dc = E.DeviceCloud.from_host(cloud.positions, np.zeros(len(cloud)), cloud.a0, dev)
    counters = E.PassCounters(dev)
    g = filter_gradient(dc, det, acq, R.device_supervision(real_k.data, det), counters)
    idx = _compact_indices(g, 0 if strict else 1)
    R._add_ops(counters.read())
    keep = idx.cpu().numpy().astype(np.int64)
    retained = cloud.subset(keep) if isinstance(cloud, PointCloud) else type(cloud).subset(cloud, keep)
    return retained, FilterReport(g=g.cpu().numpy(), n_input=len(cloud), n_retained=len(retained))


# ---------------------------------------------------------------------------
# One optimisation step (optimizer.py:266-306)
# ---------------------------------------------------------------------------


def _adam_(param: torch.Tensor, grad: torch.Tensor, m: torch.Tensor, v: torch.Tensor, lr: float, t: int,
           floor: float | None = None) -> None:
    bc1 = 1.0 - _ADAM_BETA1 ** t
    bc2 = 1.0 - _ADAM_BETA2 ** t
    call("pab_adam", ptr(param), ptr(grad), ptr(m), ptr(v), param.numel(), float(lr), bc1, bc2,
         float(floor if floor is not None else 0.0), 1 if floor is not None else 0, E._stream())


def _device_step(state: OptimState, det: E.DeviceDetectors, acq: E.Acq, real_local: torch.Tensor,
                 stage: str) -> float:
    dc = state._dc
    counters = E.PassCounters(dc.dev)
    res, loss_rows = E.forward_rows(dc, det, acq, counters, real_local=real_local)
    n_total = det.n_total * acq.n_out
    stage_code = 2 if stage == "fine" else 1
    d_p0, d_a0, d_pos = E.adjoint_grads(dc, det, acq, res, 1.0, stage_code, 2.0 / n_total, counters,
                                        loss_rows=loss_rows)
    # the one host read of the iteration: the all-reduced pass tail (loss,
    # error flags, op count), identical on every rank
    loss_sum, ops = counters.result(check_nonfinite=False)
    loss_value = loss_sum / n_total
    if not math.isfinite(loss_value) or counters.tail_flags()[1]:
        raise OptimizationError(
            f"non-finite loss or gradient at step {state.step_count}: loss={loss_value}, "
            f"balls={dc.n}, p0 range=({float(dc.p0.min())}, {float(dc.p0.max())}), "
            f"a0 range=({float(dc.a0.min())}, {float(dc.a0.max())})")
    R._add_ops(ops)
    state.step_count += 1
    t = state.step_count
    _adam_(dc.p0, d_p0, state._m["p0"], state._v["p0"], state.lr.p0, t)
    _adam_(dc.a0, d_a0, state._m["a0"], state._v["a0"], state.lr.a0, t, floor=_A0_RUNTIME_FLOOR)
    if stage == "fine":
        _adam_(dc.pos, d_pos, state._m["position"], state._v["position"], state.lr.position, t)
    state._last = _DeviceGrads(d_p0, d_a0, d_pos)
    state._touched()
    return loss_value


def step(state: OptimState, ctx, real_k, f: int, stage: str):
    """One adaptive-moment update; returns (state, pre-update loss)."""
    expected = ctx.grid.decimated(f).n_samples if f > 1 else ctx.grid.n_samples
    if real_k.data.shape[1] != expected:
        raise ValueError(f"supervision not decimated to factor {f}: has {real_k.data.shape[1]} samples, "
                         f"expected {expected}")
    if stage not in ("coarse", "fine"):
        raise ValueError(f"stage must be 'coarse' or 'fine', got {stage!r}")
    det = R.device_detectors(ctx)
    acq = R._acq(ctx, f)
    if state.n == 0:
        raise OptimizationError("all points destroyed")
    loss_value = _device_step(state, det, acq, R.device_supervision(real_k.data, det), stage)
    return state, loss_value


# ---------------------------------------------------------------------------
# Adaptive density control (optimizer.py:314-406)
# ---------------------------------------------------------------------------


def _select(x: torch.Tensor, k: int, out: torch.Tensor) -> None:
    """out[0] = k-th smallest (0-based) of x (exact radix selection on device)."""
    ws = E.workspace(x.device)
    st = ws.get("select_state", int(_lib.load().pab_select_workspace_bytes()) // 8, torch.int64)
    call("pab_select_kth_f64", ptr(x), x.numel(), int(k), ptr(out), ptr(st), E._stream())


def density_control(state: OptimState, thresholds: DensityThresholds, stage: str) -> OptimState:
    """Destroy weak / out-of-range balls, split oversized ones, duplicate the
    top decile by position-gradient norm (fine); optimizer.py:314-406.

    Runs on the GPU (``pab_select_kth_f64``, ``pab_density_*``,
    ``pab_compact``, gathers); the isotropic unit vectors are drawn from the
    reference's SplitMix64 stream (``CounterRng(seed).spawn(generation)``) on
    the host in the reference's order (split children first, then
    duplicates) and uploaded.  Outputs are bit-identical to the reference."""
    n = state.n
    if n == 0:
        state._generation += 1
        state._host_cache = None
        return state
    dev = state._dev
    dc = state._dc
    rng = CounterRng(state.seed).spawn(state._generation)
    f64 = lambda m: torch.empty(m, dtype=torch.float64, device=dev)
    up = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(dev)

    # destroy: p0 below frac * median, a0 outside [a0_min, a0_max]
    med = f64(2)
    _select(dc.p0, (n - 1) // 2, med[0:1])
    if n % 2 == 0:
        _select(dc.p0, n // 2, med[1:2])
    key = f64(n)
    call("pab_density_keep_key", ptr(dc.p0), ptr(dc.a0), n, ptr(med[0:1]), ptr(med[1:2]) if n % 2 == 0 else None,
         float(thresholds.destroy_p0_frac), float(thresholds.a0_min), float(thresholds.a0_max), ptr(key),
         E._stream())
    surv = _compact_indices(key, 0)
    ns = surv.numel()
    pos, p0, a0 = _gather(dc.pos, 3, surv).view(ns, 3), _gather(dc.p0, 1, surv), _gather(dc.a0, 1, surv)
    free = _gather(state._free, 1, surv)
    m = {"p0": _gather(state._m["p0"], 1, surv), "a0": _gather(state._m["a0"], 1, surv),
         "position": _gather(state._m["position"], 3, surv).view(ns, 3)}
    v = {"p0": _gather(state._v["p0"], 1, surv), "a0": _gather(state._v["a0"], 1, surv),
         "position": _gather(state._v["position"], 3, surv).view(ns, 3)}
    gnorm = None
    if state._last is not None and ns:
        gnorm = f64(ns)
        call("pab_row_norms", ptr(state._last.d_pos_t), ptr(surv), ns, ptr(gnorm), E._stream())

    # split: a0 > split_a0 -> two children
    skey = f64(max(ns, 1))[:ns]
    if ns:
        call("pab_density_split_key", ptr(a0), ns, float(thresholds.split_a0), ptr(skey), E._stream())
    S = _compact_indices(skey, 0)
    K = _compact_indices(skey, 3)
    nS, nK = S.numel(), K.numel()
    par_pos, par_p0, par_a0 = _gather(pos, 3, K).view(nK, 3), _gather(p0, 1, K), _gather(a0, 1, K)
    par_free = _gather(free, 1, K)
    parts_pos, parts_p0, parts_a0, parts_free = [par_pos], [par_p0], [par_a0], [par_free]
    if nS:
        unit = up(rng.unit_vectors(nS))
        cpos, cp0, ca0 = f64(2 * nS * 3), f64(2 * nS), f64(2 * nS)
        # bind gathered operands to names: a temporary freed right after ptr()
        # would be recycled by the caching allocator before the kernel runs
        s_pos, s_p0, s_a0 = _gather(pos, 3, S), _gather(p0, 1, S), _gather(a0, 1, S)
        call("pab_split_children", ptr(s_pos), ptr(s_p0), ptr(s_a0), ptr(unit), nS, ptr(cpos), ptr(cp0),
             ptr(ca0), E._stream())
        sfree = _gather(free, 1, S)
        parts_pos.append(cpos.view(2 * nS, 3))
        parts_p0.append(cp0)
        parts_a0.append(ca0)
        parts_free.append(torch.cat([sfree, sfree]))

    # duplicate (fine): top ceil((1 - q) n_live) by |grad pos|, ties by index
    if stage == "fine" and gnorm is not None and nK:
        gn = _gather(gnorm, 1, K)
        k_dup = min(math.ceil((1.0 - thresholds.duplicate_grad_quantile) * nK), nK)
        if k_dup > 0:
            t = f64(1)
            _select(gn, nK - k_dup, t)
            dkey = f64(nK)
            call("pab_density_dup_key", ptr(gn), nK, ptr(t), ptr(dkey), E._stream())
            above = _compact_indices(dkey, 0)
            ties = _compact_indices(dkey, 4)
            cnt = torch.tensor([ties.numel(), above.numel()], dtype=torch.int32, device=dev)
            call("pab_density_take_ties", ptr(ties), ptr(cnt[0:1]), ptr(cnt[1:2]), int(k_dup), nK, ptr(dkey),
                 E._stream())
            order = _compact_indices(dkey, 0)
            unit = up(rng.unit_vectors(order.numel()))
            k = order.numel()
            dpos, dp0, da0 = f64(3 * k), f64(k), f64(k)
            o_pos, o_p0, o_a0 = _gather(par_pos, 3, order), _gather(par_p0, 1, order), _gather(par_a0, 1, order)
            call("pab_duplicate", ptr(o_pos), ptr(o_p0), ptr(o_a0), ptr(unit), k, ptr(dpos), ptr(dp0), ptr(da0),
                 E._stream())
            parts_pos.append(dpos.view(k, 3))
            parts_p0.append(dp0)
            parts_a0.append(da0)
            parts_free.append(_gather(par_free, 1, order))

    new_pos = torch.cat(parts_pos).contiguous()
    n_new = new_pos.shape[0]
    state._dc = E.DeviceCloud(new_pos, torch.cat(parts_p0), torch.cat(parts_a0))
    state._free = torch.cat(parts_free)
    for src, dst in ((m, state._m), (v, state._v)):
        for key_ in _KEYS:
            kept = _gather(src[key_], 3 if key_ == "position" else 1, K)
            shape = (n_new, 3) if key_ == "position" else (n_new,)
            z = torch.zeros(shape, dtype=torch.float64, device=dev)
            z[:nK] = kept.view(nK, 3) if key_ == "position" else kept
            dst[key_] = z
    state._generation += 1
    state._host_cache = None
    state._last = None
    return state


# ---------------------------------------------------------------------------
# Hierarchical driver (optimizer.py:414-500)
# ---------------------------------------------------------------------------


@dataclass
class TraceRecord:
    step: int
    time_s: float
    loss: float
    ball_count: int
    level: int


@dataclass
class IterationTrace:
    records: list = field(default_factory=list)

    def record(self, step: int, time_s: float, loss: float, ball_count: int, level: int) -> None:
        if self.records and step <= self.records[-1].step:
            raise ValueError("trace steps must increase monotonically")
        self.records.append(TraceRecord(step, time_s, loss, ball_count, level))

    def to_csv(self, path) -> None:
        with open(path, "w", encoding="utf-8") as fh:
            fh.write("step,time_s,loss,ball_count,level\n")
            for r in self.records:
                fh.write(f"{r.step},{r.time_s:.6f},{r.loss:.12g},{r.ball_count},{r.level}\n")

    @classmethod
    def from_csv(cls, path) -> "IterationTrace":
        trace = cls()
        with open(path, "r", encoding="utf-8") as fh:
            header = fh.readline().strip()
            if header != "step,time_s,loss,ball_count,level":
                raise ValueError(f"unexpected trace header: {header!r}")
            for line in fh:
                s, t, l, b, lv = line.strip().split(",")
                trace.record(int(s), float(t), float(l), int(b), int(lv))
        return trace


def _filter_state_(state: OptimState, det, acq, real_local, strict: bool = True) -> None:
    """Builder-defined periodic filter (config 3): reference predicate
    (optimizer.py:230-258) on the current cloud at the current factor;
    survivors keep their parameters, Adam moments and last gradients.
    Reference equivalent: the ``callback`` of run_hierarchical filtering
    ``state`` in place (tests/golden/make_golden_config3.py)."""
    dc = state._dc
    probe = E.DeviceCloud(dc.pos, torch.zeros_like(dc.p0), dc.a0)
    probe.adopt_order(dc)
    if dc._adj is not None and dc._adj.perm is not None:   # the adjoint's processing order too
        probe.adjoint_cloud().adopt_order(dc._adj)
    counters = E.PassCounters(dc.dev)
    g = filter_gradient(probe, det, acq, real_local, counters)
    counters.read()
    idx = _compact_indices(g, 0 if strict else 1)
    m = idx.numel()
    if m == state.n:
        return
    ws_gather = lambda src, width: _gather(src, width, idx)
    new = E.DeviceCloud(ws_gather(dc.pos, 3).view(m, 3), ws_gather(dc.p0, 1), ws_gather(dc.a0, 1))
    state._dc = new
    for d in (state._m, state._v):
        d["p0"] = ws_gather(d["p0"], 1)
        d["a0"] = ws_gather(d["a0"], 1)
        d["position"] = ws_gather(d["position"], 3).view(m, 3)
    state._free = ws_gather(state._free, 1)
    state._host_cache = None
    last = state._last   # survivors keep their last gradients: a density-control step right after the
    #                      filter still ranks duplicates by |grad position|
    if last is not None:
        state._last = _DeviceGrads(ws_gather(last.d_p0_t, 1), ws_gather(last.d_a0_t, 1),
                                   ws_gather(last.d_pos_t, 3).view(m, 3))


def _gather(src: torch.Tensor, width: int, idx: torch.Tensor) -> torch.Tensor:
    m = idx.numel()
    out = torch.empty(m * width, dtype=torch.float64, device=src.device)
    call("pab_gather_f64", ptr(src.contiguous()), width, ptr(idx), m, ptr(out), E._stream())
    return out


def run_hierarchical(init: PointCloud, ctx, real, schedule: Schedule, thresholds: DensityThresholds, *,
                     lr: LearningRates | None = None, seed=0, callback=None, state: OptimState | None = None,
                     filter_every: int | None = None, plateau: bool = True):
    """Every schedule level in order on progressively finer supervision.

    Extensions (off by default = reference behaviour): ``filter_every`` applies
    the zero-gradient filter to the live cloud every k iterations (BASELINE
    config 3); ``plateau=False`` disables the 50-iteration plateau stop.
    """
    if state is None:
        state = create_state(init.copy(), lr=lr, seed=seed)
    trace = IterationTrace()
    t_start = time.perf_counter()
    det = R.device_detectors(ctx)
    full = R.device_supervision(real.data, det)
    global_step = 0
    for li, level in enumerate(schedule.levels):
        if state.n == 0:
            raise OptimizationError("all points destroyed")
        acq = R._acq(ctx, level.f)
        real_local = full if level.f == 1 else E.decimate_rows(full, level.f)
        period = _COARSE_DENSITY_EVERY if level.stage == "coarse" else schedule.duplication_period
        losses = []
        for it in range(level.max_iters):
            loss_value = _device_step(state, det, acq, real_local, level.stage)
            global_step += 1
            losses.append(loss_value)
            trace.record(global_step, time.perf_counter() - t_start, loss_value, state.n, li)
            if callback is not None:
                callback(state, global_step, li, loss_value)
            if filter_every and (it + 1) % filter_every == 0:
                _filter_state_(state, det, acq, real_local)
                if state.n == 0:
                    raise OptimizationError("all points destroyed")
            if (it + 1) % period == 0:
                state = density_control(state, thresholds, level.stage)
                if state.n == 0:
                    raise OptimizationError("all points destroyed")
            if plateau and len(losses) > _PLATEAU_WINDOW:
                past = losses[-1 - _PLATEAU_WINDOW]
                if abs(past - loss_value) < _PLATEAU_REL * max(abs(past), 1e-300):
                    break
    return state.cloud, trace


# ---------------------------------------------------------------------------
# Positivity-constrained refinement (optimizer.py:507-573), SURVEY §8f rank 3
# ---------------------------------------------------------------------------


def softplus(x: np.ndarray) -> np.ndarray:
    """log(1 + exp(x)) with the overflow-safe split form; always > 0
    (optimizer.py:507-510).  Host helper of the API; the refinement loop
    evaluates it on the device (``pab_softplus_f64``)."""
    x = np.asarray(x, dtype=np.float64)
    return np.log1p(np.exp(-np.abs(x))) + np.maximum(x, 0.0)


def inv_softplus(y: np.ndarray) -> np.ndarray:
    """Preimage of softplus for y > 0, accurate over many decades
    (optimizer.py:513-523)."""
    y = np.asarray(y, dtype=np.float64)
    if np.any(y <= 0.0):
        raise ValueError("inv_softplus requires strictly positive input")
    small = y < 0.7
    out = np.empty_like(y)
    out[small] = np.log(np.expm1(y[small]))
    big = ~small
    out[big] = y[big] + np.log1p(-np.exp(-y[big]))
    return out


def sigmoid(x: np.ndarray) -> np.ndarray:
    """Logistic function split by sign (optimizer.py:526-533)."""
    x = np.asarray(x, dtype=np.float64)
    pos = x >= 0.0
    out = np.empty_like(x)
    out[pos] = 1.0 / (1.0 + np.exp(-x[pos]))
    ex = np.exp(x[~pos])
    out[~pos] = ex / (1.0 + ex)
    return out


def positivity_refine(state: OptimState, ctx, real, iters: int) -> PointCloud:
    """Final fit with a0 = softplus(a0_free), density control frozen
    (optimizer.py:536-573): fresh moments, fine backward at the native rate,
    Adam on p0, a0_free (gradient d_a0 * sigmoid(a0_free)) and positions, no
    a0 floor.  The whole loop stays on the device; the entry preimage is
    taken on the host as in the reference."""
    cloud = state.cloud
    if len(cloud) and np.any(cloud.a0 <= 0.0):
        raise ValueError("positivity refinement requires a0 > 0 at entry")
    free_h = inv_softplus(cloud.a0) if len(cloud) else np.empty(0)
    refine = create_state(cloud, lr=state.lr, seed=state.seed)
    dc = refine._dc
    n = dc.n
    if n == 0 or int(iters) <= 0:
        out = PointCloud(cloud.positions.copy(), cloud.p0.copy(),
                         softplus(free_h) if n else cloud.a0.copy(), free_h.copy(), cloud.generation)
        state.cloud = out
        return out
    free = torch.from_numpy(np.ascontiguousarray(free_h)).to(dc.dev)
    g_free = torch.empty_like(free)
    det = R.device_detectors(ctx)
    acq = R._acq(ctx, 1)
    real_local = R.device_supervision(real.data, det)
    n_total = det.n_total * acq.n_out
    s = E._stream()
    for _ in range(int(iters)):
        call("pab_softplus_f64", ptr(free), n, ptr(dc.a0), s)
        dc.invalidate()
        counters = E.PassCounters(dc.dev)
        res, loss_rows = E.forward_rows(dc, det, acq, counters, real_local=real_local)
        d_p0, d_a0, d_pos = E.adjoint_grads(dc, det, acq, res, 1.0, 2, 2.0 / n_total, counters,
                                            loss_rows=loss_rows)
        loss_sum, ops = counters.result(check_nonfinite=False)
        loss_value = loss_sum / n_total
        if not math.isfinite(loss_value):
            raise OptimizationError(f"non-finite loss during refinement: {loss_value}")
        R._add_ops(ops)
        refine.step_count += 1
        t = refine.step_count
        _adam_(dc.p0, d_p0, refine._m["p0"], refine._v["p0"], refine.lr.p0, t)
        call("pab_mul_sigmoid_f64", ptr(d_a0), ptr(free), n, ptr(g_free), s)
        _adam_(free, g_free, refine._m["a0"], refine._v["a0"], refine.lr.a0, t)
        _adam_(dc.pos, d_pos, refine._m["position"], refine._v["position"], refine.lr.position, t)
    call("pab_softplus_f64", ptr(free), n, ptr(dc.a0), s)
    out = PointCloud(dc.pos.cpu().numpy(), dc.p0.cpu().numpy(), dc.a0.cpu().numpy(), free.cpu().numpy(),
                     cloud.generation)
    state.cloud = out
    return out
