"""Device-resident state and launch orchestration for the forward/adjoint path.

PyTorch is used for device memory, streams and ``torch.distributed``; all
arithmetic on the path runs in the sm_100a library (``_lib``).

Multi-GPU: one process per GPU, detectors sharded in
contiguous blocks; the ball cloud, its Adam state and every per-ball decision
are replicated.  The forward is detector-local; the one exchange per
iteration is the all-reduce (NCCL) of the per-ball gradient buffer, whose
tail carries the loss, the error flags and the op count.
"""

from __future__ import annotations

import os

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import call, ptr
from .model import OptimizationError, SimulationError
from .parallel import TAIL, Shard, allreduce_sum_, current_shard, gather_rows, read_tail  # noqa: F401


FORWARD_WARPS = int(os.environ.get("PAB_FWD_WARPS", "4"))   # 2 CTAs per SM: one sorts while the other sweeps
FORWARD_TILE_ROWS = 160   # reserved ABI argument (the library's tile height is a build constant)
ADJOINT_WARPS = int(os.environ.get("PAB_ADJ_WARPS", "1"))   # = PAB_ADJ_WARPS of the library build
GROUP = 32
A0_BUCKETS = int(os.environ.get("PAB_A0_BUCKETS", "6"))   # lane groups hold balls of similar radius (equal window lengths)
# the adjoint walks each ball's own window (no tile, no pairing): it prefers
# narrower radius buckets than the forward, so it runs on its own packing of
# the same cloud (measured adjoint at config 2: 6 / 8 / 10 / 16 buckets ->
# 20.19 / 20.02 / 19.87 / 19.75 ms)
ADJ_A0_BUCKETS = int(os.environ.get("PAB_ADJ_A0_BUCKETS", "16"))
GROUP_META_BYTES = 48


def cuda_device() -> torch.device:
    if not torch.cuda.is_available():
        raise _lib.LibraryError("a CUDA device is required: this package has no CPU path")
    _lib.load()
    return torch.device("cuda", torch.cuda.current_device())


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


_SM_COUNT: dict = {}


def sm_count(dev: torch.device) -> int:
    if dev.index not in _SM_COUNT:
        _SM_COUNT[dev.index] = torch.cuda.get_device_properties(dev).multi_processor_count
    return _SM_COUNT[dev.index]


# ---------------------------------------------------------------------------
# Acquisition / directivity parameters of one call
# ---------------------------------------------------------------------------

DIR_CODES = {"none": 0, "cos_power": 1, "element": 2}


MAX_RECORD_SAMPLES = 1 << 21   # = kMaxRecordSamples (csrc/pab_common.cuh)
# groups wider than the forward's tile listed per detector x partition for the
# wide-group kernel (more: it scans for them itself); 1 KB per CTA
WIDE_CAP = int(os.environ.get("PAB_WIDE_CAP", "255"))


@dataclass(frozen=True)
class Acq:
    v: float
    t0: float
    dt: float            # full-rate grid
    n_samples: int       # full-rate count
    f: int
    cutoff: float
    dir_kind: int
    dir_param: float

    @property
    def n_out(self) -> int:
        return -(-self.n_samples // self.f) if self.f > 1 else self.n_samples

    def __post_init__(self) -> None:
        # the kernels round sample indices with FP32 magic constants (exact
        # below 2^22; include/paball_b200.h): records up to 2^21 full-rate
        # samples (52 ms at 40 MHz)
        if self.n_out * self.f > MAX_RECORD_SAMPLES:
            raise ValueError(f"record of {self.n_out * self.f} full-rate samples exceeds the supported "
                             f"{MAX_RECORD_SAMPLES}")


def detector_aux(positions: np.ndarray, normals, directivity) -> np.ndarray:
    """[J, 9]: receive direction (-outward normal), element axes e1, e2."""
    J = positions.shape[0]
    aux = np.zeros((J, 9))
    if directivity.kind == "none":
        return aux
    if normals is None:
        raise ValueError(f"directivity {directivity.kind!r} needs SensorArray.normals")
    face = -np.asarray(normals, dtype=np.float64)
    face /= np.linalg.norm(face, axis=1, keepdims=True)
    aux[:, 0:3] = face
    ref = np.zeros_like(face)
    ref[:, 0] = 1.0
    ref[np.abs(face[:, 0]) > 0.9] = [0.0, 1.0, 0.0]
    e1 = ref - np.sum(ref * face, axis=1, keepdims=True) * face
    e1 /= np.linalg.norm(e1, axis=1, keepdims=True)
    aux[:, 3:6] = e1
    aux[:, 6:9] = np.cross(face, e1)
    return aux


class DeviceDetectors:
    """This rank's contiguous block of detectors, resident on the GPU."""

    def __init__(self, positions: np.ndarray, normals, directivity, sound_speed: float,
                 dev: torch.device, shard: Shard):
        positions = np.asarray(positions, dtype=np.float64).reshape(-1, 3)
        self.n_total = positions.shape[0]
        self.shard = shard
        lo, hi = shard.range(self.n_total)
        self.lo, self.hi = lo, hi
        self.n_local = hi - lo
        aux = detector_aux(positions, normals, directivity)
        self.pos = torch.from_numpy(np.ascontiguousarray(positions[lo:hi])).to(dev)
        self.aux = torch.from_numpy(np.ascontiguousarray(aux[lo:hi])).to(dev)
        self.sound_speed = float(sound_speed)


# ---------------------------------------------------------------------------
# Ball cloud on device
# ---------------------------------------------------------------------------


class DeviceCloud:
    """FP64 SoA cloud in caller order plus packed processing-order records."""

    def __init__(self, pos: torch.Tensor, p0: torch.Tensor, a0: torch.Tensor, buckets: int | None = None):
        self.dev = pos.device
        self.pos = pos.contiguous()
        self.p0 = p0.contiguous()
        self.a0 = a0.contiguous()
        self.buckets = A0_BUCKETS if buckets is None else buckets
        self.perm = None    # processing (sorted) order
        self.slots = None   # lane-group slots of the order: ball index or -1 (padding)
        self._ng = None
        self._packed = False
        self._adj = None

    def adopt_order(self, other: "DeviceCloud") -> None:
        """Use another cloud's processing order and lane groups (same balls)."""
        self.perm, self.slots, self._ng = other.perm, other.slots, other._ng

    def adjoint_cloud(self) -> "DeviceCloud":
        """The same balls (shared parameter tensors) packed for the adjoint
        with ADJ_A0_BUCKETS radius buckets; follows this cloud's
        invalidations.  With equal bucket counts it is this cloud."""
        if ADJ_A0_BUCKETS == self.buckets:
            return self
        if self._adj is None or self._adj.pos is not self.pos or self._adj.p0 is not self.p0 \
                or self._adj.a0 is not self.a0:
            self._adj = DeviceCloud(self.pos, self.p0, self.a0, buckets=ADJ_A0_BUCKETS)
        return self._adj

    @classmethod
    def from_host(cls, positions, p0, a0, dev) -> "DeviceCloud":
        """Upload caller arrays (FP64 numpy) as one contiguous device buffer
        through the page-locked staging slot (hostio: streaming-store host
        copy overlapped with the DMA), on the current stream."""
        from . import hostio
        (pos_d, p0_d, a0_d), _ = hostio.stager("cloud").upload(
            [(np.asarray(positions).reshape(-1, 3), torch.float64), (p0, torch.float64), (a0, torch.float64)], dev)
        return cls(pos_d, p0_d, a0_d)

    @property
    def n(self) -> int:
        return int(self.p0.shape[0])

    @property
    def n_groups(self) -> int:
        return self._ng if self._ng is not None else (self.n + GROUP - 1) // GROUP

    def invalidate(self, resort: bool = False) -> None:
        """Parameters changed: repack before the next pass (and resort)."""
        self._packed = False
        if self._adj is not None:
            self._adj.invalidate(resort)
        if resort:
            self.perm = self.slots = self._ng = None

    def sort(self) -> None:
        """Processing order on the device, no host round trip: cloud bounds,
        (a0 bucket, Hilbert) keys, stable radix sort -> perm; lane group g
        holds balls perm[32 g .. 32 g + 31].  (Measured and rejected this
        round: breaking groups at radius-bucket changes and spatial jumps
        (padded segments) and log2-spaced radius buckets were slower on
        config 2 and on the config-3 reconstruction at every setting.)"""
        n = self.n
        self._ptable_ok = False   # new units: rebuild the pairing table
        if n == 0:
            self.perm = self.slots = torch.empty(0, dtype=torch.int32, device=self.dev)
            self._ng = 0
            return
        ws = workspace(self.dev)
        lib = _lib.load()
        # scratch per bucket count: the forward's and the adjoint's packings
        # of one cloud may sort concurrently on two streams (_run_model)
        b = self.buckets
        bounds = ws.get(f"cloud_bounds{b}", 8, torch.float64)
        bws = ws.get(f"cloud_bounds_ws{b}", int(lib.pab_cloud_bounds_workspace_bytes()) // 8 + 1, torch.float64)
        keys = ws.get(f"sort_keys{b}", n, torch.int64)
        sws = ws.get(f"sort_ws{b}", int(lib.pab_sort_perm_workspace_bytes(n)) // 8 + 1, torch.int64)
        self.perm = torch.empty(n, dtype=torch.int32, device=self.dev)
        call("pab_cloud_bounds", ptr(self.pos), ptr(self.a0), n, ptr(bounds), ptr(bws), _stream())
        call("pab_sort_keys", ptr(self.pos), ptr(self.a0), n, ptr(bounds), self.buckets, ptr(keys), _stream())
        call("pab_sort_perm", ptr(keys), n, ptr(self.perm), ptr(sws), _stream())
        self.slots, self._ng = self.perm, (n + GROUP - 1) // GROUP

    def pack(self) -> None:
        if self._packed:
            return
        if self.perm is None or self.perm.shape[0] != self.n or self.slots is None:
            self.sort()
        ng = self.n_groups
        npad = ng * GROUP
        if not hasattr(self, "rec_a") or self.rec_a.numel() < npad * 16:
            self.rec_a = torch.empty(npad * 16, dtype=torch.uint8, device=self.dev)
            self.rec_b = torch.empty(npad * 16, dtype=torch.uint8, device=self.dev)
            self.gmeta = torch.empty(max(ng, 1) * GROUP_META_BYTES, dtype=torch.uint8, device=self.dev)
        if self.n:
            call("pab_pack", ptr(self.pos), ptr(self.p0), ptr(self.a0), ptr(self.slots), self.slots.numel(),
                 ptr(self.rec_a), ptr(self.rec_b), ptr(self.gmeta), _stream())
        self._packed = True

    def pack_async(self, stream: torch.cuda.Stream) -> torch.cuda.Event:
        """Sort and pack on ``stream`` (after the work queued so far on the
        current stream, e.g. the cloud upload); returns the event the
        consumer's stream waits on.  The packed tensors are marked as used by
        the current stream too (caching-allocator safety)."""
        main = torch.cuda.current_stream(self.dev)
        stream.wait_stream(main)
        with torch.cuda.stream(stream):
            self.pack()
        for t in (self.perm, self.rec_a, self.rec_b, self.gmeta):
            if t is not None:
                t.record_stream(main)
        ev = torch.cuda.Event()
        ev.record(stream)
        return ev

    def pair_table(self) -> torch.Tensor:
        """Dual-walk pairing table: which two balls of a 64-ball unit a lane
        walks together, per direction cell.  Built on first use after each
        sort (unit membership follows the processing order); repacks with
        moved balls keep it, like the sort order itself: any pairing gives
        the same sums up to FP32 rounding, a slightly stale one only walks a
        little more."""
        if not getattr(self, "_ptable_ok", False):
            nbytes = int(_lib.load().pab_pair_table_bytes(self.n_groups))
            if not hasattr(self, "ptable") or self.ptable.numel() < max(nbytes, 1):
                self.ptable = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=self.dev)
            if self.n:
                call("pab_pair_table", ptr(self.rec_a), ptr(self.gmeta), self.n_groups, ptr(self.ptable), _stream())
            self._ptable_ok = True
        return self.ptable

# ---------------------------------------------------------------------------
# Workspace and launch planning
# ---------------------------------------------------------------------------


class Workspace:
    """Grow-only scratch tensors keyed by name."""

    def __init__(self, dev):
        self.dev = dev
        self.bufs: dict = {}

    def get(self, name: str, numel: int, dtype) -> torch.Tensor:
        t = self.bufs.get(name)
        if t is None or t.numel() < numel or t.dtype != dtype:
            t = torch.empty(max(numel, 1), dtype=dtype, device=self.dev)
            self.bufs[name] = t
        return t[:numel]


_WS: dict = {}


def workspace(dev) -> Workspace:
    if dev.index not in _WS:
        _WS[dev.index] = Workspace(dev)
    return _WS[dev.index]


@dataclass
class ForwardPlan:
    groups_per_cell: int
    partitions: int
    warps: int
    tile_rows: int


def plan_forward(cloud: DeviceCloud, det: DeviceDetectors, acq: Acq) -> ForwardPlan:
    """Two CTAs (4 walker + 4 producer warps, ~110-115 KB smem each) per SM:
    detectors x partitions should cover >= 20 waves (measured with the dual
    walk: 2 / 4 / 6 / 12 partitions at config 2 give 21.16 / 21.00 / 20.81 /
    20.76 ms of forward + residual; finer partitions cost residual traffic
    and partial-row memory); each partition keeps >= 4 lane groups per warp."""
    dev = cloud.dev
    tile = FORWARD_TILE_ROWS
    warps = FORWARD_WARPS
    while warps > 1 and _lib.load().pab_forward_smem_bytes(acq.n_out, warps, tile) > 227 * 1024:
        warps -= 1
    target_ctas = 40 * sm_count(dev)   # >= 20 waves of 2 resident CTAs per SM
    parts = max(1, -(-target_ctas // max(det.n_local, 1)))
    parts = int(max(1, min(parts, cloud.n_groups // (4 * warps))))
    parts = int(os.environ.get("PAB_FWD_PARTS", parts))   # tuning override
    return ForwardPlan(0, parts, warps, tile)


ADJ_WAVES = float(os.environ.get("PAB_ADJ_WAVES", "16"))


def plan_adjoint(cloud: DeviceCloud, det: DeviceDetectors) -> int:
    """Detector chunks: at least ADJ_WAVES waves of 16 resident warps per SM
    and at most 256 detectors per chunk (finer tail; measured at config 2: 1 /
    2 / 4 / 8 chunks give 20.41 / 20.28 / 20.19 / 20.19 ms), with the FP64
    partial sums (40 B per ball and chunk) kept under 2 GiB.  Lane groups of
    different radius buckets differ 4x in work, so small clouds need many
    waves for balance: the config-3 reconstruction (4.7k-14k groups x 512
    detectors) takes 3.04 / 2.81 / 2.57 / 2.35 / 2.45 s at 2 / 4 / 8 / 16 /
    32 waves; config 2 (31k groups, 4 chunks by the detector bound) is
    unchanged."""
    ctas = -(-cloud.n_groups // ADJOINT_WARPS)
    target = int(ADJ_WAVES * 16 * sm_count(cloud.dev)) // ADJOINT_WARPS   # waves of 16 resident warps per SM
    chunks = max(1, -(-target // max(ctas, 1)), -(-det.n_local // 256))
    cap = max(1, (2 << 30) // max(40 * cloud.n_groups * GROUP, 1))
    chunks = int(max(1, min(chunks, cap, max(1, det.n_local // 16))))
    return int(os.environ.get("PAB_ADJ_CHUNKS", chunks))   # tuning override


# ---------------------------------------------------------------------------
# Passes
# ---------------------------------------------------------------------------


# Every gradient buffer ends in the pass tail (parallel.TAIL doubles, written
# by pab_pass_tail): loss sum, coincident flag, non-finite flag, op count.  It
# rides in the same all-reduce as the per-ball gradients: one collective per
# iteration, and every rank sees the same loss, error flags and op count (so
# every rank raises the same error at the same step).


class PassCounters:
    """Device op counter + status word for one API call, reduced over ranks
    through the pass tail."""

    def __init__(self, dev):
        ws = workspace(dev)
        self.dev = dev
        self.ops = ws.get("ops", 1, torch.int64)
        self.status = ws.get("status", 1, torch.int32)
        self.ops.zero_()
        self.status.zero_()
        self.tail = None   # device tail of this pass (after the all-reduce)
        self._host_tail = None

    def close(self, loss_rows: torch.Tensor | None = None, tail: torch.Tensor | None = None) -> torch.Tensor:
        """Write this rank's pass tail (device) from its loss rows, status
        word and op counter."""
        if tail is None:
            tail = workspace(self.dev).get("tail", TAIL, torch.float64)
        n_rows = 0 if loss_rows is None else int(loss_rows.numel())
        call("pab_pass_tail", ptr(loss_rows) if n_rows else None, n_rows, ptr(self.ops), ptr(self.status),
             ptr(tail), _stream())
        return tail

    def result(self, host_tail=None, check_nonfinite: bool = True) -> tuple[float, int]:
        """(loss sum, op count) of the pass summed over ranks; raises the
        reference's error classes, identically on every rank.  A pass
        without an adjoint (forward only) reduces its tail here."""
        loss_sum, coincident, nonfinite, ops = read_tail(self._host(host_tail))
        if coincident:
            raise SimulationError("ball coincident with a sensor (zero source-sensor distance)")
        if check_nonfinite and nonfinite:
            raise OptimizationError("non-finite gradient")
        return loss_sum, ops

    def _host(self, host_tail=None):
        if host_tail is None:
            if self._host_tail is not None:
                return self._host_tail
            if self.tail is None:
                t = self.close()
                if current_shard().world > 1:
                    allreduce_sum_(t)
                self.tail = t
            host_tail = self.tail.cpu().numpy()
        self._host_tail = host_tail
        return host_tail

    def tail_flags(self) -> tuple[bool, bool]:
        """(coincident, non-finite) of the reduced pass tail."""
        _, coincident, nonfinite, _ = read_tail(self._host())
        return coincident, nonfinite

    def read(self) -> int:
        return self.result()[1]


# bench hook: {"residual" | "finalize": [start, end] CUDA events} recorded on the
# launching stream around those HBM-bound kernels (None: no events)
TIMING = None


def _mark(name: str, i: int) -> None:
    if TIMING is not None and name in TIMING:
        TIMING[name][i].record(torch.cuda.current_stream())


def check_coincident(cloud: DeviceCloud, det: DeviceDetectors, counters: PassCounters) -> None:
    """Exact FP64 ball-on-sensor test (reference radiator.py:189-193) into
    the pass's status word."""
    if cloud.n_groups and det.n_local:
        call("pab_coincident", ptr(cloud.rec_b), ptr(cloud.gmeta), cloud.n_groups, ptr(cloud.pos), ptr(det.pos),
             det.n_local, ptr(counters.status), _stream())


def forward_rows(cloud: DeviceCloud, det: DeviceDetectors, acq: Acq, counters: PassCounters,
                 real_local: torch.Tensor | None = None, out: torch.Tensor | None = None,
                 real_ready: torch.cuda.Event | None = None):
    """Simulate this rank's rows.  With ``real_local`` the result is the
    residual sim - real and the per-row FP64 sum of squares is returned
    (``real_ready``: event the supervision upload records; only the residual
    epilogue waits for it, the forward kernel overlaps the copy).
    ``real_local`` may also be a callable returning (tensor, event): it is
    called right after the forward kernel is queued, so a host-side upload
    of the supervision runs while the GPU simulates.
    Returns (out [J_local, n_out] f32, loss_rows [J_local] f64 or None)."""
    ws = workspace(cloud.dev)
    n_out = acq.n_out
    J = det.n_local
    if out is None:
        out = torch.empty((J, n_out), dtype=torch.float32, device=cloud.dev)
    if J == 0:
        return out, (torch.zeros(0, dtype=torch.float64, device=cloud.dev) if real_local is not None else None)
    cloud.pack()
    check_coincident(cloud, det, counters)
    plan = plan_forward(cloud, det, acq)
    partial = ws.get("partial_rows", plan.partitions * J * n_out, torch.float32)
    loss_rows = ws.get("loss_rows", J, torch.float64) if real_local is not None else None
    if cloud.n_groups > 0:
        # the dual walk (pairing table) at the native rate (measured on the config-3 reconstruction: single
        # walks at f >= 2 are 2 % faster; windows of 8-17 samples); PAB_FORWARD_DUAL=0: single walks only
        dual = os.environ.get("PAB_FORWARD_DUAL", "1") != "0" and acq.f <= int(os.environ.get("PAB_FORWARD_DUAL_MAXF", "1"))
        ptab = ptr(cloud.pair_table()) if dual else None
        wide = ws.get("wide_list", plan.partitions * J * (WIDE_CAP + 1), torch.int32)
        call("pab_forward", ptr(cloud.rec_a), ptr(cloud.rec_b), ptr(cloud.gmeta), ptab,
             cloud.n_groups,
             ptr(det.pos), ptr(det.aux), J, det.sound_speed, acq.t0, acq.dt, acq.f, n_out, acq.cutoff,
             acq.dir_kind, acq.dir_param, plan.groups_per_cell, plan.partitions, plan.warps,
             plan.tile_rows, ptr(partial), ptr(wide), WIDE_CAP, ptr(counters.ops), ptr(counters.status), _stream())
    else:
        partial.zero_()
    if callable(real_local):
        real_local, real_ready = real_local()
    if real_ready is not None:
        torch.cuda.current_stream(cloud.dev).wait_event(real_ready)
    _mark("residual", 0)
    call("pab_residual", ptr(partial), plan.partitions, J, n_out, ptr(real_local), ptr(out),
         ptr(loss_rows), _stream())
    _mark("residual", 1)
    return out, loss_rows


def adjoint_grads(cloud: DeviceCloud, det: DeviceDetectors, acq: Acq, res: torch.Tensor, res_sign: float,
                  stage: int, scale: float, counters: PassCounters, count_ops: bool = False,
                  flat: torch.Tensor | None = None, loss_rows: torch.Tensor | None = None):
    """Per-ball loss gradients in caller order (FP64), reduced over ranks.
    stage: 0 filter (d_p0 only), 1 coarse, 2 fine.  The three fields are
    views of one contiguous buffer ``flat`` ([n] for stage 0, [5n] otherwise,
    then the TAIL-double pass tail with this pass's loss (``loss_rows``),
    error flags and op count; allocated when not given): one all-reduce,
    one host copy.  ``counters.tail`` is the reduced tail."""
    dev = cloud.dev
    n = cloud.n
    width = 1 if stage == 0 else 5
    if flat is None:
        flat = torch.zeros(width * n + TAIL, dtype=torch.float64, device=dev)
    else:
        flat = flat[: width * n + TAIL]
        flat.zero_()
    d_p0 = flat[:n]
    d_a0 = flat[n:2 * n] if stage >= 1 else None
    d_pos = flat[2 * n:5 * n].view(n, 3) if stage >= 1 else None
    tail = flat[width * n:]
    if n > 0 and det.n_local > 0:
        cloud = cloud.adjoint_cloud()   # the adjoint's own packing (radius buckets)
        cloud.pack()
        if stage == 0:   # the filter pass runs no forward
            check_coincident(cloud, det, counters)
        chunks = plan_adjoint(cloud, det)
        ws = workspace(dev)
        npad = cloud.n_groups * GROUP
        gpart = ws.get("grad_partial", chunks * 5 * npad, torch.float64)
        call("pab_adjoint", ptr(cloud.rec_a), ptr(cloud.rec_b), ptr(cloud.gmeta), cloud.n_groups,
             ptr(det.pos), ptr(det.aux), det.n_local, det.sound_speed, acq.t0, acq.dt, acq.f, acq.n_out,
             acq.cutoff, acq.dir_kind, acq.dir_param, ptr(res), float(res_sign), int(stage), chunks,
             ADJOINT_WARPS, ptr(gpart), ptr(counters.ops) if count_ops else None, ptr(counters.status),
             _stream())
        _mark("finalize", 0)
        call("pab_grad_finalize", ptr(gpart), chunks, cloud.n_groups, ptr(cloud.rec_b), float(scale), int(stage),
             ptr(d_p0), ptr(d_a0), ptr(d_pos), ptr(counters.status), _stream())
        _mark("finalize", 1)
        if TIMING is not None:
            TIMING["finalize_bytes"] = chunks * 5 * npad * 8 + npad * 16 + 5 * n * 8
    counters.close(loss_rows, tail)
    if det.shard.world > 1:
        allreduce_sum_(flat)   # gradients + loss + flags + ops: the iteration's one collective
    counters.tail = tail
    return d_p0, d_a0, d_pos


def decimate_rows(src: torch.Tensor, f: int) -> torch.Tensor:
    rows, n_in = src.shape
    n_out = -(-n_in // f)
    dst = torch.empty((rows, n_out), dtype=torch.float32, device=src.device)
    call("pab_decimate", ptr(src), rows, n_in, f, ptr(dst), _stream())
    return dst


def full_rows(local: torch.Tensor, det: DeviceDetectors) -> torch.Tensor:
    """All ranks' rows (rank order) for API results."""
    if det.shard.world == 1:
        return local
    return gather_rows(local, det.n_total)


def current_shard_for(dev) -> Shard:
    return current_shard()


def sumsq_diff(a: torch.Tensor, b: torch.Tensor | None) -> float:
    """sum (a - b)^2 over FP64 device tensors (deterministic order)."""
    ws = workspace(a.device)
    n = a.numel()
    scratch = ws.get("ssd", int(_lib.load().pab_sumsq_workspace_bytes(n)) // 8 + 1, torch.float64)
    out = ws.get("ssd_out", 1, torch.float64)
    call("pab_sumsq_diff_f64", ptr(a), ptr(b), n, ptr(out), ptr(scratch), _stream())
    return float(out.item())


def mse_device(sim: np.ndarray, real: np.ndarray) -> float:
    dev = cuda_device()
    a = torch.from_numpy(np.ascontiguousarray(sim)).to(dev)
    b = torch.from_numpy(np.ascontiguousarray(real)).to(dev)
    return sumsq_diff(a, b) / a.numel()
