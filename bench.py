"""Benchmark of the forward + adjoint hot path (BASELINE.json metric).

Workload: BASELINE config 2 ("microbench"): 1,000,000 balls uniform in a
20 mm cube, a0 ~ U[0.05, 0.2] mm, 1024 detectors on a jittered ellipsoid cap
with cos^2 directivity, 40 MHz x 4096 samples; seeded synthetic inputs
(paper_2601_00551_b200.scenes).  One step = one fine backward pass = forward
rows + residual/loss + adjoint + gradient finalisation (+ NCCL all-reduce of
the per-ball gradients for N > 1).  Metric: ball-detector pair evaluations
per second, pairs = N_balls x N_detectors per step.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Each rank owns a contiguous detector block (strong scaling: the
configuration is fixed, the per-GPU work shrinks as 1/N); the step's one
collective is the NCCL all-reduce of the per-ball gradient buffer, whose
tail carries the loss, error flags and op count.  ``--gpus N`` without a
torchrun environment re-launches itself under ``torch.distributed.run``
with N ranks (NCCL, one GPU per rank).  With fewer GPUs than ranks the
ranks share the GPUs over a gloo group ("oversubscribed": the multi-rank
code path runs, the number is not a scaling measurement).

The default line also carries BASELINE's second metric (``recon``: the
config-3 reconstruction wall time, with the CPU reference's extrapolated
time beside it) and the launch-bound config-1 toy (``config1``).
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ball-detector pair evals/s (fwd+adjoint) per iteration"
UNIT = "pairs/s"
FLOPS_FWD = 7      # per in-window sample
FLOPS_ADJ_FINE = 12
# dram__bytes_read.sum + dram__bytes_write.sum per launch from the latest
# ncu --set full capture of each kernel (profiles/)
TRAFFIC_BYTES = {"forward_kernel": 173_180_416, "adjoint_kernel": 174_639_360}
TRAFFIC_SRC = "profiles/r02_v10_ncu_summary.txt"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, choices=[2, 4, 5], default=2,
                    help="BASELINE config: 2 microbench (default, the headline), 4 planar tilted / element, "
                         "5 mouse-scale (one fwd+fine-adjoint iteration of the 256^3-in-ellipsoid grid cloud)")
    ap.add_argument("--n-balls", type=int, default=None, help="default: 1M (config 2), 4M (config 4)")
    ap.add_argument("--n-det", type=int, default=1024)
    ap.add_argument("--n-samples", type=int, default=4096, help="config 2 only (config 4: 6144)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-balls", type=int, default=50000,
                    help="CPU reference sample: balls (strided subset) x --cpu-det detectors")
    ap.add_argument("--cpu-det", type=int, default=0,
                    help="detectors of the CPU sample (0: 8 per host thread, >= 128: every thread gets a block)")
    ap.add_argument("--cpu-reps", type=int, default=3, help="CPU sample: best of this many runs")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-recon", action="store_true",
                    help="skip the config-3 reconstruction wall time (BASELINE's second metric)")
    ap.add_argument("--no-config1", action="store_true", help="skip the config-1 (launch-bound toy) timing")
    return ap.parse_args()


def make_scene(args):
    """(scene, directivity kwargs for P.Directivity, oracle kind) of the
    selected BASELINE config."""
    from paper_2601_00551_b200 import scenes
    if args.config == 5:
        sc = scenes.mouse_config()
        args.n_balls = len(sc.init)
        args.n_det, args.n_samples = sc.array.positions.shape[0], sc.grid.n_samples
        return sc, dict(kind="cos_power", power=2.0), ("cos_power", 2.0)
    if args.config == 4:
        args.n_balls = args.n_balls or 4_000_000
        args.n_det, args.n_samples = 1024, 6144
        return scenes.planar_config(n_balls=args.n_balls), dict(kind="element", width=0.5e-3), ("element", 0.5e-3)
    args.n_balls = args.n_balls or 1_000_000
    scene = scenes.microbench_config(n_balls=args.n_balls, n_det=args.n_det, n_samples=args.n_samples)
    return scene, dict(kind="cos_power", power=2.0), ("cos_power", 2.0)


def config_dict(args, world):
    if args.config == 5:
        return {"workload": "config5-mouse-scale: one fwd+fine-adjoint iteration of the initial grid cloud",
                "n_balls": args.n_balls, "n_detectors": args.n_det, "n_samples": args.n_samples,
                "sampling_hz": 40e6, "a0_mm": 0.1, "directivity": "cos^2", "parallelism": f"detector-shard x{world}",
                "l2": "inputs larger than L2", "inputs": "device-resident"}
    if args.config == 4:
        return {"workload": "config4-planar-tilted: fwd+fine-adjoint", "n_balls": args.n_balls,
                "n_detectors": 1024, "n_samples": 6144, "sampling_hz": 40e6, "a0_mm": [0.05, 0.2],
                "directivity": "element 0.5 mm", "parallelism": f"detector-shard x{world}",
                "l2": "flushed between timed steps (256 MiB write)", "inputs": "device-resident"}
    return {"workload": "config2-microbench: fwd+fine-adjoint", "n_balls": args.n_balls,
            "n_detectors": args.n_det, "n_samples": args.n_samples, "sampling_hz": 40e6,
            "a0_mm": [0.05, 0.2], "directivity": "cos^2", "parallelism": f"detector-shard x{world}",
            "l2": "flushed between timed steps (256 MiB write)", "inputs": "device-resident"}


# ---------------------------------------------------------------------------
# clocks sampler (B200_PROFILING.md recipe)
# ---------------------------------------------------------------------------

class ClockSampler:
    """SM clock and clock-event (throttle) reasons sampled during the timed
    region.  In-process NVML (the library nvidia-smi reads), initialised and
    sampled once BEFORE the timed region so no process spawn or NVML start-up
    lands inside it; falls back to the nvidia-smi CLI without pynvml."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index: int, dev=None, period: float = 0.05):
        self.index = index
        self.period = period
        self.rows = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)
        self._nv = None
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = None
            if dev is not None:
                try:
                    pr = torch_props(dev)
                    h = nv.nvmlDeviceGetHandleByPciBusId(
                        f"{pr.pci_domain_id:08X}:{pr.pci_bus_id:02X}:{pr.pci_device_id:02X}.0")
                except Exception:
                    h = None
            self._h = h if h is not None else nv.nvmlDeviceGetHandleByIndex(index)
            self._bits = [nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                          nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap]
            self._nv = nv
            self._max = float(nv.nvmlDeviceGetMaxClockInfo(self._h, nv.NVML_CLOCK_SM))
            self._sample()   # warm path, discarded
            self.rows.clear()
        except Exception:
            self._nv = None

    def _sample(self):
        if self._nv is not None:
            nv = self._nv
            sm = float(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
            r = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
            self.rows.append([str(sm), str(self._max)] + ["Active" if r & b else "Not Active" for b in self._bits])
            return
        out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True,
                             timeout=5).stdout.strip()
        if out:
            self.rows.append([x.strip() for x in out.split(",")])

    def _run(self):
        while not self._stop.is_set():
            try:
                self._sample()
            except Exception:
                pass
            self._stop.wait(self.period if self._nv is not None else 0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock sampling unavailable"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        reasons = sorted({self.NAMES[i] for r in self.rows for i in range(4) if r[2 + i].strip() == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows),
                "source": "NVML (in-process)" if self._nv is not None else "nvidia-smi"}


def torch_props(dev):
    import torch
    return torch.cuda.get_device_properties(dev)




# ---------------------------------------------------------------------------
# CPU reference (the oracle's restatement of the reference algorithm) on a
# bounded sample, with a thread sweep
# ---------------------------------------------------------------------------

def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def host_ram_bytes() -> int:
    try:
        with open("/proc/meminfo") as fh:
            for line in fh:
                if line.startswith("MemAvailable:"):
                    return int(line.split()[1]) * 1024
    except OSError:
        pass
    return 16 << 30


def load_reference_package():
    """The unmodified reference package, pip-installed once into
    baseline/_ref (git-ignored; travels to the GPU box with the snapshot),
    or None."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "paball")):
        return None
    if ref not in sys.path:
        sys.path.insert(0, ref)
    try:
        import paball  # noqa: F401
        from paball import model as M
        from paball import radiator as Rr
    except Exception:
        return None
    return M, Rr


class CpuReference:
    """The reference's CPU implementation of the path on a strided ball
    subset x a strided detector subset of the workload (cost is linear in
    N * J * W, so pairs/s carries over).

    kind "reference": the UNMODIFIED reference package (baseline/_ref),
    ``paball.radiator.backward(cloud, ctx, real, "fine")`` with
    ``set_num_threads`` (its own sensor blocks of 8 over a thread pool,
    radiator.py:316-332).  The reference has no detector directivity; the
    workload's cos^2 / element weight is one multiply per pair on top of
    ~40 window samples, so the sample is timed without it (and the stock
    backward's >1024-ball cache-key bug, changes values, not
    cost).  kind "port": oracle/radiator.py (the FP64 restatement, ~25 %
    slower than the reference) when the package is not installed.

    The thread count is swept on a small sample first; the timed sample
    then runs with the best count, and every thread has a sensor block
    (>= 8 detectors per thread)."""

    SWEEP = (1, 2, 4, 8, 16, 32, 64)

    def __init__(self, scene, kind, n_balls: int, n_det: int = 0):
        self.ref = load_reference_package()
        self.kind = "reference" if self.ref is not None else "port"
        self.dirkind = kind
        self.scene = scene
        ncpu = os.cpu_count() or 1
        J = scene.array.positions.shape[0]
        n_det = n_det or min(J, max(128, 8 * ncpu))
        stride = max(1, J // n_det)
        self.sens = scene.array.positions[::stride][:n_det]
        self.nrm = scene.array.normals[::stride][:n_det]
        self.threads_avail = ncpu
        # ~14 KB cached per ball per busy thread: stay within half the RAM
        cap = int(0.5 * host_ram_bytes() / (14e3 * max(1, min(ncpu, -(-self.sens.shape[0] // 8)))))
        self.n_balls = int(max(1000, min(n_balls, cap, len(scene.init))))
        self.sel = self._subset(self.n_balls)
        t = scene.truth
        tsel = np.linspace(0, len(t) - 1, min(len(t), self.n_balls)).astype(np.int64)
        sc = scene
        if self.kind == "reference":
            M, Rr = self.ref
            self.ctx = Rr.ForwardContext(M.SensorArray(self.sens, float(sc.array.sound_speed)),
                                         M.TimeGrid(0.0, sc.grid.dt, sc.grid.n_samples))
            Rr.set_num_threads(ncpu)
            truth = M.PointCloud(t.positions[tsel], t.p0[tsel], t.a0[tsel])
            self.real = Rr.simulate_signals(truth, self.ctx)
        else:
            from oracle import radiator as OR   # the reference's CPU algorithm (restated); baseline only
            self.OR = OR
            self.real, _, _, _ = OR.run_model(t.positions[tsel], t.p0[tsel], t.a0[tsel], self.sens, self.nrm,
                                              float(sc.array.sound_speed), 0.0, sc.grid.dt, sc.grid.n_samples, 1,
                                              kind=kind, threads=ncpu)
        self.threads = None
        self.sweep = {}

    def _subset(self, m):
        return np.linspace(0, len(self.scene.init) - 1, m).astype(np.int64)

    def _run(self, sel, threads) -> float:
        c, sc = self.scene.init, self.scene
        if self.kind == "reference":
            M, Rr = self.ref
            Rr.set_num_threads(threads)
            cloud = M.PointCloud(c.positions[sel], c.p0[sel], c.a0[sel])
            t0 = time.perf_counter()
            Rr.backward(cloud, self.ctx, self.real, stage="fine")
            return time.perf_counter() - t0
        t0 = time.perf_counter()
        self.OR.run_model(c.positions[sel], c.p0[sel], c.a0[sel], self.sens, self.nrm, float(sc.array.sound_speed),
                          0.0, sc.grid.dt, sc.grid.n_samples, 1, real=self.real, stage="fine",
                          kind=self.dirkind, threads=threads)
        return time.perf_counter() - t0

    def pick_threads(self, sweep_balls: int = 6000) -> int:
        sel = self._subset(min(sweep_balls, self.n_balls))
        blocks = -(-self.sens.shape[0] // 8)
        cands = [t for t in self.SWEEP if t <= min(self.threads_avail, blocks)]
        if min(self.threads_avail, blocks) not in cands:
            cands.append(min(self.threads_avail, blocks))
        for t in cands:
            self.sweep[t] = len(sel) * self.sens.shape[0] / self._run(sel, t)
        self.threads = max(self.sweep, key=self.sweep.get)
        return self.threads

    def pairs_per_s(self, reps: int) -> float:
        if self.threads is None:
            self.pick_threads()
        best = min(self._run(self.sel, self.threads) for _ in range(max(1, reps)))
        return self.n_balls * self.sens.shape[0] / best

    def describe(self, value: float, reps: int) -> dict:
        what = ("unmodified reference package (baseline/_ref) paball.radiator.backward, no directivity"
                if self.kind == "reference" else "oracle/radiator.py FP64 numpy restatement")
        return {"value": value, "unit": UNIT, "cores": self.threads, "kind": self.kind,
                "sample": f"{self.n_balls} balls (strided subset) x {self.sens.shape[0]} detectors of the workload, "
                          f"fine backward (fwd+adj): {what}; best of {reps} at the best thread count",
                "thread_sweep_pairs_per_s": {str(k): v for k, v in sorted(self.sweep.items())},
                "host_threads": self.threads_avail, "cpu_model": cpu_model()}


def run_reference(args, rank, world):
    """The reference arm: the reference's CPU algorithm on the host cores
    (rank 0 only; other ranks exit without work)."""
    if rank != 0:
        return
    scene, _, kind = make_scene(args)
    ref = CpuReference(scene, kind, args.cpu_balls, args.cpu_det)
    ref.pick_threads()
    vals = [ref.pairs_per_s(1) for _ in range(args.warmup + args.steps)]
    v = statistics.median(vals[args.warmup:]) if args.steps else vals[-1]
    ms = args.n_balls * args.n_det / v * 1e3
    cpu = ref.describe(v, 1)
    cpu["sample"] = cpu["sample"].replace("best of 1", f"median of {args.steps} steps after {args.warmup} warm-up")
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": f"synthetic (seeded CounterRng, BASELINE config {args.config})",
            "config": config_dict(args, world), "impl": "reference", "cpu_baseline": cpu,
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "note": "reference CPU implementation (cpu_baseline.kind: 'reference' = the unmodified paball package "
                    "pip-installed into baseline/_ref, 'port' = oracle/radiator.py); each step = one fine backward "
                    "of the sample; ms_per_step extrapolated linearly to the full N*J"}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# BASELINE's second metric and the launch-bound toy
# ---------------------------------------------------------------------------

def recon_cpu_estimate(sc, kept, sched, trace, n_sub: int = 3000, threads: int | None = None):
    """Extrapolated wall time of the same reconstruction on the reference's
    CPU implementation: one backward (the iteration's whole cost; Adam and
    density control are O(N) numpy) timed per level on a strided n_sub-ball
    subset of the filtered cloud with all detectors, scaled linearly by every
    iteration's ball count (plus the initial filter on the 96^3 grid).  The
    unmodified reference package (baseline/_ref) when installed, else the
    oracle restatement."""
    threads = threads or os.cpu_count() or 1
    n_samples = sc.grid.n_samples
    sens, v = sc.array.positions, float(sc.array.sound_speed)
    sel = np.linspace(0, len(kept) - 1, min(n_sub, len(kept))).astype(np.int64)
    ref = load_reference_package()
    per_level = []
    for lv in sched.levels:
        n_out = -(-n_samples // lv.f)
        if ref is not None:
            M, Rr = ref
            Rr.set_num_threads(threads)
            ctx = Rr.ForwardContext(M.SensorArray(sens, v), M.TimeGrid(0.0, sc.grid.dt, n_samples))
            grid_k = ctx.grid.decimated(lv.f) if lv.f > 1 else ctx.grid
            real = M.SignalSet(grid_k, np.zeros((sens.shape[0], n_out)))
            cloud = M.PointCloud(kept.positions[sel], kept.p0[sel], kept.a0[sel])
            t0 = time.perf_counter()
            Rr.backward(cloud, ctx, real, stage=lv.stage)
        else:
            from oracle import radiator as OR
            t0 = time.perf_counter()
            OR.run_model(kept.positions[sel], kept.p0[sel], kept.a0[sel], sens, None, v, 0.0, sc.grid.dt,
                         n_samples, lv.f, real=np.zeros((sens.shape[0], n_out)), stage=lv.stage, threads=threads)
        per_level.append((time.perf_counter() - t0) / len(sel))   # s per ball per iteration
    total = per_level[0] * len(sc.init)   # the initial filter pass at f = 4 (same kernel sums, p0 = 0)
    for r in trace.records:
        total += per_level[r.level] * r.ball_count
    return {"value_s": total, "kind": "reference" if ref is not None else "port", "cores": threads,
            "sample": f"one backward per level on {len(sel)} balls (strided subset of the filtered cloud) x "
                      f"{sens.shape[0]} detectors, scaled by each iteration's ball count",
            "s_per_ball_iteration": per_level}


def run_recon(world: int):
    """BASELINE config 3 end to end through the public API: zero-gradient
    filter of the 96^3 grid at f = 4, then the (4,100,coarse), (2,100,fine),
    (1,100,fine) schedule with the filter re-applied every 10 iterations and
    the reference density-control cadence; host wall clock (max over ranks)."""
    import torch

    import paper_2601_00551_b200 as P
    from paper_2601_00551_b200 import scenes
    sc = scenes.schedule_config()
    ctx = P.ForwardContext(sc.array, sc.grid)
    real = P.simulate_signals(sc.truth, ctx)
    spacing = 28e-3 / 96
    th = P.DensityThresholds.from_spacing(spacing)
    lr = P.LearningRates.from_spacing(spacing)
    sched = P.Schedule((P.Level(4, 100, "coarse"), P.Level(2, 100, "fine"), P.Level(1, 100, "fine")),
                       duplication_period=100)
    walls = []
    for _ in range(2):   # the first run pays one-off allocations (workspaces, page-locked buffers): report the second
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        kept, rep = P.zero_gradient_filter(sc.init, ctx, real, f=4)
        final, trace = P.run_hierarchical(kept, ctx, real, sched, th, lr=lr, seed=103, filter_every=10,
                                          plateau=False)
        torch.cuda.synchronize()
        walls.append(time.perf_counter() - t0)
    wall = max_over_ranks(walls[-1], world)
    out = {"workload": "config3: 512 det, 96^3 init, 50k-ball truth, 40 MHz x 4096, filter at f=4 then schedule "
                       "4/2/1 x 100 (filter every 10, density control every 100), fp32 kernels",
           "wall_s": wall, "unit": "s", "higher_is_better": False, "cold_run_wall_s": walls[0],
           "iterations": len(trace.records),
           "n_init": len(sc.init), "n_after_filter": len(kept), "n_final": len(final),
           "loss_first": trace.records[0].loss, "loss_last": trace.records[-1].loss,
           "path": "paper_2601_00551_b200.zero_gradient_filter + run_hierarchical (public API, host wall clock)"}
    return out, (sc, kept, sched, trace)


def run_config1(world: int):
    """BASELINE config 1 (launch-bound toy) through the public API: forward of
    the truth, zero-gradient filter of the 32^3 grid at f = 1, five fine Adam
    steps; host wall clock of filter + steps (max over ranks)."""
    import torch

    import paper_2601_00551_b200 as P
    from paper_2601_00551_b200 import scenes
    sc = scenes.toy_config()
    ctx = P.ForwardContext(sc.array, sc.grid)
    real = P.simulate_signals(sc.truth, ctx)
    lr = P.LearningRates.from_spacing(10e-3 / 32)

    def once():
        kept, _ = P.zero_gradient_filter(sc.init, ctx, real, f=1)
        state = P.create_state(kept, lr=lr, seed=103)
        for _ in range(5):
            state, _ = P.step(state, ctx, real, 1, "fine")
        return state

    once()
    times = []
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        state = once()
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t0)
    return {"workload": "config1 toy: 256 det, 32^3 init, filter at f=1 + 5 fine Adam steps (public API)",
            "wall_ms": 1e3 * max_over_ranks(min(times), world), "unit": "ms", "higher_is_better": False,
            "n_after_filter": state.n, "best_of": 3}


def max_over_ranks(x: float, world: int) -> float:
    if world <= 1:
        return float(x)
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], dtype=torch.float64,
                     device="cuda" if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ---------------------------------------------------------------------------
# Our arm
# ---------------------------------------------------------------------------

def relaunch_under_torchrun(args) -> int:
    """``--gpus N`` outside torchrun: run this script as N ranks."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd).returncode


def nominal_fp32_peak(sms: int) -> tuple[float, float, str]:
    """Fixed roofline denominators: the FFMA2 rate (256 FP32 flop/clk/SM)
    and MUFU ex2 rate (16/clk/SM) at the measured maximum SM clock."""
    mhz, src = 1965.0, "1965 MHz (B200 clocks.max.sm)"
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            mhz = float(json.load(fh)["sm_max_mhz"])
            src = f"{mhz:.0f} MHz (MEASURED_PEAKS.json sm_max_mhz)"
    except (OSError, KeyError, ValueError):
        pass
    return sms * 256 * mhz * 1e6, sms * 16 * mhz * 1e6, \
        f"nominal: {sms} SMs x 256 FP32 flop/clk (FFMA2) and 16 ex2/clk at {src}"


def probe_peaks():
    """Live FP32 / ex2 / shared-memory RMW probes (tools/probe), reported
    beside the fixed denominators."""
    probe = os.path.join(ROOT, "tools", "probe", "libfp32_peak.so")
    try:
        lib = ctypes.CDLL(probe)
        fl, ex, rm = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
        out = {}
        if lib.probe_fp32_peak(3, ctypes.byref(fl), ctypes.byref(ex)) == 0:
            out["fp32_tflops"], out["ex2_per_s"] = fl.value / 1e12, ex.value
        if lib.probe_smem_rmw(3, ctypes.byref(rm)) == 0:
            out["smem_rmw_per_s"] = rm.value
        return out
    except (OSError, AttributeError):
        return {}


def main():
    args = parse()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(relaunch_under_torchrun(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist

    ndev = max(1, torch.cuda.device_count())
    oversubscribed = world > ndev
    dev = torch.device("cuda", local % ndev)
    torch.cuda.set_device(dev)
    if world > 1:
        if oversubscribed:   # ranks share GPUs: gloo over host memory, no rank waits inside a kernel
            dist.init_process_group("gloo")
        else:
            os.environ.setdefault("NCCL_DEBUG", "INFO")          # init log: the driver can check nranks
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=dev)

    import paper_2601_00551_b200 as P
    from paper_2601_00551_b200 import _lib
    from paper_2601_00551_b200 import engine as E
    from paper_2601_00551_b200 import radiator as R

    scene, dirkw, kind = make_scene(args)
    ctx = P.ForwardContext(scene.array, scene.grid, directivity=P.Directivity(**dirkw))
    det = R.device_detectors(ctx)
    acq = R._acq(ctx, 1)
    n_total = det.n_total * acq.n_out

    # supervision: forward of the truth cloud, resident on device (this rank's rows)
    truth = E.DeviceCloud.from_host(scene.truth.positions, scene.truth.p0, scene.truth.a0, dev)
    counters = E.PassCounters(dev)
    real_local, _ = E.forward_rows(truth, det, acq, counters)
    real_local = real_local.clone()
    del truth
    cloud = E.DeviceCloud.from_host(scene.init.positions, scene.init.p0, scene.init.a0, dev)
    cloud.pack()
    res_buf = torch.empty_like(real_local)
    flat_buf = torch.empty(5 * cloud.n + E.TAIL, dtype=torch.float64, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()

    def one_step(ev=None):
        """forward + residual/loss + adjoint + finalize (+ the one all-reduce
        of gradients and pass tail for N > 1), inputs resident."""
        c = E.PassCounters(dev)
        cloud.invalidate()   # parameters change every iteration: repack (the optimizer's per-step cost;
        #                      the sort order and the dual-walk pairing table persist until a resort)
        if ev:
            ev[0].record(stream)
        cloud.pack()
        res, loss_rows = E.forward_rows(cloud, det, acq, c, real_local=real_local, out=res_buf)
        if ev:
            ev[1].record(stream)
        E.adjoint_grads(cloud, det, acq, res, 1.0, 2, 2.0 / n_total, c, flat=flat_buf, loss_rows=loss_rows)
        if ev:
            ev[2].record(stream)
        return c

    for k in range(args.warmup):   # exactly the timed loop's launches (flush, events), untimed
        flush.fill_(float(k))
        E.TIMING = {n: [torch.cuda.Event(enable_timing=True) for _ in range(2)] for n in ("residual", "finalize")}
        c = one_step([torch.cuda.Event(enable_timing=True) for _ in range(3)])
    E.TIMING = None
    torch.cuda.synchronize()
    _, ops_per_step = c.result()

    # kernel-level events: pack+forward+residual, adjoint+finalize(+all-reduce)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    sampler = ClockSampler(dev.index, dev, period=float(os.environ.get("PAB_BENCH_CLOCK_PERIOD", "0.05")))
    hbm_evs = []
    # the sampler thread is running (steady state) before the timed region
    # opens, so its start-up never delays a kernel launch inside it; its
    # samples span the timed region
    with sampler:
        time.sleep(0.2)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        launches0 = _lib.LAUNCHES["kernels"]
        for k in range(args.steps):
            flush.fill_(float(k))
            E.TIMING = {n: [torch.cuda.Event(enable_timing=True) for _ in range(2)] for n in ("residual", "finalize")}
            hbm_evs.append(E.TIMING)
            one_step(evs[k])
        launches = _lib.LAUNCHES["kernels"] - launches0
        torch.cuda.synchronize()
    E.TIMING = None
    if world > 1:
        dist.barrier()
    fwd_ms = [e[0].elapsed_time(e[1]) for e in evs]
    adj_ms = [e[1].elapsed_time(e[2]) for e in evs]
    step_ms = [e[0].elapsed_time(e[2]) for e in evs]
    mean_step = sum(step_ms) / len(step_ms)
    print(f"rank {rank} step_ms " + " ".join(f"{x:.2f}" for x in step_ms) + " | fwd "
          + " ".join(f"{x:.2f}" for x in fwd_ms) + " | adj " + " ".join(f"{x:.2f}" for x in adj_ms), file=sys.stderr)
    ms_max = max_over_ranks(mean_step, world)
    pairs = args.n_balls * det.n_total
    value = pairs / (ms_max * 1e-3)

    # end to end through the public API: host cloud + supervision in, loss +
    # gradients out, every step; pageable numpy arrays (what a caller of the
    # reference API holds) and, beside it, the same with page-locked arrays
    e2e = None
    if args.e2e_steps > 0:
        real_full = E.full_rows(real_local, det).double().cpu().numpy()

        def time_e2e(host_cloud, host_real):
            P.backward(host_cloud, ctx, host_real, stage="fine")
            ms = []
            for _ in range(args.e2e_steps):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                P.backward(host_cloud, ctx, host_real, stage="fine")
                torch.cuda.synchronize()
                ms.append((time.perf_counter() - t0) * 1e3)
            return max_over_ranks(statistics.median(ms), world)

        pageable_ms = time_e2e(P.PointCloud(scene.init.positions.copy(), scene.init.p0.copy(),
                                            scene.init.a0.copy()), P.SignalSet(scene.grid, real_full))
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
        pinned_ms = time_e2e(P.PointCloud(pin(scene.init.positions), pin(scene.init.p0), pin(scene.init.a0)),
                             P.SignalSet(scene.grid, pin(real_full)))
        n = args.n_balls
        h2d = n * 5 * 8 + det.n_total * acq.n_out * 4   # FP64 cloud; supervision narrowed to FP32 while staged
        d2h = (5 * n + E.TAIL) * 8
        e2e = {"value": pairs / (pageable_ms * 1e-3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": pageable_ms,
               "path": "paper_2601_00551_b200.backward(PointCloud, ForwardContext, SignalSet, 'fine') with pageable "
                       "host numpy inputs (as a reference caller holds them); cloud and supervision staged through "
                       "page-locked buffers (threaded chunked copies, DMA per chunk; the supervision upload overlaps "
                       "the forward kernel) and loss + gradients downloaded every step",
               "pinned": {"value": pairs / (pinned_ms * 1e-3), "ms_per_step": pinned_ms,
                          "path": "same call with page-locked host arrays"}}

    recon = recon_state = None
    if not args.no_recon and args.config == 2:
        recon, recon_state = run_recon(world)
    config1 = None
    if not args.no_config1 and args.config == 2:
        config1 = run_config1(world)

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    # roofline of the dominant kernel against
    # the north star's ceiling, the FP32 CUDA-core peak (fixed nominal
    # denominator; the live probes are printed beside it), with SURVEY §8d's
    # algorithmic flops per in-window sample (the reference op count): 7 for
    # the forward, 12 for the fine adjoint
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    peak_flops, peak_ex2, peak_src = nominal_fp32_peak(sms)
    fwd_mean = sum(fwd_ms) / len(fwd_ms)
    adj_mean = sum(adj_ms) / len(adj_ms)
    samples = ops_per_step   # in-window samples of the pass over all ranks (== the adjoint's)
    local_samples = samples / world
    fwd_s, adj_s = fwd_mean * 1e-3, adj_mean * 1e-3
    kernels = {"forward_kernel": (FLOPS_FWD, fwd_s, "forward+residual events; pack and residual are ~0.3%"),
               "adjoint_kernel": (FLOPS_ADJ_FINE, adj_s, "adjoint+finalize events; finalize is ~0.4%")}
    dom = max(kernels, key=lambda k: kernels[k][1])
    fl, secs, note = kernels[dom]
    ach = fl * local_samples / secs
    roofline = {"bound": "fp32", "achieved": ach / 1e12, "peak": peak_flops / 1e12, "unit": "TFLOP/s",
                "frac": ach / peak_flops, "traffic": TRAFFIC_BYTES.get(dom), "kernel": dom,
                "peak_source": peak_src, "peak_probe_live": probe_peaks(),
                "algorithmic": f"{fl} FP32 flops x {int(local_samples)} in-window samples per launch (SURVEY 8d; {note})",
                "traffic_unit": f"DRAM bytes per launch (ncu --set full, {TRAFFIC_SRC})",
                "other_bounds": {
                    "forward_fp32 (7 flops per sample)": {"frac": FLOPS_FWD * local_samples / fwd_s / peak_flops},
                    "adjoint_fp32 (12 flops per sample)": {"frac": FLOPS_ADJ_FINE * local_samples / adj_s / peak_flops},
                    "forward_ex2 (1 per sample)": {"frac": local_samples / fwd_s / peak_ex2},
                    "adjoint_ex2 (1 per sample)": {"frac": local_samples / adj_s / peak_ex2},
                    "path_fp32 (fwd+adj, 19 flops per sample)": {
                        "frac": (FLOPS_FWD + FLOPS_ADJ_FINE) * local_samples / (ms_max * 1e-3) / peak_flops},
                    "path_ex2 (fwd+adj, 2 ex2 per sample)": {"frac": 2 * local_samples / (ms_max * 1e-3) / peak_ex2}},
                "kernel_ms": {"forward+residual": fwd_mean, "adjoint+finalize": adj_mean}}

    # the HBM-bound kernels of the step (signal and gradient traffic) against
    # the measured copy bandwidth; algorithmic bytes: residual = partition
    # planes + supervision read, residual written; finalize = chunk partials
    # + ball records read, caller-order gradients written
    peak_hbm, hbm_src = 6650.0, "fallback (B200_PROFILING.md)"
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            peak_hbm, hbm_src = float(json.load(fh)["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs"
    except (OSError, KeyError, ValueError):
        pass
    parts = E.plan_forward(cloud, det, acq).partitions
    res_bytes = (parts + 2) * det.n_local * acq.n_out * 4
    hbm = {"peak_GBps": peak_hbm, "peak_source": hbm_src}
    for name, nbytes in (("residual", res_bytes), ("grad_finalize", hbm_evs[0].get("finalize_bytes", 0))):
        key = "finalize" if name == "grad_finalize" else name
        ms_k = statistics.median(t[key][0].elapsed_time(t[key][1]) for t in hbm_evs)
        gbs = nbytes / (ms_k * 1e-3) / 1e9
        hbm[name] = {"ms": ms_k, "algorithmic_bytes": int(nbytes), "GBps": gbs, "frac": gbs / peak_hbm}
    roofline["hbm_kernels"] = hbm

    cpu = None
    if world == 1 and not args.no_cpu:
        ref = CpuReference(scene, kind, args.cpu_balls, args.cpu_det)
        ref.pick_threads()
        cpu = ref.describe(ref.pairs_per_s(args.cpu_reps), args.cpu_reps)
        if recon is not None:
            sc3, kept3, sched3, trace3 = recon_state
            recon["cpu_reference"] = recon_cpu_estimate(sc3, kept3, sched3, trace3, threads=ref.threads)

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "accumulation": "f64 per ball across detectors (adjoint)",
            "data": f"synthetic (seeded CounterRng, BASELINE config {args.config})", "config": config_dict(args, world),
            "in_window_samples_per_step": samples, "samples_per_pair": samples / pairs,
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "clocks": sampler.summary(),
            "gpu_launches": int(launches),
            "gpu_launches_note": "library kernels issued inside the timed region (counted by _lib.call): per step "
                                 "pack x2 (forward and adjoint packings), coincidence test, forward sweep, forward wide groups, residual, "
                                 "adjoint, finalize, pass tail",
            "kernel_ms_min_median": {"forward+residual": [min(fwd_ms), statistics.median(fwd_ms)],
                                     "adjoint+finalize": [min(adj_ms), statistics.median(adj_ms)]}}
    if world > 1:
        line["collective"] = {"backend": dist.get_backend(), "per_step": "one all-reduce of (5 n + 4) FP64",
                              "oversubscribed": oversubscribed, "gpus_visible": ndev}
        if oversubscribed:
            line["note"] = (f"{world} ranks on {ndev} GPU(s): the multi-rank path runs (gloo all-reduce), "
                            "the number is not a scaling measurement")
    if recon is not None:
        line["recon"] = recon
    if config1 is not None:
        line["config1"] = config1
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
