"""Benchmark of the forward + adjoint hot path (BASELINE.json metric).

Workload: BASELINE config 2 ("microbench"): 1,000,000 balls uniform in a
20 mm cube, a0 ~ U[0.05, 0.2] mm, 1024 detectors on a jittered ellipsoid cap
with cos^2 directivity, 40 MHz x 4096 samples; seeded synthetic inputs
(paper_2601_00551_b200.scenes).  One step = one fine backward pass = forward
rows + residual/loss + adjoint + gradient finalisation (+ NCCL all-reduce of
the per-ball gradients for N > 1).  Metric: ball-detector pair evaluations
per second, pairs = N_balls x N_detectors per step.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Under torchrun each rank owns a contiguous detector block (strong scaling:
the configuration is fixed, the per-GPU work shrinks as 1/N).
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
TRAFFIC_FWD_BYTES = 172_755_456   # dram__bytes_read.sum + dram__bytes_write.sum, forward, profiles/r01_v12
EX2_PER_SAMPLE = 1


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
    ap.add_argument("--cpu-balls", type=int, default=20000, help="oracle sample: balls x 64 detectors")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--recon", action="store_true",
                    help="also time the full config-3 reconstruction (filter + 300 iterations)")
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
# CPU reference (oracle port of the reference algorithm) on a bounded sample
# ---------------------------------------------------------------------------

def cpu_reference_pairs_per_s(scene, n_sample: int, steps: int = 1, threads: int | None = None,
                              n_det: int = 64, kind=("cos_power", 2.0)):
    """SURVEY.md §6 microbench slice: a strided ball subset x a strided
    detector subset of config 2 (pairs/s is linear in N*J*W)."""
    from oracle import radiator as OR   # the reference's CPU algorithm (restated); baseline only
    threads = threads or os.cpu_count() or 1
    c, t = scene.init, scene.truth
    stride = max(1, scene.array.positions.shape[0] // n_det)
    sens, nrm = scene.array.positions[::stride], scene.array.normals[::stride]
    sel = np.linspace(0, len(c) - 1, n_sample).astype(np.int64)
    real, _, _, _ = OR.run_model(t.positions[sel], t.p0[sel], t.a0[sel], sens, nrm, 1500.0, 0.0, scene.grid.dt,
                                 scene.grid.n_samples, 1, kind=kind, threads=threads)
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        OR.run_model(c.positions[sel], c.p0[sel], c.a0[sel], sens, nrm, 1500.0, 0.0, scene.grid.dt,
                     scene.grid.n_samples, 1, real=real, stage="fine", kind=kind, threads=threads)
        times.append(time.perf_counter() - t0)
    pairs = n_sample * sens.shape[0]
    return pairs / min(times), threads, f"{n_sample} balls (strided subset) x {sens.shape[0]} detectors, " \
                                        f"fine backward (fwd+adj), best of {steps}"


def run_reference(args, rank, world):
    if rank != 0:
        return
    scene, _, kind = make_scene(args)
    vals = []
    for _ in range(args.warmup + args.steps):
        v, cores, sample = cpu_reference_pairs_per_s(scene, args.cpu_balls, steps=1, kind=kind)
        vals.append(v)
    v = statistics.median(vals[args.warmup:]) if args.steps else vals[-1]
    ms = args.n_balls * args.n_det / v * 1e3
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": f"synthetic (seeded CounterRng, BASELINE config {args.config})",
            "config": config_dict(args, world), "impl": "reference",
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "note": "reference CPU algorithm = oracle/radiator.py (FP64 numpy port of paball radiator, "
                    "key-fixed); ms_per_step extrapolated linearly to the full N*J"}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# Our arm
# ---------------------------------------------------------------------------

def run_recon():
    """BASELINE config 3 end to end through the public API: zero-gradient
    filter of the 96^3 grid at f = 4, then the (4,100,coarse), (2,100,fine),
    (1,100,fine) schedule with the filter re-applied every 10 iterations and
    the reference density-control cadence; host wall clock."""
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
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    kept, rep = P.zero_gradient_filter(sc.init, ctx, real, f=4)
    final, trace = P.run_hierarchical(kept, ctx, real, sched, th, lr=lr, seed=103, filter_every=10, plateau=False)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    return {"workload": "config3: 512 det, 96^3 init, 50k-ball truth, 40 MHz x 4096, schedule 4/2/1 x 100",
            "wall_s": wall, "iterations": len(trace.records), "n_init": len(sc.init), "n_after_filter": len(kept),
            "n_final": len(final), "loss_first": trace.records[0].loss, "loss_last": trace.records[-1].loss}


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)

    import paper_2601_00551_b200 as P
    from paper_2601_00551_b200 import engine as E
    from paper_2601_00551_b200 import radiator as R
    from paper_2601_00551_b200 import scenes

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
    cloud = E.DeviceCloud.from_host(scene.init.positions, scene.init.p0, scene.init.a0, dev)
    cloud.pack()
    res_buf = torch.empty_like(real_local)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()

    def one_step(ev=None):
        c = E.PassCounters(dev)
        cloud.invalidate()   # parameters change every iteration: repack (the optimizer's per-step cost;
        #                      the sort order and the dual-walk pairing table persist until a resort)
        if ev:
            ev[0].record(stream)
        cloud.pack()
        res, loss_rows = E.forward_rows(cloud, det, acq, c, real_local=real_local, out=res_buf)
        if ev:
            ev[1].record(stream)
        g = E.adjoint_grads(cloud, det, acq, res, 1.0, 2, 2.0 / n_total, c)
        if ev:
            ev[2].record(stream)
        return c, loss_rows, g

    for k in range(args.warmup):   # exactly the timed loop's launches (flush, events), untimed
        flush.fill_(float(k))
        E.TIMING = {n: [torch.cuda.Event(enable_timing=True) for _ in range(2)] for n in ("residual", "finalize")}
        c, _, _ = one_step([torch.cuda.Event(enable_timing=True) for _ in range(3)])
    E.TIMING = None
    torch.cuda.synchronize()
    ops_per_step = c.read()

    # kernel-level events: pack+forward+residual, adjoint+finalize(+allreduce)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    sampler = ClockSampler(local, dev, period=float(os.environ.get("PAB_BENCH_CLOCK_PERIOD", "0.05")))
    hbm_evs = []
    # the sampler thread is running (steady state) before the timed region
    # opens, so its start-up never delays a kernel launch inside it; its
    # samples span the timed region
    with sampler:
        time.sleep(0.2)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        for k in range(args.steps):
            flush.fill_(float(k))
            E.TIMING = {n: [torch.cuda.Event(enable_timing=True) for _ in range(2)] for n in ("residual", "finalize")}
            hbm_evs.append(E.TIMING)
            one_step(evs[k])
        torch.cuda.synchronize()
    E.TIMING = None
    if world > 1:
        dist.barrier()
    fwd_ms = [e[0].elapsed_time(e[1]) for e in evs]
    adj_ms = [e[1].elapsed_time(e[2]) for e in evs]
    step_ms = [e[0].elapsed_time(e[2]) for e in evs]
    mean_step = sum(step_ms) / len(step_ms)
    print("step_ms " + " ".join(f"{x:.2f}" for x in step_ms) + " | fwd " + " ".join(f"{x:.2f}" for x in fwd_ms)
          + " | adj " + " ".join(f"{x:.2f}" for x in adj_ms), file=sys.stderr)
    t = torch.tensor([mean_step], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    pairs = args.n_balls * det.n_total
    value = pairs / (ms_max * 1e-3)

    # end to end through the public API: host (pinned) cloud + supervision in,
    # loss + gradients out, every step
    e2e = None
    if args.e2e_steps > 0:
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
        host_cloud = P.PointCloud(pin(scene.init.positions), pin(scene.init.p0), pin(scene.init.a0))
        real_full = E.full_rows(real_local, det).double().cpu()
        host_real = P.SignalSet(scene.grid, real_full.pin_memory().numpy())
        P.backward(host_cloud, ctx, host_real, stage="fine")
        e2e_ms = []
        for _ in range(args.e2e_steps):
            R._sup_cache.clear()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            P.backward(host_cloud, ctx, host_real, stage="fine")
            torch.cuda.synchronize()
            e2e_ms.append((time.perf_counter() - t0) * 1e3)
        tt = torch.tensor([statistics.median(e2e_ms)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        n = args.n_balls
        h2d = n * 5 * 8 + det.n_total * acq.n_out * 8 // world * world
        d2h = n * 5 * 8 + 8
        e2e = {"value": pairs / (float(tt.item()) * 1e-3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": float(tt.item()),
               "path": "paper_2601_00551_b200.backward(PointCloud, ForwardContext, SignalSet, 'fine') "
                       "with pinned host numpy inputs; supervision re-uploaded every step"}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    # roofline of the dominant kernel: the
    # forward against the north star's ceiling, the FP32 CUDA-core peak, with
    # SURVEY §8d's algorithmic 7 FP32 flops per in-window sample (the
    # reference op count); the canonical ex2 (1 per sample) and shared-memory
    # RMW (8 B per sample) ceilings of the same work, and both kernels'
    # fractions, are reported beside it.  Peaks are probed live on this GPU.
    probe = os.path.join(ROOT, "tools", "probe", "libfp32_peak.so")
    peak_flops = peak_ex2 = peak_rmw = None
    peak_kind = "measured live (tools/probe: FFMA2 chains, ex2 chains, private-column smem RMW; this GPU)"
    try:
        lib = ctypes.CDLL(probe)
        fl, ex, rm = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
        if lib.probe_fp32_peak(3, ctypes.byref(fl), ctypes.byref(ex)) == 0:
            peak_flops, peak_ex2 = fl.value, ex.value
        if lib.probe_smem_rmw(3, ctypes.byref(rm)) == 0:
            peak_rmw = rm.value
    except (OSError, AttributeError):
        pass
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    if peak_flops is None or peak_rmw is None:
        peak_flops, peak_ex2, peak_rmw = sms * 256 * 1.965e9, sms * 16 * 1.965e9, sms * 14.4 * 1.965e9
        peak_kind = "nominal at 1965 MHz (FFMA2 256 flop/clk/SM, ex2 16/clk/SM, smem RMW 14.4/clk/SM)"
    fwd_mean = sum(fwd_ms) / len(fwd_ms)
    adj_mean = sum(adj_ms) / len(adj_ms)
    samples = ops_per_step   # in-window samples evaluated by the forward (== adjoint)
    fwd_s, adj_s = fwd_mean * 1e-3, adj_mean * 1e-3
    ach = FLOPS_FWD * samples / fwd_s
    roofline = {"bound": "fp32", "achieved": ach / 1e12, "peak": peak_flops / 1e12, "unit": "TFLOP/s",
                "frac": ach / peak_flops, "traffic": TRAFFIC_FWD_BYTES, "kernel": "forward_kernel",
                "peak_source": peak_kind,
                "algorithmic": f"{FLOPS_FWD} FP32 flops x {samples} in-window samples per launch (SURVEY 8d; "
                               "forward+residual events, of which pack and residual are ~0.3%)",
                "traffic_unit": "DRAM bytes per forward launch (ncu --set full, profiles/r01_v12; 6 partition planes written)",
                "other_bounds": {
                    "forward_ex2 (1 per sample)": {"frac": samples / fwd_s / peak_ex2, "peak_per_s": peak_ex2},
                    "forward_smem_rmw (8 B per sample)": {"frac": samples / fwd_s / peak_rmw,
                                                          "peak_GBps": 8.0 * peak_rmw / 1e9},
                    "adjoint_ex2 (its binding ceiling)": {"frac": samples / adj_s / peak_ex2},
                    "adjoint_fp32": {"frac": FLOPS_ADJ_FINE * samples / adj_s / peak_flops},
                    "path_fp32 (fwd+adj, 19 flops per sample)": {
                        "frac": (FLOPS_FWD + FLOPS_ADJ_FINE) * samples / (ms_max * 1e-3) / peak_flops},
                    "path_ex2 (fwd+adj, 2 ex2 per sample)": {"frac": 2 * samples / (ms_max * 1e-3) / peak_ex2}},
                "design_note": "the forward's dual walk executes 0.5 ex2, 4 FP32 lane-ops and 4 B of shared RMW per "
                               "walked ball-sample (1.28 walked per in-window sample); no pipe is saturated "
                               "(ncu r01_v12: issue slots 69%, ALU 42%, XU 40%, FMA 32%, LSU 17%)",
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
        v, cores, sample = cpu_reference_pairs_per_s(scene, args.cpu_balls, steps=1, kind=kind)
        cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample}

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "accumulation": "f64 per ball across detectors (adjoint)",
            "data": f"synthetic (seeded CounterRng, BASELINE config {args.config})", "config": config_dict(args, world),
            "in_window_samples_per_step": samples, "samples_per_pair": samples / pairs,
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "clocks": sampler.summary(),
            "gpu_launches": 5 * args.steps,   # pack, forward, residual, adjoint, finalize (pairing table: per sort)
            "kernel_ms_min_median": {"forward+residual": [min(fwd_ms), statistics.median(fwd_ms)],
                                     "adjoint+finalize": [min(adj_ms), statistics.median(adj_ms)]}}
    if args.recon:
        line["recon"] = run_recon()
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
