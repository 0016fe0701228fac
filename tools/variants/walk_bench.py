"""Forward walk loop in isolation (PAB_WALK_BENCH build): cycles per
16-sample trip per warp at 8 warps/SM vs the ex2 (XU) bound of 128.

usage: PAB_LIBRARY=tools/variants/lib_WB.so python tools/variants/walk_bench.py
"""
import ctypes
import os

import torch

lib = ctypes.CDLL(os.environ["PAB_LIBRARY"])
sms = torch.cuda.get_device_properties(0).multi_processor_count
clk = 1.965e9
out = torch.empty(sms * 2 * 128, device="cuda")
for L in (16, 48, 96):
    reps = 4000
    ms = ctypes.c_float()
    rc = lib.pab_bench_walk(sms * 2, reps, L, ctypes.c_void_p(out.data_ptr()), ctypes.byref(ms))
    trips = reps * L / 16.0
    cyc = ms.value * 1e-3 * clk / trips
    samples = sms * 2 * 128 * reps * L
    print(f"L={L}: rc={rc} {ms.value:.2f} ms, {cyc:.1f} cycles per 16-sample trip per warp "
          f"(XU bound 128 at 2 warps/SMSP -> 256 per trip pair), {samples / (ms.value * 1e-3) / 1e12:.2f} T samples/s")
for L in (48,):
    reps = 4000
    ms = ctypes.c_float()
    rc = lib.pab_bench_walk_dual(sms * 2, reps, L, ctypes.c_void_p(out.data_ptr()), ctypes.byref(ms))
    samples = 2 * sms * 2 * 128 * reps * L   # two balls per lane
    print(f"dual L={L}: rc={rc} {ms.value:.2f} ms, {samples / (ms.value * 1e-3) / 1e12:.2f} T ball-samples/s")
for L in (48, 96):
    reps = 4000
    ms = ctypes.c_float()
    rc = lib.pab_bench_walk_dualrec(sms * 2, reps, L, ctypes.c_void_p(out.data_ptr()), ctypes.byref(ms))
    samples = 2 * sms * 2 * 128 * reps * L   # two balls per lane
    print(f"dual-recurrence L={L}: rc={rc} {ms.value:.2f} ms, {samples / (ms.value * 1e-3) / 1e12:.2f} T ball-samples/s")
