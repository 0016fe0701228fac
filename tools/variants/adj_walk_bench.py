"""Adjoint moment walk in isolation (PAB_ADJ_BENCH build): lane-samples/s at
16 warps per SM vs the ex2 ceiling (4.6e12/s).
usage: PAB_LIBRARY=tools/variants/lib_AB.so python tools/variants/adj_walk_bench.py"""
import ctypes
import os

import torch

lib = ctypes.CDLL(os.environ["PAB_LIBRARY"])
sms = torch.cuda.get_device_properties(0).multi_processor_count
out = torch.empty(sms * 16 * 32, device="cuda")
for casc in (0, 1):   # direct FP32x2 moments / two-sided cascade with the ratio recurrence
    for L in (16, 40, 44, 48, 96):
        reps = 4000
        ms = ctypes.c_float()
        rc = lib.pab_bench_adj_walk(sms * 16, reps, L, casc, ctypes.c_void_p(out.data_ptr()), ctypes.byref(ms))
        samples = sms * 16 * 32 * reps * L
        print(f"adjoint walk {'cascade' if casc else 'direct '} L={L}: rc={rc} {ms.value:.2f} ms, "
              f"{samples / (ms.value * 1e-3) / 1e12:.2f} T lane-samples/s")
