"""Per-part clock breakdown of the fine adjoint kernel (PAB_ADJ_PROF build)
on config 2 (tuning aid).

usage: PAB_LIBRARY=tools/variants/lib_APROF.so python tools/variants/adj_prof.py
"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import paper_2601_00551_b200 as P  # noqa: E402
from paper_2601_00551_b200 import _lib  # noqa: E402
from paper_2601_00551_b200 import scenes  # noqa: E402

sc = scenes.microbench_config()
ctx = P.ForwardContext(sc.array, sc.grid, directivity=P.Directivity("cos_power", power=2.0))
real = P.SignalSet(sc.grid, np.random.default_rng(0).standard_normal((sc.array.n_sensors, sc.grid.n_samples)) * 1e-3)
lib = _lib.load()
buf = (C.c_ulonglong * 16)()
for _ in range(2):
    lib.pab_adj_prof(buf, 1)
    P.backward(sc.init, ctx, real, stage="fine")
    torch.cuda.synchronize()
lib.pab_adj_prof(buf, 0)
v = list(buf)
names = ["batch geometry (32 detectors)", "wait staged segments", "stage next pair + shuffles", "setups (pair)",
         "moment walks (pair)", "epilogues (pair)", "non-uniform pairs (fallback)", "total"]
for i, n in enumerate(names):
    print(f"  {n:32s} {v[i]:.3e}  {100.0 * v[i] / max(v[7], 1):5.1f}%")
print(f"  {'unaccounted':32s} {v[7] - sum(v[:7]):.3e}  {100.0 * (v[7] - sum(v[:7])) / max(v[7], 1):5.1f}%")
