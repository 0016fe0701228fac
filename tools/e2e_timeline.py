"""Host timeline of one public-API backward() at config 2 with pageable
inputs (tuning tool): where the end-to-end time goes beyond the kernels."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_00551_b200 as P  # noqa: E402
from paper_2601_00551_b200 import engine as E  # noqa: E402
from paper_2601_00551_b200 import radiator as R  # noqa: E402
from paper_2601_00551_b200 import scenes  # noqa: E402

sc = scenes.microbench_config()
ctx = P.ForwardContext(sc.array, sc.grid, directivity=P.Directivity("cos_power", power=2.0))
real = P.simulate_signals(sc.truth, ctx)
marks = []
orig = {}


def wrap(mod, name):
    f = getattr(mod, name)
    orig[name] = f

    def g(*a, **k):
        t0 = time.perf_counter()
        r = f(*a, **k)
        marks.append((name, t0, time.perf_counter()))
        return r
    setattr(mod, name, g)


for n in ("forward_rows", "adjoint_grads"):
    wrap(E, n)
wrap(E.DeviceCloud, "from_host")
for _ in range(3):
    P.backward(sc.init, ctx, real, stage="fine")
for _ in range(3):
    marks.clear()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    P.backward(sc.init, ctx, real, stage="fine")
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    print(f"total {1e3 * (t1 - t0):.2f} ms: " + ", ".join(f"{n} [{1e3 * (a - t0):.2f}, {1e3 * (b - t0):.2f}]"
                                                      for n, a, b in marks))
