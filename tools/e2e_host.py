"""Host-side time of public-API backward() calls at config 2 with pageable
inputs (tuning tool): cProfile of the Python edge; the time spent waiting for
the GPU shows up under synchronize."""
import cProfile
import os
import pstats
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_00551_b200 as P  # noqa: E402
from paper_2601_00551_b200 import scenes  # noqa: E402

sc = scenes.microbench_config()
ctx = P.ForwardContext(sc.array, sc.grid, directivity=P.Directivity("cos_power", power=2.0))
real = P.simulate_signals(sc.truth, ctx)
real = P.SignalSet(real.grid, np.array(real.data))
for _ in range(3):
    P.backward(sc.init, ctx, real, stage="fine")
torch.cuda.synchronize()
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
for _ in range(5):
    P.backward(sc.init, ctx, real, stage="fine")
pr.disable()
print(f"wall per call {(time.perf_counter() - t0) / 5 * 1e3:.2f} ms")
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
