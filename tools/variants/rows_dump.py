"""Dump forward rows and fine gradients of a reduced config-2 instance with
the library PAB_LIBRARY selects, for bitwise comparisons of kernel variants
(tuning aid): PAB_LIBRARY=... python rows_dump.py out.npz"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import paper_2601_00551_b200 as P  # noqa: E402
from paper_2601_00551_b200 import scenes  # noqa: E402

sc = scenes.microbench_config(n_balls=200_000, n_det=128, n_samples=4096)
ctx = P.ForwardContext(sc.array, sc.grid, directivity=P.Directivity("cos_power", power=2.0))
f = int(os.environ.get("F", "1"))   # decimation factor (f > 1: the single-walk sweep)
rows = P.simulate_at_rate(sc.truth, ctx, f).data
L, g = P.backward(sc.init, ctx, P.SignalSet(sc.grid.decimated(f) if f > 1 else sc.grid, rows), stage="fine")
np.savez(sys.argv[1], rows=rows, loss=L, p0=g.d_p0, a0=g.d_a0, pos=g.d_position)
print("dumped", sys.argv[1], rows.shape, L)
