"""Oversize-group statistics of a PAB_FWD_STATS build on config 2 (tuning aid).

usage: PAB_LIBRARY=tools/variants/lib_S.so python tools/variants/fwd_stats.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import paper_2601_00551_b200 as P  # noqa: E402
from paper_2601_00551_b200 import engine as E  # noqa: E402
from paper_2601_00551_b200 import radiator as R  # noqa: E402
from paper_2601_00551_b200 import scenes  # noqa: E402

if os.environ.get("CONFIG") == "4":
    sc = scenes.planar_config(n_balls=int(os.environ.get("N", "4000000")))
    ctx = P.ForwardContext(sc.array, sc.grid)
else:
    sc = scenes.microbench_config()
    ctx = P.ForwardContext(sc.array, sc.grid, directivity=P.Directivity("cos_power", power=2.0))
det = R.device_detectors(ctx)
acq = R._acq(ctx, 1)
dc = E.DeviceCloud.from_host(sc.init.positions, sc.init.p0, sc.init.a0, torch.device("cuda", 0))
c = E.PassCounters(dc.dev)
E.forward_rows(dc, det, acq, c)
torch.cuda.synchronize()
ops = int(c.ops.item())
plan = E.plan_forward(dc, det, acq)
pairs_groups = dc.n_groups * det.n_local
print(f"oversize group-detector pairs {ops >> 40} of {pairs_groups} ({100.0 * (ops >> 40) / pairs_groups:.3f}%), "
      f"partitions {plan.partitions}")
