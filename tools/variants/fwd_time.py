"""Forward-only timing on config 2 or 4 with an optional directivity
override (tuning aid): CONFIG=4 DIR=cos2|element|none python fwd_time.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import paper_2601_00551_b200 as P  # noqa: E402
from paper_2601_00551_b200 import engine as E  # noqa: E402
from paper_2601_00551_b200 import radiator as R  # noqa: E402
from paper_2601_00551_b200 import scenes  # noqa: E402

cfg = os.environ.get("CONFIG", "2")
nb = int(os.environ.get("N", "0")) or None
sc = scenes.planar_config(n_balls=nb or 4_000_000) if cfg == "4" else scenes.microbench_config(n_balls=nb or 1_000_000)
dk = os.environ.get("DIR", "element" if cfg == "4" else "cos2")
d = {"cos2": P.Directivity("cos_power", power=2.0), "element": P.Directivity("element", width=0.5e-3),
     "none": P.Directivity("none")}[dk]
ctx = P.ForwardContext(sc.array, sc.grid, directivity=d)
det = R.device_detectors(ctx)
acq = R._acq(ctx, 1)
dc = E.DeviceCloud.from_host(sc.init.positions, sc.init.p0, sc.init.a0, torch.device("cuda", 0))
dc.pack()
dc.pair_table()
c = E.PassCounters(dc.dev)
ms = []
for it in range(4):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    E.forward_rows(dc, det, acq, c)
    b.record()
    torch.cuda.synchronize()
    ms.append(a.elapsed_time(b))
print(f"config {cfg} dir {dk} dual {os.environ.get('PAB_FORWARD_DUAL', '1')}: forward {sorted(ms)[1]:.2f} ms")
