"""Per-phase clock breakdown of the forward kernel (PAB_FWD_PROF build) on
config 2 (tuning aid).

usage: PAB_LIBRARY=tools/variants/lib_PROF.so python tools/variants/fwd_prof.py
"""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import paper_2601_00551_b200 as P  # noqa: E402
from paper_2601_00551_b200 import _lib  # noqa: E402
from paper_2601_00551_b200 import engine as E  # noqa: E402
from paper_2601_00551_b200 import radiator as R  # noqa: E402
from paper_2601_00551_b200 import scenes  # noqa: E402

if os.environ.get("CONFIG") == "recon2":   # the config-3 reconstruction's f = 1 cloud (tools/recon_level2_cloud.py)
    sc = scenes.schedule_config()
    ctx = P.ForwardContext(sc.array, sc.grid)
    import numpy as np
    d = np.load(os.path.join("gpurun_out", "level2_cloud.npz"))

    class _C:
        pass
    sc.init = _C()
    sc.init.positions, sc.init.p0, sc.init.a0 = d["pos"], d["p0"], d["a0"]
elif os.environ.get("CONFIG") == "4":
    sc = scenes.planar_config(n_balls=int(os.environ.get("N", "4000000")))
    ctx = P.ForwardContext(sc.array, sc.grid, directivity=P.Directivity(
        "none") if os.environ.get("DIR") == "none" else P.Directivity("element", width=0.5e-3))
else:
    sc = scenes.microbench_config()
    ctx = P.ForwardContext(sc.array, sc.grid, directivity=P.Directivity("cos_power", power=2.0))
det = R.device_detectors(ctx)
acq = R._acq(ctx, 1)
dc = E.DeviceCloud.from_host(sc.init.positions, sc.init.p0, sc.init.a0, torch.device("cuda", 0))
lib = _lib.load()
buf = (C.c_ulonglong * 32)()
for it in range(2):
    lib.pab_fwd_prof(buf, 1)
    c = E.PassCounters(dc.dev)
    E.forward_rows(dc, det, acq, c)
    torch.cuda.synchronize()
lib.pab_fwd_prof(buf, 0)
v = list(buf)
ops = int(c.ops.item())
print(f"dual units {v[15]}, single-fallback units {v[14]} (walked lane-samples count ball-slots once per lane)")
print(f"walked lane-samples {v[11]:.4e} (regular groups {v[12]}), in-window samples {ops:.4e}: walked/useful {v[11] / ops:.3f}")
names_w = {0: "A bin", 1: "A sync", 2: "B sort+sync", 3: "D sweep", 4: "D end sync", 5: "E merge", 7: "F oversize+sync",
           6: "  D: final flush", 13: "  D: ring loop total", 8: "  D: wait full", 9: "  D: make_room flush", 10: "  D: walk"}
names_p = {16: "A bin", 17: "A sync", 18: "B sort+sync", 19: "D sweep", 20: "D end sync", 21: "E merge",
           23: "F oversize+sync", 26: "  D: batch geometry", 24: "  D: setups (2 per trip)",
           25: "  D: wait empty"}
for title, names, top in (("walkers", names_w, (0, 1, 2, 3, 4, 5, 7)), ("producers", names_p, (16, 17, 18, 19, 20, 21, 23))):
    tot = sum(v[i] for i in top)
    print(f"{title}: total {tot:.3e} warp-cycles")
    for i, n in names.items():
        print(f"  {n:28s} {v[i]:.3e}  {100.0 * v[i] / max(tot, 1):5.1f}%")
