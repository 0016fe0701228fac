import numpy as np, torch, time, sys, os
sys.path.insert(0, ".")
import paper_2601_00551_b200 as P
from paper_2601_00551_b200 import engine as E, radiator as R, scenes
sc = scenes.schedule_config(); ctx = P.ForwardContext(sc.array, sc.grid)
d = np.load("gpurun_out/level2_cloud.npz")
det = R.device_detectors(ctx); acq = R._acq(ctx, 1)
cloud = E.DeviceCloud.from_host(d["pos"], d["p0"], d["a0"], det.pos.device)
ts = []
for i in range(4):
    c = E.PassCounters(det.pos.device); cloud.invalidate(); torch.cuda.synchronize(); t = time.perf_counter()
    rows, _ = E.forward_rows(cloud, det, acq, c); torch.cuda.synchronize(); ts.append((time.perf_counter() - t) * 1e3)
print(os.environ.get("PAB_LIBRARY", "base"), "fwd ms", [round(x, 2) for x in ts], "ops", int(c.ops.item()))
np.save(sys.argv[1], rows.cpu().numpy())
