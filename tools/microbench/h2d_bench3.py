"""Cloud-sized uploads through hostio (streaming-store staging) vs pageable .to() (tuning tool)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2601_00551_b200 import hostio  # noqa: E402

dev = torch.device("cuda", 0)
rng = np.random.default_rng(0)
pos, p0, a0 = rng.standard_normal((1_000_000, 3)), rng.standard_normal(1_000_000), rng.standard_normal(1_000_000)
sup = rng.standard_normal((1024, 4096))


def t(fn, reps=7):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best * 1e3


print(f"pageable .to() x3 (cloud 40 MB)   {t(lambda: [torch.from_numpy(x).to(dev) for x in (pos, p0, a0)]):.2f} ms")
for parts in (1, 2, 4, 8):
    hostio.PARTS = parts
    st = hostio.Stager()
    print(f"hostio cloud {parts} parts              "
          f"{t(lambda: st.upload([(pos, torch.float64), (p0, torch.float64), (a0, torch.float64)], dev)):.2f} ms")
    st2 = hostio.Stager()
    print(f"hostio supervision -> f32 {parts} parts "
          f"{t(lambda: st2.upload([(sup, torch.float32)], dev)):.2f} ms")
print(f"pageable supervision f64 .to()     {t(lambda: torch.from_numpy(sup).to(dev).float()):.2f} ms")
