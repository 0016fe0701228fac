"""Host->device upload strategies for pageable numpy arrays (tuning tool):
pageable .to(), single-threaded staging + one DMA, threaded staging in
pieces (hostio), DMA only from pinned memory, and the device->pinned copy."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2601_00551_b200 import hostio  # noqa: E402

dev = torch.device("cuda", 0)
a = np.random.default_rng(0).standard_normal(5_000_000)   # 40 MB float64
pinned = torch.empty(a.size, dtype=torch.float64, pin_memory=True)


def t(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best * 1e3


def single():
    np.copyto(pinned.numpy(), a)
    return pinned.to(dev, non_blocking=True)


print(f"pageable .to()              {t(lambda: torch.from_numpy(a).to(dev)):.2f} ms")
print(f"pinned -> device (DMA only) {t(lambda: pinned.to(dev, non_blocking=True)):.2f} ms")
print(f"1-thread stage + DMA        {t(single):.2f} ms")
for parts in (1, 2, 4):
    hostio.PARTS = parts
    st = hostio.Stager()
    print(f"hostio {parts} parts            {t(lambda: st.upload([(a, torch.float64)], dev)):.2f} ms")
    st32 = hostio.Stager()
    print(f"hostio {parts} parts -> f32     {t(lambda: st32.upload([(a, torch.float32)], dev)):.2f} ms")
d = torch.empty(a.size, dtype=torch.float64, device=dev)
h = torch.empty(a.size, dtype=torch.float64, pin_memory=True)
print(f"device -> pinned            {t(lambda: h.copy_(d, non_blocking=True)):.2f} ms")
