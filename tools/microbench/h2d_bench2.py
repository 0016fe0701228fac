import time, numpy as np, torch
from concurrent.futures import ThreadPoolExecutor
dev = torch.device("cuda", 0)
a = np.random.default_rng(0).standard_normal(5_000_000)
pool = ThreadPoolExecutor(8)
buf = torch.empty(a.nbytes, dtype=torch.uint8, pin_memory=True)
pf = torch.empty(a.size, dtype=torch.float64, pin_memory=True)
d = torch.empty(a.size, dtype=torch.float64, device=dev)
def t(fn, reps=7):
    fn(); torch.cuda.synchronize(); best=1e9
    for _ in range(reps):
        t0=time.perf_counter(); fn(); torch.cuda.synchronize(); best=min(best,time.perf_counter()-t0)
    return best*1e3
def par(dst, src, casting="same_kind"):
    step = -(-src.size // 8)
    fs=[pool.submit(np.copyto, dst[i:i+step], src[i:i+step], casting=casting) for i in range(0, src.size, step)]
    [f.result() for f in fs]
print("par copy to f64 pinned", t(lambda: par(pf.numpy(), a)))
print("par copy to u8-view pinned", t(lambda: par(buf.numpy().view(np.float64), a)))
print("par copy unsafe", t(lambda: par(buf.numpy().view(np.float64), a, "unsafe")))
print("DMA f64 pinned", t(lambda: d.copy_(pf, non_blocking=True)))
print("DMA u8-view", t(lambda: d.copy_(buf.view(torch.float64), non_blocking=True)))
print("par + DMA", t(lambda: (par(pf.numpy(), a), d.copy_(pf, non_blocking=True))))
def two():
    h = a.size // 2
    par(pf.numpy()[:h], a[:h]); d[:h].copy_(pf[:h], non_blocking=True)
    par(pf.numpy()[h:], a[h:]); d[h:].copy_(pf[h:], non_blocking=True)
print("par + DMA 2 halves", t(two))
print("pageable to()", t(lambda: torch.from_numpy(a).to(dev)))
print("pageable copy_ into existing", t(lambda: d.copy_(torch.from_numpy(a))))
print("empty device alloc + pageable", t(lambda: torch.empty(a.size, dtype=torch.float64, device=dev).copy_(torch.from_numpy(a))))
