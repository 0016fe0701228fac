"""Host -> device transfers of the API edge (reference callers hold pageable
float64 numpy arrays; radiator.py:290-359 reads them on every call).

A pageable ``tensor.to(device)`` is staged by the driver through its own
pinned buffer with the calling thread blocked (40 MB float64 on the B200
host: ~2.6 ms).  A cached host copy into page-locked memory followed by the
DMA is no faster: the DMA then reads lines that sit dirty in the CPU caches
(copy ~0.9 ms + DMA 0.73 ms measured separately, 2.7 ms back to back;
tools/microbench/h2d_bench2.py).  Here the library's host stager
(csrc/pab_host.cu) copies with non-temporal stores on several threads (and
narrows the supervision to FP32 in the same pass, halving its DMA), in a
few pieces whose DMAs are queued as soon as each piece is staged; all
arrays of one upload travel as one contiguous device buffer.
"""

from __future__ import annotations

import os

import numpy as np
import torch

from . import _lib

PARTS = 1   # pieces per array (measured, cloud 40 MB: 1 / 2 / 4 / 8 pieces 1.29 / 1.48 / 2.40 / 4.05 ms; pageable .to() 2.74)
THREADS = int(os.environ.get("PAB_HOST_THREADS", max(1, min(8, os.cpu_count() or 1))))   # staging threads (tuning override)


class Stager:
    """One page-locked staging slot (grow-only), reused call after call; the
    previous upload's DMA is waited for before the slot is overwritten."""

    def __init__(self):
        self.buf = None
        self.done = None

    def _reserve(self, nbytes: int) -> torch.Tensor:
        if self.done is not None:
            self.done.synchronize()
        if self.buf is None or self.buf.numel() < nbytes:
            self.buf = torch.empty(max(nbytes, 1), dtype=torch.uint8, pin_memory=True)
        return self.buf

    def upload(self, arrays, dev, stream: torch.cuda.Stream | None = None):
        """arrays: [(numpy array, torch dtype)] (float64 sources; float32
        targets are narrowed while staged) -> device tensors of the same
        shapes, views of one contiguous device buffer.  Copies run on
        ``stream`` (default: the current stream); returns (tensors, event
        recorded after the last DMA)."""
        lib = _lib.load()
        stream = stream or torch.cuda.current_stream(dev)
        specs = []
        total = 0
        for a, dt in arrays:
            src = np.ascontiguousarray(a, dtype=np.float64)
            esz = 4 if dt == torch.float32 else 8
            specs.append((np.shape(a), src, dt, esz, total))
            total += (src.size * esz + 255) & ~255
        buf = self._reserve(total)
        base = buf.data_ptr()
        with torch.cuda.stream(stream):
            dbuf = torch.empty(max(total, 1), dtype=torch.uint8, device=dev)
            outs = [dbuf[off:off + src.size * esz].view(dt).view(shape) for shape, src, dt, esz, off in specs]
            for _, src, dt, esz, off in specs:
                piece = max(1024, ((-(-src.size // PARTS)) + 1023) & ~1023)
                for e0 in range(0, src.size, piece):
                    e1 = min(src.size, e0 + piece)
                    b0, nb = off + e0 * esz, (e1 - e0) * esz
                    sptr = src.ctypes.data + e0 * 8
                    if dt == torch.float32:
                        rc = lib.pab_host_stage_narrow(base + b0, sptr, e1 - e0, THREADS)
                    else:
                        rc = lib.pab_host_stage_copy(base + b0, sptr, nb, THREADS)
                    if rc != 0:
                        raise ValueError("pab_host_stage_*: invalid staging arguments")
                    dbuf[b0:b0 + nb].copy_(buf[b0:b0 + nb], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(stream)
        self.done = ev
        return outs, ev


_STAGERS: dict = {}


def stager(name: str) -> Stager:
    s = _STAGERS.get(name)
    if s is None:
        s = _STAGERS[name] = Stager()
    return s
