"""The processing-order sort on the device (csrc/pab_sort.cu): exact cloud
bounds, the same keys as the host-bounds entry point, and a stable radix sort
equal to a full sort of the 64-bit keys (the low 28 bits are the index)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch

    from paper_2601_00551_b200 import _lib
    from paper_2601_00551_b200 import engine as E
    E.cuda_device()
    return torch, _lib, E


def _sort(torch, _lib, keys):
    n = keys.numel()
    lib = _lib.load()
    ws = torch.empty(int(lib.pab_sort_perm_workspace_bytes(n)) // 8 + 1, dtype=torch.int64, device=keys.device)
    perm = torch.empty(n, dtype=torch.int32, device=keys.device)
    k = keys.clone()
    _lib.call("pab_sort_perm", _lib.ptr(k), n, _lib.ptr(perm), _lib.ptr(ws), torch.cuda.current_stream().cuda_stream)
    return perm


@pytest.mark.parametrize("n", [1, 5, 2047, 2048, 2049, 100_003, 1_000_000])
def test_radix_sort_equals_full_key_sort(env, n):
    torch, _lib, E = env
    rng = np.random.default_rng(n)
    hi = rng.integers(0, 1 << 34, n, dtype=np.int64)
    hi[rng.integers(0, n, n // 3 + 1)] = hi[0]   # many equal high parts: stability matters
    keys = torch.from_numpy((hi << 28) | np.arange(n, dtype=np.int64)).cuda()
    perm = _sort(torch, _lib, keys)
    want = (torch.sort(keys).values & 0xFFFFFFF).to(torch.int32)
    assert torch.equal(perm, want)


def test_cloud_sort_matches_the_host_bounds_keys(env):
    torch, _lib, E = env
    from paper_2601_00551_b200 import scenes
    sc = scenes.microbench_config(n_balls=200_000, n_det=8, n_samples=256)
    dev = torch.device("cuda", torch.cuda.current_device())
    c = E.DeviceCloud.from_host(sc.init.positions, sc.init.p0, sc.init.a0, dev)
    c.sort()
    lo = torch.amin(c.pos, dim=0)
    hi = torch.amax(c.pos, dim=0)
    ext = float(torch.max(hi - lo).item())
    a0lo, a0hi = (float(x) for x in torch.aminmax(c.a0))
    keys = torch.empty(c.n, dtype=torch.int64, device=dev)
    lo_h = lo.cpu().numpy()
    _lib.call("pab_morton_keys", _lib.ptr(c.pos), _lib.ptr(c.a0), c.n, float(lo_h[0]), float(lo_h[1]),
              float(lo_h[2]), ext, a0lo, a0hi, c.buckets, _lib.ptr(keys), torch.cuda.current_stream().cuda_stream)
    want = (torch.sort(keys).values & 0xFFFFFFF).to(torch.int32)
    assert torch.equal(c.perm, want)
