"""Multi-process detector sharding on CPU (gloo, world_size 2): the host-side
composition used by the engine (shard ranges, gradient/loss all-reduce, row
gather) reproduces the single-process result.  The per-shard compute is the
oracle here (the CUDA kernels need a GPU; the driver's GPU runs are 1-GPU)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from pab_helpers import golden


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import radiator as OR
        from paper_2601_00551_b200.parallel import Shard, current_shard, gather_rows, sharded_backward

        g = golden("radiator.npz")
        sens = g["si_sensors"]
        J, n_out = sens.shape[0], 256
        shard = current_shard()
        assert shard == Shard(rank, world)

        def compute_local(lo, hi):
            _, L, (gp0, ga0, gpos), _ = OR.run_model(g["si_cand_pos"], g["si_cand_p0"], g["si_cand_a0"],
                                                     sens[lo:hi], None, 1500.0, 0.0, 5e-8, n_out, 1,
                                                     real=g["si_real"][lo:hi], stage="fine")
            n_local = (hi - lo) * n_out
            rescale = n_local / (J * n_out)   # oracle scales by 2/N_local
            grads = tuple(torch.from_numpy(x * rescale) for x in (gp0, ga0, gpos))
            return L * n_local, grads

        loss_sum, grads = sharded_backward(compute_local, J, shard, "cpu")
        lo, hi = shard.range(J)
        rows, _, _, _ = OR.run_model(g["si_cand_pos"], g["si_cand_p0"], g["si_cand_a0"], sens[lo:hi], None,
                                     1500.0, 0.0, 5e-8, n_out, 1)
        full = gather_rows(torch.from_numpy(rows), J)
        if rank == 0:
            out_q.put((loss_sum / (J * n_out), [t.numpy() for t in grads], full.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_detector_sharding_matches_single_process():
    from oracle import radiator as OR
    g = golden("radiator.npz")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    loss, grads, rows = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want_rows, L, (gp0, ga0, gpos), _ = OR.run_model(g["si_cand_pos"], g["si_cand_p0"], g["si_cand_a0"],
                                                     g["si_sensors"], None, 1500.0, 0.0, 5e-8, 256, 1,
                                                     real=g["si_real"], stage="fine")
    assert abs(loss - L) <= 1e-13 * L
    for got, ref in zip(grads, (gp0, ga0, gpos)):
        np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-14 * np.abs(ref).max())
    np.testing.assert_array_equal(rows, OR.run_model(g["si_cand_pos"], g["si_cand_p0"], g["si_cand_a0"],
                                                     g["si_sensors"], None, 1500.0, 0.0, 5e-8, 256, 1)[0])


def test_shard_ranges_partition_detectors():
    from paper_2601_00551_b200.parallel import Shard
    for J in (1, 7, 64, 1024, 1023):
        for world in (1, 2, 3, 8):
            rng = [Shard(r, world).range(J) for r in range(world)]
            assert rng[0][0] == 0 and rng[-1][1] == J
            assert all(a[1] == b[0] for a, b in zip(rng, rng[1:]))
            sizes = [hi - lo for lo, hi in rng]
            assert max(sizes) - min(sizes) <= 1
