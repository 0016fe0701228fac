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
            _, L, (gp0, ga0, gpos), ops = OR.run_model(g["si_cand_pos"], g["si_cand_p0"], g["si_cand_a0"],
                                                     sens[lo:hi], None, 1500.0, 0.0, 5e-8, n_out, 1,
                                                     real=g["si_real"][lo:hi], stage="fine")
            n_local = (hi - lo) * n_out
            rescale = n_local / (J * n_out)   # oracle scales by 2/N_local
            grads = tuple(torch.from_numpy(x * rescale) for x in (gp0, ga0, gpos))
            return L * n_local, grads, (False, False, ops)

        loss_sum, grads, (co, nf, n_ops) = sharded_backward(compute_local, J, shard, "cpu")
        assert not co and not nf
        lo, hi = shard.range(J)
        rows, _, _, _ = OR.run_model(g["si_cand_pos"], g["si_cand_p0"], g["si_cand_a0"], sens[lo:hi], None,
                                     1500.0, 0.0, 5e-8, n_out, 1)
        full = gather_rows(torch.from_numpy(rows), J)
        if rank == 0:
            out_q.put((loss_sum / (J * n_out), [t.numpy() for t in grads], full.numpy(), n_ops))
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
    loss, grads, rows, n_ops = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want_rows, L, (gp0, ga0, gpos), want_ops = OR.run_model(g["si_cand_pos"], g["si_cand_p0"], g["si_cand_a0"],
                                                     g["si_sensors"], None, 1500.0, 0.0, 5e-8, 256, 1,
                                                     real=g["si_real"], stage="fine")
    assert abs(loss - L) <= 1e-13 * L
    assert n_ops == want_ops   # per-shard op counts sum to the single-process count
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


def _coincident_worker(rank, world, port, out_q):
    """Rank 1's detector shard holds a sensor placed on a ball: only that
    rank's pass flags it, and after the one all-reduce BOTH ranks see the
    flag (the engine then raises SimulationError on every rank, instead of
    one rank raising while the other hangs in the next collective)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import radiator as OR
        from paper_2601_00551_b200.parallel import current_shard, sharded_backward

        g = golden("radiator.npz")
        sens = g["si_sensors"].copy()
        J, n_out = sens.shape[0], 256
        sens[J - 1] = g["si_cand_pos"][0]   # last detector: rank 1's shard
        shard = current_shard()

        def compute_local(lo, hi):
            n = g["si_cand_pos"].shape[0]
            zeros = (torch.zeros(n, dtype=torch.float64), torch.zeros(n, dtype=torch.float64),
                     torch.zeros((n, 3), dtype=torch.float64))
            try:
                _, L, (gp0, ga0, gpos), ops = OR.run_model(g["si_cand_pos"], g["si_cand_p0"], g["si_cand_a0"],
                                                           sens[lo:hi], None, 1500.0, 0.0, 5e-8, n_out, 1,
                                                           real=g["si_real"][lo:hi], stage="fine")
            except OR.OracleSimulationError:
                return 0.0, zeros, (True, False, 0)
            return L, tuple(torch.from_numpy(x) for x in (gp0, ga0, gpos)), (False, False, ops)

        _, _, (co, nf, _) = sharded_backward(compute_local, J, shard, "cpu")
        out_q.put((rank, co, nf))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_error_flag_on_one_rank_reaches_every_rank():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_coincident_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict((r, (co, nf)) for r, co, nf in (q.get(timeout=240) for _ in range(2)))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert got == {0: (True, False), 1: (True, False)}


def test_tail_round_trip():
    from paper_2601_00551_b200.parallel import TAIL, read_tail, tail_values
    t = tail_values(3.5, True, False, 12345)
    assert len(t) == TAIL
    assert read_tail(t) == (3.5, True, False, 12345)
    # summed over ranks: flags become counts, still read as "set"
    s = [a + b for a, b in zip(t, tail_values(1.0, True, True, 5))]
    assert read_tail(s) == (4.5, True, True, 12350)
