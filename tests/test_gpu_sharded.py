"""The detector-sharded path on the real CUDA kernels: two
ranks (gloo process group, both on cuda:0 -- the ranks never wait on each
other inside a kernel; the only exchanges are the host-side all-reduce /
all-gather that NCCL performs on a multi-GPU node) against one process.

Checks: the sharded forward gathers the same rows, the sharded backward
gives the same loss and gradients up to FP summation order, and the
filter + Adam steps keep identical clouds on every rank."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _instance():
    import paper_2601_00551_b200 as P
    from paper_2601_00551_b200 import scenes
    sc = scenes.microbench_config(n_balls=6000, n_det=96, n_samples=1024)
    ctx = P.ForwardContext(sc.array, sc.grid, directivity=P.Directivity("cos_power", power=2.0))
    return P, sc, ctx


def _run(P, sc, ctx):
    real = P.simulate_signals(sc.truth, ctx)
    L, g = P.backward(sc.init, ctx, real, stage="fine")
    kept, rep = P.zero_gradient_filter(sc.init, ctx, real, f=2)
    state = P.create_state(kept, lr=P.LearningRates.from_spacing(4e-4), seed=3)
    losses = []
    for _ in range(3):
        state, Ls = P.step(state, ctx, real, 1, "fine")
        losses.append(Ls)
    c = state.cloud
    return {"rows": real.data, "L": L, "gp0": g.d_p0, "ga0": g.d_a0, "gpos": g.d_position,
            "kept": rep.n_retained, "losses": np.array(losses), "p0": c.p0, "pos": c.positions}


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        P, sc, ctx = _instance()
        out = _run(P, sc, ctx)
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(600)
def test_two_rank_sharded_path_matches_single_process():
    ctx_mp = mp.get_context("spawn")
    q = ctx_mp.Queue()
    port = _free_port()
    procs = [ctx_mp.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=500) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    P, sc, ctx = _instance()
    ref = _run(P, sc, ctx)
    rel = lambda a, b: np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(np.asarray(b)), 1e-300)
    for r in (0, 1):
        got = res[r]
        assert rel(got["rows"], ref["rows"]) < 1e-6          # gathered rows: same kernels, same detectors
        assert abs(got["L"] - ref["L"]) <= 1e-9 * ref["L"]
        assert rel(got["gp0"], ref["gp0"]) < 1e-6           # per-detector sums re-associated across ranks
        assert rel(got["ga0"], ref["ga0"]) < 1e-6
        assert rel(got["gpos"], ref["gpos"]) < 1e-6
        assert got["kept"] == ref["kept"]
        np.testing.assert_allclose(got["losses"], ref["losses"], rtol=1e-6)
        assert rel(got["p0"], ref["p0"]) < 1e-6
    # every rank holds the same cloud
    np.testing.assert_array_equal(res[0]["p0"], res[1]["p0"])
    np.testing.assert_array_equal(res[0]["pos"], res[1]["pos"])


def _coincident_worker(rank, world, port, q):
    """A ball sits on the last detector (rank 1's shard): only rank 1's
    kernels see it, the reduced pass tail makes BOTH ranks raise
    SimulationError at the same call (neither hangs in a later collective).
    The op count each rank adds is the global one."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        P, sc, ctx = _instance()
        real = P.simulate_signals(sc.truth, ctx)
        P.reset_op_count()
        P.backward(sc.init, ctx, real, stage="fine")
        ops = P.op_count()
        bad = sc.init.copy()
        bad.positions[0] = sc.array.positions[-1]
        raised = []
        for call in (lambda: P.backward(bad, ctx, real, stage="fine"),
                     lambda: P.step(P.create_state(bad, lr=P.LearningRates.from_spacing(4e-4)), ctx, real, 1,
                                    "fine")):
            try:
                call()
                raised.append(False)
            except P.SimulationError:
                raised.append(True)
        # both ranks are still in step: one more collective completes
        L, _ = P.backward(sc.init, ctx, real, stage="fine")
        q.put((rank, raised, ops, L))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(600)
def test_error_on_one_rank_is_raised_on_every_rank():
    ctx_mp = mp.get_context("spawn")
    q = ctx_mp.Queue()
    port = _free_port()
    procs = [ctx_mp.Process(target=_coincident_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict((r, (raised, ops, L)) for r, raised, ops, L in (q.get(timeout=500) for _ in range(2)))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    P, sc, ctx = _instance()
    real = P.simulate_signals(sc.truth, ctx)
    P.reset_op_count()
    L, _ = P.backward(sc.init, ctx, real, stage="fine")
    for r in (0, 1):
        raised, ops, Lr = res[r]
        assert raised == [True, True]
        assert ops == P.op_count()          # the global op count on every rank
        assert abs(Lr - L) <= 1e-9 * L
