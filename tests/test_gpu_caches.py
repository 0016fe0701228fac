"""In-place edits of caller-owned arrays between calls reach the device.

The reference reads ``real.data``, ``array.positions`` and ``array.normals``
on every call (reference radiator.py:316-332, :419-435); the device copies
here must never go stale: the supervision is uploaded on every call and the
detector cache is keyed on the content of the sensor arrays."""

import numpy as np
import pytest

from oracle import radiator as OR
from pab_helpers import rel_l2

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_2601_00551_b200 as P
    return P


def _instance(P):
    from paper_2601_00551_b200 import scenes
    sc = scenes.microbench_config(n_balls=3000, n_det=32, n_samples=1024)
    ctx = P.ForwardContext(sc.array, sc.grid, directivity=P.Directivity("cos_power", power=2.0))
    return sc, ctx


def _oracle_loss(sc, real, normals=None, positions=None):
    c = sc.init
    _, L, _, _ = OR.run_model(c.positions, c.p0, c.a0, sc.array.positions if positions is None else positions,
                              sc.array.normals if normals is None else normals, 1500.0, 0.0, sc.grid.dt,
                              sc.grid.n_samples, 1, real=real, stage="fine", kind=("cos_power", 2.0))
    return L


def test_in_place_edit_of_one_interior_supervision_sample(P):
    sc, ctx = _instance(P)
    real = P.simulate_signals(sc.truth, ctx)
    L1, _ = P.backward(sc.init, ctx, real, stage="fine")
    # one interior sample, not on any sampling stride a content fingerprint would use
    j, k = 17, 613
    delta = 50.0 * np.abs(real.data).max()
    real.data[j, k] += delta
    L2, g2 = P.backward(sc.init, ctx, real, stage="fine")
    want = _oracle_loss(sc, real.data)
    assert L2 != L1
    assert abs(L2 - want) <= 1e-4 * want
    # and back: the edit is undone on the device too
    real.data[j, k] -= delta
    L3, _ = P.backward(sc.init, ctx, real, stage="fine")
    assert abs(L3 - L1) <= 1e-12 * L1


def test_refilled_buffer_at_the_same_address(P):
    sc, ctx = _instance(P)
    real = P.simulate_signals(sc.truth, ctx)
    buf = real.data
    L1, _ = P.backward(sc.init, ctx, real, stage="fine")
    buf[:] = 0.5 * buf   # same array object, same address, new content
    L2, _ = P.backward(sc.init, ctx, real, stage="fine")
    want = _oracle_loss(sc, buf)
    assert abs(L2 - want) <= 1e-4 * want and abs(L2 - L1) > 1e-3 * L1


def test_in_place_edit_of_detector_positions_and_normals(P):
    sc, ctx = _instance(P)
    real = P.simulate_signals(sc.truth, ctx)
    P.backward(sc.init, ctx, real, stage="fine")
    sc.array.positions[3] += np.array([0.0, 0.0, 1e-3])   # same SensorArray object
    sc.array.normals[5] = -sc.array.normals[5]
    L, _ = P.backward(sc.init, ctx, real, stage="fine")
    want = _oracle_loss(sc, real.data)
    assert abs(L - want) <= 1e-4 * want
    rows = P.simulate_signals(sc.truth, ctx).data
    want_rows, _, _, _ = OR.run_model(sc.truth.positions, sc.truth.p0, sc.truth.a0, sc.array.positions,
                                      sc.array.normals, 1500.0, 0.0, sc.grid.dt, sc.grid.n_samples, 1,
                                      kind=("cos_power", 2.0))
    assert rel_l2(rows, want_rows) < 1e-4


def test_ball_exactly_on_a_sensor_far_from_its_group_centre(P):
    """The coincidence test is exact in FP64 (reference radiator.py:189-193)
    even when the ball sits far from its lane group's centre, where the
    kernels' FP32 offsets cannot resolve 1e-12."""
    sc, ctx = _instance(P)
    real = P.simulate_signals(sc.truth, ctx)
    bad = sc.init.copy()
    bad.positions[1234] = sc.array.positions[7]
    for call in (lambda: P.simulate_signals(bad, ctx), lambda: P.backward(bad, ctx, real, stage="fine"),
                 lambda: P.zero_gradient_filter(bad, ctx, real, f=2)):
        with pytest.raises(P.SimulationError):
            call()
    near = sc.init.copy()
    near.positions[1234] = sc.array.positions[7] + np.array([1e-9, 0.0, 0.0])   # reference: no error
    P.simulate_signals(near, ctx)


def test_adjoint_on_an_unaligned_residual_view(P):
    """pab_adjoint stages 16-byte vectors only from a 16-byte aligned
    residual; an offset view (a row slice of a larger buffer) takes the
    4-byte path and gives the same gradients up to the few overrun samples
    past a window end (finite residual in one staging, zero padding in the
    other; their Gaussian weights are below 2^-24)."""
    import torch

    from paper_2601_00551_b200 import engine as E
    from paper_2601_00551_b200 import radiator as R
    sc, ctx = _instance(P)
    det = R.device_detectors(ctx)
    acq = R._acq(ctx, 1)
    dev = det.pos.device
    cloud = E.DeviceCloud.from_host(sc.init.positions, sc.init.p0, sc.init.a0, dev)
    real = R.device_supervision(P.simulate_signals(sc.truth, ctx).data, det)
    c = E.PassCounters(dev)
    res, _ = E.forward_rows(cloud, det, acq, c, real_local=real)
    buf = torch.empty(res.numel() + 1, dtype=torch.float32, device=dev)
    buf[1:].copy_(res.reshape(-1))
    shifted = buf[1:].view(res.shape)
    assert shifted.data_ptr() % 16 != 0
    n_total = det.n_total * acq.n_out
    a = [t.clone() for t in E.adjoint_grads(cloud, det, acq, res, 1.0, 2, 2.0 / n_total, E.PassCounters(dev))]
    b = E.adjoint_grads(cloud, det, acq, shifted, 1.0, 2, 2.0 / n_total, E.PassCounters(dev))
    for x, y in zip(a, b):
        assert rel_l2(x.cpu().numpy(), y.cpu().numpy()) < 1e-6
