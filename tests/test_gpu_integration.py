"""The reference-side ctypes binding shown in INTEGRATION.md, executed as
written (library path substituted) with this package's model objects
standing in for the reference's ``paball`` modules: the documented seam
``_run_model(cloud, ctx, f, real, stage)`` must reproduce the package's own
forward, loss and gradients."""

import os
import re
import sys
import types

import numpy as np
import pytest

from pab_helpers import rel_l2

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _stub(P):
    from paper_2601_00551_b200 import _lib
    from paper_2601_00551_b200 import radiator as R
    src = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    block = re.search(r"```python\n(# paball/_b200\.py.*?)```", src, re.S).group(1)
    block = block.replace('C.CDLL("libpaball_b200.so")', f"C.CDLL({_lib.LIB_PATH!r})")
    fake_r = types.ModuleType("paball.radiator")
    fake_r.ParamGradients = R.ParamGradients
    fake_r._run_model = None
    fake_m = types.ModuleType("paball.model")
    fake_m.SimulationError = P.SimulationError
    fake = types.ModuleType("paball")
    fake.radiator, fake.model = fake_r, fake_m
    saved = {k: sys.modules.get(k) for k in ("paball", "paball.radiator", "paball.model")}
    sys.modules.update({"paball": fake, "paball.radiator": fake_r, "paball.model": fake_m})
    try:
        ns = {}
        exec(compile(block, "INTEGRATION.md", "exec"), ns)
    finally:
        for k, v in saved.items():
            if v is None:
                sys.modules.pop(k, None)
            else:
                sys.modules[k] = v
    return ns["_run_model_b200"]


def test_integration_stub_matches_package():
    import paper_2601_00551_b200 as P
    run = _stub(P)
    rng = np.random.default_rng(7)
    n = 3000
    pos = rng.uniform(-4e-3, 4e-3, (n, 3))
    cloud = P.PointCloud(pos, rng.uniform(0.2, 1.0, n), rng.uniform(0.05e-3, 0.2e-3, n))
    ang = rng.uniform(0, 2 * np.pi, 16)
    sens = np.column_stack([0.03 * np.cos(ang), 0.03 * np.sin(ang), rng.uniform(-0.01, 0.01, 16)])
    ctx = P.ForwardContext(P.SensorArray(sens, 1500.0), P.TimeGrid(0.0, 2.5e-8, 2048))
    rows, _, _, ops = run(cloud, ctx, 1)
    P.reset_op_count()
    ref = P.simulate_signals(cloud, ctx).data
    assert rel_l2(rows, ref) < 1e-5   # FP32 summation order differs (partitions, bucket count)
    assert ops == P.op_count()
    real = P.SignalSet(ctx.grid, 0.9 * ref + 0.01 * np.abs(ref).max())
    cand = P.PointCloud(pos + rng.normal(scale=2e-5, size=pos.shape), cloud.p0 * 1.1, cloud.a0 * 0.97)
    _, L, g, _ = run(cand, ctx, 1, real=real, stage="fine")
    Lp, gp = P.backward(cand, ctx, real, stage="fine")
    assert abs(L - Lp) <= 1e-6 * Lp
    assert rel_l2(g.d_p0, gp.d_p0) < 1e-5
    assert rel_l2(g.d_a0, gp.d_a0) < 1e-5
    assert rel_l2(g.d_position, gp.d_position) < 1e-5
