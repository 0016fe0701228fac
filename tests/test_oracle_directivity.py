"""Pin the oracle's directivity extension (not in the reference, SURVEY §8a
A13): (1) kind "none" equals the reference bit for bit, (2) its analytic
gradients match central finite differences in FP64 (reference pattern
test_radiator.py:177-201), (3) the zero-pressure gradient is the inner
product with the unit-pressure kernel (test_optimizer.py:94-110)."""

import numpy as np
import pytest

from oracle import radiator as OR
from pab_helpers import golden

KINDS = [("cos_power", 2.0), ("cos_power", 3.0), ("element", 5e-4)]


def instance():
    g = golden("radiator.npz")
    return (g["si_sensors"], g["si_normals"], g["si_cand_pos"], g["si_cand_p0"], g["si_cand_a0"],
            g["si_true_pos"], g["si_true_p0"], g["si_true_a0"])


def run(pos, p0, a0, sens, nrm, kind, real=None, f=1, stage="fine"):
    return OR.run_model(pos, p0, a0, sens, nrm, 1500.0, 0.0, 5e-8, 256, f, real=real, stage=stage, kind=kind)


def test_none_is_reference():
    g = golden("radiator.npz")
    sens, nrm, pos, p0, a0, *_ = instance()
    rows, _, _, _ = run(pos, p0, a0, sens, nrm, ("none",))
    assert np.array_equal(rows, g["si_cand_rows"])


@pytest.mark.parametrize("kind", KINDS)
def test_directivity_gradients_match_finite_differences(kind):
    sens, nrm, pos, p0, a0, tpos, tp0, ta0 = instance()
    real, _, _, _ = run(tpos, tp0, ta0, sens, nrm, kind)
    _, _, (gp0, ga0, gpos), _ = run(pos, p0, a0, sens, nrm, kind, real=real)

    def L(pp, pz, az):
        rows, _, _, _ = run(pp, pz, az, sens, nrm, kind)
        return float(np.sum((rows - real) ** 2) / rows.size)

    worst = 0.0
    for i in range(len(p0)):
        for which, h in (("p0", 1e-6), ("a0", 1e-9), ("x", 1e-9), ("y", 1e-9), ("z", 1e-9)):
            pp, pz, az = pos.copy(), p0.copy(), a0.copy()
            qp, qz, qa = pos.copy(), p0.copy(), a0.copy()
            if which == "p0":
                pz[i] += h; qz[i] -= h; want = gp0[i]
            elif which == "a0":
                az[i] += h; qa[i] -= h; want = ga0[i]
            else:
                ax = "xyz".index(which)
                pp[i, ax] += h; qp[i, ax] -= h; want = gpos[i, ax]
            fd = (L(pp, pz, az) - L(qp, qz, qa)) / (2 * h)
            if abs(fd) > 1e-30:
                worst = max(worst, abs(fd - want) / abs(fd))
    assert worst <= 1e-5, worst


@pytest.mark.parametrize("kind", KINDS)
def test_filter_gradient_is_inner_product(kind):
    sens, nrm, pos, p0, a0, tpos, tp0, ta0 = instance()
    real, _, _, _ = run(tpos, tp0, ta0, sens, nrm, kind, f=4)
    n = len(p0)
    _, _, (g, _, _), _ = run(pos, np.zeros(n), a0, sens, nrm, kind, real=real, f=4, stage="coarse")
    for i in range(n):
        k_i, _, _, _ = run(pos[i:i + 1], [1.0], a0[i:i + 1], sens, nrm, kind, f=4)
        ip = float(np.sum(real * k_i))
        assert abs(g[i] + 2.0 * ip / real.size) <= 1e-12 * max(abs(g[i]), 1e-300) + 1e-300
