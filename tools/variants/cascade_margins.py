import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np
import paper_2601_00551_b200 as P
from oracle import radiator as OR
from pab_helpers import rel_l2
for (a0_lo, a0_hi, n, f) in [(0.06, 0.2, 4000, 1), (0.1, 0.2, 4000, 2), (0.045, 0.25, 48, 1), (0.03, 0.05, 3000, 1), (0.12, 0.12, 2000, 1)]:
    rng = np.random.default_rng(97 + n)
    pos = rng.uniform(-3e-3, 3e-3, (n, 3)); p0 = rng.uniform(0.2, 1.0, n)
    a0 = np.exp(rng.uniform(np.log(a0_lo * 1e-3), np.log(a0_hi * 1e-3), n))
    ang = rng.uniform(0, 2 * np.pi, 16)
    sens = np.column_stack([0.03 * np.cos(ang), 0.03 * np.sin(ang), rng.uniform(-0.01, 0.01, 16)])
    nrm = sens / np.linalg.norm(sens, axis=1, keepdims=True)
    grid = P.TimeGrid(0.0, 2.5e-8, 2048); kind = ("cos_power", 2.0)
    ctx = P.ForwardContext(P.SensorArray(sens, 1500.0, normals=nrm), grid, directivity=P.Directivity("cos_power", power=2.0))
    m = max(n // 3, 16)
    real, _, _, _ = OR.run_model(pos[:m], p0[:m], 1.3 * a0[:m], sens, nrm, 1500.0, 0.0, grid.dt, grid.n_samples, f, kind=kind, threads=4)
    _, L, (gp0, ga0, gpos), _ = OR.run_model(pos, p0, a0, sens, nrm, 1500.0, 0.0, grid.dt, grid.n_samples, f, real=real, stage="fine", kind=kind, threads=4)
    sup = P.SignalSet(grid.decimated(f) if f > 1 else grid, real)
    Lg, gr = P.backward(P.PointCloud(pos, p0, a0), ctx, sup, stage="fine")
    print((a0_lo, a0_hi, n, f), f"loss {abs(Lg-L)/L:.1e} p0 {rel_l2(gr.d_p0, gp0):.2e} a0 {rel_l2(gr.d_a0, ga0):.2e} pos {rel_l2(gr.d_position, gpos):.2e}")
