import sys, numpy as np
sys.path[:0]=["/root/repo","/root/repo/tests"]
import paper_2601_00551_b200 as P
from paper_2601_00551_b200 import scenes
from pab_helpers import golden, rel_l2
from oracle import render as ORend
g = golden("toy.npz")
sc = scenes.toy_config()
ctx = P.ForwardContext(sc.array, sc.grid)
real = P.SignalSet(sc.grid, g["real"])
keep = g["filter_g"] < 0
lr = P.LearningRates(*g["lr"])
state = P.create_state(sc.init.subset(keep), lr=lr, seed=103)
losses = []
for _ in range(5):
    state, L = P.step(state, ctx, real, 1, "fine"); losses.append(L)
c = state.cloud; init = sc.init.subset(keep)
print("toy losses rel", np.max(np.abs(np.array(losses)/g["step_losses"]-1)))
print("toy dpos rel", rel_l2(c.positions - init.positions, g["final_pos"] - init.positions), "p0", rel_l2(c.p0, g["final_p0"]), "a0", rel_l2(c.a0, g["final_a0"]))
d = np.linalg.norm((c.positions - init.positions) - (g["final_pos"] - init.positions), axis=1)
print("per-ball displacement error quantiles", np.quantile(d, [0.5, 0.99, 1.0]), "lr pos", lr.position)
g = golden("schedule.npz")
ctx = P.ForwardContext(P.SensorArray(g["sensors"]), P.TimeGrid(0.0, 5e-8, 512))
real = P.SignalSet(ctx.grid, g["real"])
n = g["init_pos"].shape[0]
init = P.PointCloud(g["init_pos"], np.full(n, 0.05), np.full(n, 5e-4))
filt, rep = P.zero_gradient_filter(init, ctx, real, f=8)
sched = P.Schedule((P.Level(8, 150, "coarse"), P.Level(2, 60, "fine"), P.Level(1, 60, "fine")), duplication_period=50)
final, trace = P.run_hierarchical(filt.copy(), ctx, real, sched, P.DensityThresholds.from_spacing(4e-4), lr=P.LearningRates.from_spacing(4e-4), seed=P.RngSeed(61), plateau=False)
losses = np.array([r.loss for r in trace.records])
print("schedule loss rel max", np.max(np.abs(losses/g["losses"]-1)), "at", np.argmax(np.abs(losses/g["losses"]-1)))
vol = ORend.voxelize(final.positions, final.p0, final.a0, (31, 31, 31), 2e-4, (-3e-3,) * 3)
print("schedule volume", rel_l2(vol, g["volume"]))
