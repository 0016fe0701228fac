import numpy as np, sys, os
sys.path.insert(0, ".")
import paper_2601_00551_b200 as P
cloud = P.PointCloud([[0.0, 0.0, 0.0]], [1.0], [0.5e-3])
array = P.SensorArray(positions=[[0.03, 0.0, 0.0]], sound_speed=1500.0)
ctx = P.ForwardContext(array, P.TimeGrid(0.0, 1e-8, 4096))
s = P.simulate_signals(cloud, ctx).data[0]
np.save(sys.argv[1], s)
nz = np.nonzero(s)[0]
print(os.environ.get("PAB_LIBRARY", "base"), "nonzero", nz.min() if nz.size else None, nz.max() if nz.size else None, "nan", np.isnan(s).sum(), "argmin", np.argmin(s), "argmax", np.argmax(s), s[1990:2010:4])
