"""Interchange fixtures written by the reference's own writers
(reference formats.py:97-243), run once in this container; the tests compare
this package's writers byte for byte and its readers value for value.

  sig.pasg     3 x 5 rows, t0 = -1.25e-6, dt = 2.5e-8
  cloud.pcbg   4 balls
  vol.pavx     3 x 4 x 2 volume, origin (-1e-3, 2e-3, 0.5e-3), spacing 2.5e-4
  sensors3.csv / sensors6.csv   5 sensors without / with normals
  img.pgm / img.f32             6 x 4 image (one negative pixel)
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import load_reference  # noqa: E402

OUT = os.path.join(HERE, "formats")


def main() -> None:
    load_reference()
    from paball import formats as F
    from paball.model import CounterRng, PointCloud, SensorArray, SignalSet, TimeGrid, VoxelGrid

    r = CounterRng(31)
    os.makedirs(OUT, exist_ok=True)
    F.write_signals(os.path.join(OUT, "sig.pasg"),
                    SignalSet(TimeGrid(-1.25e-6, 2.5e-8, 5), r.uniform(-2, 2, 15).reshape(3, 5)))
    F.write_cloud(os.path.join(OUT, "cloud.pcbg"),
                  PointCloud(r.uniform(-5e-3, 5e-3, 12).reshape(4, 3), r.uniform(0.1, 2, 4), r.uniform(1e-4, 6e-4, 4)))
    F.write_volume(os.path.join(OUT, "vol.pavx"),
                   VoxelGrid((3, 4, 2), 2.5e-4, np.array([-1e-3, 2e-3, 0.5e-3]), r.uniform(-1, 1, 24).reshape(3, 4, 2)))
    pos = r.uniform(-0.02, 0.02, 15).reshape(5, 3)
    nrm = pos / np.linalg.norm(pos, axis=1, keepdims=True)
    F.write_sensors_csv(os.path.join(OUT, "sensors3.csv"), SensorArray(pos))
    F.write_sensors_csv(os.path.join(OUT, "sensors6.csv"), SensorArray(pos, normals=nrm))
    img = r.uniform(0, 3, 24).reshape(6, 4)
    img[2, 1] = -0.5
    F.write_pgm(os.path.join(OUT, "img.pgm"), img)
    F.write_float_sidecar(os.path.join(OUT, "img.f32"), img)
    np.savez(os.path.join(OUT, "values.npz"), img=img, pos=pos, nrm=nrm)


if __name__ == "__main__":
    main()
