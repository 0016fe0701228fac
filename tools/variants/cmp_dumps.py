"""Compare two rows_dump.py outputs: bitwise-equal fields and relative L2."""
import sys

import numpy as np

a, b = np.load(sys.argv[1]), np.load(sys.argv[2])
for k in a.files:
    x, y = a[k], b[k]
    same = np.array_equal(x, y)
    rel = float(np.linalg.norm(x - y) / max(np.linalg.norm(x), 1e-300))
    print(f"{k}: bitwise {'equal' if same else 'DIFFERENT'}, rel L2 {rel:.3e}")
