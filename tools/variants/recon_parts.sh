#!/bin/bash
# config-3 reconstruction wall time (min of 3) under forward-partition / adjoint-chunk overrides (tuning, on a gpurun box)
for spec in "$@"; do
  env $spec timeout 600 python -c "
import sys, json; sys.argv=['bench.py']; sys.path.insert(0,'.')
import bench
w = [bench.run_recon(1)[0]['wall_s'] for _ in range(4)]
print('$spec', ' '.join(f'{x:.3f}' for x in w), 'min', round(min(w[1:]), 3))
" 2>&1 | tail -1
done
