#!/bin/bash
# forward variant A/B on a gpurun box: rows / gradients bitwise vs the variant
# library at full rate and decimated, step times, config-3 reconstruction
#   tools/variants/run_fwd_ab.sh VARIANT
v=$1
mkdir -p gpurun_out
for f in 1 2; do
  F=$f PAB_LIBRARY=tools/variants/lib_$v.so timeout 300 python tools/variants/rows_dump.py gpurun_out/d_$v.npz > gpurun_out/dump0.log 2>&1
  F=$f timeout 300 python tools/variants/rows_dump.py gpurun_out/d_base.npz > gpurun_out/dump1.log 2>&1
  echo "f=$f"; python tools/variants/cmp_dumps.py gpurun_out/d_$v.npz gpurun_out/d_base.npz
done
rm -f gpurun_out/d_*.npz
bash tools/variants/ab.sh base $v base $v
for name in base $v; do
  if [ "$name" = base ]; then lib=""; else lib=tools/variants/lib_$name.so; fi
  PAB_LIBRARY=$lib timeout 600 python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu --no-config1 > gpurun_out/recon_$name.log 2>&1
  echo "$name recon $(tail -1 gpurun_out/recon_$name.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["recon"]["wall_s"], d["recon"]["cold_run_wall_s"])' 2>&1)"
done
