#!/bin/bash
# A/B of environment switches on the config-2 end-to-end call (tuning, on a gpurun box)
mkdir -p gpurun_out
i=0
for spec in "$@"; do
  i=$((i+1))
  env $spec timeout 600 python bench.py --steps 3 --warmup 3 --e2e-steps 6 --no-cpu --no-recon --no-config1 > gpurun_out/e2e_$i.log 2>&1
  echo "e2e [$spec] rc=$? $(tail -1 gpurun_out/e2e_$i.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["e2e"]["ms_per_step"],3), round(d["e2e"]["pinned"]["ms_per_step"],3), round(d["ms_per_step"],3))' 2>&1 | tail -1)"
done
