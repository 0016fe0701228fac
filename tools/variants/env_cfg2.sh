#!/bin/bash
# A/B of environment switches on the config-2 step (tuning, on a gpurun box):
#   tools/variants/env_cfg2.sh "PAB_ADJ_A0_BUCKETS=12" "PAB_ADJ_CHUNKS=8 PAB_A0_BUCKETS=5" ...
mkdir -p gpurun_out
i=0
for spec in "$@"; do
  i=$((i+1))
  env $spec timeout 600 python bench.py --steps 6 --warmup 3 --e2e-steps 0 --no-cpu --no-recon --no-config1 > gpurun_out/env_$i.log 2>&1
  echo "cfg2 [$spec] rc=$? $(tail -1 gpurun_out/env_$i.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],3), {k: round(v[1],3) for k,v in d["kernel_ms_min_median"].items()})' 2>&1 | tail -1)"
done
