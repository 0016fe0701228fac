#!/bin/bash
# A/B of environment switches on config 2 step times and the config-3 reconstruction (tuning, on a gpurun box)
for spec in "$@"; do
  env $spec timeout 600 python bench.py --steps 6 --warmup 3 --e2e-steps 0 --no-cpu --no-recon --no-config1 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg2 $spec', round(d['ms_per_step'],3), {k: round(v[1],3) for k,v in d['kernel_ms_min_median'].items()})"
done
tools/variants/recon_parts.sh "$@"
