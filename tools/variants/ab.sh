#!/bin/bash
# A/B step times of library variants on a gpurun box (config 2, no CPU/recon legs):
#   tools/variants/ab.sh base NAME ...     (base = the in-tree library)
mkdir -p gpurun_out
for name in "$@"; do
  if [ "$name" = base ]; then lib=""; else lib=tools/variants/lib_$name.so; fi
  PAB_LIBRARY=$lib timeout 600 python bench.py --steps 6 --warmup 3 --e2e-steps 0 --no-cpu --no-recon --no-config1 \
    > gpurun_out/ab_$name.log 2>&1
  echo "$name rc=$? $(tail -1 gpurun_out/ab_$name.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],3), {k: round(v[1],3) for k,v in d["kernel_ms_min_median"].items()})' 2>&1)"
done
