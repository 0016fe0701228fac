#!/bin/bash
# usage: tools/variants/run_variants_env.sh NAME:ENVSTRING ...  (ENVSTRING: VAR=v,VAR2=w)
mkdir -p gpurun_out
for spec in "$@"; do
  name=${spec%%:*}; envs=${spec#*:}
  env ${envs//,/ } PAB_LIBRARY=tools/variants/lib_$name.so timeout 600 python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu > gpurun_out/var_$name.log 2>&1
  echo "$name $envs rc=$? $(tail -1 gpurun_out/var_$name.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["kernel_ms_min_median"])' 2>&1)"
done
