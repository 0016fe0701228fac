mkdir -p gpurun_out
for name in base m14; do
  if [ "$name" = base ]; then lib=""; else lib=tools/variants/lib_$name.so; fi
  PAB_LIBRARY=$lib timeout 600 python bench.py --config 4 --steps 4 --warmup 3 --e2e-steps 0 --no-cpu --no-recon --no-config1 > gpurun_out/c4_$name.log 2>&1
  echo "$name c4 $(tail -1 gpurun_out/c4_$name.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],2), d["kernel_ms_min_median"])' 2>&1)"
  PAB_LIBRARY=$lib timeout 600 python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu --no-config1 > gpurun_out/recon_$name.log 2>&1
  echo "$name recon $(tail -1 gpurun_out/recon_$name.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["recon"]["wall_s"], d["recon"]["cold_run_wall_s"])' 2>&1)"
done
