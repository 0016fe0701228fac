mkdir -p gpurun_out
for m in 1 2; do
  PAB_FORWARD_DUAL_MAXF=$m timeout 600 python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu --no-config1 > gpurun_out/recon_m$m.log 2>&1
  echo "maxf=$m recon $(tail -1 gpurun_out/recon_m$m.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["recon"]["wall_s"], d["recon"]["cold_run_wall_s"], d["recon"]["n_final"], d["recon"]["loss_last"])' 2>&1)"
done
PAB_FORWARD_DUAL_MAXF=2 timeout 900 python -m pytest tests/test_gpu_optimizer.py tests/test_gpu_scale.py tests/test_gpu_radiator.py -q -m gpu -x 2>&1 | tail -3
