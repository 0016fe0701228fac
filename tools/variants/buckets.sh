for b in 4 6 8 12 16; do
  PAB_A0_BUCKETS=$b timeout 600 python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu > gpurun_out/bk_$b.log 2>&1
  echo "b=$b $(tail -1 gpurun_out/bk_$b.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["kernel_ms_min_median"])')"
done
