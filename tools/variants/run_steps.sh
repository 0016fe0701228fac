for v in "$@"; do
  if [ "$v" = base ]; then lib=""; else lib="PAB_LIBRARY=tools/variants/lib_$v.so"; fi
  echo "$v: $(env $lib timeout 300 python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu 2>&1 | grep step_ms)"
done
