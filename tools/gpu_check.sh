#!/bin/bash
# Run on a gpurun box: GPU tests, bench, launch list, ncu captures of the two hot kernels.
# usage: tools/gpu_check.sh [tests] [bench] [ncu]
set -u
mkdir -p gpurun_out
for what in "$@"; do
  case $what in
    tests)
      timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" ;;
    smoke)
      timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" ;;
    bench)
      timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" ;;
    ncu)
      SMALL="python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu --no-recon --no-config1"
      timeout 300 $SMALL > gpurun_out/bench_small.log 2>&1 && \
      timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $SMALL > gpurun_out/ncu1.log 2>&1 && \
      timeout 900 ncu --set full --clock-control none --import-source on -k regex:forward_kernel -c 1 -o gpurun_out/prof_fwd -f $SMALL > gpurun_out/ncu2.log 2>&1; \
      timeout 900 ncu --set full --clock-control none --import-source on -k regex:adjoint_kernel -c 1 -o gpurun_out/prof_adj -f $SMALL > gpurun_out/ncu3.log 2>&1; echo "ncu rc=$?" ;;
  esac
done
