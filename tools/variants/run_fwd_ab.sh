#!/bin/bash
# forward variant A/B on a gpurun box: rows bitwise vs the variant library, step times
#   tools/variants/run_fwd_ab.sh VARIANT
v=$1
mkdir -p gpurun_out
PAB_LIBRARY=tools/variants/lib_$v.so timeout 300 python tools/variants/rows_dump.py gpurun_out/d_$v.npz > gpurun_out/dump0.log 2>&1
timeout 300 python tools/variants/rows_dump.py gpurun_out/d_base.npz > gpurun_out/dump1.log 2>&1
python tools/variants/cmp_dumps.py gpurun_out/d_$v.npz gpurun_out/d_base.npz
rm -f gpurun_out/d_*.npz
bash tools/variants/ab.sh base $v base $v
