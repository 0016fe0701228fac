#!/bin/bash
# Copy the judged evidence of the last tools/gpu_check.sh run from gpurun_out/
# into profiles/ under a tag:  tools/save_profiles.sh r01_v3
set -eu
tag=$1
out=profiles
cp gpurun_out/bench.log "$out/${tag}_bench.log"
tail -1 gpurun_out/bench.log > "$out/${tag}_bench.json"
cp gpurun_out/launches.csv "$out/${tag}_launches.csv"
{
  echo "# ncu --set full --clock-control none summaries (tools/ncu_summary.py, ncu_pipes.py, ncu_sass_mix.py)"
  for k in fwd adj; do
    echo; echo "## $k"
    python tools/ncu_summary.py gpurun_out/prof_$k.ncu-rep
    python tools/ncu_pipes.py gpurun_out/prof_$k.ncu-rep
    echo "SASS mix per warp-pair (1M balls x 1024 detectors / 32 = 3.2e7 warp-pairs):"
    python tools/ncu_sass_mix.py gpurun_out/prof_$k.ncu-rep 0.5 3.2e7
  done
} > "$out/${tag}_ncu_summary.txt" 2>&1
python tools/ncu_hot_lines.py gpurun_out/prof_fwd.ncu-rep 40 > "$out/${tag}_forward_hotlines.txt" 2>&1
python tools/ncu_hot_lines.py gpurun_out/prof_adj.ncu-rep 40 > "$out/${tag}_adjoint_hotlines.txt" 2>&1
python tools/launch_share.py gpurun_out/launches.csv > "$out/${tag}_launch_share.txt" 2>&1 || true
ls -la $out | grep "$tag"
