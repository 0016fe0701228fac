mkdir -p gpurun_out
PAB_LIBRARY=tools/variants/lib_bench.so timeout 300 python tools/variants/adj_walk_bench.py > gpurun_out/walk.log 2>&1; echo "walk rc=$?"; cat gpurun_out/walk.log | tail -12
PAB_LIBRARY=tools/variants/lib_nocasc.so timeout 300 python tools/variants/rows_dump.py gpurun_out/d_nocasc.npz > gpurun_out/dump0.log 2>&1
timeout 300 python tools/variants/rows_dump.py gpurun_out/d_casc.npz > gpurun_out/dump1.log 2>&1
python tools/variants/cmp_dumps.py gpurun_out/d_nocasc.npz gpurun_out/d_casc.npz
rm -f gpurun_out/d_*.npz
bash tools/variants/ab.sh base nocasc base nocasc
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/gpu_tests.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
