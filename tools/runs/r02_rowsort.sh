mkdir -p gpurun_out
rm -f /tmp/tc_arcs_*.npz
python -m pytest tests/test_gpu_parity.py tests/test_task_queues.py tests/test_io.py -q -x -m gpu > gpurun_out/t7.log 2>&1; echo EXIT $? >> gpurun_out/t7.log
python -m pytest tests/test_gpu_large.py -q -x -k "costliest or c5" >> gpurun_out/t7.log 2>&1; echo EXIT $? >> gpurun_out/t7.log
VARIANTS="prerow sp64 wla2 tla2 ds0" CFGS="C3 C2 C4" bash tools/ab.sh > gpurun_out/ab7.log 2>&1
(echo "== torch alloc 0"; TC_TORCH_ALLOC=0 python tools/quick_time.py C3 2>&1 | tail -3 | head -2) >> gpurun_out/ab7.log
