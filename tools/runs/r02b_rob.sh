mkdir -p gpurun_out
rm -f /tmp/tc_arcs_*.npz
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_task_queues.py -q -x -m gpu > gpurun_out/rob_t.log 2>&1; echo EXIT $? >> gpurun_out/rob_t.log
timeout 600 python -m pytest tests/test_gpu_large.py -q -x -k "c4_full or costliest" > gpurun_out/rob_t4.log 2>&1; echo EXIT $? >> gpurun_out/rob_t4.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/rob_smoke.log 2>&1; echo EXIT $? >> gpurun_out/rob_smoke.log
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/rob_C3.json 2> /dev/null
