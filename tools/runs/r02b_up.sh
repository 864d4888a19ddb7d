mkdir -p gpurun_out
rm -f /tmp/tc_arcs_*.npz
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_task_queues.py -q -x > gpurun_out/up_t.log 2>&1; echo EXIT $? >> gpurun_out/up_t.log
timeout 300 python -m pytest tests/test_gpu_large.py -q -x -k "c4_full" > gpurun_out/up_t4.log 2>&1; echo EXIT $? >> gpurun_out/up_t4.log
VARIANTS="up4 base" CFGS="C3 C2 C4" timeout 900 bash tools/ab.sh > gpurun_out/up_ab.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/up_C3.csv python tools/quick_time.py C3 > gpurun_out/upn.log 2>&1
