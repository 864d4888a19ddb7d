mkdir -p gpurun_out
rm -f /tmp/tc_arcs_*.npz
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "row_sort or golden or random or single or spec or tiny or empty or closed or skewed or mixed or errors or device_arcs or relabel or range_small" > gpurun_out/one2_t.log 2>&1; echo EXIT $? >> gpurun_out/one2_t.log
timeout 300 python -m pytest tests/test_gpu_large.py -q -x -k "c4_full" > gpurun_out/one2_t4.log 2>&1; echo EXIT $? >> gpurun_out/one2_t4.log
VARIANTS="noone" CFGS="C3 C2 C4" timeout 600 bash tools/ab.sh > gpurun_out/one2_ab.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/one2_C3.csv python tools/quick_time.py C3 > gpurun_out/onen.log 2>&1
