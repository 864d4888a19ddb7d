mkdir -p gpurun_out
rm -f /tmp/tc_arcs_*.npz
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "row_sort or golden or random or single or spec or tiny or range or closed or skewed or mixed" > gpurun_out/up2_t.log 2>&1; echo EXIT $? >> gpurun_out/up2_t.log
VARIANTS="u5b2 u3b4 base" CFGS="C3" timeout 900 bash tools/ab.sh > gpurun_out/up2_ab.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/up2_C3.csv python tools/quick_time.py C3 > gpurun_out/up2n.log 2>&1
