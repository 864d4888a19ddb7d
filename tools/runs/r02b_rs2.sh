mkdir -p gpurun_out
rm -f /tmp/tc_arcs_*.npz
python -m pytest tests/test_gpu_parity.py -q -x -k "row_sort or golden or random or single or spec or tiny or empty or closed or skewed or mixed or errors or device_arcs" > gpurun_out/rs3_t.log 2>&1; echo EXIT $? >> gpurun_out/rs3_t.log
VARIANTS="base" CFGS="C3 C2" bash tools/ab.sh > gpurun_out/rs3_ab.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/rs3_launches.csv python tools/quick_time.py C3 > gpurun_out/rs3_ncu.log 2>&1
