mkdir -p gpurun_out
rm -f /tmp/tc_arcs_*.npz
TC_LIB_VARIANT=build/xnor/libtriadcensus.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "row_sort or golden or random or spec or tiny or empty or closed or skewed or mixed or device_arcs or relabel or build_sort" > gpurun_out/x_t.log 2>&1; echo EXIT $? >> gpurun_out/x_t.log
VARIANTS="xnor" CFGS="C3 C4 C2" bash tools/ab.sh > gpurun_out/x_ab.log 2>&1
TC_LIB_VARIANT=build/xnor/libtriadcensus.so timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:rs_downsweep --csv --log-file gpurun_out/x_ncu.csv python tools/quick_time.py C3 > gpurun_out/x_ncu.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:rs_downsweep --csv --log-file gpurun_out/b_ncu.csv python tools/quick_time.py C3 > gpurun_out/b_ncu.log 2>&1
