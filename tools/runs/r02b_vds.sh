mkdir -p gpurun_out
rm -f /tmp/tc_arcs_*.npz
TC_LIB_VARIANT=build/vds/libtriadcensus.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/w_t.log 2>&1; echo EXIT $? >> gpurun_out/v_t.log
VARIANTS="vds" CFGS="C3 C4" bash tools/ab.sh > gpurun_out/w_ab.log 2>&1
TC_LIB_VARIANT=build/vds/libtriadcensus.so timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:rs_downsweep --csv --log-file gpurun_out/w_ncu.csv python tools/quick_time.py C3 > gpurun_out/w_ncu.log 2>&1
