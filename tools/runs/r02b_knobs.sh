mkdir -p gpurun_out
rm -f /tmp/tc_arcs_*.npz
VARIANTS="up5 wlb8 wlb2" CFGS="C3" timeout 1500 bash tools/ab.sh > gpurun_out/knobs_ab.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/knobs_up5.csv env TC_LIB_VARIANT=build/up5/libtriadcensus.so python tools/quick_time.py C3 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/knobs_wlb8.csv env TC_LIB_VARIANT=build/wlb8/libtriadcensus.so python tools/quick_time.py C3 > /dev/null 2>&1
