mkdir -p gpurun_out
rm -f /tmp/tc_arcs_*.npz
TC_LIB_VARIANT=build/wlh2/libtriadcensus.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "row_sort or golden or random or single or spec or tiny or empty or closed or skewed or mixed or errors or device_arcs or relabel" > gpurun_out/wlh_t.log 2>&1; echo EXIT $? >> gpurun_out/wlh_t.log
VARIANTS="wlh1 wlh2" CFGS="C3 C2" bash tools/ab.sh > gpurun_out/wlh_ab.log 2>&1
for v in wlh2; do
TC_LIB_VARIANT=build/$v/libtriadcensus.so timeout 300 ncu --set full --clock-control none -k regex:k_write_lower -c 1 --csv --page raw --log-file gpurun_out/wlh_ncu_$v.csv python tools/quick_time.py C3 > gpurun_out/wlh_ncu_$v.log 2>&1
done
timeout 300 ncu --set full --clock-control none -k regex:k_upper_plan -c 1 --csv --page raw --log-file gpurun_out/up_ncu.csv python tools/quick_time.py C3 > gpurun_out/up_ncu.log 2>&1
