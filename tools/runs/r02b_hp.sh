mkdir -p gpurun_out
rm -f /tmp/tc_arcs_*.npz
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "single or spec or tiny or empty or random or golden or row_sort or closed or skewed or mixed or relabel or device_arcs" > gpurun_out/hp2_t.log 2>&1; echo EXIT $? >> gpurun_out/hp2_t.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/hp2_smoke.log 2>&1; echo EXIT $? >> gpurun_out/hp2_smoke.log
timeout 600 python tools/quick_time.py C3 > gpurun_out/hp2_qt.log 2>&1
TC_LIB_VARIANT=build/base/libtriadcensus.so timeout 600 python tools/quick_time.py C3 >> gpurun_out/hp2_qt.log 2>&1
