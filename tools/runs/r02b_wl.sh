mkdir -p gpurun_out
rm -f /tmp/tc_arcs_*.npz
python -m pytest tests/test_gpu_parity.py -q -x -k "row_sort or golden or random or single or spec or tiny or empty or closed or skewed or mixed or errors or device_arcs or relabel" > gpurun_out/wl_t.log 2>&1; echo EXIT $? >> gpurun_out/wl_t.log
VARIANTS="wl1 wl4 base" CFGS="C3" bash tools/ab.sh > gpurun_out/wl_ab.log 2>&1
python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/wl_bench_C3.json 2> gpurun_out/wl_bench_C3.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/wl_C3.csv python tools/quick_time.py C3 > gpurun_out/wln.log 2>&1
