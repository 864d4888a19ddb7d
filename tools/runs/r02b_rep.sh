mkdir -p gpurun_out
rm -f /tmp/tc_arcs_*.npz
python -m pytest tests/test_gpu_parity.py -q -x -k "row_sort or golden or random or single or spec or tiny or empty or closed or skewed or mixed or errors or device_arcs or relabel or range_small" > gpurun_out/rep_t.log 2>&1; echo EXIT $? >> gpurun_out/rep_t.log
VARIANTS="norep" CFGS="C3 C2" bash tools/ab.sh > gpurun_out/rep_ab.log 2>&1
python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/rep_bench_C3.json 2> gpurun_out/rep_bench_C3.err
ncu --set full --clock-control none --import-source on -k regex:"k_census_thread" -c 1 -o gpurun_out/rep_thread -f python tools/quick_time.py C3 > gpurun_out/rep_ncu.log 2>&1
