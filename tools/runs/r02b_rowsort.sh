mkdir -p gpurun_out
rm -f /tmp/tc_arcs_*.npz
python -m pytest tests/test_gpu_parity.py -q -x -k "row_sort or golden or random or single or spec or tiny or empty or closed or skewed or mixed or errors or device_arcs" > gpurun_out/rs_t.log 2>&1; echo EXIT $? >> gpurun_out/rs_t.log
VARIANTS="base" CFGS="C3 C2 C4" bash tools/ab.sh > gpurun_out/rs_ab.log 2>&1
python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/rs_bench_C3.json 2> gpurun_out/rs_bench_C3.err
