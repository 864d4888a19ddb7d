mkdir -p gpurun_out
rm -f /tmp/tc_arcs_*.npz
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/base_box.txt 2>&1
python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/base_gputest.log 2>&1; echo EXIT $? >> gpurun_out/base_gputest.log
python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/base_bench_C3.json 2> gpurun_out/base_bench_C3.err
for c in C3 C2 C4; do python tools/quick_time.py $c; done > gpurun_out/base_qt.log 2>&1
