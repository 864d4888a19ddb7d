mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "golden or random or row_sort or range_small or skewed or census64 or concurrent or multi" > gpurun_out/al2_t.log 2>&1; echo EXIT $? >> gpurun_out/al2_t.log
for al in pool torch; do
  timeout 600 python bench.py --config C4 --steps 3 --warmup 2 --no-cpu-baseline --alloc $al > gpurun_out/al2_C4_$al.json 2> gpurun_out/al2_C4_$al.err
  timeout 600 python bench.py --mode 64 --steps 10 --warmup 3 --no-cpu-baseline --alloc $al > gpurun_out/al2_m64_$al.json 2> gpurun_out/al2_m64_$al.err
  timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --alloc $al > gpurun_out/al2_C3_$al.json 2> gpurun_out/al2_C3_$al.err
done
