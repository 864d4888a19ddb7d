mkdir -p gpurun_out/fin2
timeout 900 python bench.py --config C5 --steps 3 --warmup 3 > gpurun_out/fin2/bench_C5.json 2> gpurun_out/fin2/bench_C5.err
timeout 600 python bench.py --config C4 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/fin2/bench_C4_recheck.json 2> /dev/null
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/fin2/bench_C3_recheck.json 2> /dev/null
