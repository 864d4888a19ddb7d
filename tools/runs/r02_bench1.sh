mkdir -p gpurun_out
(nproc; lscpu | head -20; free -g) > gpurun_out/box.txt 2>&1
python bench.py --steps 20 --warmup 3 > gpurun_out/bench_C3.json 2> gpurun_out/bench_C3.err
python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/ref_C3.json 2> gpurun_out/ref_C3.err
