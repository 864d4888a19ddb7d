mkdir -p gpurun_out
rm -f /tmp/tc_arcs_*.npz
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/f4_gputest.log 2>&1; echo EXIT $? >> gpurun_out/f4_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f4_smoke.log 2>&1; echo EXIT $? >> gpurun_out/f4_smoke.log
python bench.py --steps 20 --warmup 3 > gpurun_out/f4_bench_C3.json 2> gpurun_out/f4_bench_C3.err
python bench.py --config C2 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/f4_bench_C2.json 2> gpurun_out/f4_bench_C2.err
python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/f4_bench_C4.json 2> gpurun_out/f4_bench_C4.err
python bench.py --mode 64 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/f4_bench_C3_mode64.json 2> gpurun_out/f4_bench_C3_mode64.err
timeout 900 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/f4_bench_C5.json 2> gpurun_out/f4_bench_C5.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/f4_bench_reference_C3.json 2> gpurun_out/f4_bench_reference_C3.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f4_launches_C3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/f4_ncu.log 2>&1
