mkdir -p gpurun_out
rm -f /tmp/tc_arcs_*.npz
timeout 1500 python -m pytest tests -m gpu -q -x --durations=5 > gpurun_out/full2_gputest.log 2>&1; echo EXIT $? >> gpurun_out/full2_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/full2_smoke.log 2>&1; echo EXIT $? >> gpurun_out/full2_smoke.log
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/full2_bench_C3.json 2> gpurun_out/full2_bench_C3.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/full2_launches_C3.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
