mkdir -p gpurun_out
rm -f /tmp/tc_arcs_*.npz
timeout 1500 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/full1_gputest.log 2>&1; echo EXIT $? >> gpurun_out/full1_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/full1_smoke.log 2>&1; echo EXIT $? >> gpurun_out/full1_smoke.log
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/full1_bench_C3.json 2> gpurun_out/full1_bench_C3.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_plan_tile|k_census_thread|k_write_upper|k_row_sort_small" -c 4 -o gpurun_out/full1_ncu -f python tools/quick_time.py C3 > gpurun_out/full1_ncu.log 2>&1
