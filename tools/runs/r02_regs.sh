mkdir -p gpurun_out
rm -f /tmp/tc_arcs_*.npz
VARIANTS="minb1" CFGS="C3 C2" bash tools/ab.sh > gpurun_out/ab12.log 2>&1
python bench.py --steps 20 --warmup 3 > gpurun_out/bench_C3.json 2> gpurun_out/bench_C3.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C3.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_census_thread -c 1 -o gpurun_out/full_C3_k_census_thread -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_census_warp -c 1 -o gpurun_out/full_C3_k_census_warp -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
