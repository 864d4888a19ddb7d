# Round-2 (second session) evidence: bench lines (C3 headline with cpu_baseline,
# C2, C4, C5, C3 64-type, reference arm), ncu launch lists and --set full
# captures of the census kernels and the build kernels -> gpurun_out/
mkdir -p gpurun_out
O=gpurun_out/fin3
mkdir -p $O
rm -f /tmp/tc_arcs_*.npz
(nproc; lscpu | head -20; free -g; nvidia-smi) > $O/box.txt 2>&1
timeout 900 python bench.py --steps 20 --warmup 3 > $O/bench_C3.json 2> $O/bench_C3.err
timeout 600 python bench.py --config C2 --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_C2.json 2> $O/bench_C2.err
timeout 900 python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_C4.json 2> $O/bench_C4.err
timeout 900 python bench.py --config C5 --steps 3 --warmup 3 > $O/bench_C5.json 2> $O/bench_C5.err
timeout 600 python bench.py --mode 64 --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_C3_mode64.json 2> $O/bench_C3_mode64.err
timeout 1500 python bench.py --impl reference --steps 20 --warmup 3 > $O/bench_reference_C3.json 2> $O/bench_reference_C3.err
for c in C3 C2 C4; do
  st=2; [ $c = C4 ] && st=1
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$c.csv \
    python bench.py --config $c --steps $st --warmup 1 --no-cpu-baseline > /dev/null 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_census_thread|k_census_warp" -c 2 -o $O/full_C3 -f \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_census_warp" -c 1 -o $O/full_C4 -f \
  python bench.py --config C4 --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"rs_downsweep|k_row_sort|k_write_lower|k_head_write|k_upper_plan|k_row_bounds|k_row_classify" -c 16 -o $O/full_C3_build -f \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
ls -la $O
