#!/bin/bash
# GPU box: bench lines + ncu launch lists + ncu --set full captures of the bin
# kernels for C3 (bench workload), C2 and C4 -> gpurun_out/ (summarised into
# profiles/ by tools/make_profiles.py)
cd "$(dirname "$0")/.."
O=gpurun_out
python bench.py --steps 20 --warmup 3 > $O/bench_C3.json 2> $O/bench_C3.err
python bench.py --config C2 --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_C2.json 2> $O/bench_C2.err
python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_C4.json 2> $O/bench_C4.err
for c in C3 C2 C4; do
  st=2; [ $c = C4 ] && st=1
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$c.csv \
    python bench.py --config $c --steps $st --warmup 1 --no-cpu-baseline > /dev/null 2>&1
  for k in k_census_thread k_census_warp; do
    ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o $O/full_${c}_$k -f \
      python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
  done
done
ls $O
