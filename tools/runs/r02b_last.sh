mkdir -p gpurun_out/last
O=gpurun_out/last
rm -f /tmp/tc_arcs_*.npz
timeout 1800 python -m pytest tests -m gpu -q -x --durations=5 > $O/gputest.log 2>&1; echo EXIT $? >> $O/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo EXIT $? >> $O/smoke.log
timeout 900 python bench.py --steps 20 --warmup 3 > $O/bench_C3.json 2> $O/bench_C3.err
timeout 600 python bench.py --config C2 --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_C2.json 2> $O/bench_C2.err
timeout 900 python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_C4.json 2> $O/bench_C4.err
timeout 600 python bench.py --mode 64 --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_C3_mode64.json 2> $O/bench_C3_mode64.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C3.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
