mkdir -p gpurun_out
rm -f /tmp/tc_arcs_*.npz
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/end_smoke.log 2>&1; echo EXIT $? >> gpurun_out/end_smoke.log
for c in C3 C2 C4; do
  python bench.py --config $c --steps 20 --warmup 3 > gpurun_out/end_bench_$c.json 2> gpurun_out/end_bench_$c.err
done
