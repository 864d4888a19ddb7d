mkdir -p gpurun_out
# C4 golden ranges on the host cores in the background (reverse order; the
# container runs them forward), 14 of 16 cores
(timeout 3300 python tests/golden/make_golden_sharded.py C4 --procs 14 --chunks 448 --reverse --cache gpurun_out/c4_box.jsonl --no-write > gpurun_out/golden_box.log 2>&1 &)
python -m pytest tests/test_gpu_parity.py -q -x -k "golden or random or range or shard or closed or spec or single" > gpurun_out/t6.log 2>&1; echo EXIT $? >> gpurun_out/t6.log
VARIANTS="ds0 dsfull" CFGS="C3 C4" bash tools/ab.sh > gpurun_out/ab6.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"rs_downsweep|k_write_lower|k_head_write|k_write_upper|k_head_count" -c 9 -o gpurun_out/build_full2 -f python tools/quick_time.py C3 > gpurun_out/ncu6.log 2>&1
wait
sleep 3000
