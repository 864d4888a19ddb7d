mkdir -p gpurun_out
rm -f /tmp/tc_arcs_*.npz
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_io.py tests/test_task_queues.py -q -x -m gpu > gpurun_out/lazy_t.log 2>&1; echo EXIT $? >> gpurun_out/lazy_t.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/lazy_smoke.log 2>&1; echo EXIT $? >> gpurun_out/lazy_smoke.log
for i in 1 2; do
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/lazy_bench_$i.json 2> /dev/null
TC_LIB_VARIANT=build/base/libtriadcensus.so timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/lazy_base_$i.json 2> /dev/null
done
