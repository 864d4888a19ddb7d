mkdir -p gpurun_out
rm -f /tmp/tc_arcs_*.npz
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_task_queues.py -q -x -m gpu > gpurun_out/side_t.log 2>&1; echo EXIT $? >> gpurun_out/side_t.log
for c in C3 C2; do for i in 1 2; do
timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/side_${c}_$i.json 2> /dev/null
TC_LIB_VARIANT=build/base/libtriadcensus.so timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/sidebase_${c}_$i.json 2> /dev/null
done; done
timeout 600 python bench.py --config C4 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/side_C4.json 2> /dev/null
