mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_task_queues.py -q -x -k "skewed or mixed or golden or random or hub or shard or closed or census64" > gpurun_out/t4.log 2>&1; echo EXIT $? >> gpurun_out/t4.log
python -m pytest tests/test_gpu_large.py -q -x -k "costliest" >> gpurun_out/t4.log 2>&1; echo EXIT $? >> gpurun_out/t4.log
VARIANTS="tab0 noint nostage c1024" CFGS="C4 C2" bash tools/ab.sh > gpurun_out/ab4.log 2>&1
