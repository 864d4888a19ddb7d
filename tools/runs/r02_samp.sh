mkdir -p gpurun_out
rm -f /tmp/tc_arcs_*.npz
python -m pytest tests/test_gpu_parity.py -q -x -k "skewed or hub or mixed or closed or golden or concurrent" > gpurun_out/t11.log 2>&1; echo EXIT $? >> gpurun_out/t11.log
python -m pytest tests/test_gpu_large.py -q -x -k "c4_full or c4_every or costliest or c5" >> gpurun_out/t11.log 2>&1; echo EXIT $? >> gpurun_out/t11.log
VARIANTS="nosamp" CFGS="C4 C2 C5" bash tools/ab.sh > gpurun_out/ab11.log 2>&1
