mkdir -p gpurun_out
rm -f /tmp/tc_arcs_*.npz
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "row_sort or golden or random or single or spec or tiny or range_small or closed or skewed or mixed or census64" > gpurun_out/pipe_t.log 2>&1; echo EXIT $? >> gpurun_out/pipe_t.log
VARIANTS="nopipe wpipe0" CFGS="C3 C2 C4" timeout 900 bash tools/ab.sh > gpurun_out/pipe_ab.log 2>&1
