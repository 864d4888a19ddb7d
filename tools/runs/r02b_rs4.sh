mkdir -p gpurun_out
rm -f /tmp/tc_arcs_*.npz
python -m pytest tests/test_gpu_parity.py -q -x -k "row_sort or golden or random or single or spec or tiny or empty or closed or skewed or mixed or errors or device_arcs or relabel" > gpurun_out/rs6_t.log 2>&1; echo EXIT $? >> gpurun_out/rs6_t.log
python -m pytest tests/test_gpu_large.py -q -x -k "c4_full" > gpurun_out/rs6_t4.log 2>&1; echo EXIT $? >> gpurun_out/rs6_t4.log
VARIANTS="base" CFGS="C3 C2 C4" bash tools/ab.sh > gpurun_out/rs6_ab.log 2>&1
