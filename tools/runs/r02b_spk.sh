mkdir -p gpurun_out
rm -f /tmp/tc_arcs_*.npz
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "skewed or mixed or golden or closed or range_small" > gpurun_out/spk_t.log 2>&1; echo EXIT $? >> gpurun_out/spk_t.log
timeout 600 python -m pytest tests/test_gpu_large.py -q -x -k "c4_full or costliest" > gpurun_out/spk_t4.log 2>&1; echo EXIT $? >> gpurun_out/spk_t4.log
VARIANTS="spk1 spk4 base" CFGS="C4 C2" timeout 900 bash tools/ab.sh > gpurun_out/spk_ab.log 2>&1
