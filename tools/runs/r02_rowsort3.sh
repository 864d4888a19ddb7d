mkdir -p gpurun_out
rm -f /tmp/tc_arcs_*.npz
python -m pytest tests/test_gpu_parity.py -q -x -k "golden or random or range_small or closed or spec or single or skewed or mixed or tiny or empty" > gpurun_out/t9.log 2>&1; echo EXIT $? >> gpurun_out/t9.log
VARIANTS="prerow" CFGS="C3 C2 C4" bash tools/ab.sh > gpurun_out/ab9.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_row_sort" -c 1 -o gpurun_out/rowsort3 -f python tools/quick_time.py C3 > gpurun_out/ncu9.log 2>&1
