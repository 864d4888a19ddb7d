mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -q -x -k "single or random or golden or range_small or mixed or skewed or spec" > gpurun_out/t2.log 2>&1; echo EXIT $? >> gpurun_out/t2.log
VARIANTS="tab0 reg5" CFGS="C3 C2" bash tools/ab.sh > gpurun_out/ab2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"rs_downsweep|k_write_lower|k_head_write|rs_upsweep|k_census_thread" -c 16 -o gpurun_out/build_full -f python tools/quick_time.py C3 > gpurun_out/ncu2.log 2>&1
ls -la gpurun_out
