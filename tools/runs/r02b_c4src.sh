mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_census_warp" -c 1 -o gpurun_out/c4_warp -f python tools/quick_time.py C4 > gpurun_out/c4src.log 2>&1
