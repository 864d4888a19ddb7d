mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:"k_census_warp" -c 1 -o gpurun_out/c4_warp -f python tools/quick_time.py C4 > gpurun_out/ncu_c4.log 2>&1
python tools/quick_time.py C4 > gpurun_out/qt_c4.log 2>&1
