mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_census_hp" -c 1 -o gpurun_out/hp_ncu -f python tools/quick_time.py C3 > gpurun_out/hp_ncu.log 2>&1
