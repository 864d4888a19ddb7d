mkdir -p gpurun_out
VARIANTS="nol1" CFGS="C3 C2 C4" bash tools/ab.sh > gpurun_out/l1_ab.log 2>&1
ncu --section LaunchStats --section MemoryWorkloadAnalysis -k regex:"k_census_thread|k_census_warp" -c 2 python tools/quick_time.py C3 > gpurun_out/l1_ncu.txt 2>&1
TC_LIB_VARIANT=build/nol1/libtriadcensus.so ncu --section LaunchStats -k regex:"k_census_thread|k_census_warp" -c 2 python tools/quick_time.py C3 > gpurun_out/l1_ncu_nol1.txt 2>&1
