mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/rs_launches.csv python tools/quick_time.py C3 > gpurun_out/rs_ncu.log 2>&1
TC_LIB_VARIANT=build/base/libtriadcensus.so ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/base_launches.csv python tools/quick_time.py C3 > gpurun_out/base_ncu.log 2>&1
