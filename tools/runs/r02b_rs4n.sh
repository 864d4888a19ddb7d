mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/rs4_C4.csv python tools/quick_time.py C4 > gpurun_out/rs4n.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/rs4_C2.csv python tools/quick_time.py C2 >> gpurun_out/rs4n.log 2>&1
