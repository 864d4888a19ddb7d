bash tools/runs/r02b_rs4.sh
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/rs6_C3.csv python tools/quick_time.py C3 > gpurun_out/rs6n.log 2>&1
