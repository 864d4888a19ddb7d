mkdir -p gpurun_out
rm -f /tmp/tc_arcs_*.npz
for v in rs8m6 rs8m4; do
TC_LIB_VARIANT=build/$v/libtriadcensus.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "row_sort or golden or random or spec or tiny or empty or closed or skewed or mixed or device_arcs or relabel or build_sort" > gpurun_out/rs_t_$v.log 2>&1; echo EXIT $? >> gpurun_out/rs_t_$v.log
done
VARIANTS="rs8m4 rs8m6 rs8m8 rs16m5" CFGS="C3 C4" bash tools/ab.sh > gpurun_out/rs_ab.log 2>&1
