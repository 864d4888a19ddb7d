mkdir -p gpurun_out
rm -f /tmp/tc_arcs_*.npz
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "row_sort or golden or random or single or spec or tiny or closed or skewed or mixed" > gpurun_out/rside_t.log 2>&1; echo EXIT $? >> gpurun_out/rside_t.log
for i in 1 2 3; do
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/rside_$i.json 2> /dev/null
TC_LIB_VARIANT=build/base/libtriadcensus.so timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/rsidebase_$i.json 2> /dev/null
done
