mkdir -p gpurun_out
rm -f /tmp/tc_arcs_*.npz
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/hwnd_t.log 2>&1; echo EXIT $? >> gpurun_out/hwnd_t.log
timeout 600 python -m pytest tests/test_gpu_large.py -q -x -k "c4_full" > gpurun_out/hwnd_t4.log 2>&1; echo EXIT $? >> gpurun_out/hwnd_t4.log
for i in 1 2 3; do
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/hwnd_$i.json 2> /dev/null

TC_LIB_VARIANT=build/base/libtriadcensus.so timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/hwnd_base_$i.json 2> /dev/null
done
