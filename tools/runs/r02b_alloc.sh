mkdir -p gpurun_out
for al in pool torch; do
  timeout 600 python bench.py --config C4 --steps 3 --warmup 2 --no-cpu-baseline --alloc $al > gpurun_out/al_C4_$al.json 2> gpurun_out/al_C4_$al.err
  timeout 600 python bench.py --mode 64 --steps 5 --warmup 3 --no-cpu-baseline --alloc $al > gpurun_out/al_m64_$al.json 2> gpurun_out/al_m64_$al.err
done
TC_LIB_VARIANT=build/base/libtriadcensus.so timeout 600 python bench.py --config C4 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/al_C4_base.json 2> gpurun_out/al_C4_base.err
