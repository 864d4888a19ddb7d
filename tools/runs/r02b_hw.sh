mkdir -p gpurun_out
rm -f /tmp/tc_arcs_*.npz
VARIANTS="hw5 hw6" CFGS="C3 C4" bash tools/ab.sh > gpurun_out/hw_ab.log 2>&1
