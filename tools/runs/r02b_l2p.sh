mkdir -p gpurun_out
rm -f /tmp/tc_arcs_*.npz
VARIANTS="l2p" CFGS="C3 C4" timeout 1200 bash tools/ab.sh > gpurun_out/l2p_ab.log 2>&1
