mkdir -p gpurun_out
rm -f /tmp/tc_arcs_*.npz
python -m pytest tests -m gpu -q --durations=20 > gpurun_out/gputest_full.log 2>&1; echo EXIT $? >> gpurun_out/gputest_full.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo EXIT $? >> gpurun_out/smoke.log
bash tools/runs/r02_final.sh
