mkdir -p gpurun_out/fin3
rm -f /tmp/tc_arcs_*.npz
timeout 1800 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/fin3/gputest.log 2>&1; echo EXIT $? >> gpurun_out/fin3/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin3/smoke.log 2>&1; echo EXIT $? >> gpurun_out/fin3/smoke.log
bash tools/runs/r02b_final.sh
