python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
python scripts/probe_snap.py > gpurun_out/probe_snap.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_snap_yi_reg" -s 4 -c 2 -o gpurun_out/prof_yireg python scripts/probe_snap.py > gpurun_out/ncu_yireg.log 2>&1
tail -2 gpurun_out/pytest_gpu.log; grep -B2 -A15 "Error\|assert" gpurun_out/pytest_gpu.log | head -40; cat gpurun_out/probe_snap.log; tail -2 gpurun_out/ncu_yireg.log
