python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
python scripts/probe_snap.py > gpurun_out/probe_snap.log 2>&1
PL_SNAP_YI=3 python scripts/probe_snap.py > gpurun_out/probe_snap_yi3.log 2>&1
tail -2 gpurun_out/pytest_gpu.log; grep -B2 -A12 "Error\|assert" gpurun_out/pytest_gpu.log | head -30; cat gpurun_out/probe_snap.log gpurun_out/probe_snap_yi3.log
