python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
for v in 3 5 6; do PL_SNAP_YI=$v python scripts/probe_snap.py > gpurun_out/probe_snap_yi$v.log 2>&1; done
PL_SNAP_YI=6 python -m pytest tests/test_gpu_manybody.py -m gpu -q -x -k "snap and not window" > gpurun_out/pytest_yi6.log 2>&1
tail -2 gpurun_out/pytest_gpu.log; grep -B2 -A15 "Error\|assert" gpurun_out/pytest_gpu.log | head -40; tail -1 gpurun_out/pytest_yi6.log; cat gpurun_out/probe_snap_yi*.log
