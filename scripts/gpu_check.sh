python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
python scripts/probe_snap.py > gpurun_out/probe_snap.log 2>&1
PL_SNAP_YI=3 python scripts/probe_snap.py > gpurun_out/probe_snap_yi3.log 2>&1
PL_SNAP_YI=3 python -m pytest tests/test_gpu_manybody.py -m gpu -q -x -k snap > gpurun_out/pytest_gpu_yi3.log 2>&1
tail -2 gpurun_out/pytest_gpu.log; tail -1 gpurun_out/pytest_gpu_yi3.log; cat gpurun_out/probe_snap.log gpurun_out/probe_snap_yi3.log
