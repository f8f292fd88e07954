python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
PL_SNAP_RR=0 python -m pytest tests/test_gpu_manybody.py -m gpu -q -x -k snap > gpurun_out/pytest_gpu_norr.log 2>&1
python scripts/probe_snap.py > gpurun_out/probe_snap.log 2>&1
PL_SNAP_RR=0 python scripts/probe_snap.py > gpurun_out/probe_snap_norr.log 2>&1
tail -2 gpurun_out/pytest_gpu.log gpurun_out/pytest_gpu_norr.log; cat gpurun_out/probe_snap.log gpurun_out/probe_snap_norr.log
