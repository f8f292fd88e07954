python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
for v in 6 7; do PL_SNAP_YI=$v python scripts/probe_snap.py > gpurun_out/probe_snap_yi$v.log 2>&1; done
PL_SNAP_YI=7 python -m pytest tests/test_gpu_manybody.py -m gpu -q -x -k "snap and not window" > gpurun_out/pytest_yi7.log 2>&1
tail -1 gpurun_out/pytest_gpu.log; tail -1 gpurun_out/pytest_yi7.log; grep SNAP gpurun_out/probe_snap_yi*.log
