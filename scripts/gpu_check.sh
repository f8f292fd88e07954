for v in 3 6; do PL_SNAP_YI=$v python scripts/probe_snap.py > gpurun_out/probe_snap_yi$v.log 2>&1; done
PL_SNAP_YI=6 python -m pytest tests/test_gpu_manybody.py -m gpu -q -x -k "snap and not window" > gpurun_out/pytest_yi6.log 2>&1
tail -1 gpurun_out/pytest_yi6.log; grep SNAP gpurun_out/probe_snap_yi*.log
