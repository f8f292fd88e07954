python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
python scripts/probe_sweep.py > gpurun_out/probe_sweep.log 2>&1
python scripts/probe_snap.py > gpurun_out/probe_snap.log 2>&1
tail -1 gpurun_out/pytest_gpu.log; grep -B2 -A15 "Error\|assert" gpurun_out/pytest_gpu.log | head -30; grep N_atoms gpurun_out/probe_sweep.log; grep SNAP gpurun_out/probe_snap.log
