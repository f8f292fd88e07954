python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
python scripts/probe_sweep.py > gpurun_out/probe_sweep.log 2>&1
tail -1 gpurun_out/pytest_gpu.log; grep N_atoms gpurun_out/probe_sweep.log
