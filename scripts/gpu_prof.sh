# correctness + stage timing + ncu full capture of the SNAP kernels on the probe
python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
python scripts/probe_snap.py > gpurun_out/probe_snap.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_snap_ -s 12 -c 4 -o gpurun_out/prof_snap2 python scripts/probe_snap.py > gpurun_out/ncu_full2.log 2>&1
tail -2 gpurun_out/pytest_gpu.log; cat gpurun_out/probe_snap.log; tail -3 gpurun_out/ncu_full2.log
