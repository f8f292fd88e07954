python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
PL_SNAP_YI=5 python scripts/probe_snap.py > gpurun_out/probe5.log 2>&1 && PL_SNAP_YI=6 python scripts/probe_snap.py > gpurun_out/probe6.log 2>&1 && \
PL_SNAP_YI=5 ncu --set full --clock-control none --import-source on -k regex:"k_snap_yi" -s 7 -c 1 -o gpurun_out/prof_yi5_large python scripts/probe_snap.py > gpurun_out/ncu5.log 2>&1 && \
PL_SNAP_YI=6 ncu --set full --clock-control none --import-source on -k regex:"k_snap_yi" -s 7 -c 1 -o gpurun_out/prof_yi6_large python scripts/probe_snap.py > gpurun_out/ncu6.log 2>&1
tail -2 gpurun_out/pytest_gpu.log; grep -B2 -A15 "Error\|assert" gpurun_out/pytest_gpu.log | head -30; tail -1 gpurun_out/ncu5.log gpurun_out/ncu6.log
