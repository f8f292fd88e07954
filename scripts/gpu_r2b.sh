# round 2b: minimisation probe, the previously failing tests, ncu --set full of the three SNAP kernels
timeout 600 python scripts/probe_minimize.py > gpurun_out/r2b_min.log 2>&1; echo "probe rc=$?"; cat gpurun_out/r2b_min.log | tail -12
timeout 900 python -m pytest tests/test_gpu_ensemble.py::test_sequential_batch_equals_single_chains tests/test_gpu_manybody.py::test_heavy_system_sweeps_batch_equals_single -q -p no:cacheprovider -rf > gpurun_out/r2b_pytest.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/r2b_pytest.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_snap_(yi_p|deidrj_run|ui_r4)" -s 4 -c 3 \
    -o gpurun_out/r2b_prof_larger python scripts/probe_eval.py > gpurun_out/r2b_ncu_full.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/r2b_ncu_full.log
