timeout 900 python -m pytest tests/test_gpu_manybody.py tests/test_gpu_core.py -q -p no:cacheprovider -rf -x > gpurun_out/ab_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/ab_pytest.log
timeout 300 python scripts/probe_sweep.py 2>&1 | tail -2
timeout 300 python scripts/bench_configs.py pr1 2>&1 | tail -1 | cut -c1-200
