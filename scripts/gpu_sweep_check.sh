timeout 900 python -m pytest tests/test_gpu_manybody.py tests/test_gpu_core.py tests/test_gpu_ensemble.py -q -p no:cacheprovider -rf -x > gpurun_out/sw_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/sw_pytest.log
timeout 600 python scripts/probe_sweep.py 2>&1 | tail -3
timeout 900 python scripts/bench_configs.py pr1 larger_parareal > gpurun_out/sw_configs.jsonl 2>&1; cut -c1-500 gpurun_out/sw_configs.jsonl
