# round 2c: peaks, ensemble statistical-parity test, BASELINE configs
timeout 300 python scripts/probe_peaks.py > gpurun_out/r2c_peaks.json 2>&1; cat gpurun_out/r2c_peaks.json
timeout 1200 python -m pytest tests/test_gpu_ensemble.py -q -p no:cacheprovider -rf > gpurun_out/r2c_pytest.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/r2c_pytest.log
timeout 2400 python scripts/bench_configs.py sweep pr1 heavy larger_parareal heavy_parareal > gpurun_out/r2c_configs.jsonl 2> gpurun_out/r2c_configs.err; echo "configs rc=$?"
cut -c1-700 gpurun_out/r2c_configs.jsonl
