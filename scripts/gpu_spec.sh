# speculative parareal pipeline: bitwise test, engine tests, then PR1 / larger wall-clock with and without
timeout 900 python -m pytest tests/test_gpu_manybody.py tests/test_gpu_core.py -q -p no:cacheprovider -rf -x > gpurun_out/spec_pytest.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/spec_pytest.log
for m in 0 1; do PL_PARAREAL_SPEC=$m timeout 900 python scripts/bench_configs.py larger_parareal > gpurun_out/spec_larger_$m.jsonl 2>&1; echo "spec=$m"; cut -c1-400 gpurun_out/spec_larger_$m.jsonl; done
