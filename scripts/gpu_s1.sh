# round-2 check: GPU tests (all, no -x), then a short bench
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > gpurun_out/s1_pytest.log 2>&1; echo "pytest rc=$?"
tail -25 gpurun_out/s1_pytest.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/s1_bench.log 2>&1; echo "bench rc=$?"
tail -c 3000 gpurun_out/s1_bench.log
