# round-2 session 2: full GPU tests, bench, BASELINE configs (incl. heavy parareal, full ensemble)
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > gpurun_out/s2_pytest.log 2>&1; echo "pytest rc=$?"
tail -8 gpurun_out/s2_pytest.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/s2_bench.log 2>&1; echo "bench rc=$?"
tail -c 600 gpurun_out/s2_bench.log
timeout 2400 python scripts/bench_configs.py sweep pr1 heavy heavy_parareal ensemble > gpurun_out/s2_configs.jsonl 2> gpurun_out/s2_configs.err; echo "configs rc=$?"
cut -c1-600 gpurun_out/s2_configs.jsonl
