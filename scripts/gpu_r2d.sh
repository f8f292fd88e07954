bash scripts/gpu_quick.sh
timeout 2400 python scripts/bench_configs.py sweep pr1 heavy larger_parareal heavy_parareal > gpurun_out/r2d_configs.jsonl 2> gpurun_out/r2d_configs.err; echo "configs rc=$?"
cut -c1-700 gpurun_out/r2d_configs.jsonl
