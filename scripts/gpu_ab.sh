for i in 1 2 3; do timeout 300 python scripts/bench_configs.py pr1 2>&1 | cut -c80-200; done
for i in 1 2; do PL_SWEEP_FULL=1 timeout 300 python scripts/bench_configs.py pr1 2>&1 | cut -c80-200; done
