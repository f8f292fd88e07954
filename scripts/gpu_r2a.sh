# round 2 check: all GPU tests (no -x), default bench, reference arm, launch list
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > gpurun_out/r2a_pytest.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/r2a_pytest.log
timeout 1200 python bench.py > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2a_bench_ref.json 2> gpurun_out/r2a_bench_ref.err; echo "ref rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 1500 -c 1500 --csv \
    --log-file gpurun_out/r2a_launches_larger.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-parareal --no-hbm \
    > gpurun_out/r2a_ncu_launch.log 2>&1; echo "ncu rc=$?"
head -c 2500 gpurun_out/r2a_bench.json; echo; head -c 800 gpurun_out/r2a_bench_ref.json
