# round measurement: full GPU tests, default bench line, reference arm, launch list, one ncu --set full capture, configs
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > gpurun_out/v11_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/v11_pytest.log
timeout 1500 python bench.py > gpurun_out/v11_bench.json 2> gpurun_out/v11_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/v11_bench_ref.json 2> gpurun_out/v11_bench_ref.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 1500 -c 1500 --csv \
    --log-file gpurun_out/v11_launches_larger.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-parareal --no-hbm \
    > gpurun_out/v11_ncu_launch.log 2>&1; echo "ncu launch rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_snap_(yi_p|deidrj_tm|ui_r4)" -s 4 -c 3 \
    -o gpurun_out/v11_snap python scripts/probe_eval.py > gpurun_out/v11_ncu_full.log 2>&1; echo "ncu full rc=$?"
timeout 2400 python scripts/bench_configs.py sweep pr1 heavy larger_parareal heavy_parareal > gpurun_out/v11_configs.jsonl 2> gpurun_out/v11_configs.err; echo "configs rc=$?"
head -c 1500 gpurun_out/v11_bench.json; echo; head -c 400 gpurun_out/v11_bench_ref.json; echo; cut -c1-400 gpurun_out/v11_configs.jsonl
