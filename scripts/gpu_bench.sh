# round measurement, part A: GPU tests, default bench line, ncu launch list
# (part B, scripts/gpu_ncu.sh, is the one ncu --set full capture: one ncu run per gpurun call)
python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
python bench.py --steps 1 --warmup 1 --no-cpu --no-parareal > gpurun_out/plain_larger.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 1500 -c 1500 --csv \
    --log-file gpurun_out/launches_larger.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-parareal \
    > gpurun_out/ncu_launch.log 2>&1
tail -2 gpurun_out/pytest_gpu.log; cat gpurun_out/bench.json | head -c 3000; echo; cat gpurun_out/bench_ref.json | head -c 1500
