# round measurement: GPU tests, default bench line, launch list + one ncu --set full capture
python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python bench.py --steps 1 --warmup 1 --no-cpu --no-parareal > gpurun_out/plain_larger.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 1500 -c 1500 --csv \
    --log-file gpurun_out/launches_larger.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-parareal \
    > gpurun_out/ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_snap_(yi_box|deidrj_adj|ui_rr)" -s 3 -c 3 \
    -o gpurun_out/prof_larger python bench.py --steps 1 --warmup 1 --no-cpu --no-parareal > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/pytest_gpu.log; cat gpurun_out/bench.json | head -c 1500; tail -2 gpurun_out/ncu_full.log
