# round measurement, part B: one ncu --set full capture of the three SNAP kernels (larger config)
python bench.py --steps 1 --warmup 1 --no-cpu --no-parareal > gpurun_out/plain_larger.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_snap_(yi_box|deidrj_run|ui_r4)" -s 4 -c 3 \
    -o gpurun_out/prof_larger python bench.py --steps 1 --warmup 1 --no-cpu --no-parareal > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log
