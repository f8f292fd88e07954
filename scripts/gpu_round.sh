# full round measurement: GPU tests, bench (+ reference arm), ncu launch list, one ncu --set full
# capture of the three SNAP kernels, then every BASELINE config (ensemble: all 7 segments)
bash scripts/gpu_bench.sh
bash scripts/gpu_ncu.sh
PL_ENSEMBLE_SEGMENTS=7 python scripts/bench_configs.py sweep pr1 heavy larger_parareal ensemble > gpurun_out/configs.jsonl 2> gpurun_out/configs.err
cat gpurun_out/configs.jsonl | cut -c1-400
