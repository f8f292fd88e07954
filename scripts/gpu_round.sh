# full round measurement: GPU tests, bench (+ reference arm), ncu launch list, one ncu --set full
# capture of the three SNAP kernels, then the BASELINE configs (PL_ENSEMBLE_SEGMENTS segments, default 1)
bash scripts/gpu_bench.sh
bash scripts/gpu_ncu.sh
python scripts/bench_configs.py sweep pr1 heavy larger_parareal ensemble > gpurun_out/configs.jsonl 2> gpurun_out/configs.err
cut -c1-400 gpurun_out/configs.jsonl
