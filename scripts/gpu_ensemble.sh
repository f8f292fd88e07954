# configs[3] residence-time ensemble: full protocol (minimise, thermalise, sequential fine + adaptive parareal
# per member over the same plans, quenched labels, min_run 2, compare_ensembles)
PL_ENSEMBLE_SEGMENTS=${PL_ENSEMBLE_SEGMENTS:-7} timeout 3000 python scripts/bench_configs.py ensemble > gpurun_out/r2_ensemble.jsonl 2> gpurun_out/r2_ensemble.err; echo "rc=$?"
cut -c1-1500 gpurun_out/r2_ensemble.jsonl; tail -3 gpurun_out/r2_ensemble.err
