timeout 900 python -m pytest tests/test_gpu_manybody.py tests/test_gpu_core.py -q -p no:cacheprovider -rf -x > gpurun_out/ab_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/ab_pytest.log
for m in 2 4; do
  TAG="split<=$m 1 window" NCELL=4 BATCH=1 PL_YI_SPLIT_MAX=$m timeout 300 python scripts/probe_yi.py 2>&1 | tail -1
  TAG="split<=$m 4 windows" NCELL=4 BATCH=4 PL_YI_SPLIT_MAX=$m timeout 300 python scripts/probe_yi.py 2>&1 | tail -1
  TAG="split<=$m 1 larger" NCELL=8 BATCH=1 PL_YI_SPLIT_MAX=$m timeout 300 python scripts/probe_yi.py 2>&1 | tail -1
  PL_YI_SPLIT_MAX=$m timeout 300 python scripts/bench_configs.py pr1 2>&1 | cut -c80-150
done
