timeout 900 python -m pytest tests/test_gpu_manybody.py -q -p no:cacheprovider -rf -x > gpurun_out/ab_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/ab_pytest.log
for t in 0 1; do
  TAG="tmem=$t PR1 batch" NCELL=4 BATCH=16 PL_SNAP_TMEM=$t timeout 300 python scripts/probe_yi.py 2>&1 | tail -1
  TAG="tmem=$t 1 window" NCELL=4 BATCH=1 PL_SNAP_TMEM=$t timeout 300 python scripts/probe_yi.py 2>&1 | tail -1
  TAG="tmem=$t 8 larger" NCELL=8 BATCH=8 PL_SNAP_TMEM=$t timeout 300 python scripts/probe_yi.py 2>&1 | tail -1
done
