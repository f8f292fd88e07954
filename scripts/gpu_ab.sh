timeout 900 python -m pytest tests/test_gpu_manybody.py tests/test_gpu_core.py -q -p no:cacheprovider -rf -x > gpurun_out/ab_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/ab_pytest.log
for nw in 8 12; do
  TAG="small nw=$nw PR1 batch" NCELL=4 BATCH=16 PL_YI_SMALL_NW=$nw timeout 300 python scripts/probe_yi.py 2>&1 | tail -1
  TAG="small nw=$nw 4 windows larger" NCELL=8 BATCH=4 PL_YI_SMALL_NW=$nw timeout 300 python scripts/probe_yi.py 2>&1 | tail -1
done
TAG="large" timeout 300 python scripts/probe_yi.py 2>&1 | tail -1
