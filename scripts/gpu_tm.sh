timeout 600 python -m pytest tests/test_gpu_manybody.py -q -p no:cacheprovider -rf -x -k "specialised or production or heavy_system_vs or snap_vs_oracle or window_vs" > gpurun_out/tm_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/tm_pytest.log
for t in 0 1; do TAG="tmem=$t" PL_SNAP_TMEM=$t timeout 300 python scripts/probe_yi.py 2>&1 | tail -1; done
TAG="pair PR1" NCELL=4 BATCH=16 timeout 300 python scripts/probe_yi.py 2>&1 | tail -1
