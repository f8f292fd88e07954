# A/B of SNAP kernel variants: GPU SNAP tests, then stage timings per env value
# usage: bash scripts/gpu_ab.sh VAR v1 v2 ...
V=${1:-PL_SNAP_PAIR}; shift
python -m pytest tests/test_gpu_manybody.py -q -x > gpurun_out/pytest_mb.log 2>&1; tail -1 gpurun_out/pytest_mb.log
for x in "$@"; do echo "== $V=$x"; env $V=$x python scripts/probe_snap.py 2>&1 | tail -2; done
