# GPU tests against the bounds-checked build (device asserts, PL_CHECKS) and the default build
PL_LIB_VARIANT=checks timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > gpurun_out/checks_pytest.log 2>&1; echo "checks pytest rc=$?"; tail -3 gpurun_out/checks_pytest.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > gpurun_out/default_pytest.log 2>&1; echo "default pytest rc=$?"; tail -3 gpurun_out/default_pytest.log
