# quick check: all GPU tests + bench without the CPU / parareal / HBM legs
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rf -x > gpurun_out/q_pytest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/q_pytest.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-parareal --no-hbm > gpurun_out/q_bench.log 2>&1; echo "bench rc=$?"
python - <<'PY'
import json
l = json.loads(open("gpurun_out/q_bench.log").read().strip().splitlines()[-1])
r = l["roofline"]
print("value", l["value"], "ms/step", l["ms_per_step"], "e2e", l["e2e"]["value"])
print({k: (v["avg_launch_ms"], v["frac"]) for k, v in r["kernels"].items()})
print(r["stage_share"])
PY
