timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rf -x > gpurun_out/ab_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/ab_pytest.log
for sk in 0 0.3; do PL_SNAP_SKIN=$sk timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu --no-parareal --no-hbm > gpurun_out/ab_bench_$sk.log 2>&1; python - <<PY
import json
l = json.loads(open("gpurun_out/ab_bench_$sk.log").read().strip().splitlines()[-1])
print("skin=$sk value", round(l["value"]/1e6, 3), "M e2e", round(l["e2e"]["value"]/1e6, 3), {k: v["avg_launch_ms"] for k, v in l["roofline"]["kernels"].items()}, l["roofline"]["stage_share"]["neigh"])
PY
done
for sk in 0 0.3; do TAG="skin=$sk PR1 parareal" PL_SNAP_SKIN=$sk timeout 600 python scripts/bench_configs.py pr1 2>&1 | tail -1 | cut -c1-200; done
