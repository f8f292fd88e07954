NCELL=4 timeout 300 python scripts/probe_sweep_one.py > /dev/null 2>&1 || exit 1
NCELL=4 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_sweep_cluster -s 1 -c 1 -o gpurun_out/r2_sweep129 python scripts/probe_sweep_one.py > gpurun_out/r2_sweep129.log 2>&1; echo "ncu rc=$?"
