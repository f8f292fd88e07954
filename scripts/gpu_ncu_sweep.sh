timeout 300 python scripts/probe_sweep_one.py > gpurun_out/r2_sweep_plain.log 2>&1 || exit 1
timeout 300 python scripts/probe_hbm.py > gpurun_out/r2_hbm_plain.log 2>&1 || exit 1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_sweep_cluster -s 1 -c 1 -o gpurun_out/r2_sweep python scripts/probe_sweep_one.py > gpurun_out/r2_sweep_ncu.log 2>&1; echo "ncu sweep rc=$?"
timeout 900 ncu --set full --clock-control none -k regex:"k_eam|k_open|k_close" -o gpurun_out/r2_hbm python scripts/probe_hbm.py > gpurun_out/r2_hbm_ncu.log 2>&1; echo "ncu hbm rc=$?"
tail -2 gpurun_out/r2_hbm_ncu.log
