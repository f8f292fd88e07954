timeout 300 python scripts/probe_eval.py > /dev/null 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_snap_(yi_p|deidrj_run|deidrj_tm|ui_r4)" -s 4 -c 3 \
    -o gpurun_out/$1 python scripts/probe_eval.py > gpurun_out/$1.log 2>&1; echo "ncu rc=$?"
