# ncu --set full of the force kernels (pair form and ordered form), larger config
python scripts/probe_eval.py > /dev/null 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"k_snap_deidrj" -s 1 -c 1 -o gpurun_out/de_pair python scripts/probe_eval.py > gpurun_out/ncu_de1.log 2>&1
PL_SNAP_PAIR=0 ncu --set full --clock-control none --import-source on -k regex:"k_snap_deidrj" -s 1 -c 1 -o gpurun_out/de_adj4 python scripts/probe_eval.py > gpurun_out/ncu_de2.log 2>&1
tail -1 gpurun_out/ncu_de1.log gpurun_out/ncu_de2.log
