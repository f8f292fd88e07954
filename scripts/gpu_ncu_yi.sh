export PL_YI_PHASE_KB=${PL_YI_PHASE_KB:-100}
python scripts/probe_eval.py > /dev/null 2>&1 || exit 1
ncu --set full --import-source on --clock-control none -k regex:"k_snap_yi" -s 1 -c 1 -o gpurun_out/$1 python scripts/probe_eval.py > gpurun_out/$1.log 2>&1
tail -n 2 gpurun_out/$1.log
