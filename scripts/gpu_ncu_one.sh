# ncu --set full of one kernel (regex $1) of probe_eval.py, env from the caller; output gpurun_out/$2
python scripts/probe_eval.py > /dev/null 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"$1" -s 1 -c 1 -o gpurun_out/$2 python scripts/probe_eval.py > gpurun_out/$2.log 2>&1
tail -n 2 gpurun_out/$2.log
