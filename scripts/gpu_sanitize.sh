# compute-sanitizer runs (one tool per invocation), summaries under gpurun_out/
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  PL_SNAP_PAIR_RUN=2 timeout 1200 $CS --tool $tool --print-limit 50 python scripts/sanitize_case.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; tail -4 gpurun_out/sanitize_$tool.log
done
