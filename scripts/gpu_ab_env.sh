# A/B of runtime switches: per-stage SNAP times of the larger config and of a PR1
# batch, alternating, for each environment setting in ENVS ("-" = none), e.g.
# ENVS="- PL_YI_YT=0"
ENVS=${ENVS:--}
for rep in 1 2; do
  for e in $ENVS; do
    if [ "$e" = "-" ]; then E=""; else E="$e"; fi
    env $E TAG="$e larger" timeout 300 python scripts/probe_yi.py 2>&1 | tail -1
    env $E TAG="$e pr1x16" NCELL=4 BATCH=16 timeout 300 python scripts/probe_yi.py 2>&1 | tail -1
  done
done
