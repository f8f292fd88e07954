# A/B of library variants (build.py --variant NAME -D...): per-stage SNAP times of the
# larger config (probe_yi) and of one PR1 window batch, alternating, VARIANTS="default a b"
VARIANTS=${VARIANTS:-default}
for rep in 1 2; do
  for v in $VARIANTS; do
    if [ "$v" = default ]; then unset PL_LIB_VARIANT; else export PL_LIB_VARIANT=$v; fi
    TAG="$v larger" timeout 300 python scripts/probe_yi.py 2>&1 | tail -1
    TAG="$v pr1x16" NCELL=4 BATCH=16 timeout 300 python scripts/probe_yi.py 2>&1 | tail -1
  done
done
unset PL_LIB_VARIANT
