# A/B of library variants (build.py --variant NAME -D...): per-stage SNAP times at the larger config
for v in "" peel; do for kb in 100 130; do
  TAG="variant=${v:-base} kb=$kb" PL_LIB_VARIANT=$v PL_YI_PHASE_KB=$kb timeout 300 python scripts/probe_yi.py 2>&1 | tail -1
done; done
for v in "" peel; do
  TAG="variant=${v:-base} PR1 batch" NCELL=4 BATCH=16 PL_LIB_VARIANT=$v timeout 300 python scripts/probe_yi.py 2>&1 | tail -1
done
