# A/B of the Y-kernel phase budget
for kb in 100000 170 100 60 40 25; do
  TAG="kb=$kb" PL_YI_PHASE_KB=$kb timeout 300 python scripts/probe_yi.py 2>&1 | tail -1
done
