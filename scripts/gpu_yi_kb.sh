# A/B of the Y kernel's phase code budget (PL_YI_PHASE_KB)
for kb in ${KBS:-24 28 32 40 48 64 80 100}; do
  PL_YI_PHASE_KB=$kb TAG="kb=$kb larger" timeout 300 python scripts/probe_yi.py 2>&1 | tail -1 | cut -c1-90
done
