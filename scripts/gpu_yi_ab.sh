# A/B of the Y kernel: warps per CTA x phase code budget
for nw in 8; do for kb in 170 100 70; do
  TAG="nw=$nw kb=$kb" PL_YI_NW=$nw PL_YI_PHASE_KB=$kb timeout 300 python scripts/probe_yi.py 2>&1 | tail -1
done; done
