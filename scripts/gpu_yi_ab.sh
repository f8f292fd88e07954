# A/B of the Y kernel: warps per CTA x phase code budget
for kb in 80 100 120 140; do
  TAG="nw=8 kb=$kb" PL_YI_NW=8 PL_YI_PHASE_KB=$kb timeout 300 python scripts/probe_yi.py 2>&1 | tail -1
done
TAG="nw=12 kb=100" PL_YI_NW=12 PL_YI_PHASE_KB=100 timeout 300 python scripts/probe_yi.py 2>&1 | tail -1
