PL_LIB_VARIANT=timing timeout 300 python scripts/probe_yi_phases.py | tail -1
PL_LIB_VARIANT=timing PL_YI_MODEL_COST=1 timeout 300 python scripts/probe_yi_phases.py | tail -1
TAG="measured" timeout 300 python scripts/probe_yi.py 2>&1 | tail -1
TAG="model" PL_YI_MODEL_COST=1 timeout 300 python scripts/probe_yi.py 2>&1 | tail -1
TAG="measured PR1" NCELL=4 BATCH=16 timeout 300 python scripts/probe_yi.py 2>&1 | tail -1
TAG="model PR1" NCELL=4 BATCH=16 PL_YI_MODEL_COST=1 timeout 300 python scripts/probe_yi.py 2>&1 | tail -1
