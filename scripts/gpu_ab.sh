for v in nopf "" nopf ""; do TAG="variant=${v:-pf}" PL_LIB_VARIANT=$v timeout 300 python scripts/probe_yi.py 2>&1 | tail -1; done
