"""Measured FP64 vector (DFMA) and FP64 tensor-core (DMMA m8n8k4) peaks of this device."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2212_10508_b200 import _lib

lib, ctx = _lib.load(), _lib.context()
out = np.zeros(1)
res = {}
for name in ("pl_fp64_peak", "pl_dmma_peak"):
    best = 0.0
    for _ in range(5):
        _lib.check(getattr(lib, name)(ctx.handle, _lib.dptr(out)))
        best = max(best, float(out[0]))
    res[name] = round(best, 3)
print(json.dumps(res))
