"""Per-stage SNAP kernel times (live CUDA events) of the larger config, for A/B runs.

    PL_YI_PHASE_KB=60 python scripts/probe_yi.py
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2212_10508_b200 import _lib, tungsten as W

ncell, B = int(os.environ.get("NCELL", 8)), int(os.environ.get("BATCH", 64))
q0, box = W.bcc_sia(ncell)
rs = np.random.default_rng(0)
Q = torch.from_numpy(q0[None] + 0.05 * rs.normal(size=(B, q0.shape[0]))).cuda()
pot = W.make_snap(q0.shape[0] // 3, box)
for _ in range(2):
    E0, G0, _ = pot.evaluate(Q, True, True)
torch.cuda.synchronize()
lib, ctx = _lib.load(), _lib.context()
reps = int(os.environ.get("REPS", 10))
_lib.check(lib.pl_prof_begin(ctx.handle))
for _ in range(reps):
    pot.evaluate(Q, True, True)
torch.cuda.synchronize()
ms = np.zeros(8)
n = np.zeros(8, dtype=np.int64)
_lib.check(lib.pl_prof_end(ctx.handle, 8, _lib.dptr(ms), n.ctypes.data_as(_lib.pi64)))
names = ["neigh", "ui", "yi", "deidrj", "gather"]
print(os.environ.get("TAG", ""), " ".join(f"{names[i]}={ms[i] / max(n[i], 1):.4f}" for i in range(5)),
      f"E0={float(E0[0]):.15e}", f"G00={float(G0[0, 0]):.15e}", flush=True)
