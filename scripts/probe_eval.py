"""One batched SNAP evaluation of the larger config (for ncu captures)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2212_10508_b200 import tungsten as W

ncell, B = int(os.environ.get("NCELL", 8)), int(os.environ.get("BATCH", 64))
q0, box = W.bcc_sia(ncell)
rs = np.random.default_rng(0)
Q = torch.from_numpy(q0[None] + 0.05 * rs.normal(size=(B, q0.shape[0]))).cuda()
pot = W.make_snap(q0.shape[0] // 3, box)
for _ in range(int(os.environ.get("REPS", 3))):
    pot.evaluate(Q, False, True)
torch.cuda.synchronize()
print("ok")
