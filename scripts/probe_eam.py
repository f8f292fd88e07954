"""EAM force sweep of configs[1] (4096 x 129 atoms): per-stage times (live events) and wall."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2212_10508_b200 import _lib, tungsten as W

q0, box = W.bcc_sia(4)
n = q0.shape[0] // 3
Q = torch.from_numpy(q0[None] + 0.1 * np.random.default_rng(2212).normal(size=(4096, q0.shape[0]))).cuda()
eam = W.make_eam(n, box)
for _ in range(2):
    eam.evaluate(Q, True, True, True)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(3):
    eam.evaluate(Q, True, True, True)
torch.cuda.synchronize()
wall = (time.perf_counter() - t) / 3
lib, ctx = _lib.load(), _lib.context()
_lib.check(lib.pl_prof_begin(ctx.handle))
for _ in range(3):
    eam.evaluate(Q, True, True, True)
torch.cuda.synchronize()
ms = np.zeros(8); cnt = np.zeros(8, dtype=np.int64)
_lib.check(lib.pl_prof_end(ctx.handle, 8, _lib.dptr(ms), cnt.ctypes.data_as(_lib.pi64)))
print(f"wall {wall*1e3:.3f} ms  neigh {ms[0]/3:.3f} ms  eam {ms[5]/3:.3f} ms", flush=True)
