"""SNAP kernel stage timing probe (live CUDA events per stage)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2212_10508_b200 import _lib, tungsten as W

names = ["neigh", "ui", "yi", "deidrj", "gather", "eam", "int"]
for ncell, B in ((4, 16), (8, 64)):
    q0, box = W.bcc_sia(ncell)
    n = q0.shape[0] // 3
    rs = np.random.default_rng(0)
    Q = torch.from_numpy(q0[None] + 0.05 * rs.normal(size=(B, q0.shape[0]))).cuda()
    pot = W.make_snap(n, box)
    for _ in range(2):
        pot.evaluate(Q, False, True)
    torch.cuda.synchronize()
    lib, ctx = _lib.load(), _lib.context()
    _lib.check(lib.pl_prof_begin(ctx.handle))
    t = time.perf_counter()
    reps = 5
    for _ in range(reps):
        pot.evaluate(Q, False, True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / reps
    ms = np.zeros(8); cnt = np.zeros(8, dtype=np.int64)
    _lib.check(lib.pl_prof_end(ctx.handle, 8, _lib.dptr(ms), cnt.ctypes.data_as(_lib.pi64)))
    print(f"SNAP N={n} B={B}: {dt*1e3:.3f} ms/eval, {n*B/dt:.3e} atom-evals/s | " +
          " ".join(f"{names[i]}={ms[i]/reps:.3f}ms" for i in range(5)), flush=True)
