import os, sys, time
sys.path.insert(0, '/root/repo') if os.path.exists('/root/repo') else None
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2212_10508_b200 import tungsten as W
for ncell, B in ((20, 1), (16, 2)):
    q0, box = W.bcc_sia(ncell)
    rs = np.random.default_rng(0)
    Q = torch.from_numpy(q0[None] + 0.05 * rs.normal(size=(B, q0.shape[0]))).cuda()
    pot = W.make_snap(q0.shape[0] // 3, box)
    for _ in range(2): pot.evaluate(Q, False, True)
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(5): pot.evaluate(Q, False, True)
    torch.cuda.synchronize(); dt = (time.perf_counter() - t) / 5
    print(f"N={q0.shape[0]//3} B={B}: {dt*1e3:.3f} ms/eval")
