"""Steepest descent of the W+SIA start on the SNAP (fine) and EAM surfaces: iterations per tolerance."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2212_10508_b200 import tungsten as W
from paper_2212_10508_b200.potentials import minimize_batch

q0, box = W.bcc_sia(4)
n = q0.shape[0] // 3
for name, pot in (("snap", W.make_snap(n, box)), ("eam", W.make_eam(n, box))):
    x = q0
    for tol in (1e-1, 1e-2, 1e-3, 1e-4, 1e-6):
        t = time.perf_counter()
        X, st, it, e = minimize_batch(pot, x[None], tol=tol, max_iter=20000)
        g = pot.gradient(X[0]) if hasattr(pot, "gradient") else None
        gn = float(np.linalg.norm(g)) if g is not None else float("nan")
        print(f"{name} tol={tol:g} status={st[0]} iters={it[0]} E={e[0]:.6f} |g|={gn:.3e} "
              f"max|dx|={np.abs(X[0]-q0).max():.3f} {time.perf_counter()-t:.1f}s", flush=True)
        x = X[0]
