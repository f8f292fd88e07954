"""Phase balance of the Y kernel (diagnostic build: build.py --variant timing -DPL_YI_TIMING,
run with PL_LIB_VARIANT=timing): per phase, mean / max warp time and the barrier loss."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2212_10508_b200 import _lib, tungsten as W

q0, box = W.bcc_sia(8)
Q = torch.from_numpy(q0[None] + 0.05 * np.random.default_rng(0).normal(size=(64, q0.shape[0]))).cuda()
pot = W.make_snap(q0.shape[0] // 3, box)
for _ in range(2):
    pot.evaluate(Q, False, True)
torch.cuda.synchronize()
buf = np.zeros(4096 * 24 * 24 + 2 * 125 * 5, dtype=np.int64)
assert _lib.load().pl_yi_timing(buf.ctypes.data_as(_lib.vp)) == 0, "not a PL_YI_TIMING build"
items = buf[4096 * 24 * 24:]
cyc, cnt = items[:625].reshape(125, 5), items[625:].reshape(125, 5)
buf = buf[:4096 * 24 * 24].reshape(4096, 24, 24)
nb = (Q.shape[0] * Q.shape[1] // 3 + 31) // 32
t = buf[:nb, :, :8].astype(float)
ph_used = [p for p in range(24) if t[:, p, :].max() > 0]
tot_max = tot_mean = 0.0
for p in ph_used:
    mx = t[:, p, :].max(axis=1)
    mn = t[:, p, :].mean(axis=1)
    tot_max += mx.mean()
    tot_mean += mn.mean()
    print(f"phase {p:2d}: mean warp {mn.mean():9.0f} cyc, max warp {mx.mean():9.0f} cyc, balance {mn.mean() / mx.mean():.3f}")
print(f"all phases: sum of max {tot_max:.0f} cyc, sum of mean {tot_mean:.0f} cyc, balance {tot_mean / tot_max:.3f}")
