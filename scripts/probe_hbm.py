"""ncu target for the HBM-bound kernels: the EAM force sweep of configs[1] (4096 x 129
atoms, E + F + virial) and a batched EAM window (64 x 1025 atoms, L = 3) whose
k_open / k_close_open / k_close stream the integrator state."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2212_10508_b200 as pl
from paper_2212_10508_b200 import tungsten as W
from paper_2212_10508_b200.integrator import WindowKernel

q0, box = W.bcc_sia(4)
n = q0.shape[0] // 3
Q = torch.from_numpy(q0[None] + 0.1 * np.random.default_rng(2212).normal(size=(4096, q0.shape[0]))).cuda()
eam = W.make_eam(n, box)
for _ in range(2):
    eam.evaluate(Q, True, True, True)
q1, box1 = W.bcc_sia(8)
n1 = q1.shape[0] // 3
L = 3
params = pl.LangevinParams(1.0, W.KB * 1000.0, 0.001, L, mass=np.full(3 * n1, W.MASS_W))
k = WindowKernel(W.make_eam(n1, box1), params, pl.TemperatureSchedule.robust(L), 3 * n1)
Q1 = torch.from_numpy(q1[None] + 0.05 * np.random.default_rng(1).normal(size=(64, q1.shape[0]))).cuda()
P1 = torch.zeros_like(Q1)
noise = k.noise(pl.derive_seeds(5, 64))
k.run(Q1, P1, noise)
torch.cuda.synchronize()
print("ok")
