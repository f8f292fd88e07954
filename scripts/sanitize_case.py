"""Small workloads for compute-sanitizer (racecheck / memcheck / synccheck) runs.

Covers every kernel family of the hot path: neighbour lists (brute force and
cell lists), SNAP ui / Y (split and non-split) / ytrans / force (2-atom pair
warps and 8-atom runs, PL_SNAP_PAIR_RUN=2) / gather, EAM, the BBK integrator
kernels, the noise generator, the cluster coarse sweep and bootstrap.
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2212_10508_b200 as pl
from paper_2212_10508_b200 import tungsten as W

# PR1 system: adaptive parareal, SNAP fine / EAM coarse (cluster sweep), 3 windows x 2 substeps
q0, box = W.bcc_sia(4)
n = q0.shape[0] // 3
L, N = 2, 3
params = pl.LangevinParams(1.0, W.KB * 1000.0, 0.001, L, mass=np.full(3 * n, W.MASS_W))
sched = pl.TemperatureSchedule.robust(L)
pair = pl.PropagatorPair(W.make_snap(n, box), W.make_eam(n, box), 100.0, 1.0)
res = pl.parareal_adaptive(pl.PhaseState(q=q0, p=W.maxwell_boltzmann(n, 1000.0, 11)), pair, params, sched,
                           pl.NoisePlan.for_windows(11, N), pl.PararealConfig(N, 1e-10, 0.35))
print("parareal", res.n_slab, res.total_iterations, flush=True)
# larger batch: cell lists, non-split Y kernel, run force kernel
q1, box1 = W.bcc_sia(8)
n1 = q1.shape[0] // 3
Q = torch.from_numpy(q1[None] + 0.05 * np.random.default_rng(0).normal(size=(5, q1.shape[0]))).cuda()
E, G, V = W.make_snap(n1, box1).evaluate(Q, True, True, True)
torch.cuda.synchronize()
print("snap batch", float(E.sum()), flush=True)
