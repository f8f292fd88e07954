"""One coarse sweep (persistent cluster kernel) of NCELL (default 8: 1025 atoms), 16 windows x L=200 (ncu target)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2212_10508_b200 as pl
from paper_2212_10508_b200 import tungsten as W
from paper_2212_10508_b200.parareal import DevicePropagator, _DeviceRun

ncell, N, L = int(os.environ.get("NCELL", 8)), 16, 200
q0, box = W.bcc_sia(ncell)
n = q0.shape[0] // 3
params = pl.LangevinParams(1.0, W.KB * 1000.0, 0.001, L, mass=np.full(3 * n, W.MASS_W))
sched = pl.TemperatureSchedule.robust(L)
plan = pl.NoisePlan.for_windows(11, N)
f = DevicePropagator(W.make_snap(n, box), params, sched, plan, 3 * n)
c = DevicePropagator(W.make_eam(n, box), params, sched, plan, 3 * n)
run = _DeviceRun(pl.PhaseState(q=q0, p=W.maxwell_boltzmann(n, 1000.0, 11)), f, c, N)
run.bootstrap(0)
run.jumps(0, N, 1)
run.snapshot_prev(0, N)
run.sweep(0, N, False, 0.0, 1)
torch.cuda.synchronize()
print("ok")
