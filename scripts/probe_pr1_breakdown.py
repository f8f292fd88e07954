"""Adaptive parareal wall-clock split into bootstrap / fine jumps / sweep (synchronised timers).

    python scripts/probe_pr1_breakdown.py [ncell N L]   (default PR1: 4 16 100)
"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2212_10508_b200 as pl
from paper_2212_10508_b200 import parareal as pp, tungsten as W

acc = {"bootstrap": 0.0, "jumps": 0.0, "sweep": 0.0}
cnt = {k: 0 for k in acc}
for name in acc:
    orig = getattr(pp._DeviceRun, name)

    def wrap(self, *a, _o=orig, _n=name, **k):
        torch.cuda.synchronize()
        t = time.perf_counter()
        r = _o(self, *a, **k)
        torch.cuda.synchronize()
        acc[_n] += time.perf_counter() - t
        cnt[_n] += 1
        return r
    setattr(pp._DeviceRun, name, wrap)

ncell, N, L = (int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (4, 16, 100)
q0, box = W.bcc_sia(ncell)
n = q0.shape[0] // 3
params = pl.LangevinParams(1.0, W.KB * 1000.0, 0.001, L, mass=np.full(3 * n, W.MASS_W))
sched = pl.TemperatureSchedule.robust(L)
init = pl.PhaseState(q=q0, p=W.maxwell_boltzmann(n, 1000.0, 11))
pair = pl.PropagatorPair(W.make_snap(n, box), W.make_eam(n, box), 100.0, 1.0)
cfg = pl.PararealConfig(N, 1e-10, 0.35)
plan = pl.NoisePlan.for_windows(11, N)
if n < 500:
    pl.parareal_adaptive(init, pair, params, sched, plan, cfg)  # warm
for k in acc:
    acc[k] = 0.0
    cnt[k] = 0
torch.cuda.synchronize()
t = time.perf_counter()
res = pl.parareal_adaptive(init, pair, params, sched, plan, cfg)
torch.cuda.synchronize()
print(f"wall {time.perf_counter() - t:.3f} s, slabs {res.n_slab}, sum_k {res.total_iterations};",
      {k: (round(v, 3), cnt[k]) for k, v in acc.items()})
