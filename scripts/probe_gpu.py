"""Quick GPU timing probe of the current kernels (not the bench)."""

import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_2212_10508_b200 as pl
from paper_2212_10508_b200 import tungsten as W
from paper_2212_10508_b200.integrator import WindowKernel


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps


def main():
    for ncell, W_ in ((4, 16), (8, 64)):
        q0, box = W.bcc_sia(ncell)
        n = q0.shape[0] // 3
        pot = W.make_eam(n, box)
        L = 100
        params = pl.LangevinParams(1.0, W.KB * 1000.0, 0.001, L, mass=np.full(3 * n, W.MASS_W))
        k = WindowKernel(pot, params, pl.TemperatureSchedule.robust(L), 3 * n)
        seeds = pl.derive_seeds(11, W_)
        t0 = time.perf_counter()
        noise = k.noise(seeds)
        torch.cuda.synchronize()
        tn = time.perf_counter() - t0
        Q0 = torch.from_numpy(np.repeat(q0[None], W_, 0)).cuda()
        P0 = torch.zeros_like(Q0)
        dt = timeit(lambda: k.run(Q0, P0, noise))
        print(f"EAM N={n} W={W_} L={L}: {dt*1e3:.2f} ms/window-batch, "
              f"{n*W_*L/dt:.3e} atom-steps/s, {dt/L*1e6:.1f} us/step, noise gen {tn*1e3:.1f} ms")
    # DW adaptive config end to end
    params = pl.LangevinParams(0.5, 0.4, 0.05, 2)
    sched = pl.TemperatureSchedule.robust(2)
    plan = pl.NoisePlan.for_windows(11, 800)
    pair = pl.PropagatorPair(pl.DoubleWell(1.0, 1.0), pl.DoubleWell(0.8, 1.0), 175.0, 1.0)
    t = time.perf_counter()
    res = pl.parareal_adaptive(pl.PhaseState(q=[-1.0], p=[0.0]), pair, params, sched, plan,
                               pl.PararealConfig(800, 1e-10, 0.35))
    print(f"adaptive.json: {time.perf_counter()-t:.2f} s, N_slab {res.n_slab}, sum k {res.total_iterations}")


if __name__ == "__main__":
    main()
