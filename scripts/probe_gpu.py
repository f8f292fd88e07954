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


def timeit(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps


def main():
    for ncell, B in ((4, 16), (8, 64)):
        q0, box = W.bcc_sia(ncell)
        n = q0.shape[0] // 3
        rs = np.random.default_rng(0)
        Q = torch.from_numpy(q0[None] + 0.05 * rs.normal(size=(B, q0.shape[0]))).cuda()
        for name, pot in (("EAM", W.make_eam(n, box)), ("SNAP", W.make_snap(n, box))):
            dt = timeit(lambda: pot.evaluate(Q, False, True))
            print(f"{name} grad N={n} B={B}: {dt*1e3:.3f} ms/eval, {n*B/dt:.3e} atom-evals/s", flush=True)
    for ncell, W_, L in ((4, 16, 100), (8, 64, 20)):
        q0, box = W.bcc_sia(ncell)
        n = q0.shape[0] // 3
        pot = W.make_snap(n, box)
        params = pl.LangevinParams(1.0, W.KB * 1000.0, 0.001, L, mass=np.full(3 * n, W.MASS_W))
        k = WindowKernel(pot, params, pl.TemperatureSchedule.robust(L), 3 * n)
        noise = k.noise(pl.derive_seeds(11, W_))
        Q0 = torch.from_numpy(np.repeat(q0[None], W_, 0)).cuda()
        P0 = torch.from_numpy(np.stack([W.maxwell_boltzmann(n, 1000.0, s) for s in range(W_)])).cuda()
        dt = timeit(lambda: k.run(Q0, P0, noise), reps=2)
        Q1, P1, blow = k.run(Q0, P0, noise)
        ke = (P1 ** 2).sum().item() / (2 * W.MASS_W) / (1.5 * W_ * n) / W.KB
        print(f"SNAP window N={n} W={W_} L={L}: {dt*1e3:.1f} ms, {n*W_*L/dt:.3e} atom-steps/s, "
              f"{dt/L*1e6:.0f} us/step, blowups={int((blow!=0).sum())}, T_kin={ke:.0f} K", flush=True)
    # DW adaptive config end to end
    params = pl.LangevinParams(0.5, 0.4, 0.05, 2)
    sched = pl.TemperatureSchedule.robust(2)
    plan = pl.NoisePlan.for_windows(11, 800)
    pair = pl.PropagatorPair(pl.DoubleWell(1.0, 1.0), pl.DoubleWell(0.8, 1.0), 175.0, 1.0)
    t = time.perf_counter()
    res = pl.parareal_adaptive(pl.PhaseState(q=[-1.0], p=[0.0]), pair, params, sched, plan,
                               pl.PararealConfig(800, 1e-10, 0.35))
    print(f"adaptive.json: {time.perf_counter()-t:.2f} s, N_slab {res.n_slab}, sum k {res.total_iterations}")
    # PR1 parareal: SNAP fine, EAM coarse, 16 x 100
    q0, box = W.bcc_sia(4)
    n = q0.shape[0] // 3
    mass = np.full(3 * n, W.MASS_W)
    params = pl.LangevinParams(1.0, W.KB * 1000.0, 0.001, 100, mass=mass)
    sched = pl.TemperatureSchedule.robust(100)
    plan = pl.NoisePlan.for_windows(11, 16)
    init = pl.PhaseState(q=q0, p=W.maxwell_boltzmann(n, 1000.0, 11))
    for lam in (1.0, None):
        eam = W.make_eam(n, box)
        snap = W.make_snap(n, box)
        fine = snap if lam is None else pl.Perturbed(eam, snap, 0.1)
        pair = pl.PropagatorPair(fine, eam, 100.0, 1.0)
        t = time.perf_counter()
        try:
            res = pl.parareal_adaptive(init, pair, params, sched, plan, pl.PararealConfig(16, 1e-10, 0.35))
            print(f"PR1 parareal fine={'SNAP' if lam is None else 'EAM+0.1SNAP'}: {time.perf_counter()-t:.2f} s, "
                  f"N_slab {res.n_slab}, sum k {res.total_iterations}, converged {res.converged}", flush=True)
        except Exception as e:
            print("PR1 parareal failed:", type(e).__name__, e, flush=True)


if __name__ == "__main__":
    main()
