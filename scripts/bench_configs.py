"""One-off measurements of the other BASELINE configs (bench.py covers configs[2]).

    python scripts/bench_configs.py [sweep] [pr1] [ensemble] [heavy] [larger_parareal]

Prints one JSON line per config.  Synthetic inputs; timing by
CUDA-synchronised wall clock around the measured call.
"""

import json
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_2212_10508_b200 as pl
from paper_2212_10508_b200 import sia, tungsten as W


def timed(fn, reps=1):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        out = fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps, out


def force_sweep():
    """configs[1]: 4096 x 129-atom W+SIA, sigma = 0.1 A, SNAP and EAM E/F/virial in one batch each."""
    q0, box = W.bcc_sia(4)
    n = q0.shape[0] // 3
    rs = np.random.default_rng(2212)
    Q = torch.from_numpy(q0[None] + 0.1 * rs.normal(size=(4096, q0.shape[0]))).cuda()
    snap, eam = W.make_snap(n, box), W.make_eam(n, box)
    ts, _ = timed(lambda: snap.evaluate(Q, True, True, True), 3)
    te, _ = timed(lambda: eam.evaluate(Q, True, True, True), 3)
    return {"config": "force_sweep: 4096 x 129-atom W+SIA, sigma 0.1 A, E + F + virial",
            "snap_s": ts, "snap_atom_evals_per_s": 4096 * n / ts, "eam_s": te,
            "eam_atom_evals_per_s": 4096 * n / te}


def _pr1(T=1000.0, N=16, L=100, seed=11):
    q0, box = W.bcc_sia(4)
    n = q0.shape[0] // 3
    mass = np.full(3 * n, W.MASS_W)
    params = pl.LangevinParams(1.0, W.KB * T, 0.001, L, mass=mass)
    sched = pl.TemperatureSchedule.robust(L)
    return q0, box, n, params, sched


def pr1_parareal():
    q0, box, n, params, sched = _pr1()
    init = pl.PhaseState(q=q0, p=W.maxwell_boltzmann(n, 1000.0, 11))
    pair = pl.PropagatorPair(W.make_snap(n, box), W.make_eam(n, box), 100.0, 1.0)
    plan = pl.NoisePlan.for_windows(11, 16)
    cfg = pl.PararealConfig(16, 1e-10, 0.35)
    t, res = timed(lambda: pl.parareal_adaptive(init, pair, params, sched, plan, cfg))
    seq_t, _ = timed(lambda: pl.sequential_propagate(init, 16, pair.fine, params, sched, plan))
    return {"config": "PR1 adaptive parareal: 129 atoms, 16 x 100, SNAP/EAM, 1000 K", "wall_s": t,
            "n_slab": res.n_slab, "sum_k": res.total_iterations, "sequential_fine_s": seq_t}


def ensemble(R=256, N=32, L=100, T=1200.0, segments=1):
    """configs[3] (one 3.2 ps segment per replica by default): batched replicas + SIA hops."""
    q0, box, n, params, sched = _pr1(T=T, N=N, L=L)
    pair = pl.PropagatorPair(W.make_snap(n, box), W.make_eam(n, box), 100.0, 1.0)
    cfg = pl.PararealConfig(N, 1e-5, 0.35)  # delta_conv of configs/ensemble.json
    rs = np.random.default_rng(7)
    inits = [pl.PhaseState(q=q0 + 0.03 * rs.normal(size=q0.shape),
                           p=math.sqrt(W.MASS_W * W.KB * T) * rs.normal(size=q0.shape)) for _ in range(R)]
    plans = [pl.NoisePlan.for_windows(pl.derive_seed(77, 10 ** 9 + i), N) for i in range(R)]
    t0 = time.perf_counter()
    res = pl.parareal_adaptive_batch(inits, pair, params, sched, plans, cfg)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    labels = sia.sia_site_labels(np.stack([r.trajectory.positions() for r in res]), 4, W.A0)
    hops = int(sum(np.count_nonzero(np.diff(lab)) for lab in labels))
    fine_windows = sum(sum(a.iterations * (a.n_final - s.n_init) for a in s.attempts) for r in res for s in r.slabs)
    return {"config": f"ensemble: {R} replicas x {N} slices x {L} steps, T = {T:g} K, SNAP/EAM",
            "wall_s": wall, "converged": int(sum(r.converged for r in res)),
            "mean_sum_k": float(np.mean([r.total_iterations for r in res])),
            "fine_atom_steps_per_s": fine_windows * n * L / wall, "sia_hops": hops}


def heavy(L=100):
    q0, box = W.bcc_sia(20)
    n = q0.shape[0] // 3
    params = pl.LangevinParams(1.0, W.KB * 1000.0, 0.001, L, mass=np.full(3 * n, W.MASS_W))
    sched = pl.TemperatureSchedule.robust(L)
    st = pl.PhaseState(q=q0, p=W.maxwell_boltzmann(n, 1000.0, 11))
    snap = W.make_snap(n, box)
    t, _ = timed(lambda: pl.propagate_windows([st], snap, params, sched, [pl.derive_seed(11, 1)]))
    return {"config": f"heavy: {n} atoms, one SNAP window of {L} substeps (cell lists)", "wall_s": t,
            "atom_steps_per_s": n * L / t}


def larger_parareal(N=64, L=200):
    q0, box = W.bcc_sia(8)
    n = q0.shape[0] // 3
    params = pl.LangevinParams(1.0, W.KB * 1000.0, 0.001, L, mass=np.full(3 * n, W.MASS_W))
    sched = pl.TemperatureSchedule.robust(L)
    init = pl.PhaseState(q=q0, p=W.maxwell_boltzmann(n, 1000.0, 11))
    pair = pl.PropagatorPair(W.make_snap(n, box), W.make_eam(n, box), 100.0, 1.0)
    plan = pl.NoisePlan.for_windows(11, N)
    t, res = timed(lambda: pl.parareal_adaptive(init, pair, params, sched, plan,
                                                pl.PararealConfig(N, 1e-10, 0.35)))
    return {"config": f"larger adaptive parareal: {n} atoms, {N} x {L}, SNAP/EAM", "wall_s": t,
            "n_slab": res.n_slab, "sum_k": res.total_iterations}


def main():
    which = sys.argv[1:] or ["sweep", "pr1", "heavy"]
    fns = {"sweep": force_sweep, "pr1": pr1_parareal, "ensemble": ensemble, "heavy": heavy,
           "larger_parareal": larger_parareal}
    for w in which:
        try:
            print(json.dumps(fns[w]()), flush=True)
        except Exception as exc:  # report and continue
            print(json.dumps({"config": w, "error": f"{type(exc).__name__}: {exc}"}), flush=True)


if __name__ == "__main__":
    main()
