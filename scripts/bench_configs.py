"""One-off measurements of the other BASELINE configs (bench.py covers configs[2]).

    python scripts/bench_configs.py [sweep] [pr1] [ensemble] [heavy] [larger_parareal] [heavy_parareal]

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


def ensemble(R=256, N=32, L=100, T=1200.0, segments=None):
    """configs[3]: the reference ensemble protocol (cli.py:986-1050, paper_2212_10508_b200.ensemble)
    with R replicas of the 129-atom W + SIA system at 1200 K: minimise on the fine (SNAP) surface,
    thermalise 10 windows, then per member a sequential fine chain and adaptive parareal (32 slices
    x 100 steps = 3.2 ps per segment, delta from configs/ensemble.json) over the same plans,
    chained for ``segments`` segments (20 ps / 3.2 ps = 6.25: 7 segments = 22.4 ps), SIA site
    labels of quenched nodes, min_run 2, compare_ensembles of the two pooled CIs."""
    from paper_2212_10508_b200.ensemble import run_ensemble
    segments = int(os.environ.get("PL_ENSEMBLE_SEGMENTS", "7")) if segments is None else segments
    R = int(os.environ.get("PL_ENSEMBLE_SIZE", R))
    q0, box, n, params, sched = _pr1(T=T, N=N, L=L)
    pair = pl.PropagatorPair(W.make_snap(n, box), W.make_eam(n, box), 100.0, 1.0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = run_ensemble(pair, params, sched, pl.PhaseState(q=q0, p=np.zeros_like(q0)),
                       pl.PararealConfig(N, 1e-5, 0.35), size=R, master_seed=77, n_cells=4, a=W.A0,
                       segments=segments, thermalization_windows=10, min_run=2, quench=True)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    out = {"config": f"ensemble: {R} replicas x {segments} segments x {N} slices x {L} steps, T = {T:g} K, "
                     "SNAP fine / EAM coarse, quenched SIA site labels, min_run 2", "wall_s": wall}
    out.update(res.as_dict())
    return out


def heavy_parareal(N=8, L=1000):
    """configs[4] end to end on one GPU: adaptive parareal, 16,001 atoms, 8 slices x 1000 steps,
    SNAP fine (8 windows batched, cell lists) / EAM coarse sweep on the device (per-window path)."""
    q0, box = W.bcc_sia(20)
    n = q0.shape[0] // 3
    params = pl.LangevinParams(1.0, W.KB * 1000.0, 0.001, L, mass=np.full(3 * n, W.MASS_W))
    sched = pl.TemperatureSchedule.robust(L)
    init = pl.PhaseState(q=q0, p=W.maxwell_boltzmann(n, 1000.0, 11))
    pair = pl.PropagatorPair(W.make_snap(n, box), W.make_eam(n, box), 100.0, 1.0)
    plan = pl.NoisePlan.for_windows(11, N)
    torch.cuda.synchronize()
    t = time.perf_counter()
    res = pl.parareal_adaptive(init, pair, params, sched, plan, pl.PararealConfig(N, 1e-10, 0.35))
    torch.cuda.synchronize()
    wall = time.perf_counter() - t
    t = time.perf_counter()
    pl.sequential_propagate(init, N, pair.fine, params, sched, plan)
    torch.cuda.synchronize()
    seq = time.perf_counter() - t
    return {"config": f"heavy adaptive parareal: {n} atoms, {N} x {L}, SNAP/EAM", "wall_s": wall,
            "n_slab": res.n_slab, "sum_k": res.total_iterations, "converged": res.converged,
            "sequential_fine_s": seq}


def heavy(L=1000):
    """configs[4] on one GPU: one 16001-atom SNAP window of L = 1000 substeps (cell lists),
    with the per-kernel FP64 roofline fractions the config asks for (live stage events)."""
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    from paper_2212_10508_b200 import _lib
    q0, box = W.bcc_sia(20)
    n = q0.shape[0] // 3
    params = pl.LangevinParams(1.0, W.KB * 1000.0, 0.001, L, mass=np.full(3 * n, W.MASS_W))
    sched = pl.TemperatureSchedule.robust(L)
    st = pl.PhaseState(q=q0, p=W.maxwell_boltzmann(n, 1000.0, 11))
    snap = W.make_snap(n, box)
    from paper_2212_10508_b200.integrator import WindowKernel
    k = WindowKernel(snap, params, sched, 3 * n)
    Q0 = torch.from_numpy(q0[None].copy()).to(k.device)
    P0 = torch.from_numpy(st.p[None].copy()).to(k.device)
    noise = k.noise([pl.derive_seed(11, 1)])
    k.run(Q0, P0, noise)  # warm (also the neighbour/cell buffers)
    torch.cuda.synchronize()
    lib, ctx = _lib.load(), _lib.context()
    _lib.check(lib.pl_prof_begin(ctx.handle))
    t = time.perf_counter()
    k.run(Q0, P0, noise)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t
    ms = np.zeros(8)
    cnt = np.zeros(8, dtype=np.int64)
    _lib.check(lib.pl_prof_end(ctx.handle, 8, _lib.dptr(ms), cnt.ctypes.data_as(_lib.pi64)))
    fl = bench.snap_flops_per_eval(snap, Q0)
    peak = bench.ctypes_peak()
    per_kernel = {}
    for name, i, f in (("k_snap_ui_r4", 1, fl["ui"]), ("k_snap_yi_p", 2, fl["yi"]),
                       ("k_snap_deidrj_tm", 3, fl["deidrj"])):
        t_launch = ms[i] / max(cnt[i], 1) * 1e-3
        tf = f / t_launch / 1e12
        per_kernel[name] = {"ms_per_launch": round(ms[i] / max(cnt[i], 1), 4), "tflops": round(tf, 3),
                            "frac": round(tf / peak, 4)}
    per_kernel["neighbours_ms_per_launch"] = round(ms[0] / max(cnt[0], 1), 4)
    per_kernel["gather_ms_per_launch"] = round(ms[4] / max(cnt[4], 1), 4)
    return {"config": f"heavy: {n} atoms, one SNAP window of {L} substeps (cell lists)", "wall_s": wall,
            "atom_steps_per_s": n * L / wall, "fp64_peak_tflops": round(peak, 3), "per_kernel": per_kernel}


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
    from paper_2212_10508_b200 import parareal as par
    return {"config": f"larger adaptive parareal: {n} atoms, {N} x {L}, SNAP/EAM", "wall_s": t,
            "n_slab": res.n_slab, "sum_k": res.total_iterations, **par.LAST_RUN_STATS}


def main():
    which = sys.argv[1:] or ["sweep", "pr1", "heavy"]
    fns = {"sweep": force_sweep, "pr1": pr1_parareal, "ensemble": ensemble, "heavy": heavy,
           "larger_parareal": larger_parareal, "heavy_parareal": heavy_parareal}
    for w in which:
        try:
            print(json.dumps(fns[w]()), flush=True)
        except Exception as exc:  # report and continue
            print(json.dumps({"config": w, "error": f"{type(exc).__name__}: {exc}"}), flush=True)


if __name__ == "__main__":
    main()
