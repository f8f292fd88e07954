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


def ensemble(R=256, N=32, L=100, T=1200.0, segments=None):
    """configs[3]: R replicas x N slices x L steps at 1200 K, chained 3.2 ps segments.

    20 ps / 3.2 ps = 6.25: the full config is 7 segments (the 7th overruns to
    22.4 ps).  ``segments`` (env PL_ENSEMBLE_SEGMENTS, default 1) segments are
    run, each from the previous segment's final states with fresh window seeds;
    the wall-clock of the full config is extrapolated linearly from them and
    labelled as such.  SIA site labels of every node feed the residence times.
    """
    segments = int(os.environ.get("PL_ENSEMBLE_SEGMENTS", "1")) if segments is None else segments
    q0, box, n, params, sched = _pr1(T=T, N=N, L=L)
    pair = pl.PropagatorPair(W.make_snap(n, box), W.make_eam(n, box), 100.0, 1.0)
    cfg = pl.PararealConfig(N, 1e-5, 0.35)  # delta_conv of configs/ensemble.json
    rs = np.random.default_rng(7)
    states = [pl.PhaseState(q=q0 + 0.03 * rs.normal(size=q0.shape),
                            p=math.sqrt(W.MASS_W * W.KB * T) * rs.normal(size=q0.shape)) for _ in range(R)]
    walls, conv, sumk, fine_windows = [], 0, [], 0
    label_chunks = []
    for seg in range(segments):
        plans = [pl.NoisePlan.for_windows(pl.derive_seed(77, 10 ** 9 + seg * R + i), N) for i in range(R)]
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = pl.parareal_adaptive_batch(states, pair, params, sched, plans, cfg)
        torch.cuda.synchronize()
        walls.append(time.perf_counter() - t0)
        conv += int(sum(r.converged for r in res))
        sumk += [r.total_iterations for r in res]
        fine_windows += sum(sum(a.iterations * (a.n_final - s.n_init) for a in s.attempts)
                            for r in res for s in r.slabs)
        pos = np.stack([r.trajectory.positions() for r in res])  # (R, N+1, d)
        label_chunks.append(sia.sia_site_labels(pos if seg == 0 else pos[:, 1:], 4, W.A0))
        states = [r.trajectory[r.trajectory.n_windows] for r in res]
    labels = np.concatenate(label_chunks, axis=1)
    hops = int(sum(np.count_nonzero(np.diff(lab)) for lab in labels))
    events = [e for lab in labels for e in sia.residence_times(lab)]
    done = [e.duration for e in events if not e.censored]
    mean, lo, hi = sia.mean_ci(done) if len(done) >= 2 else (float("nan"),) * 3
    wall = float(sum(walls))
    return {"config": f"ensemble: {R} replicas x {N} slices x {L} steps per 3.2 ps segment, T = {T:g} K, SNAP/EAM",
            "segments_run": segments, "segment_wall_s": walls, "wall_s": wall,
            "full_config_wall_s_extrapolated": wall / segments * 7,
            "converged": conv, "mean_sum_k": float(np.mean(sumk)),
            "fine_atom_steps_per_s": fine_windows * n * L / wall, "sia_hops": hops,
            "residence_windows_mean_ci": [mean, lo, hi], "residence_events": len(done)}


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
    for name, i, f in (("k_snap_ui_r4", 1, fl["ui"]), ("k_snap_yi_box", 2, fl["yi"]),
                       ("k_snap_deidrj_pair", 3, fl["deidrj"])):
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
