"""Benchmark: SNAP Langevin atom-steps/s over batched parareal slices (+ parareal wall-clock).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config larger]

A "step" is the fine stage of one parareal iteration: every slice of the
workload propagated through one window of L BBK substeps with the SNAP
(twojmax = 8, fp64) potential, batched in one ``pl_propagate_windows`` call,
followed (N > 1) by the NCCL all-gather of the slice endpoints that the
coarse sweep consumes.  Default workload = BASELINE configs[2]
("larger"): BCC W 8x8x8 + <111> SIA = 1025 atoms, 64 slices x L = 200, per
rank (weak scaling: every rank owns its own 64 slices).

value     fine atom-steps/s of the whole job, inputs resident in HBM
e2e       the same through the public API (host PhaseStates in, host states
          out, H2D/D2H and device noise generation inside the timed region)
roofline  dominant kernel (k_snap_yi / k_snap_deidrj / ...) algorithmic FP64
          FLOPs per launch / live CUDA-event duration, against the DFMA peak
          measured on this device by pl_fp64_peak (FP64 is not in
          MEASURED_PEAKS.json)
cpu_baseline  the C oracle (oracle/native, "port") on the host cores, bounded
          sample, rank 0 only
parareal  wall-clock of one adaptive parareal run of BASELINE configs[0] (PR1:
          129 atoms, 16 slices x 100, SNAP fine / EAM coarse), fine stage
          sharded over all ranks (max over ranks)
--impl reference  the CPU reference arm: the oracle port of the reference
          path (oracle/: BBK integrator + C SNAP) on all host cores.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np

CONFIGS = {
    # name: (cells, slices per rank, substeps L, temperature K)
    "larger": (8, 64, 200, 1000.0),
    "pr1": (4, 16, 100, 1000.0),
    "heavy": (20, 1, 1000, 1000.0),
}
GAMMA, DT = 1.0, 0.001  # ps^-1, ps


def _env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


# ---------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index, self.samples, self.proc = index, [], None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 6:
                self.samples.append(parts)

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(sm)}


# ---------------------------------------------------------------- workload
def build_inputs(cfg_name, rank, world):
    from paper_2212_10508_b200 import tungsten as W
    cells, slices, L, T = CONFIGS[cfg_name]
    q0, box = W.bcc_sia(cells)
    n = q0.shape[0] // 3
    rs = np.random.default_rng(1000 + rank)
    # slice start states: thermalised-looking lattice (0.05 A jitter) + MB momenta
    Q = q0[None, :] + 0.05 * rs.normal(size=(slices, q0.shape[0]))
    P = math.sqrt(W.MASS_W * W.KB * T) * rs.normal(size=(slices, q0.shape[0]))  # Maxwell-Boltzmann
    seeds = [int(x) for x in __import__("paper_2212_10508_b200").derive_seeds(11 + rank, slices)]
    return dict(q0=q0, box=box, n=n, Q=Q, P=P, seeds=seeds, L=L, T=T, slices=slices, cells=cells)


def snap_flops_per_eval(pot, Qdev):
    """Algorithmic FLOPs of one SNAP force evaluation over the batch Qdev (B, 3N)."""
    import ctypes as C
    import torch
    from paper_2212_10508_b200 import _lib
    ctx = _lib.context()
    lib = _lib.load()
    counts = np.zeros(5, dtype=np.int32)
    fl = np.zeros(3)
    _lib.check(lib.pl_snap_info(pot.handle(ctx), counts.ctypes.data_as(_lib.pi32), _lib.dptr(fl)))
    B, d = Qdev.shape
    n = d // 3
    maxn = 64
    nbr = torch.zeros((B, n, maxn), dtype=torch.int32, device=Qdev.device)
    cnt = torch.zeros((B, n), dtype=torch.int32, device=Qdev.device)
    _lib.check(lib.pl_neighbours(ctx.handle, pot.handle(ctx), B, _lib.ptr(Qdev), maxn,
                                 _lib.ptr(nbr), _lib.ptr(cnt)))
    pairs = float(cnt.sum().item())
    atoms = float(B * n)
    return dict(ui=pairs * fl[0], yi=atoms * fl[1], deidrj=pairs * fl[2], pairs=pairs, atoms=atoms,
                per_pair_ui=fl[0], per_atom_yi=fl[1], per_pair_de=fl[2])


def run_ours(args, rank, world, local_rank):
    import torch
    import paper_2212_10508_b200 as pl
    from paper_2212_10508_b200 import _lib, tungsten as W
    from paper_2212_10508_b200.integrator import WindowKernel

    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    inp = build_inputs(args.config, rank, world)
    n, L, T = inp["n"], inp["L"], inp["T"]
    slices = inp["slices"]
    d = 3 * n
    mass = np.full(d, W.MASS_W)
    params = pl.LangevinParams(GAMMA, W.KB * T, DT, L, mass=mass)
    sched = pl.TemperatureSchedule.robust(L)
    pot = W.make_snap(n, inp["box"])
    k = WindowKernel(pot, params, sched, d)
    dev = k.device
    Q0 = torch.from_numpy(inp["Q"]).to(dev)
    P0 = torch.from_numpy(inp["P"]).to(dev)
    noise = k.noise(inp["seeds"])           # iteration-invariant: generated once (HBM resident)
    Q1 = torch.empty_like(Q0)
    P1 = torch.empty_like(P0)
    gathered = torch.empty((world, 2, slices, d), dtype=torch.float64, device=dev) if world > 1 else None
    ends = torch.empty((2, slices, d), dtype=torch.float64, device=dev)

    def step():
        k.run(Q0, P0, noise, Q1, P1)
        if world > 1:
            ends[0].copy_(Q1)
            ends[1].copy_(P1)
            dist.all_gather_into_tensor(gathered.view(-1), ends.view(-1))

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local_rank)
    clocks.start()
    lib, ctx = _lib.load(), _lib.context()
    _lib.check(lib.pl_prof_begin(ctx.handle))
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(st)
    for _ in range(args.steps):
        step()
    e1.record(st)
    torch.cuda.synchronize()
    stage_ms = np.zeros(8)
    stage_n = np.zeros(8, dtype=np.int64)
    _lib.check(lib.pl_prof_end(ctx.handle, 8, _lib.dptr(stage_ms), stage_n.ctypes.data_as(_lib.pi64)))
    clk = clocks.stop()
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    blow = int((k.run(Q0, P0, noise, Q1, P1)[2] != 0).sum().item())

    atom_steps = float(world) * slices * n * L * args.steps
    value = atom_steps / (ms * 1e-3)

    # ---- roofline of the dominant kernel (live CUDA events over the timed region)
    fl = snap_flops_per_eval(pot, Q0)
    names = ["neigh", "snap_ui", "snap_yi", "snap_deidrj", "snap_gather", "eam", "integrator"]
    flops_per_launch = {"snap_ui": fl["ui"], "snap_yi": fl["yi"], "snap_deidrj": fl["deidrj"]}
    share = {names[i]: stage_ms[i] / max(stage_ms.sum(), 1e-30) for i in range(7)}
    dom = max(flops_per_launch, key=lambda s: stage_ms[names.index(s)])
    di = names.index(dom)
    avg_launch_s = stage_ms[di] / max(stage_n[di], 1) * 1e-3
    peak = ctypes_peak()
    achieved = flops_per_launch[dom] / avg_launch_s / 1e12
    snap_ms = stage_ms[1:5].sum()
    snap_flops_total = (fl["ui"] + fl["yi"] + fl["deidrj"]) * stage_n[2]
    roof = {"bound": "fp64", "kernel": f"k_{dom}", "achieved": round(achieved, 3),
            "peak": round(peak, 3), "unit": "TFLOP/s", "frac": round(achieved / peak, 4),
            "peak_source": "measured DFMA (pl_fp64_peak) on this B200; FP64 absent from MEASURED_PEAKS.json",
            "traffic": ncu_traffic(f"k_{dom}"),
            "flops_per_launch": fl[{"snap_ui": "ui", "snap_yi": "yi", "snap_deidrj": "deidrj"}[dom]],
            "snap_all_kernels_tflops": round(snap_flops_total / (snap_ms * 1e-3) / 1e12, 3),
            "stage_share": {k_: round(v, 4) for k_, v in share.items()},
            "flop_model": {"per_pair_ui": fl["per_pair_ui"], "per_atom_yi": fl["per_atom_yi"],
                           "per_pair_deidrj": fl["per_pair_de"],
                           "pairs_per_eval": fl["pairs"], "atoms_per_eval": fl["atoms"]}}

    # ---- e2e through the public API (host states in / out, noise generated in the call)
    states = [pl.PhaseState(q=inp["Q"][i], p=inp["P"][i]) for i in range(slices)]
    pl.propagate_windows(states, pot, params, sched, inp["seeds"])  # warm
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e2e_steps = max(1, min(args.steps, 3))
    for _ in range(e2e_steps):
        outs = pl.propagate_windows(states, pot, params, sched, inp["seeds"])
    torch.cuda.synchronize()
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    if world > 1:
        t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e = {"value": float(world) * slices * n * L / e2e_s, "unit": "atom-steps/s",
           "h2d_bytes_per_step": int(2 * slices * d * 8 + slices * 8),
           "d2h_bytes_per_step": int(2 * slices * d * 8 + slices * 4),
           "api": "paper_2212_10508_b200.propagate_windows(host PhaseStates, SNAP, ...)"}
    del outs

    cpu = None
    parareal = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(args, inp, pot, budget_s=args.cpu_seconds)
    if not args.no_parareal:
        # every rank runs the engine: the fine stage is sharded over ranks with one
        # NCCL all-gather per iteration (distributed.sharded_fine)
        parareal = parareal_run()
        if world > 1 and isinstance(parareal, dict) and "wall_s" in parareal:
            t = torch.tensor([parareal["wall_s"]], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            parareal["wall_s"] = float(t.item())
            parareal["ranks"] = world

    if rank == 0:
        # L+1 SNAP evaluations per window batch, each: neighbours (cell lists at >= 512
        # atoms and >= 3 cells per axis: count, scan, fill, list; else one brute-force
        # kernel), ui, yi (+ k_box_energy when a batch has fewer 32-atom blocks than SMs
        # and the Y rows are split over 2 CTAs), ytrans, deidrj (pair form), gather;
        # + open/close per substep
        cells = n >= 512 and min(inp["box"]) / 4.73 >= 3
        split = (slices * n + 31) // 32 < 148
        launches_per_step = (L + 1) * ((4 if cells else 1) + 5 + (1 if split else 0)) + 2 * L
        line = {
            "metric": "SNAP Langevin atom-steps/s over batched parareal slices",
            "value": value, "unit": "atom-steps/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.config}: BCC W {inp['cells']}^3 + <111> SIA = {n} atoms, "
                                   f"{slices} slices/rank x L={L} BBK substeps, SNAP twojmax=8 fp64, "
                                   f"T={T:g} K, gamma=1/ps, dt=1 fs",
                       "slices_per_rank": slices, "atoms": n, "substeps": L,
                       "l2": "inputs larger than L2 (noise blocks "
                             f"{noise.numel() * 8 / 1e6:.0f} MB per rank)",
                       "parallelism": f"slices sharded over {world} rank(s), NCCL all-gather of endpoints"},
            "clocks": clk, "e2e": e2e, "roofline": roof, "cpu_baseline": cpu,
            "gpu_launches": int(launches_per_step * args.steps),
            "blowups": blow,
            "parareal": parareal,
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


def ctypes_peak():
    from paper_2212_10508_b200 import _lib
    out = np.zeros(1)
    best = 0.0
    for _ in range(3):
        _lib.check(_lib.load().pl_fp64_peak(_lib.context().handle, _lib.dptr(out)))
        best = max(best, float(out[0]))
    return best


# ---------------------------------------------------------------- CPU arms
def _cpu_windows(inp, slices_sample, substeps, threads):
    """Oracle BBK + C SNAP on host threads; returns (atom-steps, seconds)."""
    from concurrent.futures import ThreadPoolExecutor
    from oracle import integrator as oint, native, rng as orng
    from paper_2212_10508_b200 import tungsten as W
    n, box = inp["n"], inp["box"]
    d = 3 * n
    mass = np.full(d, W.MASS_W)
    pot = W.make_snap(n, box)
    grad = native.snap_fn(pot)
    native.load()
    sched = oint.robust(substeps)

    def one(i):
        noise = orng.gaussian_stream(inp["seeds"][i % len(inp["seeds"])], (substeps + 1) * d)
        oint.propagate_window(inp["Q"][i % inp["slices"]], inp["P"][i % inp["slices"]], grad, GAMMA,
                              W.KB * inp["T"], DT, substeps, sched, 0, mass=mass, noise=noise)

    t = time.perf_counter()
    with ThreadPoolExecutor(max_workers=threads) as ex:
        list(ex.map(one, range(slices_sample)))
    return float(n * substeps * slices_sample), time.perf_counter() - t


def cpu_baseline(args, inp, pot, budget_s=20.0):
    threads = os.cpu_count() or 1
    # calibrate: one substep window on one thread
    s1, t1 = _cpu_windows(inp, 1, 1, 1)
    per_eval = t1 / 2.0
    substeps = max(1, min(inp["L"], int(budget_s / max(per_eval, 1e-9) / 2) // 1))
    substeps = max(1, min(substeps, 4))
    windows = threads
    steps, secs = _cpu_windows(inp, windows, substeps, threads)
    return {"value": steps / secs, "unit": "atom-steps/s", "cores": threads, "kind": "port",
            "sample": f"{windows} slices x {substeps} BBK substeps of the {inp['n']}-atom SNAP window "
                      f"(oracle/native C SNAP + oracle BBK, one slice per thread), {secs:.1f} s"}


def run_reference(args, rank, world):
    if rank != 0:
        return
    inp = build_inputs(args.config, 0, 1)
    threads = os.cpu_count() or 1
    _cpu_windows(inp, 1, 1, 1)  # warm (loads liboracle)
    per = []
    for _ in range(args.warmup):
        _cpu_windows(inp, threads, 1, threads)
    for _ in range(args.steps):
        steps, secs = _cpu_windows(inp, threads, 1, threads)
        per.append((steps, secs))
    steps = sum(s for s, _ in per)
    secs = sum(t for _, t in per)
    v = steps / secs
    line = {"impl": "reference", "metric": "SNAP Langevin atom-steps/s over batched parareal slices",
            "value": v, "unit": "atom-steps/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": secs / max(len(per), 1) * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": f"{args.config}: {inp['n']} atoms SNAP twojmax=8 fp64 BBK windows",
                       "sample": f"{threads} slices x 1 substep per step"},
            "cpu_baseline": {"value": v, "unit": "atom-steps/s", "cores": threads, "kind": "port",
                             "sample": f"{threads} slices x 1 BBK substep per step "
                                       "(reference path restated in oracle/: BBK integrator + C SNAP)"},
            "e2e": {"value": v, "unit": "atom-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def ncu_traffic(kernel):
    """DRAM bytes (read + write) per launch of the dominant kernel from the committed
    ncu --set full capture of this config (profiles/r1_traffic.json), else None."""
    try:
        with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r1_traffic.json")) as f:
            t = json.load(f)
        return t["kernels"].get(kernel)
    except (OSError, ValueError, KeyError):
        return None


# ---------------------------------------------------------------- parareal wall-clock (PR1)
def parareal_run():
    import torch
    import paper_2212_10508_b200 as pl
    from paper_2212_10508_b200 import tungsten as W
    q0, box = W.bcc_sia(4)
    n = q0.shape[0] // 3
    mass = np.full(3 * n, W.MASS_W)
    L, N = 100, 16
    params = pl.LangevinParams(GAMMA, W.KB * 1000.0, DT, L, mass=mass)
    sched = pl.TemperatureSchedule.robust(L)
    plan = pl.NoisePlan.for_windows(11, N)
    init = pl.PhaseState(q=q0, p=W.maxwell_boltzmann(n, 1000.0, 11))
    eam = W.make_eam(n, box)
    snap = W.make_snap(n, box)
    pair = pl.PropagatorPair(snap, eam, 100.0, 1.0)
    cfg = pl.PararealConfig(N, 1e-10, 0.35)   # delta_conv / delta_expl of configs/adaptive.json
    # the first run pays the one-time setup (SNAP index tables and Y-row schedules,
    # buffer allocations); wall_s is a second, warm run (every engine run starts
    # from an empty fine-window cache, so nothing carries over but the setup)
    walls = []
    for _ in range(2):
        torch.cuda.synchronize()
        t = time.perf_counter()
        try:
            res = pl.parareal_adaptive(init, pair, params, sched, plan, cfg)
        except Exception as exc:  # report, do not fail the bench
            return {"error": f"{type(exc).__name__}: {exc}"}
        torch.cuda.synchronize()
        walls.append(time.perf_counter() - t)
    wall = walls[1]
    # measured per-window costs C_f / C_c (one window, device-resident, CUDA events)
    # and the reference cost model's gain Gamma (accounting.py:141-159)
    from paper_2212_10508_b200 import accounting
    from paper_2212_10508_b200.integrator import WindowKernel

    def window_ms(pot, reps=5):
        k = WindowKernel(pot, params, sched, 3 * n)
        Q0 = torch.from_numpy(q0[None].copy()).to(k.device)
        P0 = torch.from_numpy(init.p[None].copy()).to(k.device)
        noise = k.noise([plan.window_seeds[0]])
        k.run(Q0, P0, noise)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record()
        for _ in range(reps):
            k.run(Q0, P0, noise)
        ev[1].record()
        torch.cuda.synchronize()
        return ev[0].elapsed_time(ev[1]) / reps

    cf, cc = window_ms(snap), window_ms(eam)
    g = accounting.adaptive_gain(res.slabs, N, cf, cc)
    return {"config": "PR1: 129 atoms, 16 slices x 100, SNAP fine / EAM coarse, delta_conv 1e-10, "
                      "delta_expl 0.35", "wall_s": wall, "wall_s_cold": walls[0], "n_slab": res.n_slab,
            "sum_k": res.total_iterations, "converged": res.converged,
            "cf_ms": cf, "cc_ms": cc, "gain_model": g.gain, "gain_ideal": g.ideal_gain,
            "sequential_fine_s": N * cf / 1e3, "speedup_vs_sequential_fine": (N * cf / 1e3) / wall}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="larger", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-parareal", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=20.0)
    args = ap.parse_args()
    rank = _env_int("RANK", 0)
    world = _env_int("WORLD_SIZE", 1)
    local_rank = _env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
