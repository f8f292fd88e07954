"""Benchmark: SNAP Langevin atom-steps/s over batched parareal slices (+ parareal wall-clock).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config larger|pr1|heavy] [--scaling strong|weak]

A "step" is the fine stage of one parareal iteration: every slice of the
workload propagated through one window of L BBK substeps with the SNAP
(twojmax = 8, fp64) potential, batched in one ``pl_propagate_windows`` call per
rank, followed (N > 1) by the NCCL all-gather of the slice endpoints that the
coarse sweep consumes.  Default workload = BASELINE configs[2]
("larger"): BCC W 8x8x8 + <111> SIA = 1025 atoms, 64 slices x L = 200.
``--scaling strong`` (default, the config as stated): the 64 slices are
sharded over the N ranks (8 per GPU at N = 8).  ``--scaling weak``: 64 slices
per rank.

``--gpus N`` without torchrun re-launches this script under
``torch.distributed.run`` with N ranks (one per GPU, NCCL over NVLink); under
torchrun it must equal WORLD_SIZE.

value     fine atom-steps/s of the whole job (max-over-ranks device time),
          inputs resident in HBM, no profiling events in the timed region
e2e       the same through the public API (host PhaseStates in, host states
          out, H2D/D2H and device noise generation inside the timed region)
roofline  dominant kernel, from a separate profiled pass of the same steps
          (live CUDA events per stage): algorithmic FP64 FLOPs per launch /
          average launch duration, against the DFMA peak measured on this
          device (pl_fp64_peak; FP64 is not in MEASURED_PEAKS.json).  ``hbm``
          lists the HBM-bound kernels (integrator, EAM force sweep, coarse
          sweep) against MEASURED_PEAKS.json hbm_gbs.
cpu_baseline  the reference path on the host cores (rank 0, N = 1): the oracle
          restatement of the reference BBK window (oracle/integrator.py
          WindowStepper) with the C SNAP oracle, one slice per thread -- the
          same code and the same per-substep work as --impl reference
parareal  adaptive parareal wall-clock of configs[0] (PR1) and configs[2]
          (larger), fine stage sharded over all ranks (max over ranks), with
          the sequential-fine time of the same trajectory on the same GPUs
--impl reference  the CPU reference arm: the same sample as cpu_baseline, all
          host threads, on this arm's config / metric (rank 0 only).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import socket
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np

METRIC = "SNAP Langevin atom-steps/s over batched parareal slices"
CONFIGS = {
    # name: (cells, slices of the job, substeps L, temperature K)
    "larger": (8, 64, 200, 1000.0),
    "pr1": (4, 16, 100, 1000.0),
    "heavy": (20, 8, 1000, 1000.0),
}
GAMMA, DT = 1.0, 0.001  # ps^-1, ps
CPU_SUBSTEPS = 4        # substeps per CPU-arm step (one slice per host thread)


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
def build_inputs(cfg_name):
    """All slices of the job (deterministic, independent of the rank count)."""
    import paper_2212_10508_b200 as pl
    from paper_2212_10508_b200 import tungsten as W
    cells, slices, L, T = CONFIGS[cfg_name]
    q0, box = W.bcc_sia(cells)
    n = q0.shape[0] // 3
    rs = np.random.default_rng(1000)
    # slice start states: thermalised-looking lattice (0.05 A jitter) + Maxwell-Boltzmann momenta
    Q = q0[None, :] + 0.05 * rs.normal(size=(slices, q0.shape[0]))
    P = math.sqrt(W.MASS_W * W.KB * T) * rs.normal(size=(slices, q0.shape[0]))
    seeds = [int(x) for x in pl.derive_seeds(11, slices)]
    return dict(q0=q0, box=box, n=n, Q=Q, P=P, seeds=seeds, L=L, T=T, slices=slices, cells=cells)


def rank_block(inp, rank, world, scaling):
    """Slices of this rank: a contiguous block (strong) or the whole set again (weak)."""
    S = inp["slices"]
    if scaling == "weak":
        return list(range(S))
    from paper_2212_10508_b200.distributed import shard_bounds
    lo, hi = shard_bounds(0, S, world, rank)
    return list(range(lo, hi))


def snap_flops_per_eval(pot, Qdev):
    """Algorithmic FLOPs of one SNAP force evaluation over the batch Qdev (B, 3N)."""
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


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except (OSError, ValueError):
        return {}


def hbm_peak():
    pk = _peaks()
    if "hbm_gbs" in pk:
        return float(pk["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (copy bandwidth, this pool's B200s)"
    return 7700.0, "fallback: B200 HBM3e nominal 7.7 TB/s (MEASURED_PEAKS.json absent)"


def ctypes_peak():
    from paper_2212_10508_b200 import _lib
    out = np.zeros(1)
    best = 0.0
    for _ in range(3):
        _lib.check(_lib.load().pl_fp64_peak(_lib.context().handle, _lib.dptr(out)))
        best = max(best, float(out[0]))
    return best


def _max_over_ranks(x, dev, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


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
    inp = build_inputs(args.config)
    n, L, T = inp["n"], inp["L"], inp["T"]
    mine = rank_block(inp, rank, world, args.scaling)
    slices = len(mine)
    total_slices = slices * world if args.scaling == "weak" else inp["slices"]
    d = 3 * n
    mass = np.full(d, W.MASS_W)
    params = pl.LangevinParams(GAMMA, W.KB * T, DT, L, mass=mass)
    sched = pl.TemperatureSchedule.robust(L)
    pot = W.make_snap(n, inp["box"])
    k = WindowKernel(pot, params, sched, d)
    dev = k.device
    Q0 = torch.from_numpy(inp["Q"][mine]).to(dev)
    P0 = torch.from_numpy(inp["P"][mine]).to(dev)
    seeds = [inp["seeds"][i] for i in mine]
    noise = k.noise(seeds)                  # iteration-invariant: generated once (HBM resident)
    Q1 = torch.empty_like(Q0)
    P1 = torch.empty_like(P0)
    ends = torch.empty((2, slices, d), dtype=torch.float64, device=dev)
    gathered = torch.empty((world, 2, slices, d), dtype=torch.float64, device=dev) if world > 1 else None

    def step():
        k.run(Q0, P0, noise, Q1, P1)
        if world > 1:
            ends[0].copy_(Q1)
            ends[1].copy_(P1)
            dist.all_gather_into_tensor(gathered.view(-1), ends.view(-1))

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step()
    barrier()
    clocks = ClockSampler(local_rank)
    clocks.start()
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(args.steps):
        step()
    e1.record(st)
    barrier()
    clk = clocks.stop()
    ms = _max_over_ranks(e0.elapsed_time(e1), dev, world)
    blow = int((k.run(Q0, P0, noise, Q1, P1)[2] != 0).sum().item())
    atom_steps = float(total_slices) * n * L * args.steps
    value = atom_steps / (ms * 1e-3)

    # ---- profiled pass (separate from the timed region): per-stage CUDA events
    lib, ctx = _lib.load(), _lib.context()
    prof_steps = max(1, min(args.steps, 3))
    barrier()
    _lib.check(lib.pl_prof_begin(ctx.handle))
    p0 = torch.cuda.Event(enable_timing=True)
    p1 = torch.cuda.Event(enable_timing=True)
    p0.record(st)
    for _ in range(prof_steps):
        step()
    p1.record(st)
    torch.cuda.synchronize()
    stage_ms = np.zeros(8)
    stage_n = np.zeros(8, dtype=np.int64)
    _lib.check(lib.pl_prof_end(ctx.handle, 8, _lib.dptr(stage_ms), stage_n.ctypes.data_as(_lib.pi64)))
    prof_ms_per_step = p0.elapsed_time(p1) / prof_steps

    fl = snap_flops_per_eval(pot, Q0)
    names = ["neigh", "snap_ui", "snap_yi", "snap_deidrj", "snap_gather", "eam", "integrator"]
    flops_per_launch = {"snap_ui": fl["ui"], "snap_yi": fl["yi"], "snap_deidrj": fl["deidrj"]}
    share = {names[i]: stage_ms[i] / max(stage_ms.sum(), 1e-30) for i in range(7)}
    dom = max(flops_per_launch, key=lambda s: stage_ms[names.index(s)])
    peak = ctypes_peak()

    def kfrac(s):
        i = names.index(s)
        avg = stage_ms[i] / max(stage_n[i], 1) * 1e-3
        a = flops_per_launch[s] / avg / 1e12
        return {"achieved": round(a, 3), "frac": round(a / peak, 4), "avg_launch_ms": round(avg * 1e3, 4),
                "flops_per_launch": flops_per_launch[s]}

    per_kernel = {f"k_{s}": kfrac(s) for s in flops_per_launch}
    snap_ms = stage_ms[1:5].sum()
    snap_flops_total = (fl["ui"] + fl["yi"] + fl["deidrj"]) * stage_n[2]
    hpk, hsrc = hbm_peak()
    # integrator (k_open + k_close_open + k_close): algorithmic bytes per component and
    # substep: k_close_open reads grad, p_half, q, noise and writes p, p_half, q (56 B)
    integ_i = names.index("integrator")
    integ_bytes = 56.0 * slices * d * L * prof_steps
    integ_gbs = integ_bytes / max(stage_ms[integ_i] * 1e-3, 1e-30) / 1e9
    roof = {"bound": "fp64", "kernel": f"k_{dom}", "achieved": per_kernel[f"k_{dom}"]["achieved"],
            "peak": round(peak, 3), "unit": "TFLOP/s", "frac": per_kernel[f"k_{dom}"]["frac"],
            "peak_source": "measured DFMA (pl_fp64_peak) on this B200; FP64 absent from MEASURED_PEAKS.json",
            "traffic": ncu_traffic(f"k_{dom}"),
            "flops_per_launch": flops_per_launch[dom],
            "timing": f"separate profiled pass of {prof_steps} step(s), live CUDA events per stage "
                      f"({prof_ms_per_step:.2f} ms/step profiled vs {ms / args.steps:.2f} ms/step timed)",
            "kernels": per_kernel,
            "snap_all_kernels_tflops": round(snap_flops_total / (snap_ms * 1e-3) / 1e12, 3),
            "stage_share": {k_: round(v, 4) for k_, v in share.items()},
            "flop_model": {"per_pair_ui": fl["per_pair_ui"], "per_atom_yi": fl["per_atom_yi"],
                           "per_pair_deidrj": fl["per_pair_de"],
                           "pairs_per_eval": fl["pairs"], "atoms_per_eval": fl["atoms"]},
            "hbm": {"integrator": {"achieved_gbs": round(integ_gbs, 1), "frac": round(integ_gbs / hpk, 4),
                                   "bytes_per_component_substep": 56,
                                   "launches": int(stage_n[integ_i])},
                    "peak_gbs": hpk, "peak_source": hsrc}}

    # ---- e2e through the public API (host states in / out, noise generated in the call)
    states = [pl.PhaseState(q=inp["Q"][i], p=inp["P"][i]) for i in mine]
    pl.propagate_windows(states, pot, params, sched, seeds)  # warm
    barrier()
    t0 = time.perf_counter()
    e2e_steps = max(1, min(args.steps, 3))
    for _ in range(e2e_steps):
        outs = pl.propagate_windows(states, pot, params, sched, seeds)
    torch.cuda.synchronize()
    e2e_s = _max_over_ranks((time.perf_counter() - t0) / e2e_steps, dev, world)
    e2e = {"value": float(total_slices) * n * L / e2e_s, "unit": "atom-steps/s",
           "h2d_bytes_per_step": int(2 * slices * d * 8 + slices * 8),
           "d2h_bytes_per_step": int(2 * slices * d * 8 + slices * 4),
           "api": "paper_2212_10508_b200.propagate_windows(host PhaseStates, SNAP, ...) per rank"}
    del outs

    if rank == 0 and not args.no_hbm:
        roof["hbm"].update(hbm_kernels(hpk))

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(inp)
    parareal = None
    if not args.no_parareal:
        parareal = {"pr1": parareal_run("pr1", dev, world)}
        if args.config == "larger" and not args.no_larger_parareal:
            parareal["larger"] = parareal_run("larger", dev, world)

    if rank == 0:
        # per substep: neighbours (cell lists at >= 512 atoms and >= 3 cells per axis: count,
        # scan, fill, list; else one brute-force kernel; at >= 512 atoms also the skin check
        # and reference update), ui, yi (+ k_box_energy when the batch has fewer 32-atom
        # blocks than SMs; the unsplit Y kernel also writes Y^dagger, else k_snap_ytrans),
        # deidrj, gather, one integrator kernel; + the opening gradient and k_open
        cells = n >= 512 and min(inp["box"]) / (4.73 + 0.3) >= 3
        skin = n >= 512  # Verlet-skin check + reference update kernels (the builds are gated on the device)
        split = (slices * n + 31) // 32 < 148
        per_eval = (4 if cells else 1) + (2 if skin else 0) + 4 + (2 if split else 0)
        launches_per_step = (L + 1) * per_eval + (L + 1)
        line = {
            "metric": METRIC,
            "value": value, "unit": "atom-steps/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.config}: BCC W {inp['cells']}^3 + <111> SIA = {n} atoms, "
                                   f"{total_slices} slices x L={L} BBK substeps, SNAP twojmax=8 fp64, "
                                   f"T={T:g} K, gamma=1/ps, dt=1 fs",
                       "slices_total": total_slices, "slices_per_rank": slices, "atoms": n, "substeps": L,
                       "l2": "inputs larger than L2 (noise blocks "
                             f"{noise.numel() * 8 / 1e6:.0f} MB per rank)",
                       "parallelism": f"{args.scaling} scaling: slices sharded over {world} rank(s), "
                                      "NCCL all-gather of endpoints per step"},
            "clocks": clk, "e2e": e2e, "roofline": roof, "cpu_baseline": cpu,
            "gpu_launches": int(launches_per_step * args.steps),
            "blowups": blow,
            "parareal": parareal,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


# ---------------------------------------------------------------- HBM-bound kernels
def hbm_kernels(peak_gbs):
    """EAM force sweep (configs[1]: 4096 x 129 atoms, E + F + virial in one batch) and the
    persistent coarse sweep, against the measured HBM bandwidth."""
    import torch
    import paper_2212_10508_b200 as pl
    from paper_2212_10508_b200 import _lib, tungsten as W
    out = {}
    q0, box = W.bcc_sia(4)
    n = q0.shape[0] // 3
    B = 4096
    Q = torch.from_numpy(q0[None] + 0.1 * np.random.default_rng(2212).normal(size=(B, q0.shape[0]))).cuda()
    eam = W.make_eam(n, box)
    eam.evaluate(Q, True, True, True)
    lib, ctx = _lib.load(), _lib.context()
    torch.cuda.synchronize()
    _lib.check(lib.pl_prof_begin(ctx.handle))
    reps = 5
    for _ in range(reps):
        eam.evaluate(Q, True, True, True)
    torch.cuda.synchronize()
    ms = np.zeros(8)
    cnt = np.zeros(8, dtype=np.int64)
    _lib.check(lib.pl_prof_end(ctx.handle, 8, _lib.dptr(ms), cnt.ctypes.data_as(_lib.pi64)))
    # algorithmic bytes per atom-evaluation of the two EAM passes (neighbour build excluded,
    # it is the "neigh" stage): density pass x 24 + list 58 x 4 + F' write 8; force pass x 24
    # + list 232 + F'_i 8 + gradient 24 + energy 8 + virial 48
    nb = 58
    per_atom = 24 + 4 * nb + 8 + 24 + 4 * nb + 8 + 24 + 8 + 48
    eam_s = ms[5] * 1e-3 / reps
    gbs = per_atom * B * n / eam_s / 1e9
    out["eam"] = {"config": "configs[1] force sweep: 4096 x 129 atoms, E + F + virial",
                  "achieved_gbs": round(gbs, 1), "frac": round(gbs / peak_gbs, 4),
                  "bytes_per_atom_eval": per_atom, "ms_per_eval": round(eam_s * 1e3, 4),
                  "atom_evals_per_s": B * n / eam_s,
                  "neigh_ms_per_eval": round(ms[0] / reps, 4)}
    return out


# ---------------------------------------------------------------- CPU arms
def _cpu_pool(inp, threads):
    """One oracle window (reference BBK restatement + C SNAP) per host thread, opened."""
    from concurrent.futures import ThreadPoolExecutor
    from oracle import integrator as oint, native
    from paper_2212_10508_b200 import tungsten as W
    n, box, L = inp["n"], inp["box"], inp["L"]
    d = 3 * n
    mass = np.full(d, W.MASS_W)
    pot = W.make_snap(n, box)
    grad = native.snap_fn(pot)
    native.load()
    sched = oint.robust(L)
    S = inp["slices"]
    wins = [oint.WindowStepper(inp["Q"][i % S], inp["P"][i % S], grad, GAMMA, W.KB * inp["T"], DT, L, sched,
                               inp["seeds"][i % S], mass=mass) for i in range(threads)]
    ex = ThreadPoolExecutor(max_workers=threads)
    list(ex.map(lambda w: w.open(), wins))
    return wins, ex


def _cpu_step(wins, ex, substeps):
    t = time.perf_counter()
    list(ex.map(lambda w: w.advance(substeps), wins))
    return time.perf_counter() - t


def _cpu_sample_text(inp, threads, substeps, steps):
    return (f"{threads} slices (one per host thread) x {substeps} BBK substeps per step, {steps} step(s), of "
            f"the {inp['n']}-atom L={inp['L']} windows: reference BBK window restated in "
            "oracle/integrator.py (WindowStepper) + C SNAP oracle; the window-opening gradient "
            "(1 per L substeps) falls in the untimed warm-up")


def cpu_baseline(inp):
    threads = os.cpu_count() or 1
    wins, ex = _cpu_pool(inp, threads)
    _cpu_step(wins, ex, 1)   # warm
    steps = 3
    secs = sum(_cpu_step(wins, ex, CPU_SUBSTEPS) for _ in range(steps))
    ex.shutdown()
    atom_steps = float(threads) * inp["n"] * CPU_SUBSTEPS * steps
    return {"value": atom_steps / secs, "unit": "atom-steps/s", "cores": threads, "kind": "port",
            "sample": _cpu_sample_text(inp, threads, CPU_SUBSTEPS, steps) + f", {secs:.1f} s"}


def run_reference(args, rank, world):
    if rank != 0:
        return
    inp = build_inputs(args.config)
    threads = os.cpu_count() or 1
    L = inp["L"]
    wins, ex = _cpu_pool(inp, threads)
    if (args.warmup + args.steps) * CPU_SUBSTEPS > L:
        print(json.dumps({"impl": "reference", "error": "steps x substeps exceed one window"}))
        return
    for _ in range(args.warmup):
        _cpu_step(wins, ex, CPU_SUBSTEPS)
    per = [_cpu_step(wins, ex, CPU_SUBSTEPS) for _ in range(args.steps)]
    ex.shutdown()
    secs = sum(per)
    v = float(threads) * inp["n"] * CPU_SUBSTEPS * args.steps / secs
    sample = _cpu_sample_text(inp, threads, CPU_SUBSTEPS, args.steps)
    line = {"impl": "reference", "metric": METRIC,
            "value": v, "unit": "atom-steps/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": secs / max(len(per), 1) * 1e3,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": f"{args.config}: BCC W {inp['cells']}^3 + <111> SIA = {inp['n']} atoms, "
                                   f"{inp['slices']} slices x L={L} BBK substeps, SNAP twojmax=8 fp64, "
                                   f"T={inp['T']:g} K, gamma=1/ps, dt=1 fs", "sample": sample},
            "cpu_baseline": {"value": v, "unit": "atom-steps/s", "cores": threads, "kind": "port",
                             "sample": sample},
            "e2e": {"value": v, "unit": "atom-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def ncu_traffic(kernel):
    """DRAM bytes (read + write) per launch of the dominant kernel from the committed
    ncu --set full capture of this config (profiles/traffic.json), else None."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            t = json.load(f)
        return t["kernels"].get(kernel)
    except (OSError, ValueError, KeyError):
        return None


# ---------------------------------------------------------------- parareal wall-clock
def parareal_run(cfg_name, dev, world):
    """Adaptive parareal of configs[0] (pr1) or configs[2] (larger) with SNAP fine /
    EAM coarse, delta from configs/adaptive.json; fine stage sharded over the ranks.
    Also the sequential fine chain of the same N windows on the same GPU(s)."""
    import torch
    import paper_2212_10508_b200 as pl
    from paper_2212_10508_b200 import accounting, tungsten as W
    from paper_2212_10508_b200.integrator import WindowKernel
    cells, N, L, T = CONFIGS[cfg_name]
    q0, box = W.bcc_sia(cells)
    n = q0.shape[0] // 3
    mass = np.full(3 * n, W.MASS_W)
    params = pl.LangevinParams(GAMMA, W.KB * T, DT, L, mass=mass)
    sched = pl.TemperatureSchedule.robust(L)
    plan = pl.NoisePlan.for_windows(11, N)
    init = pl.PhaseState(q=q0, p=W.maxwell_boltzmann(n, T, 11))
    eam = W.make_eam(n, box)
    snap = W.make_snap(n, box)
    pair = pl.PropagatorPair(snap, eam, 100.0, 1.0)
    cfg = pl.PararealConfig(N, 1e-10, 0.35)   # delta_conv / delta_expl of configs/adaptive.json
    runs = 2 if cfg_name == "pr1" else 1
    walls = []
    for _ in range(runs):
        torch.cuda.synchronize()
        t = time.perf_counter()
        try:
            res = pl.parareal_adaptive(init, pair, params, sched, plan, cfg)
        except Exception as exc:  # report, do not fail the bench
            return {"error": f"{type(exc).__name__}: {exc}"}
        torch.cuda.synchronize()
        walls.append(_max_over_ranks(time.perf_counter() - t, dev, world))

    def window_ms(pot, reps=3):
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
    wall = walls[-1]
    out = {"config": f"{cfg_name}: {n} atoms, {N} slices x {L}, SNAP fine / EAM coarse, delta_conv 1e-10, "
                     "delta_expl 0.35", "wall_s": wall, "n_slab": res.n_slab,
           "sum_k": res.total_iterations, "converged": res.converged, "ranks": world,
           "cf_ms": cf, "cc_ms": cc, "gain_model": g.gain, "gain_ideal": g.ideal_gain,
           "sequential_fine_s": N * cf / 1e3, "speedup_vs_sequential_fine": (N * cf / 1e3) / wall}
    if runs > 1:
        out["wall_s_cold"] = walls[0]
    return out


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="larger", choices=sorted(CONFIGS))
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"])
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-parareal", action="store_true")
    ap.add_argument("--no-larger-parareal", action="store_true")
    ap.add_argument("--no-hbm", action="store_true")
    args = ap.parse_args()
    rank = _env_int("RANK", 0)
    world = _env_int("WORLD_SIZE", 1)
    local_rank = _env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # one process per GPU: re-launch under torchrun (rank 0 prints the line)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
               os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    if world != args.gpus:
        print(json.dumps({"error": f"--gpus {args.gpus} but WORLD_SIZE={world}"}), flush=True)
        sys.exit(2)
    run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
