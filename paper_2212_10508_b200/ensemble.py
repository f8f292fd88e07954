"""Residence-time ensemble on the device (BASELINE configs[3]).

The reference's ensemble protocol (cli.py:986-1050) with the W + SIA system:

1. minimise the initial configuration on the FINE surface (``local_minima``,
   one batched ``pl_minimize``), zero momenta;
2. per member i (seed ``derive_seed(master, 10**9 + i)``): thermalise with a
   sequential fine chain (plan ``derive_seed(member_seed, 1)``);
3. from the thermalised state, run the sequential FINE reference chain and
   adaptive parareal over the SAME segment plans (segment s uses
   ``derive_seed(member_seed, 2 + s)``; s = 0 is the reference's single
   segment), each chain continuing from its own end state;
4. label every node by the SIA's Wigner-Seitz site (``pl_sia_sites``),
   optionally after quenching the node (steepest descent on the fine surface,
   so thermal flicker of the dumbbell does not count as a hop), encode
   residence times with the hysteresis ``min_run`` (analysis.py:114-156),
   pool over members and compare the two 95 % intervals
   (``compare_ensembles``, analysis.py:232-238).

All members run together: the sequential chains are batched over members
(one launch per window for all members), the parareal runs are one
``parareal_adaptive_batch`` per segment.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import accounting, sia
from .distributed import sharded_fine, world
from .integrator import TemperatureSchedule, WindowKernel, _raise_first_blowup
from .model import LangevinParams, PhaseState
from .parareal import PararealConfig, parareal_adaptive_batch
from .potentials import PropagatorPair, local_minima, minimize_batch
from .rng import NoisePlan, derive_seed

MEMBER_SEED_OFFSET = 10 ** 9  # cli.py:88


def sequential_propagate_batch(initials, n_windows: int, pot, params: LangevinParams,
                               schedule: TemperatureSchedule, plans):
    """Sequential fine chains of R members at once: (Q, P) of shape (R, n_windows + 1, d).

    Member r's window m uses ``plans[r].seed_for(m + 1)`` exactly like
    ``sequential_propagate``; every window step is one batched launch over
    the members (independent chains), so each chain equals its single run.
    Under torch.distributed the members of each step are sharded over the
    ranks and all-gathered.
    """
    import torch
    R, d = len(initials), initials[0].dim
    k = WindowKernel(pot, params, schedule, d)
    seeds = np.array([[p.window_seeds[m] for p in plans] for m in range(n_windows)], dtype=np.uint64)
    noise = k.noise(seeds.reshape(-1)).reshape(n_windows, R, -1)
    Q = torch.empty((n_windows + 1, R, d), dtype=torch.float64, device=k.device)
    P = torch.empty_like(Q)
    Q[0] = torch.from_numpy(np.stack([s.q for s in initials]))
    P[0] = torch.from_numpy(np.stack([s.p for s in initials]))
    blow = torch.zeros((n_windows, R), dtype=torch.int32, device=k.device)
    for m in range(n_windows):
        if world()[1] == 1:
            k.run(Q[m], P[m], noise[m], Q[m + 1], P[m + 1], blow[m])
            continue

        def run_block(lo, hi, m=m):  # members sharded over the ranks, gathered
            return k.run(Q[m][lo:hi].contiguous(), P[m][lo:hi].contiguous(), noise[m][lo:hi].contiguous())
        FQ, FP, b = sharded_fine(run_block, 0, R)
        Q[m + 1].copy_(FQ)
        P[m + 1].copy_(FP)
        blow[m].copy_(b)
    b = blow.cpu().numpy()
    if b.any():
        m = int(np.nonzero(b.any(axis=1))[0][0])
        _raise_first_blowup(blow[m], windows=[m + 1] * R)
    return Q.permute(1, 0, 2).cpu().numpy(), P.permute(1, 0, 2).cpu().numpy()


@dataclass
class EnsembleResult:
    fine: sia.ResidenceStats
    adaptive: sia.ResidenceStats
    comparison: sia.EnsembleComparison
    mean_gain: float
    converged: int
    runs: int
    sum_k: list = field(default_factory=list)
    fine_labels: np.ndarray | None = None
    adaptive_labels: np.ndarray | None = None

    def as_dict(self) -> dict:
        return {"fine": self.fine.as_dict(), "adaptive": self.adaptive.as_dict(),
                "comparison": {"overlap": self.comparison.overlap, "intervals": self.comparison.intervals},
                "mean_gain": self.mean_gain, "converged": self.converged, "runs": self.runs,
                "mean_sum_k": float(np.mean(self.sum_k)) if self.sum_k else None}


def _labels(Qnodes, n_cells, a, quench_pot, quench_tol, quench_iters):
    """(R, T) SIA site labels of node positions (R, T, d), optionally quenched first
    (a bounded steepest descent: it only has to remove the thermal vibration)."""
    R, T, d = Qnodes.shape
    X = Qnodes.reshape(R * T, d)
    if quench_pot is not None:
        X = minimize_batch(quench_pot, X, tol=quench_tol, max_iter=quench_iters)[0]
    return sia.sia_site_labels(X, n_cells, a).reshape(R, T)


def run_ensemble(pair: PropagatorPair, params: LangevinParams, schedule: TemperatureSchedule,
                 initial: PhaseState, config: PararealConfig, *, size: int, master_seed: int,
                 n_cells: int, a: float, segments: int = 1, thermalization_windows: int = 0,
                 min_run: int = 1, quench: bool = False, quench_tol: float = 1e-3, quench_iters: int = 300,
                 minimize_start: bool = True, minimize_tol: float = 1e-4,
                 keep_labels: bool = False) -> EnsembleResult:
    """The ensemble protocol above; returns pooled fine / adaptive residence statistics.

    ``minimize_tol`` (eV/A, |grad| of the start): the reference minimises with
    its default 1e-8 (cli.py:991), which steepest descent on the synthetic
    random-beta SNAP surface does not reach (|grad| 1e-4 after 5 iterations,
    then ~2e-6 after 20,000: scripts/probe_minimize.py); the start only has to
    be a relaxed lattice, so 1e-4 is the default here.
    """
    n = config.n_windows
    q0 = np.asarray(initial.q, dtype=float)
    if minimize_start:
        q0 = local_minima(pair.fine, [q0], tol=minimize_tol)[0]
    start = PhaseState(q=q0, p=np.zeros_like(q0))
    member_seeds = [derive_seed(master_seed, MEMBER_SEED_OFFSET + i) for i in range(size)]
    states = [start] * size
    if thermalization_windows:
        plans = [NoisePlan.for_windows(derive_seed(s, 1), thermalization_windows) for s in member_seeds]
        Q, P = sequential_propagate_batch(states, thermalization_windows, pair.fine, params, schedule, plans)
        states = [PhaseState(q=Q[r, -1], p=P[r, -1]) for r in range(size)]
    fine_states, par_states = list(states), list(states)
    fine_nodes, par_nodes = [], []
    gains, sum_k, conv, runs = [], [], 0, 0
    for s in range(segments):
        plans = [NoisePlan.for_windows(derive_seed(ms, 2 + s), n) for ms in member_seeds]
        Q, P = sequential_propagate_batch(fine_states, n, pair.fine, params, schedule, plans)
        fine_nodes.append(Q if s == 0 else Q[:, 1:])
        fine_states = [PhaseState(q=Q[r, -1], p=P[r, -1]) for r in range(size)]
        res = parareal_adaptive_batch(par_states, pair, params, schedule, plans, config)
        par_nodes.append(np.stack([r.trajectory.positions() if s == 0 else r.trajectory.positions()[1:]
                                   for r in res]))
        par_states = [r.trajectory[r.trajectory.n_windows] for r in res]
        for r in res:
            runs += 1
            conv += int(r.converged)
            sum_k.append(r.total_iterations)
            gains.append(accounting.adaptive_gain(r.slabs, n, pair.cost_fine, pair.cost_coarse).gain)
    qp = pair.fine if quench else None
    lf = _labels(np.concatenate(fine_nodes, axis=1), n_cells, a, qp, quench_tol, quench_iters)
    la = _labels(np.concatenate(par_nodes, axis=1), n_cells, a, qp, quench_tol, quench_iters)
    ev_f = [e for lab in lf for e in sia.residence_times(lab, min_run=min_run)]
    ev_a = [e for lab in la for e in sia.residence_times(lab, min_run=min_run)]
    fs, as_ = sia.residence_stats(ev_f), sia.residence_stats(ev_a)
    return EnsembleResult(fs, as_, sia.compare_ensembles(fs, as_), float(np.mean(gains)), conv, runs, sum_k,
                          lf if keep_labels else None, la if keep_labels else None)
