"""Modified-BBK Langevin windows on the GPU, API-compatible with the reference.

Mirrors /root/reference/pkg/src/paralangevin/integrator.py:
  TemperatureSchedule / solve_schedule    integrator.py:95-153
  _amplitude                              integrator.py:156-160
  BlowUpError                             integrator.py:50-57
  propagate_window                        integrator.py:292-308
``propagate_windows`` is the batched form the engines use: W windows in one
``pl_propagate_windows`` call, states and noise resident in HBM.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from .model import LangevinParams, PhaseState
from .potentials import Potential, PotentialError
from .rng import device_streams

BLOWUP_LIMIT = 1e12


class BlowUpError(RuntimeError):
    """A propagated state left the trusted numerical range."""

    def __init__(self, message: str, substep=None, window=None, iteration=None):
        super().__init__(message)
        self.substep = substep
        self.window = window
        self.iteration = iteration


class InfeasibleScheduleError(ValueError):
    def __init__(self, message: str, index: int):
        super().__init__(message)
        self.index = index


@dataclass(frozen=True)
class TemperatureSchedule:
    """Fluctuation weights C_0..C_L, one per Gaussian block of a window."""

    coefficients: tuple

    def __post_init__(self) -> None:
        coeffs = tuple(float(c) for c in self.coefficients)
        if len(coeffs) < 2:
            raise ValueError("a schedule needs at least C_0 and C_1 (substeps >= 1)")
        for i, c in enumerate(coeffs):
            if not (np.isfinite(c) and c > 0.0):
                raise ValueError(f"schedule weight C_{i} must be positive, got {c}")
        object.__setattr__(self, "coefficients", coeffs)

    @property
    def substeps(self) -> int:
        return len(self.coefficients) - 1

    @classmethod
    def identity(cls, substeps: int) -> "TemperatureSchedule":
        return cls(coefficients=(1.0,) * (substeps + 1))

    @classmethod
    def robust(cls, substeps: int) -> "TemperatureSchedule":
        return solve_schedule(substeps, 3.0)

    @classmethod
    def flat_pair(cls) -> "TemperatureSchedule":
        return solve_schedule(1, 2.0)


def solve_schedule(substeps: int, c0: float) -> TemperatureSchedule:
    """C_1 = 4 - C_0, C_l = 4 - 3 C_{l-1}; every weight must stay positive."""
    if substeps < 1:
        raise ValueError(f"substeps must be >= 1, got {substeps}")
    if not (np.isfinite(c0) and c0 > 0.0):
        raise InfeasibleScheduleError(f"schedule infeasible: C_0 = {c0} is not positive", index=0)
    coeffs = [float(c0), 4.0 - float(c0)]
    for l in range(2, substeps + 1):
        coeffs.append(4.0 - 3.0 * coeffs[l - 1])
    for i, c in enumerate(coeffs):
        if not c > 0.0:
            raise InfeasibleScheduleError(
                f"schedule infeasible for C_0 = {c0}: C_{i} = {c} is not positive", index=i)
    return TemperatureSchedule(coefficients=tuple(coeffs))


def amplitude(params: LangevinParams, c: float) -> float:
    if not c > 0.0:
        raise ValueError(f"schedule weight must be positive, got {c}")
    return 0.5 * math.sqrt(2.0 * params.gamma * c * params.inv_beta * params.dt)


class WindowKernel:
    """Frozen per-(potential, params, schedule) launch arguments of pl_propagate_windows."""

    def __init__(self, pot: Potential, params: LangevinParams, schedule: TemperatureSchedule, d: int):
        if not isinstance(pot, Potential):
            raise TypeError("propagation needs a device Potential from paper_2212_10508_b200")
        if schedule.substeps != params.substeps:
            raise ValueError(
                f"schedule has {schedule.substeps} substeps, params have {params.substeps}")
        import torch
        self.pot, self.params, self.schedule, self.d = pot, params, schedule, d
        self.L = params.substeps
        amp = np.array([amplitude(params, c) for c in schedule.coefficients], dtype=float)
        # pinned host copy: the library uploads it with cudaMemcpyAsync, which from
        # pageable memory may synchronise with the stream (speculative launches
        # on a second stream must not block the host)
        try:
            self._amp_pinned = torch.from_numpy(amp).pin_memory()
            self.amp = self._amp_pinned.numpy()
        except RuntimeError:  # no CUDA: plain host memory (the library refuses to run anyway)
            self.amp = amp
        self.dt = float(params.dt)
        self.h = 0.5 * params.dt                      # `0.5 * dt * grad` (integrator.py:174)
        self.hg = 0.5 * params.dt * params.gamma      # `0.5 * dt * gamma * p`
        ctx = _lib.context()
        self.device = torch.device("cuda", ctx.device)
        self.mass = None
        if params.mass is not None:
            m = params.mass_vector(d)
            self.mass = torch.from_numpy(np.array(m, dtype=float)).to(self.device)

    def noise(self, seeds):
        """(W, (L+1)*d) device noise blocks for the given window seeds."""
        return device_streams(seeds, (self.L + 1) * self.d)

    def run(self, Q0, P0, noise, Q1=None, P1=None, blow=None, moments=None):
        """Propagate W windows: Q0/P0 (W, d) device tensors; returns (Q1, P1, blowup).

        ``moments=(S1, S2)`` ((W, L, d) device tensors) also accumulates the
        full-step momentum moments (pl_propagate_windows_moments).
        """
        import torch
        W = Q0.shape[0]
        Q1 = torch.empty_like(Q0) if Q1 is None else Q1
        P1 = torch.empty_like(P0) if P1 is None else P1
        if blow is None:
            blow = torch.zeros(W, dtype=torch.int32, device=Q0.device)
        ctx = _lib.context()
        lib = _lib.load()
        args = (ctx.handle, self.pot.handle(ctx), W, self.d, self.L, _lib.ptr(Q0), _lib.ptr(P0),
                _lib.ptr(noise), _lib.dptr(self.amp), _lib.ptr(self.mass), self.dt, self.h, self.hg,
                _lib.ptr(Q1), _lib.ptr(P1), _lib.ptr(blow))
        try:
            if moments is None:
                _lib.check(lib.pl_propagate_windows(*args))
            else:
                _lib.check(lib.pl_propagate_windows_moments(*args, _lib.ptr(moments[0]), _lib.ptr(moments[1])))
        except _lib.CallError as err:
            if err.code in (_lib.PL_EARG, _lib.PL_EPOT):
                raise PotentialError(err.message) from None
            raise
        return Q1, P1, blow


def _raise_first_blowup(blow, windows=None):
    b = blow.cpu().numpy()
    bad = np.nonzero(b)[0]
    if bad.size:
        i = int(bad[0])
        raise BlowUpError(
            f"state left the trusted range (|component| > {BLOWUP_LIMIT:g} or non-finite) "
            f"at substep {int(b[i])}", substep=int(b[i]),
            window=None if windows is None else windows[i])


def propagate_windows(states, pot: Potential, params: LangevinParams,
                      schedule: TemperatureSchedule, seeds, noise=None):
    """Batched ``propagate_window`` over W independent windows (one device call).

    ``states`` is a list of PhaseState; ``seeds`` one window seed each;
    ``noise`` optionally injects the (W, (L+1)*d) Gaussian blocks.
    """
    import torch
    d = states[0].dim
    k = WindowKernel(pot, params, schedule, d)
    Q0 = torch.from_numpy(np.stack([s.q for s in states])).to(k.device)
    P0 = torch.from_numpy(np.stack([s.p for s in states])).to(k.device)
    if noise is None:
        noise = k.noise(seeds)
    else:
        noise = torch.as_tensor(np.asarray(noise, dtype=float)).reshape(len(states), -1).to(k.device)
    Q1, P1, blow = k.run(Q0, P0, noise.contiguous())
    _raise_first_blowup(blow)
    Q1, P1 = Q1.cpu().numpy(), P1.cpu().numpy()
    return [PhaseState(q=Q1[i], p=P1[i]) for i in range(len(states))]


def propagate_window(state: PhaseState, pot: Potential, params: LangevinParams,
                     schedule: TemperatureSchedule, seed: int) -> PhaseState:
    """Advance one window of ``params.substeps`` steps (integrator.py:292-308)."""
    return propagate_windows([state], pot, params, schedule, [seed])[0]


# ---------------------------------------------------------------- kinetic temperature
ALL_SUBSTEPS = "all_substeps"
WINDOW_ENDS = "window_ends"


def predicted_kinetic_temperature(substeps: int, inv_beta: float) -> float:
    """Leading-order stationary kinetic temperature (integrator.py:316-320)."""
    if substeps < 1:
        raise ValueError(f"substeps must be >= 1, got {substeps}")
    return inv_beta * (1.0 - 1.0 / (2.0 * substeps))


@dataclass(frozen=True)
class TemperatureReport:
    """Outcome of a kinetic-temperature measurement (integrator.py:337-346)."""

    k_eq_empirical: float
    k_eq_predicted: float
    per_substep_variance: tuple
    n_windows: int
    n_burn_in: int
    sampling: str


def _variance(s1, s2, count, mass) -> float:
    # mass-weighted, component-averaged variance from running moments (integrator.py:349-353)
    mean = s1 / count
    var = s2 / count - mean * mean
    return float(np.mean(var / mass))


def measure_kinetic_temperature_batch(pot: Potential, params: LangevinParams, schedule: TemperatureSchedule,
                                      n_windows: int, master_seeds, sampling: str = ALL_SUBSTEPS,
                                      burn_in: float = 0.1, initial: PhaseState | None = None) -> list:
    """``measure_kinetic_temperature`` for R independent chains in one device pass.

    Chain r starts cold (q = p = 0, or ``initial`` -- an extension for lattice
    systems, where q = 0 stacks every atom on one site) and runs ``n_windows`` windows, window n
    with seed ``derive_seeds(master_seeds[r], n_windows)[n]``; each window is
    one ``pl_propagate_windows_moments`` launch over all R chains, the moments
    of windows n >= n_burn accumulate on the device (integrator.py:355-365,
    430-482).  Returns one TemperatureReport per chain.
    """
    import torch
    from .rng import derive_seeds
    if sampling not in (ALL_SUBSTEPS, WINDOW_ENDS):
        raise ValueError(f"unknown sampling mode: {sampling!r}")
    if not 0.0 <= burn_in < 1.0:
        raise ValueError(f"burn_in must lie in [0, 1), got {burn_in}")
    if n_windows < 1:
        raise ValueError("n_windows must be >= 1")
    n_burn = int(round(burn_in * n_windows))
    if n_burn >= n_windows:
        n_burn = n_windows - 1
    d = params.mass.shape[0] if params.mass is not None else 1
    mass = params.mass_vector(d)
    seeds = np.stack([np.asarray(derive_seeds(int(m), n_windows), dtype=np.uint64) for m in master_seeds])
    R, L = seeds.shape[0], params.substeps
    k = WindowKernel(pot, params, schedule, d)
    Q = [torch.zeros((R, d), dtype=torch.float64, device=k.device) for _ in range(2)]
    P = [torch.zeros((R, d), dtype=torch.float64, device=k.device) for _ in range(2)]
    if initial is not None:
        if initial.dim != d:
            raise ValueError(f"initial state has dimension {initial.dim}, expected {d}")
        Q[0].copy_(torch.from_numpy(np.array(initial.q, dtype=float))[None].expand(R, d))
        P[0].copy_(torch.from_numpy(np.array(initial.p, dtype=float))[None].expand(R, d))
    S1 = torch.zeros((R, L, d), dtype=torch.float64, device=k.device)
    S2 = torch.zeros_like(S1)
    blows = torch.zeros((n_windows, R), dtype=torch.int32, device=k.device)
    for n in range(n_windows):
        a, b = n % 2, (n + 1) % 2
        noise = k.noise([int(x) for x in seeds[:, n]])
        k.run(Q[a], P[a], noise, Q[b], P[b], blows[n], moments=(S1, S2) if n >= n_burn else None)
    bl = blows.cpu().numpy()
    if bl.any():
        n, r = (int(v[0]) for v in np.nonzero(bl))
        raise BlowUpError(f"chain {r} left the trusted range at substep {int(bl[n, r])}",
                          substep=int(bl[n, r]), window=n)
    s1, s2 = S1.cpu().numpy(), S2.cpu().numpy()
    count = n_windows - n_burn
    k_pred = predicted_kinetic_temperature(L, params.inv_beta)
    out = []
    for r in range(R):
        per = tuple(_variance(s1[r, l], s2[r, l], count, mass) for l in range(L))
        k_emp = (_variance(s1[r].sum(axis=0), s2[r].sum(axis=0), count * L, mass)
                 if sampling == ALL_SUBSTEPS else per[-1])
        out.append(TemperatureReport(k_emp, k_pred, per, n_windows, n_burn, sampling))
    return out


def measure_kinetic_temperature(pot: Potential, params: LangevinParams, schedule: TemperatureSchedule,
                                n_windows: int, master_seed: int, sampling: str = ALL_SUBSTEPS,
                                burn_in: float = 0.1) -> TemperatureReport:
    """Chain windows from a cold start and report the stationary temperature (integrator.py:430-482)."""
    return measure_kinetic_temperature_batch(pot, params, schedule, n_windows, [master_seed], sampling,
                                             burn_in)[0]
