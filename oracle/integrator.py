"""Oracle restatement of the modified-BBK window propagator (TEST INFRASTRUCTURE).

Follows /root/reference/pkg/src/paralangevin/integrator.py:
  * amplitude 0.5*sqrt(2*gamma*c*inv_beta*dt) ...... integrator.py:156-160
  * blow-up check |x| <= 1e12 on (q, p) per substep .. integrator.py:163-170
  * first substep (friction on p) ................... integrator.py:173-178
  * later substeps (friction on p_half_prev) ........ integrator.py:181-186
  * window: L+1 noise blocks, block l closes substep l and reopens l+1
    ................................................. integrator.py:259-289
  * schedules  robust C0=3, C_l = 4-3C_{l-1} ......... integrator.py:114-153
numpy evaluates each expression left to right with one rounding per
operation and no FMA; this restatement keeps exactly that order so it is
bitwise equal to the reference (pinned by tests/golden/window_golden.npz).
"""

from __future__ import annotations

import math

import numpy as np

from . import rng

BLOWUP_LIMIT = 1e12


class OracleBlowUp(RuntimeError):
    def __init__(self, substep):
        super().__init__(f"blow-up at substep {substep}")
        self.substep = substep


def amplitude(gamma, inv_beta, dt, c):
    return 0.5 * math.sqrt(2.0 * gamma * c * inv_beta * dt)


def solve_schedule(substeps, c0):
    coeffs = [float(c0), 4.0 - float(c0)]
    for l in range(2, substeps + 1):
        coeffs.append(4.0 - 3.0 * coeffs[l - 1])
    return tuple(coeffs)


def robust(substeps):
    return solve_schedule(substeps, 3.0)


def identity(substeps):
    return (1.0,) * (substeps + 1)


def _bounded(q, p):
    return bool((np.abs(q) <= BLOWUP_LIMIT).all() and (np.abs(p) <= BLOWUP_LIMIT).all())


class WindowStepper:
    """One window advanced in chunks of substeps (the bench's bounded CPU samples).

    Exactly the arithmetic of ``propagate_window`` (integrator.py:259-289):
    ``open()`` evaluates grad(q0); ``advance(k)`` runs the next k substeps.
    propagate_window below is open() + advance(L), so the goldens pin both.
    """

    def __init__(self, q, p, grad_fn, gamma, inv_beta, dt, substeps, schedule, seed,
                 mass=None, noise=None):
        self.q = np.asarray(q, dtype=float)
        self.p = np.asarray(p, dtype=float)
        d = self.q.shape[0]
        self.mass = np.ones(d) if mass is None else np.asarray(mass, dtype=float)
        sqrt_m = np.sqrt(self.mass)
        self.amps = [amplitude(gamma, inv_beta, dt, c) * sqrt_m for c in schedule]
        if noise is None:
            noise = rng.gaussian_stream(seed, (substeps + 1) * d)
        self.g = np.asarray(noise, dtype=float).reshape(substeps + 1, d)
        self.grad_fn, self.gamma, self.dt, self.L = grad_fn, gamma, dt, substeps
        self.l = 0
        self.grad = None
        self.p_ref = self.p

    def open(self):
        self.grad = self.grad_fn(self.q)

    def advance(self, k):
        q, p, grad, p_ref = self.q, self.p, self.grad, self.p_ref
        dt, gamma, mass, amps, g = self.dt, self.gamma, self.mass, self.amps, self.g
        for l in range(self.l, min(self.L, self.l + k)):
            p_half = p - 0.5 * dt * grad - 0.5 * dt * gamma * p_ref + amps[l] * g[l]
            q = q + dt * (p_half / mass)
            grad = self.grad_fn(q)
            p = p_half - 0.5 * dt * grad - 0.5 * dt * gamma * p_half + amps[l + 1] * g[l + 1]
            if not _bounded(q, p):
                raise OracleBlowUp(l + 1)
            p_ref = p_half
            self.l = l + 1
        self.q, self.p, self.grad, self.p_ref = q, p, grad, p_ref
        return self.l == self.L


def propagate_window(q, p, grad_fn, gamma, inv_beta, dt, substeps, schedule, seed,
                     mass=None, noise=None):
    """One window; returns (q, p).  ``noise`` ((L+1)*d) may be injected."""
    w = WindowStepper(q, p, grad_fn, gamma, inv_beta, dt, substeps, schedule, seed, mass=mass, noise=noise)
    w.open()
    w.advance(substeps)
    return w.q, w.p
