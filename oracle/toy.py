"""Oracle restatement of the reference's analytic potentials (TEST INFRASTRUCTURE).

Follows /root/reference/pkg/src/paralangevin/potentials.py:
  * Harmonic   grad = k*q ........................... potentials.py:93-95
  * DoubleWell grad = 4*a*q*(q*q-b) ................. potentials.py:126-128
  * LennardJonesCluster all-pairs, atom-major ....... potentials.py:156-180
  * Perturbed  base + lam*delta, lam == 0 -> base ... potentials.py:206-214
Each returns ``grad_fn(q)`` closures (and energies) evaluated with numpy in
the reference's own operation order.
"""

from __future__ import annotations

import numpy as np


def harmonic(k):
    return lambda q: k * q


def harmonic_energy(k):
    return lambda q: float(0.5 * np.sum(k * q * q))


def double_well(a, b):
    return lambda q: 4.0 * a * q * (q * q - b)


def double_well_energy(a, b):
    def e(q):
        w = q * q - b
        return float(np.sum(a * w * w))
    return e


def lj(epsilon, sigma, n_atoms, space_dim):
    def grad(q):
        x = q.reshape(n_atoms, space_dim)
        diff = x[:, None, :] - x[None, :, :]
        r2 = np.sum(diff * diff, axis=-1)
        np.fill_diagonal(r2, 1.0)
        u3 = (sigma * sigma / r2) ** 3
        coeff = (24.0 * epsilon * u3 - 48.0 * epsilon * u3 * u3) / r2
        np.fill_diagonal(coeff, 0.0)
        return np.sum(coeff[:, :, None] * diff, axis=1).reshape(-1)
    return grad


def lj_energy(epsilon, sigma, n_atoms, space_dim):
    def e(q):
        x = q.reshape(n_atoms, space_dim)
        diff = x[:, None, :] - x[None, :, :]
        r2 = np.sum(diff * diff, axis=-1)
        iu = np.triu_indices(n_atoms, k=1)
        u3 = (sigma * sigma / r2[iu]) ** 3
        return float(np.sum(4.0 * epsilon * (u3 * u3 - u3)))
    return e


def perturbed(base, delta, lam):
    if lam == 0.0:
        return base
    return lambda q: base(q) + lam * delta(q)
