"""Synthetic W + SIA systems of the BASELINE configs (inputs, not the hot path).

* BCC tungsten, a = 3.1652 A, n^3 cubic cells (2 n^3 sites) plus one
  self-interstitial as a <111> dumbbell (one site replaced by two atoms
  displaced +-DUMBBELL/2 along [111]); periodic orthorhombic box n*a.
* Units: eV, Angstrom, ps.  Mass of W = 183.84 amu = 0.0190537 eV ps^2 / A^2
  (SURVEY.md 8d); k_B = 8.617333262e-5 eV/K.
* Coarse potential: Finnis-Sinclair W (Phil. Mag. A 50, 45 (1984)
  parameters): rho(r) = (r - d)^2 for r < d, phi(r) = (r - c)^2 (c0 + c1 r +
  c2 r^2) for r < c, F(rho) = -A sqrt(rho); tabulated as cubic-Hermite pieces
  on 5000-point grids over [0, 5.5 A] (BASELINE config, cutoff 5.5 A).  It
  reproduces E_coh = 8.90 eV, B = 310 GPa, C' = 159 GPa, C44 = 161 GPa at
  a = 3.1652 A.  (A Morse pair term fitted to the same targets gives C' < 0,
  i.e. an unstable bcc lattice, so the FS polynomial pair term is used.)
* Fine potential: SNAP, twojmax = 8 (55 bispectrum components + constant),
  rcut = 4.73 A, rfac0 = 0.99363, rmin0 = 0, cosine switch, wself = 1,
  beta_k = 0.05 * N(0,1) from ``gaussian`` stream derive_seed(seed, 1).
"""

from __future__ import annotations

import math

import numpy as np

A0 = 3.1652
AMU = 1.0364269e-4           # eV ps^2 / A^2 per amu
MASS_W = 183.84 * AMU
KB = 8.617333262e-5          # eV / K
DUMBBELL = 2.20              # A, <111> dumbbell separation

# Finnis-Sinclair W
FS_D, FS_A, FS_C = 4.400224, 1.896373, 3.25
FS_C0, FS_C1, FS_C2 = 47.1346499, -33.7665655, 6.2541999
EAM_RCUT = 5.5
EAM_KNOTS = 5000
RHO_MAX = 100.0

SNAP_TWOJMAX = 8
SNAP_RCUT = 4.73
SNAP_RFAC0 = 0.99363


def bcc_sia(n: int, a: float = A0, sia: bool = True):
    """Positions (flat atom-major, 3N) and box of n^3 BCC cells (+ <111> dumbbell)."""
    g = np.arange(n, dtype=float)
    I, J, K = np.meshgrid(g, g, g, indexing="ij")
    corner = np.stack([I.ravel(), J.ravel(), K.ravel()], axis=1)
    sites = np.concatenate([corner, corner + 0.5]) * a
    if sia:
        c = n // 2
        host = int(np.argmin(np.linalg.norm(sites - np.array([c, c, c]) * a, axis=1)))
        centre = sites[host].copy()
        u = np.ones(3) / math.sqrt(3.0)
        sites = np.delete(sites, host, axis=0)
        sites = np.concatenate([sites, [centre - 0.5 * DUMBBELL * u, centre + 0.5 * DUMBBELL * u]])
    box = (n * a, n * a, n * a)
    return sites.reshape(-1).copy(), box


def hermite_table(f, df, x_max: float, knots: int):
    """Cubic Hermite pieces on [0, x_max]: (n_pieces x 4) coefficients and spacing."""
    n = knots - 1
    h = x_max / n
    x = np.arange(knots) * h
    y = f(x)
    dy = df(x)
    y0, y1 = y[:-1], y[1:]
    d0, d1 = dy[:-1] * h, dy[1:] * h
    c = np.empty((n, 4))
    c[:, 0] = y0
    c[:, 1] = d0
    c[:, 2] = 3.0 * (y1 - y0) - 2.0 * d0 - d1
    c[:, 3] = 2.0 * (y0 - y1) + d0 + d1
    return c, h


def _fs_rho(r):
    return np.where(r < FS_D, (r - FS_D) ** 2, 0.0)


def _fs_drho(r):
    return np.where(r < FS_D, 2.0 * (r - FS_D), 0.0)


def _fs_phi(r):
    return np.where(r < FS_C, (r - FS_C) ** 2 * (FS_C0 + FS_C1 * r + FS_C2 * r * r), 0.0)


def _fs_dphi(r):
    p = FS_C0 + FS_C1 * r + FS_C2 * r * r
    return np.where(r < FS_C, 2.0 * (r - FS_C) * p + (r - FS_C) ** 2 * (FS_C1 + 2.0 * FS_C2 * r), 0.0)


def _fs_F(rho):
    return -FS_A * np.sqrt(np.maximum(rho, 0.0))


def _fs_dF(rho):
    out = np.empty_like(rho)
    pos = rho > 0
    out[pos] = -0.5 * FS_A / np.sqrt(rho[pos])
    # rho = 0 knot: slope of the first piece's chord keeps the table finite
    h = rho[1] - rho[0] if rho.size > 1 else 1.0
    out[~pos] = (_fs_F(np.array([h]))[0] - 0.0) / h
    return out


def eam_tables(knots: int = EAM_KNOTS, rcut: float = EAM_RCUT, rho_max: float = RHO_MAX):
    rho_c, dr = hermite_table(_fs_rho, _fs_drho, rcut, knots)
    phi_c, _ = hermite_table(_fs_phi, _fs_dphi, rcut, knots)
    F_c, drho = hermite_table(_fs_F, _fs_dF, rho_max, knots)
    return dict(rcut=rcut, dr=dr, rho=rho_c, phi=phi_c, drho=drho, F=F_c)


def make_eam(n_atoms: int, box, **kw):
    from .potentials import EAM
    t = eam_tables(**kw)
    return EAM(n_atoms=n_atoms, box=box, rcut=t["rcut"], dr=t["dr"], rho=t["rho"], phi=t["phi"],
               drho=t["drho"], F=t["F"])


def n_bispectrum(twojmax: int) -> int:
    n = 0
    for j1 in range(twojmax + 1):
        for j2 in range(j1 + 1):
            for j in range(j1 - j2, min(twojmax, j1 + j2) + 1, 2):
                if j >= j1:
                    n += 1
    return n


def snap_beta(seed: int, twojmax: int = SNAP_TWOJMAX, scale: float = 0.05) -> np.ndarray:
    """beta_0..beta_K = scale * N(0,1) from the counter stream of derive_seed(seed, 1).

    Host-side restatement of the polar stream (a handful of variates of the
    plan; the GPU generator produces the same numbers up to log()'s ulp).
    """
    from .rng import derive_seed
    count = n_bispectrum(twojmax) + 1
    s = derive_seed(seed, 1)
    mask = (1 << 64) - 1
    golden = 0x9E3779B97F4A7C15

    def mix(z):
        z &= mask
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & mask
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & mask
        return z ^ (z >> 31)

    out, j = [], 0
    while len(out) < count:
        u1 = (mix(s + (j + 1) * golden) >> 11) * 2.0 ** -53
        u2 = (mix(s + (j + 2) * golden) >> 11) * 2.0 ** -53
        j += 2
        x, y = 2.0 * u1 - 1.0, 2.0 * u2 - 1.0
        r = x * x + y * y
        if 0.0 < r < 1.0:
            f = math.sqrt(-2.0 * math.log(r) / r)
            out.append(x * f)
            out.append(y * f)
    return scale * np.array(out[:count])


def make_snap(n_atoms: int, box, seed: int = 11, twojmax: int = SNAP_TWOJMAX, beta=None,
              scale: float = 0.05):
    from .potentials import SNAP
    if beta is None:
        beta = snap_beta(seed, twojmax, scale)
    return SNAP(n_atoms=n_atoms, box=box, beta=beta, twojmax=twojmax, rcut=SNAP_RCUT,
                rfac0=SNAP_RFAC0, rmin0=0.0, switchflag=1, wself=1.0)


def maxwell_boltzmann(n_atoms: int, temperature: float, seed: int, mass: float = MASS_W):
    """p ~ N(0, m k_B T) per component (derive_seed(seed, 10^9) stream)."""
    from .rng import derive_seed, gaussian_stream
    g = gaussian_stream(derive_seed(seed, 10 ** 9), 3 * n_atoms)
    return g * math.sqrt(mass * KB * temperature)


def displaced(q0: np.ndarray, sigma: float, seed: int, count: int):
    """count configurations q0 + N(0, sigma^2) displacements (force-sweep config)."""
    from .rng import derive_seeds, gaussian_streams
    g = gaussian_streams(derive_seeds(seed, count), q0.shape[0])
    return q0[None, :] + sigma * g
