"""External pins of the C SNAP oracle (oracle/native/snap_oracle.c), CPU only.

The reference package has no SNAP, so the oracle is pinned to
definitions computed by independent code, as SURVEY.md 8(c) asks:

* Clebsch-Gordan coefficients: ``orc_cg`` (Racah formula in C) against
  ``sympy.physics.wigner.clebsch_gordan`` (exact arithmetic), every coefficient
  with 2j <= 8 that the twojmax = 8 contraction touches;
* the U recursion: the oracle's U^J of a neighbour is the spin-J/2 irreducible
  representation of its SU(2) element U^1.  The representation is built here
  from explicit polynomials (symmetric tensor power on normalised monomials),
  and that construction is itself checked against sympy's Wigner-D matrices
  ``wigner_d(J/2, alpha, beta, gamma)`` for several Euler angles;
* the bispectrum: a slow numpy evaluation B = Re <Utot^J, C^T (Utot^j1 (x)
  Utot^j2) C> on small clusters, with Utot from the polynomial representation
  (no recursion), C from sympy, against the oracle's per-atom B.

The device is checked against this oracle in tests/test_gpu_manybody.py.
"""

import math

import numpy as np
import pytest

sympy = pytest.importorskip("sympy")
from sympy import Rational as R  # noqa: E402
from sympy.physics import wigner  # noqa: E402

TJ = 8
RFAC0, RMIN0, RCUT = 0.99363, 0.0, 4.73


@pytest.fixture(scope="module")
def native():
    from oracle import native as nat
    nat.load()
    return nat


def _sym_rep(g, J):
    """Spin-J/2 representation of the 2x2 matrix g on the normalised monomials
    e_k = x^(J-k) y^k / sqrt((J-k)! k!): column l is the image of e_l."""
    out = np.zeros((J + 1, J + 1), complex)
    for l in range(J + 1):
        for a in range(J - l + 1):
            for b in range(l + 1):
                c = (math.comb(J - l, a) * math.comb(l, b) * g[0, 0] ** (J - l - a) * g[1, 0] ** a
                     * g[0, 1] ** (l - b) * g[1, 1] ** b)
                k = a + b
                out[k, l] += c * math.sqrt(math.factorial(J - k) * math.factorial(k)
                                           / (math.factorial(J - l) * math.factorial(l)))
    return out


def _u1(rv):
    """U^1 of a neighbour vector from the Cayley-Klein parameters (a, b):
    theta0 = rfac0 pi (r - rmin0) / (rcut - rmin0), a = cos theta0 - i (z/r) sin theta0,
    b = sin theta0 (y - i x) / r, U^1 = [[conj a, b], [-conj b, a]] ([ma][mb])."""
    x, y, z = rv
    r = math.sqrt(x * x + y * y + z * z)
    th = RFAC0 * math.pi * (r - RMIN0) / (RCUT - RMIN0)
    a = complex(math.cos(th), -z / r * math.sin(th))
    b = complex(y / r * math.sin(th), -x / r * math.sin(th))
    return np.array([[a.conjugate(), b], [-b.conjugate(), a]])


def _sympy_cg(j1, m1, j2, m2, J, M):
    return float(wigner.clebsch_gordan(R(j1, 2), R(j2, 2), R(J, 2), R(m1, 2), R(m2, 2), R(M, 2)))


def test_cg_matches_sympy(native):
    n = 0
    for j1 in range(TJ + 1):
        for j2 in range(TJ + 1):
            for J in range(abs(j1 - j2), min(TJ, j1 + j2) + 1, 2):
                for m1 in range(-j1, j1 + 1, 2):
                    for m2 in range(-j2, j2 + 1, 2):
                        M = m1 + m2
                        if abs(M) > J:
                            continue
                        ref = _sympy_cg(j1, m1, j2, m2, J, M)
                        got = native.cg(j1, m1, j2, m2, J, M)
                        assert got == pytest.approx(ref, rel=1e-13, abs=1e-14), (j1, m1, j2, m2, J, M)
                        n += 1
    assert n == 4451  # every (j1, j2, J) triple with 2j <= 8 and all (m1, m2)


@pytest.mark.parametrize("ang", [(R(3, 10), R(7, 10), R(11, 10)), (R(-2), R(5, 2), R(1, 7)),
                                 (R(0), R(31, 10), R(-9, 10))])
def test_polynomial_rep_is_wigner_d(ang):
    """sympy's D^{j}(alpha, beta, gamma) == the polynomial representation of D^{1/2}."""
    d12 = np.array(wigner.wigner_d(R(1, 2), *ang).evalf(30), dtype=complex)
    for J in range(1, TJ + 1):
        dj = np.array(wigner.wigner_d(R(J, 2), *ang).evalf(30), dtype=complex)
        np.testing.assert_allclose(_sym_rep(d12, J), dj, rtol=0, atol=2e-15 * (J + 1))


@pytest.mark.parametrize("rv", [(1.0, 0.5, -2.0), (-2.2, 1.3, 0.4), (0.1, -0.2, 3.9), (2.74, 0.0, 0.0)])
def test_u_recursion_is_the_irreducible_representation(native, rv):
    """Oracle U^J (recursion) == spin-J/2 representation of U^1, U^1 from (a, b)."""
    U = native.ulist(TJ, RFAC0, RMIN0, RCUT, rv)
    g = _u1(rv)
    np.testing.assert_allclose(U[1], g, rtol=0, atol=1e-15)
    for J in range(TJ + 1):
        np.testing.assert_allclose(U[J], _sym_rep(g, J), rtol=0, atol=5e-15 * (J + 1))
        # unitary
        np.testing.assert_allclose(U[J] @ U[J].conj().T, np.eye(J + 1), atol=1e-13)


def _cg_matrix(j1, j2, J, cg):
    """C[(a1, a2), ma] = <j1 m1 j2 m2 | J M>, rows in np.kron order (a1 major)."""
    C = np.zeros(((j1 + 1) * (j2 + 1), J + 1))
    for a1 in range(j1 + 1):
        for a2 in range(j2 + 1):
            m1, m2 = 2 * a1 - j1, 2 * a2 - j2
            M = m1 + m2
            if abs(M) <= J:
                C[a1 * (j2 + 1) + a2, (M + J) // 2] = cg(j1, m1, j2, m2, J, M)
    return C


def _slow_bispectrum(X, i, wself=1.0):
    """B_{j1 j2 J} of atom i of the open cluster X (canonical j1 >= j2, J >= j1)."""
    ut = [wself * np.eye(J + 1, dtype=complex) for J in range(TJ + 1)]
    for k in range(len(X)):
        if k == i:
            continue
        rv = X[k] - X[i]
        r = float(np.linalg.norm(rv))
        if r >= RCUT:
            continue
        fc = 0.5 * (math.cos(math.pi * (r - RMIN0) / (RCUT - RMIN0)) + 1.0)
        g = _u1(rv)
        for J in range(TJ + 1):
            ut[J] = ut[J] + fc * _sym_rep(g, J)
    cache = {}
    out = []
    for j1 in range(TJ + 1):
        for j2 in range(j1 + 1):
            for J in range(j1 - j2, min(TJ, j1 + j2) + 1, 2):
                if J < j1:
                    continue
                key = (j1, j2, J)
                if key not in cache:
                    cache[key] = _cg_matrix(j1, j2, J, _sympy_cg)
                C = cache[key]
                Z = C.T @ np.kron(ut[j1], ut[j2]) @ C   # Z[ma][mb]
                out.append(float(np.real(np.sum(np.conj(ut[J]) * Z))))
    return np.array(out)


@pytest.mark.parametrize("seed", [1, 2])
def test_bispectrum_slow_evaluation(native, seed):
    """Oracle per-atom B (55 components) == slow sympy-CG / polynomial-rep evaluation,
    on 4-atom open clusters (large box, no periodic images)."""
    from paper_2212_10508_b200.potentials import SNAP
    rs = np.random.default_rng(seed)
    X = rs.normal(size=(4, 3)) * 1.4 + 20.0
    beta = np.concatenate([[0.0], rs.normal(size=55) * 0.05])
    pot = SNAP(n_atoms=4, box=(40.0, 40.0, 40.0), beta=beta, twojmax=TJ, rcut=RCUT, rfac0=RFAC0,
               rmin0=RMIN0)
    _, _, _, B = native.snap(X.ravel(), pot.box, pot, want_bispectrum=True)
    assert B.shape == (4, 55)
    for i in range(4):
        slow = _slow_bispectrum(X, i)
        np.testing.assert_allclose(B[i], slow, rtol=1e-11, atol=1e-12 * np.abs(slow).max())


def _cluster_pot(n, seed, box=40.0):
    from paper_2212_10508_b200.potentials import SNAP
    rs = np.random.default_rng(seed)
    beta = np.concatenate([[0.3], rs.normal(size=55) * 0.05])
    return SNAP(n_atoms=n, box=(box, box, box), beta=beta, twojmax=TJ, rcut=RCUT, rfac0=RFAC0, rmin0=RMIN0)


def test_oracle_forces_are_energy_derivatives(native):
    """Oracle gradient (forward-mode dU, dE_k/dr_ka - dE_a/dr_ak gather) == central
    differences of the oracle energy; Sum F = 0."""
    rs = np.random.default_rng(4)
    X = rs.normal(size=(6, 3)) * 1.5 + 20.0
    pot = _cluster_pot(6, 4)
    q = X.ravel()
    e, g, _ = native.snap(q, pot.box, pot)
    h = 1e-5
    fd = np.zeros_like(q)
    for k in range(q.shape[0]):
        qp, qm = q.copy(), q.copy()
        qp[k] += h
        qm[k] -= h
        fd[k] = (native.snap(qp, pot.box, pot)[0] - native.snap(qm, pot.box, pot)[0]) / (2 * h)
    np.testing.assert_allclose(g, fd, rtol=0, atol=1e-7 * max(1.0, np.abs(g).max()))
    assert np.abs(g.reshape(-1, 3).sum(axis=0)).max() < 1e-12 * max(1.0, np.abs(g).max())


def test_oracle_rotation_invariance(native):
    """E(R X) == E(X), grad(R X) == R grad(X), virial(R X) == R virial R^T."""
    rs = np.random.default_rng(9)
    X = rs.normal(size=(7, 3)) * 1.6
    pot = _cluster_pot(7, 9)
    th, ax = 0.83, np.array([1.0, 2.0, -2.0]) / 3.0
    K = np.array([[0, -ax[2], ax[1]], [ax[2], 0, -ax[0]], [-ax[1], ax[0], 0]])
    Rm = np.eye(3) + np.sin(th) * K + (1 - np.cos(th)) * K @ K
    ea, ga, va = native.snap((X + 20.0).ravel(), pot.box, pot)
    eb, gb, vb = native.snap((X @ Rm.T + 20.0).ravel(), pot.box, pot)
    assert eb == pytest.approx(ea, rel=1e-12)
    np.testing.assert_allclose(gb.reshape(-1, 3), ga.reshape(-1, 3) @ Rm.T, atol=1e-11)

    def full(v):
        return np.array([[v[0], v[3], v[4]], [v[3], v[1], v[5]], [v[4], v[5], v[2]]])
    np.testing.assert_allclose(full(vb), Rm @ full(va) @ Rm.T, atol=1e-11)


def test_oracle_periodic_lattice_fd(native):
    """129-atom W + SIA periodic cell: oracle gradient == central differences on a
    sample of components (minimum image, neighbours across the boundary)."""
    from paper_2212_10508_b200 import tungsten as W
    q0, box = W.bcc_sia(4)
    n = q0.shape[0] // 3
    q = q0 + 0.1 * np.random.default_rng(2).normal(size=q0.shape)
    pot = W.make_snap(n, box)
    _, g, _ = native.snap(q, box, pot)
    h = 1e-5
    for k in (0, 1, 2, 200, 3 * n - 1, 3 * n - 5):
        qp, qm = q.copy(), q.copy()
        qp[k] += h
        qm[k] -= h
        fd = (native.snap(qp, box, pot)[0] - native.snap(qm, box, pot)[0]) / (2 * h)
        assert g[k] == pytest.approx(fd, abs=2e-7 * max(1.0, np.abs(g).max()))
