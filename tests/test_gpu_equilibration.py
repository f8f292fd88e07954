"""GPU parity of the equilibration / measurement callers around the hot path
(SURVEY.md 8(f) rows 2-3): batched local minimisation (pl_minimize, the
reference's _descend / local_minima, potentials.py:231-287) and the batched
kinetic-temperature measurement (pl_propagate_windows_moments, the reference's
measure_kinetic_temperature, integrator.py:430-482), against golden vectors
the reference produced here (scripts/make_golden.py) and the CPU oracle.

Tolerances: the Gaussian generator may differ from numpy by the 1-ulp freedom
of log() and device energies / norms by reduction order, so chains and
descents agree to ~1e-12 relative, not bitwise.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pl():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2212_10508_b200 as pl
    return pl


TEMP_CASES = {
    "harm": lambda pl: (pl.Harmonic(k=np.array([1.0, 3.0, 0.5])),
                        pl.LangevinParams(1.0, 0.7, 0.05, 5, mass=[1.0, 2.0, 0.5]), 40, 123),
    "dw": lambda pl: (pl.DoubleWell(1.0, 1.0), pl.LangevinParams(0.5, 0.4, 0.05, 3), 60, 7),
}


@pytest.mark.parametrize("case", sorted(TEMP_CASES))
@pytest.mark.parametrize("sampling", ["all_substeps", "window_ends"])
def test_kinetic_temperature_vs_reference(pl, golden, case, sampling):
    pot, params, nw, seed = TEMP_CASES[case](pl)
    ref = golden("temperature_golden.npz")[f"{case}_{sampling}"]
    r = pl.measure_kinetic_temperature(pot, params, pl.TemperatureSchedule.robust(params.substeps), nw, seed,
                                       sampling=sampling, burn_in=0.2)
    assert (r.n_windows, r.n_burn_in) == (int(ref[2]), int(ref[3]))
    assert r.k_eq_predicted == ref[1]
    np.testing.assert_allclose(r.k_eq_empirical, ref[0], rtol=1e-10)
    np.testing.assert_allclose(r.per_substep_variance, ref[4:], rtol=1e-10)


def test_kinetic_temperature_batch_equals_single_chains(pl):
    pot = pl.Harmonic(k=np.array([1.0, 3.0, 0.5]))
    params = pl.LangevinParams(1.0, 0.7, 0.05, 5, mass=[1.0, 2.0, 0.5])
    sched = pl.TemperatureSchedule.robust(5)
    seeds = [3, 123, 2**40 + 7]
    batch = pl.measure_kinetic_temperature_batch(pot, params, sched, 30, seeds, burn_in=0.1)
    for s, rb in zip(seeds, batch):
        r1 = pl.measure_kinetic_temperature(pot, params, sched, 30, s, burn_in=0.1)
        assert rb == r1  # chains are independent columns of one launch: bitwise equal


def test_kinetic_temperature_w_eam_batched(pl):
    """W + SIA (129 atoms, EAM), 4 replica chains started on the lattice (the
    reference's cold start q = 0 would put every atom on one site): the
    measured kinetic temperature approaches k_B T (1 - 1/(2L)) (integrator.py:316-320)."""
    from paper_2212_10508_b200 import tungsten as W
    q0, box = W.bcc_sia(4)
    n = q0.shape[0] // 3
    eam = W.make_eam(n, box)
    L, T = 20, 1000.0
    params = pl.LangevinParams(10.0, W.KB * T, 0.002, L, mass=np.full(3 * n, W.MASS_W))
    start = pl.PhaseState(q=q0, p=np.zeros_like(q0))
    reps = pl.measure_kinetic_temperature_batch(eam, params, pl.TemperatureSchedule.robust(L), 40,
                                                [1, 2, 3, 4], burn_in=0.5, initial=start)
    k = np.mean([r.k_eq_empirical for r in reps])
    assert abs(k / reps[0].k_eq_predicted - 1.0) < 0.1


def test_local_minima_double_well_vs_reference(pl, golden):
    z = golden("minima_golden.npz")
    got = pl.local_minima(pl.DoubleWell(1.0, 1.0), list(z["dw_starts"]), tol=1e-9)
    assert len(got) == len(z["dw_minima"])
    np.testing.assert_allclose(np.stack(got), z["dw_minima"], atol=1e-12)


def test_local_minima_lj7_vs_reference(pl, golden):
    z = golden("minima_golden.npz")
    lj = pl.LennardJonesCluster(1.0, 1.0, 7, 2)
    got = pl.local_minima(lj, list(z["lj_starts"]), tol=1e-6)
    assert len(got) == len(z["lj_minima"])
    # same basin reached from every start: positions to the descent tolerance, energies tightly
    np.testing.assert_allclose(np.stack(got), z["lj_minima"], atol=1e-5)
    np.testing.assert_allclose(lj.energies(np.stack(got)), z["lj_energy"], rtol=1e-12)
    for x in got:
        assert np.linalg.norm(lj.gradient(x)) <= 1e-6


def test_minimization_errors_mirror_reference(pl):
    with pytest.raises(pl.MinimizationError, match="no convergence"):
        pl.local_minima(pl.DoubleWell(1.0, 1.0), [np.array([0.3])], tol=1e-12, max_iter=3)
    with pytest.raises(ValueError):
        pl.local_minima(pl.DoubleWell(1.0, 1.0), [np.array([0.3])], tol=0.0)


def test_minimize_w_sia_eam_vs_oracle(pl):
    """Relax 8 perturbed W + SIA configurations (129 atoms, EAM) in one batch; the
    oracle EAM confirms the relaxed energies and the force tolerance."""
    from oracle import native
    from paper_2212_10508_b200 import tungsten as W
    q0, box = W.bcc_sia(4)
    n = q0.shape[0] // 3
    eam = W.make_eam(n, box)
    rs = np.random.default_rng(8)
    starts = q0[None] + 0.05 * rs.normal(size=(8, q0.shape[0]))
    X, status, iters, E = pl.minimize_batch(eam, starts, tol=1e-4, max_iter=50000)
    assert (status == 0).all(), status
    tables = W.eam_tables()
    for b in range(8):
        e_o, g_o, _ = native.eam(X[b], box, tables)
        assert np.linalg.norm(g_o) <= 1.01e-4
        np.testing.assert_allclose(E[b], e_o, rtol=1e-10)
        assert E[b] < eam.energies(starts[b:b + 1])[0]
