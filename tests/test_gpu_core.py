"""GPU parity of the noise, the BBK window kernels and the parareal engines
against the reference's own golden vectors (tests/golden, produced by
scripts/make_golden.py from /root/reference) and the CPU oracle.

Bitwise where the arithmetic allows it (DoubleWell / Harmonic windows with
injected noise; 1-D engines); the Gaussian generator may differ from numpy by
the 1-ulp freedom of log() (SURVEY.md finding 4), and multi-dimensional error
norms by reduction order (OpenBLAS ddot vs a fixed device tree).
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


def test_device_seeds(pl):
    import torch
    from paper_2212_10508_b200 import _lib
    ctx = _lib.context()
    out = torch.zeros(1000, dtype=torch.int64, device="cuda")
    _lib.check(_lib.load().pl_derive_seeds(ctx.handle, 11, 1000, _lib.ptr(out)))
    got = out.cpu().numpy().view(np.uint64)
    assert np.array_equal(got, pl.derive_seeds(11, 1000))


def test_gaussian_streams_vs_reference(pl, golden):
    z = golden("rng_golden.npz")
    total = mism = 0
    for c in z["counts"]:
        for i, sd in enumerate(z["stream_seeds"]):
            ref = z[f"stream_c{int(c)}_s{i}"]
            got = pl.gaussian_stream(int(sd), int(c))
            assert got.shape == ref.shape
            rel = np.abs(got - ref) / np.maximum(np.abs(ref), 1e-300)
            assert rel.max() < 1e-14, (c, i, rel.max())  # only log()'s last-ulp freedom
            total += ref.size
            mism += int(np.count_nonzero(got != ref))
    assert mism / total < 0.02
    got = pl.gaussian_streams(z["batch_seeds"], 387)
    np.testing.assert_allclose(got, z["batch_c387"], rtol=1e-14, atol=0)


def test_gaussian_stream_prefix_stable_and_large(pl):
    s = pl.derive_seed(3, 9)
    a = pl.gaussian_stream(s, 1_000_001)
    b = pl.gaussian_stream(s, 999)
    assert np.array_equal(a[:999], b)
    assert abs(a.mean()) < 5e-3 and abs(a.std() - 1.0) < 5e-3


def _grad_pot(pl, name):
    if name == "dw1":
        return pl.DoubleWell(1.0, 1.0)
    if name == "dw5":
        return pl.DoubleWell(np.array([1.0, 0.5, 2.0, 1.5, 0.8]), np.array([1.0, 2.0, 0.5, 1.0, 1.5]))
    if name == "harm4":
        return pl.Harmonic(k=np.array([1.0, 3.0, 0.5, 2.0]))
    if name == "lj7":
        return pl.LennardJonesCluster(1.0, 1.0, 7, 2)
    if name == "lj13":
        return pl.LennardJonesCluster(1.0, 1.0, 13, 3)


@pytest.mark.parametrize("name", ["dw1", "dw5", "harm4", "lj7", "lj13"])
def test_window_injected_noise_vs_reference(pl, golden, name):
    z = golden("window_golden.npz")
    gamma, inv_beta, dt, L = z[f"{name}_meta"]
    mass = z[f"{name}_mass"] if f"{name}_mass" in z else None
    params = pl.LangevinParams(gamma, inv_beta, dt, int(L), mass=mass)
    sched = pl.TemperatureSchedule(tuple(z[f"{name}_sched"]))
    st = pl.PhaseState(q=z[f"{name}_q0"], p=z[f"{name}_p0"])
    out = pl.propagate_windows([st], _grad_pot(pl, name), params, sched, [0],
                               noise=z[f"{name}_noise"][None, :])[0]
    if name.startswith("lj"):
        np.testing.assert_allclose(out.q, z[f"{name}_q1"], rtol=1e-12, atol=1e-13)
        np.testing.assert_allclose(out.p, z[f"{name}_p1"], rtol=1e-12, atol=1e-13)
    else:
        assert out.q.tobytes() == z[f"{name}_q1"].tobytes()
        assert out.p.tobytes() == z[f"{name}_p1"].tobytes()


def test_window_device_noise_appendix_a(pl):
    out = pl.propagate_window(pl.PhaseState(q=[-1.0], p=[0.0]), pl.DoubleWell(1.0, 1.0),
                              pl.LangevinParams(0.5, 0.4, 0.05, 2), pl.TemperatureSchedule.robust(2),
                              pl.derive_seed(11, 1))
    assert out.q[0] == pytest.approx(-1.0118800384813031, rel=1e-14)
    assert out.p[0] == pytest.approx(-0.19175494361365208, rel=1e-14)


def test_batched_windows_match_single(pl):
    pot = pl.LennardJonesCluster(1.0, 1.0, 13, 3)
    params = pl.LangevinParams(1.0, 0.2, 0.002, 10)
    sched = pl.TemperatureSchedule.robust(10)
    rs = np.random.default_rng(0)
    g = np.array([[i, j, k] for i in range(3) for j in range(3) for k in range(2)], float)[:13]
    states = [pl.PhaseState(q=(g * 1.12 + 0.01 * rs.normal(size=g.shape)).ravel(), p=np.zeros(39))
              for _ in range(5)]
    seeds = [pl.derive_seed(4, n) for n in range(1, 6)]
    batch = pl.propagate_windows(states, pot, params, sched, seeds)
    for s, sd, b in zip(states, seeds, batch):
        one = pl.propagate_window(s, pot, params, sched, sd)
        assert one.q.tobytes() == b.q.tobytes() and one.p.tobytes() == b.p.tobytes()


# ------------------------------------------------------------------ blow-up parity
# The reference's own failure tests (test_integrator.py:602-627,
# test_parareal.py:238-244, 397-422), run through the device path.
def _st(q, p=None):
    q = np.asarray(q, dtype=float)
    return q, (np.zeros_like(q) if p is None else np.asarray(p, dtype=float))


def test_blow_up_raises_with_substep(pl):
    """omega*dt = 100: the splitting is unstable; first bad substep is 2, no window context."""
    params = pl.LangevinParams(0.0, 0.0, 0.1, 20)
    sched = pl.TemperatureSchedule.identity(20)
    q, p = _st([1.0])
    with pytest.raises(pl.BlowUpError, match="substep") as ei:
        pl.propagate_window(pl.PhaseState(q=q, p=p), pl.Harmonic(k=1e6), params, sched, 1)
    assert ei.value.substep == 2
    assert ei.value.window is None


def test_blow_up_on_out_of_range_start(pl):
    params = pl.LangevinParams(0.0, 0.0, 0.1, 2)
    q, p = _st([10.0 * 1e12])
    with pytest.raises(pl.BlowUpError) as ei:
        pl.propagate_window(pl.PhaseState(q=q, p=p), pl.Free(), params, pl.TemperatureSchedule.identity(2), 1)
    assert ei.value.substep == 1


def test_blow_up_on_non_finite(pl):
    """A gradient that overflows to inf at the first substep: 'non-finite', substep 1."""
    params = pl.LangevinParams(0.0, 0.0, 0.1, 2)
    q, p = _st([1.0])
    with pytest.raises(pl.BlowUpError, match="non-finite") as ei:
        pl.propagate_window(pl.PhaseState(q=q, p=p), pl.Harmonic(k=1e308), params,
                            pl.TemperatureSchedule.identity(2), 1)
    assert ei.value.substep == 1


def test_blow_up_in_batch_reports_first_window(pl):
    """Batched windows: the first blown-up row raises, with its own substep."""
    params = pl.LangevinParams(0.0, 0.0, 0.1, 20)
    sched = pl.TemperatureSchedule.identity(20)
    states = [pl.PhaseState(q=[1e-9], p=[0.0]), pl.PhaseState(q=[1.0], p=[0.0])]
    with pytest.raises(pl.BlowUpError) as ei:
        pl.propagate_windows(states, pl.Harmonic(k=1e6), params, sched, [1, 2])
    assert ei.value.substep >= 2


def test_blow_up_sequential_reports_window(pl):
    params = pl.LangevinParams(0.0, 0.0, 0.1, 20)
    sched = pl.TemperatureSchedule.identity(20)
    plan = pl.NoisePlan.for_windows(3, 4)
    q, p = _st([1.0])
    with pytest.raises(pl.BlowUpError) as ei:
        pl.sequential_propagate(pl.PhaseState(q=q, p=p), 4, pl.Harmonic(k=1e6), params, sched, plan)
    assert ei.value.window == 1
    assert ei.value.substep == 2


def test_blow_up_during_jump_reports_context(pl):
    params = pl.LangevinParams(0.0, 0.0, 0.1, 20)
    sched = pl.TemperatureSchedule.identity(20)
    plan = pl.NoisePlan.for_windows(3, 3)
    pair = pl.PropagatorPair(fine=pl.Harmonic(k=1e6), coarse=pl.Harmonic(k=1.0), cost_fine=2.0,
                             cost_coarse=1.0)
    q, p = _st([1.0])
    cfg = pl.PararealConfig(n_windows=3, delta_conv=1e-8)
    with pytest.raises(pl.BlowUpError) as ei:
        pl.parareal_classic(pl.PhaseState(q=q, p=p), pair, params, sched, plan, cfg)
    assert ei.value.window == 1
    assert ei.value.iteration == 1
    assert ei.value.substep is not None
    with pytest.raises(pl.BlowUpError) as ei:
        pl.parareal_adaptive(pl.PhaseState(q=q, p=p), pair, params, sched, plan,
                             pl.PararealConfig(n_windows=3, delta_conv=1e-8, delta_expl=0.35))
    assert ei.value.window == 1
    assert ei.value.iteration == 1


def test_blow_up_during_bootstrap_is_iteration_zero(pl):
    params = pl.LangevinParams(0.0, 0.0, 0.1, 20)
    sched = pl.TemperatureSchedule.identity(20)
    plan = pl.NoisePlan.for_windows(3, 3)
    pair = pl.PropagatorPair(fine=pl.Harmonic(k=1.0), coarse=pl.Harmonic(k=1e6), cost_fine=2.0,
                             cost_coarse=1.0)
    q, p = _st([1.0])
    cfg = pl.PararealConfig(n_windows=3, delta_conv=1e-8, delta_expl=0.35)
    for engine in (pl.parareal_classic, pl.parareal_adaptive):
        with pytest.raises(pl.BlowUpError) as ei:
            engine(pl.PhaseState(q=q, p=p), pair, params, sched, plan, cfg)
        assert ei.value.window == 1
        assert ei.value.iteration == 0


# ------------------------------------------------------------------ engines
def _inject(prop, noise_rows):
    import torch
    prop._noise = torch.from_numpy(np.ascontiguousarray(noise_rows)).to(prop.kernel.device)


def _dw_engine_setup(pl, cfg):
    from oracle import rng as orng
    gamma, inv_beta, dt, L, seed, n = cfg[:6]
    params = pl.LangevinParams(gamma, inv_beta, dt, int(L))
    sched = pl.TemperatureSchedule.robust(int(L))
    plan = pl.NoisePlan.for_windows(int(seed), int(n))
    noise = orng.gaussian_streams(orng.derive_seeds(int(seed), int(n)), (int(L) + 1) * 1)
    from paper_2212_10508_b200.parareal import DevicePropagator
    fine = DevicePropagator(pl.DoubleWell(1.0, 1.0), params, sched, plan, 1)
    coarse = DevicePropagator(pl.DoubleWell(0.8, 1.0), params, sched, plan, 1)
    _inject(fine, noise)
    _inject(coarse, noise)
    return fine, coarse


def _check(res, z, prefix, bitwise=True):
    Q, P = res.trajectory.positions(), res.trajectory.momenta()
    if bitwise:
        assert Q.tobytes() == z[f"{prefix}_Q"].tobytes()
        assert P.tobytes() == z[f"{prefix}_P"].tobytes()
        hist = np.array(res.error_history, float)
        assert hist.tobytes() == z[f"{prefix}_hist"].tobytes()
    rows = [[s.slab_index, s.n_init, s.n_final, s.k_conv, a.n_final, a.iterations]
            for s in res.slabs for a in s.attempts]
    assert np.array_equal(np.array(rows, dtype=np.int64), z[f"{prefix}_slabs"])
    assert bool(res.converged) == bool(z[f"{prefix}_converged"])


def test_adaptive_engine_config_bitwise(pl, golden):
    z = golden("parareal_golden.npz")
    cfg = z["adaptive_cfg"]
    fine, coarse = _dw_engine_setup(pl, cfg)
    init = pl.PhaseState(q=[-1.0], p=[0.0])
    res = pl.parareal_adaptive_engine(init, fine, coarse, pl.PararealConfig(int(cfg[5]), cfg[6], cfg[7]))
    _check(res, z, "adaptive")
    assert res.n_slab == 4 and res.total_iterations == 92


def test_classic_engine_config_bitwise(pl, golden):
    z = golden("parareal_golden.npz")
    cfg = z["parareal_cfg"]
    fine, coarse = _dw_engine_setup(pl, cfg)
    res = pl.parareal_classic_engine(pl.PhaseState(q=[-1.0], p=[0.0]), fine, coarse,
                                     pl.PararealConfig(int(cfg[5]), cfg[6]))
    _check(res, z, "parareal")


def test_adaptive_device_rng_matches_oracle_on_same_noise(pl):
    """Device RNG + device engine == oracle engine driven by the device's noise."""
    from oracle import integrator as oint, parareal as opar, toy
    params = pl.LangevinParams(0.5, 0.4, 0.05, 2)
    sched = pl.TemperatureSchedule.robust(2)
    n = 300
    plan = pl.NoisePlan.for_windows(11, n)
    pair = pl.PropagatorPair(pl.DoubleWell(1.0, 1.0), pl.DoubleWell(0.8, 1.0), 175.0, 1.0)
    res = pl.parareal_adaptive(pl.PhaseState(q=[-1.0], p=[0.0]), pair, params, sched, plan,
                               pl.PararealConfig(n, 1e-10, 0.35))
    noise = pl.gaussian_streams(np.array(plan.window_seeds, dtype=np.uint64), 3)

    def mk(a):
        g = toy.double_well(a, 1.0)
        return lambda s, m: oint.propagate_window(s[0], s[1], g, 0.5, 0.4, 0.05, 2, oint.robust(2),
                                                  0, noise=noise[m])
    ref = opar.adaptive((np.array([-1.0]), np.zeros(1)), mk(1.0), mk(0.8), n, 1e-10, 0.35)
    assert np.array([s[0] for s in ref["trajectory"]]).tobytes() == res.trajectory.positions().tobytes()
    assert np.array(ref["history"], float).tobytes() == np.array(res.error_history, float).tobytes()
    assert len(ref["slabs"]) == res.n_slab


def test_sequential_config_bitwise(pl, golden):
    z = golden("parareal_golden.npz")
    fine, _ = _dw_engine_setup(pl, np.array([0.5, 0.4, 0.05, 2, 11, 500]))
    # sequential chain through the device propagator with injected noise
    st = pl.PhaseState(q=[-1.0], p=[0.0])
    Q = [st.q]
    for m in range(500):
        st = fine(st, m)
        Q.append(st.q)
    assert np.array(Q).tobytes() == z["sequential_Q"].tobytes()


def test_lj13_adaptive_vs_reference(pl, golden):
    from oracle import rng as orng
    from paper_2212_10508_b200.parareal import DevicePropagator
    z = golden("parareal_golden.npz")
    lj = pl.LennardJonesCluster(1.0, 1.0, 13, 3)
    coarse = pl.Perturbed(base=lj, delta=pl.Harmonic(k=1.0), lam=0.05)
    params = pl.LangevinParams(1.0, 0.2, 0.002, 10)
    sched = pl.TemperatureSchedule.robust(10)
    plan = pl.NoisePlan.for_windows(5, 24)
    noise = orng.gaussian_streams(orng.derive_seeds(5, 24), 11 * 39)
    f = DevicePropagator(lj, params, sched, plan, 39)
    c = DevicePropagator(coarse, params, sched, plan, 39)
    _inject(f, noise)
    _inject(c, noise)
    res = pl.parareal_adaptive_engine(pl.PhaseState(q=z["lj13_q0"], p=np.zeros(39)), f, c,
                                      pl.PararealConfig(24, 1e-10, 0.05))
    _check(res, z, "lj13", bitwise=False)
    np.testing.assert_allclose(res.trajectory.positions(), z["lj13_Q"], rtol=0, atol=1e-10)
    h = np.array(res.error_history, float)
    np.testing.assert_allclose(h[:, 2], z["lj13_hist"][:, 2], rtol=1e-6, atol=1e-13)


def test_batched_replicas_equal_single_runs_dw(pl):
    """parareal_adaptive_batch == per-replica parareal_adaptive, bit for bit (adaptive.json params)."""
    params = pl.LangevinParams(0.5, 0.4, 0.05, 2)
    sched = pl.TemperatureSchedule.robust(2)
    n = 200
    pair = pl.PropagatorPair(pl.DoubleWell(1.0, 1.0), pl.DoubleWell(0.8, 1.0), 175.0, 1.0)
    cfg = pl.PararealConfig(n, 1e-10, 0.35)
    plans = [pl.NoisePlan.for_windows(pl.derive_seed(77, 10**9 + i), n) for i in range(5)]
    inits = [pl.PhaseState(q=[-1.0 + 0.1 * i], p=[0.0]) for i in range(5)]
    batch = pl.parareal_adaptive_batch(inits, pair, params, sched, plans, cfg)
    for i in range(5):
        one = pl.parareal_adaptive(inits[i], pair, params, sched, plans[i], cfg)
        assert one.slabs == batch[i].slabs
        assert one.error_history == batch[i].error_history
        assert one.trajectory.positions().tobytes() == batch[i].trajectory.positions().tobytes()
