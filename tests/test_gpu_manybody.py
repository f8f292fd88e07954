"""GPU parity of the periodic neighbour lists and EAM against the C oracle
(oracle/native), on the BASELINE W + SIA systems.

Bar: neighbour pair sets bit-exact; energies/forces/virials <= 1e-10 relative
(fp64; the device uses FMA, the oracle does not); short trajectories <= 1e-8 A.
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


def _configs(n, count, sigma=0.1, seed=3):
    from paper_2212_10508_b200 import tungsten as W
    q0, box = W.bcc_sia(n)
    rs = np.random.default_rng(seed)
    Q = q0[None, :] + sigma * rs.normal(size=(count, q0.shape[0]))
    # unwrapped coordinates: shift some atoms by whole box vectors
    Q[:, :6] += box[0]
    return Q, box


def _device_neighbours(pl, pot, Q, maxn=128):
    import torch
    from paper_2212_10508_b200 import _lib
    ctx = _lib.context()
    B, d = Q.shape
    n = d // 3
    q = torch.from_numpy(Q).cuda()
    nbr = torch.zeros((B, n, maxn), dtype=torch.int32, device="cuda")
    cnt = torch.zeros((B, n), dtype=torch.int32, device="cuda")
    _lib.check(_lib.load().pl_neighbours(ctx.handle, pot.handle(ctx), B, _lib.ptr(q), maxn,
                                         _lib.ptr(nbr), _lib.ptr(cnt)))
    nbr, cnt = nbr.cpu().numpy(), cnt.cpu().numpy()
    return [[sorted(nbr[b, i, :cnt[b, i]].tolist()) for i in range(n)] for b in range(B)]


@pytest.mark.parametrize("ncell,rcut", [(4, 5.5), (4, 4.73), (8, 5.5)])
def test_neighbour_lists_bit_exact(pl, ncell, rcut):
    from oracle import native
    from paper_2212_10508_b200 import tungsten as W
    Q, box = _configs(ncell, 3)
    n = Q.shape[1] // 3
    pot = W.make_eam(n, box, ) if rcut == 5.5 else W.make_snap(n, box)
    dev = _device_neighbours(pl, pot, Q)
    for b in range(Q.shape[0]):
        assert dev[b] == native.neighbours(Q[b], box, rcut)


def test_eam_vs_oracle(pl):
    from oracle import native
    from paper_2212_10508_b200 import tungsten as W
    Q, box = _configs(4, 16)
    n = Q.shape[1] // 3
    pot = W.make_eam(n, box)
    t = W.eam_tables()
    E, G, V = (x.cpu().numpy() for x in pot.evaluate(Q, True, True, True))
    for b in range(Q.shape[0]):
        e, g, v = native.eam(Q[b], box, t)
        assert E[b] == pytest.approx(e, rel=1e-10)
        np.testing.assert_allclose(G[b], g, rtol=1e-10, atol=1e-10 * np.abs(g).max())
        np.testing.assert_allclose(V[b], v, rtol=1e-10, atol=1e-10 * np.abs(v).max())


def test_eam_gradient_check_and_momentum(pl):
    from paper_2212_10508_b200 import tungsten as W
    Q, box = _configs(4, 1)
    pot = W.make_eam(Q.shape[1] // 3, box)
    assert pl.gradient_check(pot, Q[0], h=1e-5) < 1e-6
    g = pot.gradient(Q[0]).reshape(-1, 3)
    assert np.abs(g.sum(axis=0)).max() < 1e-10


def test_eam_window_vs_oracle(pl):
    """100 BBK substeps of EAM W+SIA at 1000 K: device vs oracle integrator + C EAM."""
    from oracle import integrator as oint, native, rng as orng
    from paper_2212_10508_b200 import tungsten as W
    q0, box = W.bcc_sia(4)
    n = q0.shape[0] // 3
    t = W.eam_tables()
    pot = W.make_eam(n, box)
    mass = np.full(3 * n, W.MASS_W)
    params = pl.LangevinParams(1.0, W.KB * 1000.0, 0.001, 100, mass=mass)
    sched = pl.TemperatureSchedule.robust(100)
    p0 = W.maxwell_boltzmann(n, 1000.0, 11)
    seed = pl.derive_seed(11, 1)
    noise = orng.gaussian_stream(seed, 101 * 3 * n)
    out = pl.propagate_windows([pl.PhaseState(q=q0, p=p0)], pot, params, sched, [seed],
                               noise=noise[None, :])[0]
    grad = lambda q: native.eam(q, box, t)[1]
    q1, p1 = oint.propagate_window(q0, p0, grad, 1.0, W.KB * 1000.0, 0.001, 100, sched.coefficients,
                                   0, mass=mass, noise=noise)
    assert np.abs(out.q - q1).max() < 1e-8
    assert np.abs(out.p - p1).max() < 1e-8 * np.abs(p1).max()


# ------------------------------------------------------------------ SNAP
def _snap_bispectrum(pl, pot, Q):
    import torch
    from paper_2212_10508_b200 import _lib
    ctx = _lib.context()
    B, d = Q.shape
    n = d // 3
    nb = pot.beta.shape[0] - 1
    q = torch.from_numpy(Q).cuda()
    out = torch.zeros((B, n, nb), dtype=torch.float64, device="cuda")
    _lib.check(_lib.load().pl_snap_bispectrum(ctx.handle, pot.handle(ctx), B, _lib.ptr(q), _lib.ptr(out)))
    return out.cpu().numpy()


def test_snap_bispectrum_vs_oracle(pl):
    from oracle import native
    from paper_2212_10508_b200 import tungsten as W
    Q, box = _configs(4, 3)
    n = Q.shape[1] // 3
    pot = W.make_snap(n, box)
    Bd = _snap_bispectrum(pl, pot, Q)
    for b in range(Q.shape[0]):
        _, _, _, Bo = native.snap(Q[b], box, pot, want_bispectrum=True)
        np.testing.assert_allclose(Bd[b], Bo, rtol=1e-10, atol=1e-10 * np.abs(Bo).max())


@pytest.mark.parametrize("ncell,count", [(4, 6), (8, 1)])
def test_snap_vs_oracle(pl, ncell, count):
    from oracle import native
    from paper_2212_10508_b200 import tungsten as W
    Q, box = _configs(ncell, count)
    n = Q.shape[1] // 3
    pot = W.make_snap(n, box)
    E, G, V = (x.cpu().numpy() for x in pot.evaluate(Q, True, True, True))
    for b in range(Q.shape[0]):
        e, g, v = native.snap(Q[b], box, pot)
        assert E[b] == pytest.approx(e, rel=1e-10)
        np.testing.assert_allclose(G[b], g, rtol=1e-10, atol=1e-10 * np.abs(g).max())
        np.testing.assert_allclose(V[b], v, rtol=1e-10, atol=1e-10 * np.abs(v).max())


def _snap_oracle_check(native, Q, box, pot, E, G, V, systems):
    for b in systems:
        e, g, v = native.snap(Q[b], box, pot)
        assert E[b] == pytest.approx(e, rel=1e-10)
        np.testing.assert_allclose(G[b], g, rtol=1e-10, atol=1e-10 * np.abs(g).max())
        np.testing.assert_allclose(V[b], v, rtol=1e-10, atol=1e-10 * np.abs(v).max())


def test_snap_production_batch_vs_oracle(pl):
    """220 x 129 atoms = 28,380 atoms (887 blocks of 32 atoms, > 148 SMs; 444 run CTAs =
    three full waves): the batch sizes of the bench, force sweep and ensemble, which
    dispatch the non-split Y kernel k_snap_yi_p<8,0,1> and the run force kernel
    (k_snap_deidrj_tm<8,8>, chosen when its waves are >= 84 % full) naturally.  Sampled systems vs the oracle (<= 1e-10), and
    each sampled system bitwise equal to its single-system evaluation (split Y
    kernel k_snap_yi_p<8,1,2> + 2-atom pair kernel): the batch never changes the
    arithmetic."""
    from oracle import native
    from paper_2212_10508_b200 import tungsten as W
    Q, box = _configs(4, 220, seed=11)
    n = Q.shape[1] // 3
    pot = W.make_snap(n, box)
    E, G, V = (x.cpu().numpy() for x in pot.evaluate(Q, True, True, True))
    sample = (0, 1, 109, 110, 218, 219)
    _snap_oracle_check(native, Q, box, pot, E, G, V, sample)
    for b in sample:
        e1, g1, v1 = (x.cpu().numpy() for x in pot.evaluate(Q[b:b + 1], True, True, True))
        assert e1[0].tobytes() == E[b].tobytes()
        assert g1[0].tobytes() == G[b].tobytes()
        assert v1[0].tobytes() == V[b].tobytes()


def test_snap_heavy_system_vs_oracle(pl):
    """Two 16,001-atom systems (BASELINE configs[4] cell; cell-list neighbours,
    32,002 atoms = four run-kernel waves at 84.5 % fill dispatch the run force kernel):
    system 0 vs the oracle <= 1e-10."""
    from oracle import native
    from paper_2212_10508_b200 import tungsten as W
    Q, box = _configs(20, 2, sigma=0.08, seed=13)
    n = Q.shape[1] // 3
    assert n == 16001
    pot = W.make_snap(n, box)
    E, G, V = (x.cpu().numpy() for x in pot.evaluate(Q, True, True, True))
    _snap_oracle_check(native, Q, box, pot, E, G, V, (0,))


_AB_SCRIPT = """
import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2212_10508_b200 import tungsten as W
q0, box = W.bcc_sia(4)
rs = np.random.default_rng(5)
import os
Q = torch.from_numpy(q0[None] + 0.1 * rs.normal(size=(int(os.environ.get('AB_BATCH', 6)), q0.shape[0]))).cuda()
E, G, V = (x.cpu().numpy() for x in W.make_snap(q0.shape[0] // 3, box).evaluate(Q, True, True, True))
np.savez(sys.argv[1], E=E, G=G, V=V)
"""


def test_snap_specialised_matches_general_kernels(pl, tmp_path):
    """twojmax-8 kernels (k_snap_ui_r4, box-form Y, pair-symmetric reverse-mode forces
    with 2-atom warps, 8-atom runs, or runs with the history in tensor memory) against the general-twojmax kernels (k_snap_ui,
    k_snap_yi, forward-mode k_snap_deidrj; PL_SNAP_GENERIC=1): energies, forces and
    virials to 1e-12; the two pair-kernel forms agree bit for bit."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = {}
    for mode, env_add in (("gen", {"PL_SNAP_GENERIC": "1"}),
                          ("pair", {"PL_SNAP_PAIR_RUN": "0", "PL_SNAP_TMEM": "0"}),   # k_snap_deidrj_pair
                          ("tm2", {"PL_SNAP_PAIR_RUN": "0", "PL_SNAP_TMEM": "1"}),    # k_snap_deidrj_tm<2>
                          ("run", {"PL_SNAP_PAIR_RUN": "2", "PL_SNAP_TMEM": "0"}),    # k_snap_deidrj_run<8>
                          ("tm", {"PL_SNAP_PAIR_RUN": "2", "PL_SNAP_TMEM": "1"}),     # k_snap_deidrj_tm<8, 8>
                          ("tm4", {"PL_SNAP_PAIR_RUN": "2", "PL_SNAP_TMEM": "1",      # k_snap_deidrj_tm<8, 4>
                                   "PL_SNAP_TM8": "0"})):
        f = str(tmp_path / f"ab_{mode}.npz")
        env = dict(os.environ, **env_add)
        subprocess.run([sys.executable, "-c", _AB_SCRIPT, f], cwd=root, env=env, check=True)
        out[mode] = np.load(f)
    a = out["gen"]
    for m in ("pair", "tm2", "run", "tm", "tm4"):
        b = out[m]
        np.testing.assert_allclose(b["E"], a["E"], rtol=1e-12)
        np.testing.assert_allclose(b["G"], a["G"], rtol=1e-12, atol=1e-12 * np.abs(a["G"]).max())
        np.testing.assert_allclose(b["V"], a["V"], rtol=1e-12, atol=1e-12 * np.abs(a["V"]).max())
    # the pair gather sums each pair once, in list order: runs and 2-atom warps agree bit for bit
    np.testing.assert_array_equal(out["pair"]["G"], out["run"]["G"])
    np.testing.assert_array_equal(out["pair"]["E"], out["run"]["E"])
    # history in tensor memory + staged Y_k^dagger: the same arithmetic, bit for bit
    np.testing.assert_array_equal(out["tm"]["G"], out["run"]["G"])
    np.testing.assert_array_equal(out["tm"]["V"], out["run"]["V"])
    np.testing.assert_array_equal(out["tm4"]["G"], out["run"]["G"])  # one 8-warp CTA per SM or two of 4
    np.testing.assert_array_equal(out["tm4"]["V"], out["run"]["V"])
    np.testing.assert_array_equal(out["tm2"]["G"], out["pair"]["G"])
    np.testing.assert_array_equal(out["tm2"]["V"], out["pair"]["V"])


def test_snap_fused_ydagger_store_is_bitwise_ytrans(pl, tmp_path):
    """At >= 148 blocks the unsplit Y kernel writes S (.) Y^dagger itself (no k_snap_ytrans
    launch); PL_YI_YT=0 keeps the separate kernel.  Same bits in E, forces and virials."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = {}
    for mode, env_add in (("fused", {}), ("separate", {"PL_YI_YT": "0"})):
        f = str(tmp_path / f"yt_{mode}.npz")
        env = dict(os.environ, AB_BATCH="40", **env_add)   # 5160 atoms = 162 blocks
        subprocess.run([sys.executable, "-c", _AB_SCRIPT, f], cwd=root, env=env, check=True)
        out[mode] = np.load(f)
    for k in ("E", "G", "V"):
        np.testing.assert_array_equal(out["fused"][k], out["separate"][k])


@pytest.mark.parametrize("twojmax", [2, 4, 6])
def test_snap_other_twojmax_vs_oracle(pl, twojmax):
    """General-twojmax kernels (paper Strategy I coarse SNAP-6 is twojmax 2) vs the oracle."""
    from oracle import native
    from paper_2212_10508_b200.potentials import SNAP
    from paper_2212_10508_b200 import tungsten as W
    Q, box = _configs(4, 3, seed=21)
    n = Q.shape[1] // 3
    nb = {2: 5, 4: 14, 6: 30}[twojmax]
    beta = np.concatenate([[0.1], 0.05 * np.random.default_rng(twojmax).normal(size=nb)])
    pot = SNAP(n_atoms=n, box=box, beta=beta, twojmax=twojmax)
    E, G, V = (x.cpu().numpy() for x in pot.evaluate(Q, True, True, True))
    _snap_oracle_check(native, Q, box, pot, E, G, V, range(3))


def test_snap_invariances_on_device(pl):
    """Sum F = 0, rotation invariance of E (cluster in a large box), FD gradient."""
    from paper_2212_10508_b200.potentials import SNAP
    from paper_2212_10508_b200 import tungsten as W
    rs = np.random.default_rng(7)
    X = rs.normal(size=(14, 3)) * 1.7
    big = (60.0, 60.0, 60.0)
    pot = SNAP(n_atoms=14, box=big, beta=W.snap_beta(11))
    th, ax = 1.1, np.array([3.0, -1.0, 2.0]) / np.sqrt(14.0)
    K = np.array([[0, -ax[2], ax[1]], [ax[2], 0, -ax[0]], [-ax[1], ax[0], 0]])
    R = np.eye(3) + np.sin(th) * K + (1 - np.cos(th)) * K @ K
    qa, qb = (X + 30).ravel(), (X @ R.T + 30).ravel()
    E, G, _ = pot.evaluate(np.stack([qa, qb]), True, True)
    E, G = E.cpu().numpy(), G.cpu().numpy()
    assert E[0] == pytest.approx(E[1], rel=1e-12)
    np.testing.assert_allclose(G[1].reshape(-1, 3), G[0].reshape(-1, 3) @ R.T, atol=1e-10)
    assert np.abs(G[0].reshape(-1, 3).sum(axis=0)).max() < 1e-10
    assert pl.gradient_check(pot, qa, h=1e-5) < 1e-6


def test_snap_deterministic_rerun(pl):
    from paper_2212_10508_b200 import tungsten as W
    Q, box = _configs(4, 8)
    pot = W.make_snap(Q.shape[1] // 3, box)
    a = pot.evaluate(Q)[1].cpu().numpy()
    b = pot.evaluate(Q)[1].cpu().numpy()
    assert a.tobytes() == b.tobytes()


@pytest.mark.parametrize("ncell,B", [(4, 150), (8, 24)])
def test_snap_repeated_evaluations_are_bitwise_stable(pl, ncell, B):
    """Race detector stand-in (compute-sanitizer is closed on this pool): ten
    evaluations of a production-size batch (150 x 129 atoms: non-split Y kernel,
    TMEM run force kernel; 24 x 1025 atoms: cell lists) interleaved with other
    batch shapes must give the same bits every time.  A missing barrier, a ring
    or staging buffer overwritten early, or a TMEM/mbarrier ordering bug would
    show up as run-to-run differences."""
    from paper_2212_10508_b200 import tungsten as W
    Q, box = _configs(ncell, B, seed=29)
    pot = W.make_snap(Q.shape[1] // 3, box)
    ref = [x.cpu().numpy().tobytes() for x in pot.evaluate(Q, True, True, True)]
    for r in range(9):
        pot.evaluate(Q[: 1 + r % 3], True, True, True)  # other shapes in between (buffers reused)
        out = [x.cpu().numpy().tobytes() for x in pot.evaluate(Q, True, True, True)]
        assert out == ref, f"repeat {r} differs"


def test_snap_window_vs_oracle(pl):
    """20 BBK substeps of SNAP W+SIA at 1000 K: device vs oracle integrator + C SNAP."""
    from oracle import integrator as oint, native, rng as orng
    from paper_2212_10508_b200 import tungsten as W
    q0, box = W.bcc_sia(4)
    n = q0.shape[0] // 3
    pot = W.make_snap(n, box)
    L = 20
    mass = np.full(3 * n, W.MASS_W)
    params = pl.LangevinParams(1.0, W.KB * 1000.0, 0.001, L, mass=mass)
    sched = pl.TemperatureSchedule.robust(L)
    p0 = W.maxwell_boltzmann(n, 1000.0, 11)
    seed = pl.derive_seed(11, 2)
    noise = orng.gaussian_stream(seed, (L + 1) * 3 * n)
    out = pl.propagate_windows([pl.PhaseState(q=q0, p=p0)], pot, params, sched, [seed],
                               noise=noise[None, :])[0]
    q1, p1 = oint.propagate_window(q0, p0, native.snap_fn(pot), 1.0, W.KB * 1000.0, 0.001, L,
                                   sched.coefficients, 0, mass=mass, noise=noise)
    assert np.abs(out.q - q1).max() < 1e-8
    assert np.abs(out.p - p1).max() < 1e-8 * np.abs(p1).max()


# ------------------------------------------------------------------ W + SIA parareal
def _w_pr1_setup(pl, L=5, N=4, T=1000.0):
    from paper_2212_10508_b200 import tungsten as W
    q0, box = W.bcc_sia(4)
    n = q0.shape[0] // 3
    mass = np.full(3 * n, W.MASS_W)
    params = pl.LangevinParams(1.0, W.KB * T, 0.001, L, mass=mass)
    sched = pl.TemperatureSchedule.robust(L)
    p0 = np.sqrt(W.MASS_W * W.KB * T) * np.random.default_rng(5).normal(size=3 * n)
    return q0, box, n, mass, params, sched, p0


def test_w_sia_adaptive_parareal_vs_oracle(pl):
    """SNAP fine / EAM coarse adaptive parareal (persistent EAM sweep) vs the oracle engine."""
    import torch
    from oracle import integrator as oint, native, parareal as opar, rng as orng
    from paper_2212_10508_b200 import tungsten as W
    from paper_2212_10508_b200.parareal import DevicePropagator
    L, N = 5, 4
    q0, box, n, mass, params, sched, p0 = _w_pr1_setup(pl, L, N)
    snap, eam = W.make_snap(n, box), W.make_eam(n, box)
    plan = pl.NoisePlan.for_windows(11, N)
    noise = orng.gaussian_streams(orng.derive_seeds(11, N), (L + 1) * 3 * n)
    f = DevicePropagator(snap, params, sched, plan, 3 * n)
    c = DevicePropagator(eam, params, sched, plan, 3 * n)
    for prop in (f, c):
        prop._noise = torch.from_numpy(noise).cuda()
    cfg = pl.PararealConfig(N, 1e-10, 0.35)
    res = pl.parareal_adaptive_engine(pl.PhaseState(q=q0, p=p0), f, c, cfg)
    t = W.eam_tables()
    sg, eg = native.snap_fn(snap), (lambda q: native.eam(q, box, t)[1])

    def mk(g):
        return lambda s, m: oint.propagate_window(s[0], s[1], g, 1.0, params.inv_beta, 0.001, L,
                                                  sched.coefficients, 0, mass=mass, noise=noise[m])
    ref = opar.adaptive((q0, p0), mk(sg), mk(eg), N, 1e-10, 0.35)
    Qr = np.array([s[0] for s in ref["trajectory"]])
    assert np.abs(res.trajectory.positions() - Qr).max() < 1e-8
    assert [(s.slab_index, s.n_init, s.n_final, s.k_conv) for s in res.slabs] == \
        [(s[0], s[1], s[3], s[4]) for s in ref["slabs"]]
    h = np.array(res.error_history)[:, 2]
    hr = np.array(ref["history"])[:, 2]
    assert h.shape == hr.shape
    big = hr > 1e-6
    np.testing.assert_allclose(h[big], hr[big], rtol=1e-6)


def test_persistent_sweep_matches_generic(pl, monkeypatch):
    """Persistent single-CTA sweep == per-window generic sweep (EAM coarse)."""
    import torch
    from paper_2212_10508_b200 import tungsten as W
    L, N = 10, 6
    q0, box, n, mass, params, sched, p0 = _w_pr1_setup(pl, L, N)
    pair = pl.PropagatorPair(W.make_eam(n, box), W.make_eam(n, box), 1.0, 1.0)
    fine_pert = pl.Perturbed(W.make_eam(n, box), W.make_snap(n, box), 0.1)
    pair = pl.PropagatorPair(fine_pert, W.make_eam(n, box), 10.0, 1.0)
    plan = pl.NoisePlan.for_windows(3, N)
    cfg = pl.PararealConfig(N, 1e-9, 0.35)
    init = pl.PhaseState(q=q0, p=p0)
    a = pl.parareal_adaptive(init, pair, params, sched, plan, cfg)
    monkeypatch.setenv("PL_SWEEP_GENERIC", "1")
    b = pl.parareal_adaptive(init, pair, params, sched, plan, cfg)
    assert a.slabs == b.slabs
    np.testing.assert_allclose(a.trajectory.positions(), b.trajectory.positions(), rtol=0, atol=1e-9)


def test_speculative_pipeline_is_bitwise_neutral(pl, monkeypatch):
    """Chunked sweep + speculative fine windows on a second stream (PL_PARAREAL_SPEC=1)
    give bit-for-bit the records and trajectory of the plain engine, and the
    speculative windows are actually used (fewer windows propagated in jumps)."""
    from paper_2212_10508_b200 import parareal as par, tungsten as W
    L, N = 10, 12
    q0, box, n, mass, params, sched, p0 = _w_pr1_setup(pl, L, N)
    pair = pl.PropagatorPair(W.make_snap(n, box), W.make_eam(n, box), 100.0, 1.0)
    plan = pl.NoisePlan.for_windows(13, N)
    cfg = pl.PararealConfig(N, 1e-10, 0.35)
    init = pl.PhaseState(q=q0, p=p0)
    monkeypatch.setenv("PL_PARAREAL_SPEC", "0")
    a = pl.parareal_adaptive(init, pair, params, sched, plan, cfg)
    plain = dict(par.LAST_RUN_STATS)
    monkeypatch.setenv("PL_PARAREAL_SPEC", "1")
    b = pl.parareal_adaptive(init, pair, params, sched, plan, cfg)
    spec = dict(par.LAST_RUN_STATS)
    assert a.slabs == b.slabs
    assert a.error_history == b.error_history
    assert a.trajectory.positions().tobytes() == b.trajectory.positions().tobytes()
    assert a.trajectory.momenta().tobytes() == b.trajectory.momenta().tobytes()
    assert not plain["speculation"] and spec["speculation"] and spec["speculative_windows"] > 0
    assert spec["fine_windows_propagated"] < plain["fine_windows_propagated"]


@pytest.mark.parametrize("ncell", [4, 8])
def test_cluster_sweep_thread_count_is_bitwise_neutral(pl, monkeypatch, ncell):
    """The cluster sweep runs only the threads its atoms use; with the full
    1024-thread CTAs (PL_SWEEP_FULL=1) every node, slab record and error value is
    the same bit for bit (129 atoms: 8 CTAs x 17 atoms; 1025 atoms: 16 x 65)."""
    from paper_2212_10508_b200 import tungsten as W
    q0, box = W.bcc_sia(ncell)
    n = q0.shape[0] // 3
    L, N = 10, 6
    params = pl.LangevinParams(1.0, W.KB * 1000.0, 0.001, L, mass=np.full(3 * n, W.MASS_W))
    sched = pl.TemperatureSchedule.robust(L)
    init = pl.PhaseState(q=q0, p=W.maxwell_boltzmann(n, 1000.0, 3))
    pair = pl.PropagatorPair(W.make_snap(n, box), W.make_eam(n, box), 100.0, 1.0)
    plan = pl.NoisePlan.for_windows(17, N)
    cfg = pl.PararealConfig(N, 1e-10, 0.35)
    a = pl.parareal_adaptive(init, pair, params, sched, plan, cfg)
    monkeypatch.setenv("PL_SWEEP_FULL", "1")
    b = pl.parareal_adaptive(init, pair, params, sched, plan, cfg)
    assert a.slabs == b.slabs and a.error_history == b.error_history
    assert a.trajectory.positions().tobytes() == b.trajectory.positions().tobytes()


def test_degenerate_pair_converges_in_one_iteration(pl):
    """coarse == fine: jumps are exactly zero, k_conv = 1 (acceptance criterion 5)."""
    from paper_2212_10508_b200 import tungsten as W
    L, N = 5, 5
    q0, box, n, mass, params, sched, p0 = _w_pr1_setup(pl, L, N)
    eam = W.make_eam(n, box)
    pair = pl.PropagatorPair(eam, eam, 1.0, 1.0)
    plan = pl.NoisePlan.for_windows(7, N)
    res = pl.parareal_adaptive(pl.PhaseState(q=q0, p=p0), pair, params, sched, plan,
                               pl.PararealConfig(N, 1e-10, 0.35))
    assert res.converged and res.n_slab == 1 and res.total_iterations == 1
    # batched EAM (fine) and the persistent sweep (coarse) are bitwise identical:
    # every jump is exactly zero, so the error history is exactly zero
    assert all(e == 0.0 for _, _, e in res.error_history)


@pytest.mark.parametrize("rcut_kind", ["snap", "eam"])
def test_cell_list_matches_brute_force(pl, rcut_kind):
    """4395 atoms (>= CELL_MIN_ATOMS): cell-list lists == oracle brute force, bit for bit."""
    from oracle import native
    from paper_2212_10508_b200 import tungsten as W
    Q, box = _configs(13, 2, sigma=0.08)
    n = Q.shape[1] // 3
    pot = W.make_snap(n, box) if rcut_kind == "snap" else W.make_eam(n, box)
    rc = 4.73 if rcut_kind == "snap" else 5.5
    dev = _device_neighbours(pl, pot, Q)
    for b in range(Q.shape[0]):
        assert dev[b] == native.neighbours(Q[b], box, rc)


def test_batched_replicas_equal_single_runs_snap_eam(pl):
    """Replica batch (SNAP fine / EAM coarse) == single runs, bit for bit."""
    from paper_2212_10508_b200 import tungsten as W
    L, N = 5, 4
    q0, box, n, mass, params, sched, p0 = _w_pr1_setup(pl, L, N)
    pair = pl.PropagatorPair(W.make_snap(n, box), W.make_eam(n, box), 100.0, 1.0)
    cfg = pl.PararealConfig(N, 1e-10, 0.35)
    rs = np.random.default_rng(3)
    inits = [pl.PhaseState(q=q0 + 0.02 * rs.normal(size=q0.shape), p=p0) for _ in range(3)]
    plans = [pl.NoisePlan.for_windows(pl.derive_seed(5, 10**9 + i), N) for i in range(3)]
    batch = pl.parareal_adaptive_batch(inits, pair, params, sched, plans, cfg)
    for i in range(3):
        one = pl.parareal_adaptive(inits[i], pair, params, sched, plans[i], cfg)
        assert one.slabs == batch[i].slabs
        assert one.error_history == batch[i].error_history
        assert one.trajectory.positions().tobytes() == batch[i].trajectory.positions().tobytes()


def test_sia_site_labels(pl):
    """Wigner-Seitz SIA site: dumbbell site found, moves with a lattice translation, PBC-invariant."""
    from paper_2212_10508_b200 import sia, tungsten as W
    n = 4
    q0, box = W.bcc_sia(n)
    a = W.A0
    # the removed host site of bcc_sia is the site nearest (n/2, n/2, n/2) a
    lab = sia.sia_site_labels(q0[None, :], n, a)[0]
    c = n // 2
    host = n ** 3 + ((c % n) * n + (c % n)) * n + (c % n) if False else None
    X = q0.reshape(-1, 3)
    mid = X[-2:].mean(axis=0)  # dumbbell centre = host site
    u = mid / a
    if np.allclose(u, np.round(u)):
        i, j, k = (np.round(u).astype(int) % n)
        host = (i * n + j) * n + k
    else:
        i, j, k = (np.floor(u).astype(int) % n)
        host = n ** 3 + (i * n + j) * n + k
    assert lab == host
    # unwrapped copy (+ box) and a whole-lattice translation by one cubic cell
    shifted = (X + np.array(box)).ravel()
    moved = (X + np.array([a, 0.0, 0.0])).ravel()
    labs = sia.sia_site_labels(np.stack([q0, shifted, moved]), n, a)
    i2 = ((lab // n ** 2 % n) + 1) % n if lab < n ** 3 else None
    assert labs[0] == labs[1] == lab
    assert labs[2] != lab


def test_heavy_system_sweeps_batch_equals_single(pl):
    """16,001 atoms (BASELINE configs[4] cell): too large for the persistent sweeps, the
    coarse sweep runs the per-window device path; replica batches (pl_sweep_batch) equal
    single runs bit for bit, and a degenerate EAM/EAM pair converges in one iteration
    with exactly zero jumps."""
    from paper_2212_10508_b200 import tungsten as W
    q0, box = W.bcc_sia(20)
    n = q0.shape[0] // 3
    L, N = 2, 3
    params = pl.LangevinParams(1.0, W.KB * 1000.0, 0.001, L, mass=np.full(3 * n, W.MASS_W))
    sched = pl.TemperatureSchedule.robust(L)
    eam = W.make_eam(n, box)
    inits = [pl.PhaseState(q=q0, p=W.maxwell_boltzmann(n, 1000.0, s)) for s in (1, 2)]
    plans = [pl.NoisePlan.for_windows(pl.derive_seed(9, i + 1), N) for i in range(2)]
    cfg = pl.PararealConfig(N, 1e-10, 0.35)
    deg = pl.parareal_adaptive_batch(inits, pl.PropagatorPair(eam, eam, 1.0, 1.0), params, sched, plans, cfg)
    for r in deg:
        assert r.converged and r.total_iterations == 1
        assert all(e == 0.0 for _, _, e in r.error_history)
    pair = pl.PropagatorPair(W.make_snap(n, box), eam, 100.0, 1.0)
    batch = pl.parareal_adaptive_batch(inits, pair, params, sched, plans, cfg)
    for i in range(2):
        one = pl.parareal_adaptive(inits[i], pair, params, sched, plans[i], cfg)
        assert one.slabs == batch[i].slabs
        assert one.error_history == batch[i].error_history
        assert one.trajectory.positions().tobytes() == batch[i].trajectory.positions().tobytes()


@pytest.mark.parametrize("kind", ["eam", "snap"])
def test_many_body_blow_up_substep_matches_oracle(pl, kind):
    """The fused close kernels' trusted-range check on a many-body potential
    (integrator.py:163-170): one atom placed beyond 1e12 A fails the check at the
    first substep in the oracle's restatement of the reference window and on the
    device (batched with a healthy window, in either order)."""
    from oracle import integrator as oint, native, rng as orng
    from paper_2212_10508_b200 import tungsten as W
    L = 4
    q_ok, box, n, mass, params, sched, _ = _w_pr1_setup(pl, L, 1)
    q0 = q_ok.copy()
    q0[0] = 2e12
    p0 = np.zeros_like(q0)
    pot = W.make_eam(n, box) if kind == "eam" else W.make_snap(n, box)
    seed = pl.derive_seed(3, 1)
    noise = orng.gaussian_stream(seed, (L + 1) * 3 * n)
    grad = (lambda q: native.eam(q, box, W.eam_tables())[1]) if kind == "eam" else native.snap_fn(pot)
    with pytest.raises(oint.OracleBlowUp) as oe:
        oint.propagate_window(q0, p0, grad, params.gamma, params.inv_beta, params.dt, L, sched.coefficients, 0,
                              mass=mass, noise=noise)
    assert oe.value.substep == 1
    good, bad = pl.PhaseState(q=q_ok, p=np.zeros_like(q0)), pl.PhaseState(q=q0, p=p0)
    for states in ([good, bad], [bad, good]):
        with pytest.raises(pl.BlowUpError) as ei:
            pl.propagate_windows(states, pot, params, sched, [seed, seed], noise=np.stack([noise, noise]))
        assert ei.value.substep == oe.value.substep


@pytest.mark.parametrize("ncell,W", [(4, 3), (8, 2)])
def test_verlet_skin_lists_are_bitwise_neutral(pl, monkeypatch, ncell, W):
    """SNAP windows keep Verlet-skin neighbour lists (rcut + 0.3 A, rebuilt on the
    device when an atom moved more than half the skin); every SNAP kernel compacts
    the exact pairs in list order, so trajectories equal the exact-list ones bit for
    bit (PL_SNAP_SKIN=0), for brute-force (129 atoms) and cell lists (1025 atoms)."""
    from paper_2212_10508_b200 import tungsten as W_
    q0, box = W_.bcc_sia(ncell)
    n = q0.shape[0] // 3
    L = 40
    params = pl.LangevinParams(1.0, W_.KB * 1500.0, 0.001, L, mass=np.full(3 * n, W_.MASS_W))
    sched = pl.TemperatureSchedule.robust(L)
    states = [pl.PhaseState(q=q0, p=W_.maxwell_boltzmann(n, 1500.0, s)) for s in range(1, W + 1)]
    seeds = [pl.derive_seed(21, s) for s in range(1, W + 1)]
    out = {}
    for skin in ("0", "0.3"):
        monkeypatch.setenv("PL_SNAP_SKIN", skin)
        pot = W_.make_snap(n, box)
        out[skin] = pl.propagate_windows(states, pot, params, sched, seeds)
    for a, b in zip(out["0"], out["0.3"]):
        assert a.q.tobytes() == b.q.tobytes()
        assert a.p.tobytes() == b.p.tobytes()
