"""Pin the CPU oracle against golden vectors produced by the reference itself.

The fixtures in tests/golden/ were produced by scripts/make_golden.py, which
imports /root/reference/pkg/src/paralangevin read-only.  Every comparison here
is bitwise (``tobytes`` / ``array_equal``), except where noted.
"""

import numpy as np
import pytest

from oracle import integrator as oint
from oracle import parareal as opar
from oracle import rng as orng
from oracle import toy


def test_derive_seed_known_answers(golden):
    z = golden("rng_golden.npz")
    for i, m in enumerate(z["masters"]):
        for j, n in enumerate(z["ns"]):
            assert orng.derive_seed(int(m), int(n)) == int(z["seeds"][i, j])
    # SURVEY.md Appendix A
    assert orng.derive_seed(0, 1) == 0xE220A8397B1DCDAF
    assert orng.derive_seed(11, 1) == 0xAEAF52FEBE706064
    seeds = orng.derive_seeds(11, 5)
    assert [int(s) for s in seeds] == [orng.derive_seed(11, n) for n in range(1, 6)]


def test_uniforms_known_answers(golden):
    z = golden("rng_golden.npz")
    u = orng.uniforms(int(z["unif_seed"]), 0, 64)
    assert u.tobytes() == z["unif"].tobytes()
    assert u[:4].tolist() == [0.8966974976375901, 0.08945914244836006,
                              0.10994182492417715, 0.12251322416769694]


def test_gaussian_streams_bitwise(golden):
    z = golden("rng_golden.npz")
    for c in z["counts"]:
        for i, sd in enumerate(z["stream_seeds"]):
            ref = z[f"stream_c{int(c)}_s{i}"]
            got = orng.gaussian_stream(int(sd), int(c))
            assert got.tobytes() == ref.tobytes(), (c, i)
    got = orng.gaussian_streams(z["batch_seeds"], 387)
    assert got.tobytes() == z["batch_c387"].tobytes()


def test_gaussian_known_answers():
    s = orng.derive_seed(11, 1)
    want = [-1.119631577941788, 0.21533440370020615, -1.3428654143366536,
            1.7490062375691953, 0.49776881118104765, 1.144446641366192]
    assert orng.gaussian_stream(s, 6).tolist() == want
    assert orng.gaussian_stream(s, 16)[:6].tolist() == want


def _grad_for(name, z):
    if name == "dw1":
        return toy.double_well(1.0, 1.0)
    if name == "dw5":
        return toy.double_well(np.array([1.0, 0.5, 2.0, 1.5, 0.8]),
                               np.array([1.0, 2.0, 0.5, 1.0, 1.5]))
    if name == "harm4":
        return toy.harmonic(np.array([1.0, 3.0, 0.5, 2.0]))
    if name == "lj7":
        return toy.lj(1.0, 1.0, 7, 2)
    if name == "lj13":
        return toy.lj(1.0, 1.0, 13, 3)
    raise KeyError(name)


@pytest.mark.parametrize("name", ["dw1", "dw5", "harm4", "lj7", "lj13"])
def test_window_bitwise(golden, name):
    z = golden("window_golden.npz")
    gamma, inv_beta, dt, L = z[f"{name}_meta"]
    mass = z[f"{name}_mass"] if f"{name}_mass" in z else None
    q, p = oint.propagate_window(z[f"{name}_q0"], z[f"{name}_p0"], _grad_for(name, z),
                                 gamma, inv_beta, dt, int(L), tuple(z[f"{name}_sched"]),
                                 int(z[f"{name}_seed"]), mass=mass)
    assert q.tobytes() == z[f"{name}_q1"].tobytes()
    assert p.tobytes() == z[f"{name}_p1"].tobytes()
    # the injected-noise path is the same computation
    q2, p2 = oint.propagate_window(z[f"{name}_q0"], z[f"{name}_p0"], _grad_for(name, z),
                                   gamma, inv_beta, dt, int(L), tuple(z[f"{name}_sched"]),
                                   0, mass=mass, noise=z[f"{name}_noise"])
    assert q2.tobytes() == q.tobytes() and p2.tobytes() == p.tobytes()


def test_window_appendix_a():
    q, p = oint.propagate_window([-1.0], [0.0], toy.double_well(1.0, 1.0), 0.5, 0.4, 0.05, 2,
                                 oint.robust(2), orng.derive_seed(11, 1))
    assert q[0] == -1.0118800384813031 and p[0] == -0.19175494361365208


def _dw_props(cfg):
    gamma, inv_beta, dt, L, seed, n = cfg[:6]
    seeds = orng.derive_seeds(int(seed), int(n))
    sched = oint.robust(int(L))

    def make(a):
        g = toy.double_well(a, 1.0)

        def prop(state, m):
            return oint.propagate_window(state[0], state[1], g, gamma, inv_beta, dt, int(L),
                                         sched, int(seeds[m]))
        return prop
    return make(1.0), make(0.8)


def _check_result(res, z, prefix):
    Q = np.array([s[0] for s in res["trajectory"]])
    P = np.array([s[1] for s in res["trajectory"]])
    assert Q.tobytes() == z[f"{prefix}_Q"].tobytes()
    assert P.tobytes() == z[f"{prefix}_P"].tobytes()
    hist = np.array(res["history"], float)
    assert hist.tobytes() == z[f"{prefix}_hist"].tobytes()
    rows = [[s[0], s[1], s[3], s[4], a[0], a[1]] for s in res["slabs"] for a in s[2]]
    assert np.array_equal(np.array(rows, dtype=np.int64), z[f"{prefix}_slabs"])
    assert bool(res["converged"]) == bool(z[f"{prefix}_converged"])


def test_adaptive_engine_config(golden):
    z = golden("parareal_golden.npz")
    cfg = z["adaptive_cfg"]
    fine, coarse = _dw_props(cfg)
    init = (np.array([-1.0]), np.zeros(1))
    res = opar.adaptive(init, fine, coarse, int(cfg[5]), cfg[6], cfg[7])
    _check_result(res, z, "adaptive")
    # N_slab 4, sum k 92
    assert len(res["slabs"]) == 4 and sum(s[4] for s in res["slabs"]) == 92


def test_classic_engine_config(golden):
    z = golden("parareal_golden.npz")
    cfg = z["parareal_cfg"]
    fine, coarse = _dw_props(cfg)
    res = opar.classic((np.array([-1.0]), np.zeros(1)), fine, coarse, int(cfg[5]), cfg[6])
    _check_result(res, z, "parareal")
    assert res["slabs"][0][4] == 13


def test_sequential_config(golden):
    z = golden("parareal_golden.npz")
    fine, _ = _dw_props(np.array([0.5, 0.4, 0.05, 2, 11, 500]))
    states = opar.sequential((np.array([-1.0]), np.zeros(1)), fine, 500)
    assert np.array([s[0] for s in states]).tobytes() == z["sequential_Q"].tobytes()
    assert np.array([s[1] for s in states]).tobytes() == z["sequential_P"].tobytes()


def test_lj13_adaptive(golden):
    z = golden("parareal_golden.npz")
    lj = toy.lj(1.0, 1.0, 13, 3)
    coarse_g = toy.perturbed(lj, toy.harmonic(1.0), 0.05)
    seeds = orng.derive_seeds(5, 24)
    sched = oint.robust(10)

    def mk(g):
        return lambda s, m: oint.propagate_window(s[0], s[1], g, 1.0, 0.2, 0.002, 10, sched,
                                                  int(seeds[m]))
    res = opar.adaptive((z["lj13_q0"], np.zeros(39)), mk(lj), mk(coarse_g), 24, 1e-10, 0.05)
    _check_result(res, z, "lj13")
