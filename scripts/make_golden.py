"""Generate tests/golden/*.npz by running the REFERENCE package itself.

Run in the build container only (the GPU box has no /root/reference):

    python scripts/make_golden.py

Imports /root/reference/pkg/src/paralangevin read-only and freezes:
  rng_golden.npz       derive_seed(s), uniforms, gaussian_stream(s) on both
                       the scalar (<16) and batched code paths
  window_golden.npz    propagate_window on DoubleWell / Harmonic(+mass) /
                       LJ7-2D / LJ13-3D, robust and identity schedules, with
                       the exact noise block each window consumed
  parareal_golden.npz  parareal_adaptive on configs/adaptive.json (N=800, L=2),
                       parareal_classic on configs/parareal.json (N=100),
                       sequential_propagate on configs/sequential.json, and a
                       small LJ13-3D adaptive run (fine LJ, coarse Perturbed)
numpy / OpenBLAS versions are recorded in each file (the batched Gaussian
path uses numpy's SIMD log, so absolute variates depend on the host build).
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
import paralangevin as pl  # noqa: E402
from paralangevin import rng as prng  # noqa: E402

OUT = os.path.join(os.path.dirname(__file__), "..", "tests", "golden")
CFG = "/root/reference/pkg/configs"


def _versions():
    import scipy
    return dict(numpy=np.__version__, scipy=scipy.__version__)


def make_rng():
    masters = np.array([0, 1, 11, 77, 2**64 - 1, 0x123456789ABCDEF], dtype=np.uint64)
    ns = np.array([1, 2, 3, 16, 1000, 10**9], dtype=np.int64)
    seeds = np.array([[pl.derive_seed(int(m), int(n)) for n in ns] for m in masters],
                     dtype=np.uint64)
    s = pl.derive_seed(11, 1)
    unif = np.array([prng._uniform(s, j) for j in range(64)])
    counts = [1, 2, 5, 15, 16, 17, 33, 100, 1001, 39087]
    stream_seeds = [pl.derive_seed(11, n) for n in (1, 2, 3)] + [0, 2**64 - 1]
    streams = {}
    for c in counts:
        for i, sd in enumerate(stream_seeds):
            streams[f"stream_c{c}_s{i}"] = pl.gaussian_stream(sd, c)
    batch_seeds = pl.derive_seeds(5, 7)
    streams["batch_c387"] = pl.gaussian_streams(batch_seeds, 387)
    np.savez_compressed(
        os.path.join(OUT, "rng_golden.npz"),
        masters=masters, ns=ns, seeds=seeds, unif_seed=np.uint64(s), unif=unif,
        stream_seeds=np.array(stream_seeds, dtype=np.uint64), counts=np.array(counts),
        batch_seeds=batch_seeds, versions=json.dumps(_versions()), **streams,
    )


def _window_case(name, pot, params, sched, q0, p0, seed, out):
    st = pl.PhaseState(q=q0, p=p0)
    end = pl.propagate_window(st, pot, params, sched, seed)
    d = st.dim
    noise = pl.gaussian_stream(seed, (params.substeps + 1) * d)
    out[f"{name}_q0"] = np.asarray(q0, float)
    out[f"{name}_p0"] = np.asarray(p0, float)
    out[f"{name}_q1"] = end.q
    out[f"{name}_p1"] = end.p
    out[f"{name}_noise"] = noise
    out[f"{name}_meta"] = np.array([params.gamma, params.inv_beta, params.dt,
                                    params.substeps], dtype=float)
    out[f"{name}_seed"] = np.uint64(seed)
    out[f"{name}_sched"] = np.array(sched.coefficients)
    if params.mass is not None:
        out[f"{name}_mass"] = params.mass


def make_window():
    out = {}
    rs = np.random.default_rng(1234)
    # Appendix A pin: DW 1-D, adaptive.json params
    _window_case("dw1", pl.DoubleWell(1.0, 1.0), pl.LangevinParams(0.5, 0.4, 0.05, 2),
                 pl.TemperatureSchedule.robust(2), [-1.0], [0.0], pl.derive_seed(11, 1), out)
    # DW 5-D vector coefficients, long window, identity schedule
    a = np.array([1.0, 0.5, 2.0, 1.5, 0.8]); b = np.array([1.0, 2.0, 0.5, 1.0, 1.5])
    _window_case("dw5", pl.DoubleWell(a, b), pl.LangevinParams(0.7, 0.3, 0.02, 37),
                 pl.TemperatureSchedule.identity(37), rs.normal(size=5), rs.normal(size=5),
                 pl.derive_seed(3, 7), out)
    # Harmonic with mass vector
    mass = np.array([1.0, 2.5, 0.5, 4.0])
    _window_case("harm4", pl.Harmonic(k=np.array([1.0, 3.0, 0.5, 2.0])),
                 pl.LangevinParams(1.0, 0.5, 0.05, 10, mass=mass),
                 pl.TemperatureSchedule.robust(10), rs.normal(size=4), rs.normal(size=4),
                 pl.derive_seed(9, 2), out)
    # LJ7 2-D
    lj7 = pl.LennardJonesCluster(1.0, 1.0, 7, 2)
    ang = np.linspace(0, 2 * np.pi, 7, endpoint=False)
    q7 = np.concatenate([[0.0, 0.0]] + [[1.12 * np.cos(t), 1.12 * np.sin(t)] for t in ang[:6]])
    _window_case("lj7", lj7, pl.LangevinParams(1.0, 0.1, 0.005, 20),
                 pl.TemperatureSchedule.robust(20), q7, np.zeros(14), pl.derive_seed(11, 4), out)
    # LJ13 3-D (icosahedron-ish start from jittered cubic positions)
    g = np.array([[i, j, k] for i in range(3) for j in range(3) for k in range(2)], float)[:13]
    q13 = (g * 1.12 + 0.01 * rs.normal(size=g.shape)).reshape(-1)
    _window_case("lj13", pl.LennardJonesCluster(1.0, 1.0, 13, 3),
                 pl.LangevinParams(1.0, 0.2, 0.002, 25), pl.TemperatureSchedule.robust(25),
                 q13, 0.1 * rs.normal(size=39), pl.derive_seed(21, 5), out)
    np.savez_compressed(os.path.join(OUT, "window_golden.npz"),
                        versions=json.dumps(_versions()), **out)


def _res_arrays(prefix, res, out):
    traj = res.trajectory
    out[f"{prefix}_Q"] = traj.positions()
    out[f"{prefix}_P"] = traj.momenta()
    out[f"{prefix}_hist"] = np.array([[s, k, e] for s, k, e in res.error_history], float)
    slabs = []
    for sl in res.slabs:
        for a in sl.attempts:
            slabs.append([sl.slab_index, sl.n_init, sl.n_final, sl.k_conv, a.n_final, a.iterations])
    out[f"{prefix}_slabs"] = np.array(slabs, dtype=np.int64)
    out[f"{prefix}_converged"] = np.array(res.converged)


def _cfg_pair(cfg):
    from paralangevin.cli import validate_config
    return validate_config(cfg)


def make_parareal():
    out = {}
    for name in ("adaptive", "parareal", "sequential"):
        with open(os.path.join(CFG, f"{name}.json")) as fh:
            raw = json.load(fh)
        p = raw["params"]
        params = pl.LangevinParams(p["gamma"], p["inv_beta"], p["dt"], p["substeps"])
        sched = pl.TemperatureSchedule.robust(p["substeps"])
        fine = pl.DoubleWell(**{k: v for k, v in raw["potential"]["fine"].items() if k != "kind"})
        n = raw["parareal"]["n_windows"]
        plan = pl.NoisePlan.for_windows(raw["master_seed"], n)
        init = pl.PhaseState(q=np.array(raw["initial"]["q"]), p=np.zeros(1))
        if name == "sequential":
            traj = pl.sequential_propagate(init, n, fine, params, sched, plan)
            out["sequential_Q"] = traj.positions()
            out["sequential_P"] = traj.momenta()
            continue
        coarse = pl.DoubleWell(**{k: v for k, v in raw["potential"]["coarse"].items() if k != "kind"})
        pair = pl.PropagatorPair(fine, coarse, 175.0, 1.0)
        pr = raw["parareal"]
        cfg = pl.PararealConfig(n, pr["delta_conv"], pr.get("delta_expl"))
        if name == "adaptive":
            res = pl.parareal_adaptive(init, pair, params, sched, plan, cfg)
        else:
            res = pl.parareal_classic(init, pair, params, sched, plan, cfg)
        _res_arrays(name, res, out)
        out[f"{name}_cfg"] = np.array([params.gamma, params.inv_beta, params.dt, params.substeps,
                                       raw["master_seed"], n, pr["delta_conv"],
                                       pr.get("delta_expl") or 0.0])
    # LJ13 3-D adaptive: fine LJ, coarse Perturbed(LJ, Harmonic, lam)
    rs = np.random.default_rng(99)
    g = np.array([[i, j, k] for i in range(3) for j in range(3) for k in range(2)], float)[:13]
    q13 = (g * 1.12 + 0.01 * rs.normal(size=g.shape)).reshape(-1)
    lj = pl.LennardJonesCluster(1.0, 1.0, 13, 3)
    coarse = pl.Perturbed(base=lj, delta=pl.Harmonic(k=1.0), lam=0.05)
    params = pl.LangevinParams(1.0, 0.2, 0.002, 10)
    sched = pl.TemperatureSchedule.robust(10)
    n = 24
    plan = pl.NoisePlan.for_windows(5, n)
    cfg = pl.PararealConfig(n, 1e-10, 0.05)
    res = pl.parareal_adaptive(pl.PhaseState(q=q13, p=np.zeros(39)),
                               pl.PropagatorPair(lj, coarse, 10.0, 1.0), params, sched, plan, cfg)
    _res_arrays("lj13", res, out)
    out["lj13_q0"] = q13
    np.savez_compressed(os.path.join(OUT, "parareal_golden.npz"),
                        versions=json.dumps(_versions()), **out)


def make_residence():
    from paralangevin import analysis as an
    rs = np.random.default_rng(42)
    labels = np.repeat(rs.integers(0, 4, size=60), rs.integers(1, 7, size=60))
    out = {"labels": labels}
    for mr in (1, 3):
        ev = an.residence_times(labels, min_run=mr)
        out[f"events_{mr}"] = np.array([[e.basin, e.duration, int(e.censored)] for e in ev], dtype=np.int64)
        done = [e.duration for e in ev if not e.censored]
        out[f"ci_{mr}"] = np.array(an.mean_ci(done))
    np.savez_compressed(os.path.join(OUT, "residence_golden.npz"), versions=json.dumps(_versions()), **out)


def make_accounting():
    """classic_gain / adaptive_gain on hand-built slab records (accounting.py:99-159)."""
    from paralangevin import accounting as acc
    from paralangevin.parareal import SlabAttempt, SlabRecord
    slabsets = [
        [SlabRecord(1, 0, (SlabAttempt(16, 3),), 16, 3)],
        [SlabRecord(1, 0, (SlabAttempt(16, 2), SlabAttempt(9, 4)), 9, 6),
         SlabRecord(2, 9, (SlabAttempt(16, 5),), 16, 5)],
        [SlabRecord(1, 0, (SlabAttempt(64, 1), SlabAttempt(20, 3)), 20, 4),
         SlabRecord(2, 20, (SlabAttempt(41, 7),), 41, 7),
         SlabRecord(3, 41, (SlabAttempt(64, 2), SlabAttempt(63, 1), SlabAttempt(50, 9)), 50, 12),
         SlabRecord(4, 50, (SlabAttempt(64, 3),), 64, 3)],
    ]
    costs = [(1.0, 0.0), (100.0, 1.0), (37.5, 0.8125), (1.0, 1.0)]
    rows_a, rows_c = [], []
    for si, slabs in enumerate(slabsets):
        n = slabs[-1].n_final
        for cf, cc in costs:
            r = acc.adaptive_gain(slabs, n, cf, cc)
            rows_a.append([si, cf, cc, r.total_cost, r.sequential_cost, r.gain, r.ideal_gain, r.n_slab,
                           r.total_iterations])
    for n, k in ((16, 3), (100, 7), (64, 64)):
        for cf, cc in costs:
            r = acc.classic_gain(n, k, cf, cc)
            rows_c.append([n, k, cf, cc, r.total_cost, r.sequential_cost, r.gain, r.ideal_gain, r.total_effort])
    enc = [[(s.slab_index, s.n_init, s.n_final, s.k_conv, [(a.n_final, a.iterations) for a in s.attempts])
            for s in slabs] for slabs in slabsets]
    np.savez_compressed(os.path.join(OUT, "accounting_golden.npz"), versions=json.dumps(_versions()),
                        slabsets=json.dumps(enc), adaptive=np.array(rows_a), classic=np.array(rows_c))


def make_temperature():
    """measure_kinetic_temperature (integrator.py:430-482) on small systems."""
    from paralangevin import integrator as integ
    out = {}
    cases = {
        "harm": (pl.Harmonic(k=np.array([1.0, 3.0, 0.5])), pl.LangevinParams(1.0, 0.7, 0.05, 5, mass=[1.0, 2.0, 0.5]),
                 40, 123),
        "dw": (pl.DoubleWell(1.0, 1.0), pl.LangevinParams(0.5, 0.4, 0.05, 3), 60, 7),
        "lj7": (pl.LennardJonesCluster(1.0, 1.0, 7, 2), pl.LangevinParams(1.0, 0.3, 0.005, 4, mass=[1.0] * 14),
                25, 99),
    }
    for name, (pot, params, nw, seed) in cases.items():
        sched = pl.TemperatureSchedule.robust(params.substeps)
        for sampling in (integ.ALL_SUBSTEPS, integ.WINDOW_ENDS):
            if name == "lj7":
                # a cold LJ start has coincident atoms: chain from the reference's own minimiser output
                continue
            r = integ.measure_kinetic_temperature(pot, params, sched, nw, seed, sampling=sampling, burn_in=0.2)
            out[f"{name}_{sampling}"] = np.array([r.k_eq_empirical, r.k_eq_predicted, r.n_windows, r.n_burn_in]
                                                 + list(r.per_substep_variance))
    np.savez_compressed(os.path.join(OUT, "temperature_golden.npz"), versions=json.dumps(_versions()), **out)


def make_minima():
    """local_minima (potentials.py:268-287): double well, harmonic and LJ7-2D starts."""
    from paralangevin import potentials as pots
    rs = np.random.default_rng(5)
    out = {}
    dw = pl.DoubleWell(1.0, 1.0)
    starts = [np.array([x]) for x in (-1.7, -0.3, 0.2, 0.9, 2.5, -1.0)]
    out["dw_starts"] = np.stack(starts)
    out["dw_minima"] = np.stack(pots.local_minima(dw, starts, tol=1e-9))
    lj = pl.LennardJonesCluster(1.0, 1.0, 7, 2)
    base = np.array([[0.0, 0.0], [1.12, 0.0], [0.56, 0.97], [-0.56, 0.97], [-1.12, 0.0], [-0.56, -0.97],
                     [0.56, -0.97]]).ravel()
    ljs = [base + 0.05 * rs.normal(size=base.shape) for _ in range(4)]
    out["lj_starts"] = np.stack(ljs)
    out["lj_minima"] = np.stack(pots.local_minima(lj, ljs, tol=1e-6))
    out["lj_energy"] = np.array([lj.energy(m) for m in out["lj_minima"]])
    np.savez_compressed(os.path.join(OUT, "minima_golden.npz"), versions=json.dumps(_versions()), **out)


def make_reports():
    """The reference's own report files (cli._run_parareal: trajectory.csv,
    history.csv, result.json) for configs/adaptive.json and configs/parareal.json."""
    import tempfile
    from paralangevin import cli
    out = {}
    for name in ("adaptive", "parareal"):
        cfg = cli.validate_config(os.path.join(CFG, f"{name}.json"))
        with tempfile.TemporaryDirectory() as tmp:
            outputs = []
            cli._run_parareal(cfg, __import__("pathlib").Path(tmp), 1, outputs)
            for f in ("trajectory.csv", "history.csv", "result.json"):
                out[f"{name}_{f.replace('.', '_')}"] = np.array(open(os.path.join(tmp, f)).read())
    np.savez_compressed(os.path.join(OUT, "reports_golden.npz"), versions=json.dumps(_versions()), **out)


if __name__ == "__main__":
    os.makedirs(OUT, exist_ok=True)
    which = sys.argv[1:] or ["rng", "window", "parareal", "residence", "accounting", "temperature", "minima",
                             "reports"]
    for w in which:
        globals()[f"make_{w}"]()
    for f in sorted(os.listdir(OUT)):
        print(f, os.path.getsize(os.path.join(OUT, f)))
