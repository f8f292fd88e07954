"""CPU-only checks: the C ABI library loads and exports every declared symbol,
host-side types/plans follow the reference, synthetic W inputs are sane.
No compute call reaches the device here."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "paralangevin_b200.h")


def _declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|double|const char\*)\s+(pl_\w+)\(", src, re.M)))


def test_library_exports_every_declared_symbol():
    from paper_2212_10508_b200 import _lib
    lib = _lib.load()
    declared = _declared()
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(lib, name), name
    assert set(declared) == set(_lib.SIGNATURES), "ctypes table out of sync with header"
    assert lib.pl_version() == 100


def test_library_is_sm100a():
    from paper_2212_10508_b200 import _lib
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_no_gpu_raises_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2212_10508_b200 as pl
    from paper_2212_10508_b200._lib import LibraryError
    with pytest.raises(LibraryError):
        pl.DoubleWell(1.0, 1.0).gradient(np.array([0.5]))


def test_seeds_match_oracle():
    from oracle import rng as orng
    import paper_2212_10508_b200 as pl
    for m in (0, 11, 77, 2**64 - 1):
        assert [int(s) for s in pl.derive_seeds(m, 20)] == [int(s) for s in orng.derive_seeds(m, 20)]
    plan = pl.NoisePlan.for_windows(11, 5)
    assert plan.seed_for(1) == 0xAEAF52FEBE706064
    with pytest.raises(ValueError):
        pl.NoisePlan(11, (1, 2))


def test_types_validation_mirrors_reference():
    import paper_2212_10508_b200 as pl
    with pytest.raises(ValueError):
        pl.LangevinParams(gamma=1.0, inv_beta=1.0, dt=2.0)
    with pytest.raises(ValueError):
        pl.PhaseState(q=[np.nan], p=[0.0])
    s = pl.TemperatureSchedule.robust(4)
    assert s.coefficients == (3.0, 1.0, 1.0, 1.0, 1.0)
    with pytest.raises(pl.InfeasibleScheduleError):
        pl.solve_schedule(3, 0.5)
    with pytest.raises(ValueError):
        pl.PararealConfig(10, 1e-3, 1e-4)


def test_lattice_sizes():
    from paper_2212_10508_b200 import tungsten as W
    for n, natoms in ((4, 129), (8, 1025), (20, 16001)):
        q, box = W.bcc_sia(n)
        assert q.shape[0] == 3 * natoms
        assert box[0] == pytest.approx(n * W.A0)
    assert [W.n_bispectrum(t) for t in (2, 4, 6, 8, 10, 12, 14)] == [5, 14, 30, 55, 91, 140, 204]


def test_snap_beta_matches_oracle_stream():
    from oracle import rng as orng
    from paper_2212_10508_b200 import tungsten as W
    b = W.snap_beta(11)
    g = orng.gaussian_stream(orng.derive_seed(11, 1), 56)
    assert b.shape == (56,)
    np.testing.assert_allclose(b, 0.05 * g, rtol=1e-15, atol=0)


def test_eam_tables_reproduce_fs_tungsten():
    from oracle import native
    from paper_2212_10508_b200 import tungsten as W
    q, box = W.bcc_sia(4, sia=False)
    e, g, v = native.eam(q, box, W.eam_tables())
    assert e / 128 == pytest.approx(-8.90, abs=1e-3)
    assert np.abs(g).max() < 1e-10
    # virial of the perfect lattice at the equilibrium constant ~ 0 (zero pressure)
    assert abs(v[0]) < 1e-3


def test_oracle_neighbour_counts():
    from oracle import native
    from paper_2212_10508_b200 import tungsten as W
    q, box = W.bcc_sia(4, sia=False)
    assert {len(x) for x in native.neighbours(q, box, 4.73)} == {26}
    assert {len(x) for x in native.neighbours(q, box, 5.5)} == {58}


def test_residence_times_match_reference(golden):
    from paper_2212_10508_b200 import sia
    z = golden("residence_golden.npz")
    for mr in (1, 3):
        ev = sia.residence_times(z["labels"], min_run=mr)
        got = np.array([[e.basin, e.duration, int(e.censored)] for e in ev], dtype=np.int64)
        assert np.array_equal(got, z[f"events_{mr}"])
        ci = sia.mean_ci([e.duration for e in ev if not e.censored])
        assert np.array(ci).tobytes() == z[f"ci_{mr}"].tobytes()


def test_gain_accounting_matches_reference(golden):
    """accounting.adaptive_gain / classic_gain vs the reference (accounting.py:99-159)."""
    import json

    from paper_2212_10508_b200 import accounting as acc
    from paper_2212_10508_b200.parareal import SlabAttempt, SlabRecord
    z = golden("accounting_golden.npz")
    sets = [[SlabRecord(i, n0, tuple(SlabAttempt(a, k) for a, k in att), n1, kc)
             for i, n0, n1, kc, att in slabs] for slabs in json.loads(str(z["slabsets"]))]
    for row in z["adaptive"]:
        si, cf, cc = int(row[0]), row[1], row[2]
        r = acc.adaptive_gain(sets[si], sets[si][-1].n_final, cf, cc)
        assert [r.total_cost, r.sequential_cost, r.gain, r.ideal_gain] == list(row[3:7])
        assert (r.n_slab, r.total_iterations) == (int(row[7]), int(row[8]))
    for row in z["classic"]:
        r = acc.classic_gain(int(row[0]), int(row[1]), row[2], row[3])
        assert [r.total_cost, r.sequential_cost, r.gain, r.ideal_gain, r.total_effort] == list(row[4:9])
    with pytest.raises(ValueError):
        acc.adaptive_gain(sets[1][:1], 16, 1.0, 0.0)  # does not tile the window range
    with pytest.raises(ValueError):
        acc.classic_gain(16, 3, 0.0, 1.0)


@pytest.mark.parametrize("name", ["adaptive", "parareal"])
def test_report_files_match_reference(golden, tmp_path, name):
    """trajectory.csv / history.csv / result.json byte-identical to the reference's
    own report writers (cli.py:888-930) for the reference's parareal result."""
    from paper_2212_10508_b200 import reports
    from paper_2212_10508_b200.model import LangevinParams, NodeTrajectory
    from paper_2212_10508_b200.parareal import PararealConfig, PararealResult, SlabAttempt, SlabRecord
    z, ref = golden("parareal_golden.npz"), golden("reports_golden.npz")
    cfg = z[f"{name}_cfg"]
    slabs, by = [], {}
    for si, n0, n1, kc, af, ai in z[f"{name}_slabs"]:
        by.setdefault((int(si), int(n0), int(n1), int(kc)), []).append(SlabAttempt(int(af), int(ai)))
    for (si, n0, n1, kc), att in sorted(by.items()):
        slabs.append(SlabRecord(si, n0, tuple(att), n1, kc))
    res = PararealResult(trajectory=NodeTrajectory.from_arrays(z[f"{name}_Q"], z[f"{name}_P"]), slabs=slabs,
                         error_history=[tuple(r) for r in z[f"{name}_hist"]],
                         converged=bool(z[f"{name}_converged"]))
    params = LangevinParams(cfg[0], cfg[1], cfg[2], int(cfg[3]))
    config = PararealConfig(int(cfg[5]), cfg[6], cfg[7] if name == "adaptive" else None)

    class Pair:
        cost_fine, cost_coarse = 175.0, 1.0

    exp = "parareal_adaptive" if name == "adaptive" else "parareal_classic"
    paths = reports.write_parareal_report(tmp_path, res, exp, params, config, Pair)
    for p in paths:
        assert p.read_text() == str(ref[f"{name}_{p.name.replace('.', '_')}"]), p.name
