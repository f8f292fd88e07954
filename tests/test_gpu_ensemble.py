"""Statistical parity of long chaotic runs (north star, 4th correctness bullet;
SURVEY.md 8f rank 1): the reference's ensemble protocol (cli.py:986-1050) on
the W + SIA system, reduced in size.  The SIA mean residence time of adaptive
parareal must fall inside the confidence interval of the sequential fine
reference run with the same noise plans (compare_ensembles, analysis.py:232-238;
acceptance criterion 8, test_acceptance.py:373-422)."""

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


def test_sequential_batch_equals_single_chains(pl):
    from paper_2212_10508_b200 import tungsten as W
    from paper_2212_10508_b200.ensemble import sequential_propagate_batch
    q0, box = W.bcc_sia(4)
    n = q0.shape[0] // 3
    L, N = 5, 3
    params = pl.LangevinParams(1.0, W.KB * 1200.0, 0.001, L, mass=np.full(3 * n, W.MASS_W))
    sched = pl.TemperatureSchedule.robust(L)
    eam = W.make_eam(n, box)
    inits = [pl.PhaseState(q=q0, p=W.maxwell_boltzmann(n, 1200.0, s)) for s in (1, 2, 3)]
    plans = [pl.NoisePlan.for_windows(pl.derive_seed(5, i + 1), N) for i in range(3)]
    Q, P = sequential_propagate_batch(inits, N, eam, params, sched, plans)
    for r in range(3):
        one = pl.sequential_propagate(inits[r], N, eam, params, sched, plans[r])
        assert one.positions().tobytes() == Q[r].tobytes()
        assert one.momenta().tobytes() == P[r].tobytes()


def test_residence_time_ensemble_overlap(pl):
    """8 members x 2 segments x 16 windows x 100 substeps at 1200 K, SNAP fine / EAM
    coarse, delta_conv 1e-5 (configs/ensemble.json), quenched node labels, min_run 2."""
    from paper_2212_10508_b200 import tungsten as W
    from paper_2212_10508_b200.ensemble import run_ensemble
    q0, box = W.bcc_sia(4)
    n = q0.shape[0] // 3
    L, N, T = 100, 16, 1200.0
    params = pl.LangevinParams(1.0, W.KB * T, 0.001, L, mass=np.full(3 * n, W.MASS_W))
    sched = pl.TemperatureSchedule.robust(L)
    pair = pl.PropagatorPair(W.make_snap(n, box), W.make_eam(n, box), 100.0, 1.0)
    res = run_ensemble(pair, params, sched, pl.PhaseState(q=q0, p=np.zeros_like(q0)),
                       pl.PararealConfig(N, 1e-5, 0.35), size=8, master_seed=77, n_cells=4, a=W.A0,
                       segments=2, thermalization_windows=2, min_run=2, quench=True)
    assert res.converged == res.runs == 16
    assert res.fine.n_events >= 5 and res.adaptive.n_events >= 5
    assert res.comparison.overlap, res.as_dict()
