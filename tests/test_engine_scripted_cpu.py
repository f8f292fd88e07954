"""The adaptive state machine (``_adaptive_machine``) on the reference's own
scripted traces, CPU only.

Both the device engines and the host-callable engine answer the same machine;
here it is driven by plain Python propagators (no GPU), against the frozen
hand traces of the reference's test suite (test_parareal.py:425-533): identity
fine, halving coarse, N = 4, delta_conv = 1e-3, delta_expl = 1.  The values are
exact dyadic fractions, so the histories are compared with ==.
"""

import itertools

import numpy as np
import pytest

import paper_2212_10508_b200 as pl
from paper_2212_10508_b200.parareal import parareal_adaptive_engine, parareal_classic_engine


def _state(q):
    q = np.asarray(q, dtype=float)
    return pl.PhaseState(q=q, p=np.zeros_like(q))


def _halving_coarse(state, m):
    return pl.PhaseState(q=0.5 * state.q, p=state.p)


def _identity_fine(state, m):
    return pl.PhaseState(q=state.q, p=state.p)


def _config(**kw):
    return pl.PararealConfig(**{"n_windows": 4, "delta_conv": 1e-3, "delta_expl": 1.0, **kw})


def test_frozen_slab_records_and_history():
    res = parareal_adaptive_engine(_state([1.0]), _identity_fine, _halving_coarse, _config())
    assert res.converged
    assert [(s.slab_index, s.n_init, tuple((a.n_final, a.iterations) for a in s.attempts), s.n_final, s.k_conv)
            for s in res.slabs] == [(1, 0, ((4, 1), (1, 1)), 1, 2), (2, 1, ((4, 4),), 4, 4)]
    assert res.error_history == (
        (1, 1, 1.0), (1, 1, 1.0 / 0.75), (1, 2, 0.0),
        (2, 1, 0.5 / 1.5), (2, 1, 1.0 / 1.75), (2, 1, 1.375 / 1.875),
        (2, 2, 0.0), (2, 2, 0.25 / 2.75), (2, 2, 0.625 / 3.25),
        (2, 3, 0.0), (2, 3, 0.0), (2, 3, 0.125 / 3.875),
        (2, 4, 0.0), (2, 4, 0.0), (2, 4, 0.0))
    assert [s.q[0] for s in res.trajectory] == [1.0] * 5


def test_huge_explosion_threshold_reduces_to_classic():
    a = parareal_adaptive_engine(_state([1.0]), _identity_fine, _halving_coarse, _config(delta_expl=1e12))
    c = parareal_classic_engine(_state([1.0]), _identity_fine, _halving_coarse, _config())
    assert a.converged and c.converged and a.slabs == c.slabs
    assert a.error_history[3::4] == c.error_history


def test_slab_collapse_raises():
    with pytest.raises(pl.SlabCollapseError) as exc:
        parareal_adaptive_engine(_state([1.0]), _identity_fine, _halving_coarse, _config(delta_expl=0.3))
    assert exc.value.slab_index == 1 and exc.value.n_init == 0


def test_iteration_cap_aborts_with_partial_slabs():
    counter = itertools.count(1)

    def drifting_fine(state, m):
        return pl.PhaseState(q=state.q + 1e-3 * next(counter), p=state.p)

    with pytest.warns(RuntimeWarning, match="width"):
        res = parareal_adaptive_engine(_state([1.0]), drifting_fine, _identity_fine,
                                       _config(delta_conv=1e-12, delta_expl=1e6, k_max=6))
    assert not res.converged
    assert [(a.n_final, a.iterations) for a in res.slabs[-1].attempts] == [(4, 6)]


def test_degenerate_normalisation_raises():
    with pytest.raises(pl.DegenerateNormalizationError):
        parareal_adaptive_engine(_state([0.0]), _identity_fine, _identity_fine, _config())


def test_requires_explosion_threshold():
    with pytest.raises(ValueError, match="delta_expl"):
        parareal_adaptive_engine(_state([1.0]), _identity_fine, _halving_coarse,
                                 pl.PararealConfig(n_windows=4, delta_conv=1e-3))


def test_blow_up_context_in_host_engine():
    def bad_fine(state, m):
        raise pl.BlowUpError("boom at substep 3", substep=3)

    with pytest.raises(pl.BlowUpError) as exc:
        parareal_adaptive_engine(_state([1.0]), bad_fine, _halving_coarse, _config())
    assert exc.value.window == 1 and exc.value.iteration == 1 and exc.value.substep == 3

    def bad_coarse(state, m):
        raise pl.BlowUpError("boom", substep=1)

    with pytest.raises(pl.BlowUpError) as exc:
        parareal_adaptive_engine(_state([1.0]), _identity_fine, bad_coarse, _config())
    assert exc.value.window == 1 and exc.value.iteration == 0
