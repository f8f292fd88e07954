"""CPU oracle for the parareal / SNAP hot path -- TEST INFRASTRUCTURE ONLY.

Nothing in ``paper_2212_10508_b200`` imports this package.  Only ``tests/``,
``__graft_entry__.smoke()`` and the ``cpu_baseline`` / ``--impl reference``
legs of ``bench.py`` may use it, and only as the checker or as the timed CPU
reference arm -- never as the product path.

Contents
--------
``rng``         SplitMix64 seeds + Marsaglia-polar Gaussian streams
                (restates /root/reference/pkg/src/paralangevin/rng.py:31-185).
``integrator``  modified-BBK window propagator with noise-block reuse
                (restates integrator.py:156-308).
``parareal``    classic / adaptive engines, error metric, sequential chain
                (restates parareal.py:195-475).
``toy``         DoubleWell / Harmonic / LennardJonesCluster / Perturbed
                gradients (restates potentials.py:62-214).
``native``      ctypes front-end of ``liboracle.so`` -- plain C restatements
                of the periodic neighbour list, tabulated EAM and fp64 SNAP
                (no reference exists for these: see DESIGN.md "parity").

Parity pins: ``rng``/``integrator``/``parareal``/``toy`` are checked bit for
bit against golden vectors produced by the reference itself in the build
container (``scripts/make_golden.py`` -> ``tests/golden/``).  SNAP/EAM/neighbour
lists have no reference implementation ("parity unpinned" w.r.t. the
reference); the C SNAP oracle is pinned externally by
``tests/test_snap_oracle_pin.py``: its Clebsch-Gordan coefficients against
``sympy.physics.wigner.clebsch_gordan`` (all 4,451 with 2j <= 8), its U
recursion against the spin-J/2 representation built from explicit polynomials
(itself checked against sympy's ``wigner_d``), its per-atom bispectrum against
a slow numpy/sympy evaluation on open clusters, its forces against central
differences and rotation covariance.  Neighbour lists are checked by counts on
the perfect lattice and EAM by the FS-W cohesive energy.
"""
