"""ctypes front-end of oracle/native/liboracle.so (TEST INFRASTRUCTURE ONLY).

Plain-C CPU restatements of the periodic neighbour list, tabulated EAM and
fp64 SNAP (see the .c headers).  Built by ``make -C oracle/native``
(``__graft_entry__.build()`` does it); used only by tests/, smoke() and the
bench's CPU-baseline / reference arms.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "native")
LIB = os.path.join(HERE, "liboracle.so")
_lib = None
pd = C.POINTER(C.c_double)
pi = C.POINTER(C.c_int32)


def build(force=False):
    srcs = [os.path.join(HERE, f) for f in os.listdir(HERE) if f.endswith(".c")]
    stale = not os.path.exists(LIB) or any(os.path.getmtime(s) > os.path.getmtime(LIB) for s in srcs)
    if force or stale:
        subprocess.run(["make", "-s", "-B", "-C", HERE], check=True)
    return LIB


def load():
    global _lib
    if _lib is None:
        build()
        _lib = C.CDLL(LIB)
        _lib.orc_neighbours.restype = C.c_int
        _lib.orc_neighbours.argtypes = [C.c_int, pd, C.c_double, pd, C.c_int, pi, pi]
        _lib.orc_eam.restype = C.c_int
        _lib.orc_eam.argtypes = [C.c_int, pd, C.c_double, C.c_int, C.c_double, pd, pd, C.c_int,
                                 C.c_double, pd, pd, pd, pd, pd]
        if hasattr(_lib, "orc_snap"):
            _lib.orc_snap.restype = C.c_int
            _lib.orc_snap.argtypes = [C.c_int, pd, C.c_int, C.c_double, C.c_double, C.c_double,
                                      C.c_int, C.c_double, pd, C.c_int, pd, pd, pd, pd, pd]
        if hasattr(_lib, "orc_ulist"):
            _lib.orc_ulist.restype = C.c_int
            _lib.orc_ulist.argtypes = [C.c_int, C.c_double, C.c_double, C.c_double, pd, pd]
        _lib.orc_cg.restype = C.c_double
        _lib.orc_cg.argtypes = [C.c_int] * 6
    return _lib


def _d(a):
    return np.ascontiguousarray(a, dtype=np.float64).ctypes.data_as(pd)


def neighbours(q, box, rcut, maxn=256):
    lib = load()
    q = np.ascontiguousarray(q, dtype=np.float64)
    n = q.shape[0] // 3
    nbr = np.zeros((n, maxn), dtype=np.int32)
    cnt = np.zeros(n, dtype=np.int32)
    box = np.ascontiguousarray(box, dtype=np.float64)
    lib.orc_neighbours(n, _d(box), float(rcut), _d(q), maxn, nbr.ctypes.data_as(pi),
                       cnt.ctypes.data_as(pi))
    return [sorted(nbr[i, :cnt[i]].tolist()) for i in range(n)]


def eam(q, box, tables):
    """(energy, gradient, virial) of one system with EAM tables (tungsten.eam_tables)."""
    lib = load()
    q = np.ascontiguousarray(q, dtype=np.float64)
    n = q.shape[0] // 3
    e = np.zeros(1)
    g = np.zeros(3 * n)
    v = np.zeros(6)
    rho, phi, F = (np.ascontiguousarray(tables[k]) for k in ("rho", "phi", "F"))
    box = np.ascontiguousarray(box, dtype=np.float64)
    rc = lib.orc_eam(n, _d(box), float(tables["rcut"]), rho.shape[0], float(tables["dr"]), _d(rho),
                     _d(phi), F.shape[0], float(tables["drho"]), _d(F), _d(q), _d(e), _d(g), _d(v))
    if rc != 0:
        raise RuntimeError("oracle EAM failed (neighbour overflow)")
    return e[0], g, v


def _snap_args(pot):
    return (int(pot.twojmax), float(pot.rcut), float(pot.rfac0), float(pot.rmin0), int(pot.switchflag),
            float(pot.wself))


def snap(q, box, pot, want_bispectrum=False):
    """(energy, gradient, virial[, B (n x nB)]) of one system for a SNAP parameter set."""
    lib = load()
    q = np.ascontiguousarray(q, dtype=np.float64)
    n = q.shape[0] // 3
    beta = np.ascontiguousarray(pot.beta, dtype=np.float64)
    e = np.zeros(1)
    g = np.zeros(3 * n)
    v = np.zeros(6)
    nb = beta.shape[0] - 1
    bs = np.zeros((n, nb))
    tj, rc, rf, rm, sw, ws = _snap_args(pot)
    box = np.ascontiguousarray(box, dtype=np.float64)
    rcode = lib.orc_snap(n, _d(box), tj, rc, rf, rm, sw, ws, _d(beta), beta.shape[0], _d(q), _d(e),
                         _d(g), _d(v), _d(bs) if want_bispectrum else None)
    if rcode < 0:
        raise RuntimeError(f"oracle SNAP failed ({rcode})")
    return (e[0], g, v, bs) if want_bispectrum else (e[0], g, v)


def ulist(twojmax, rfac0, rmin0, rcut, rv):
    """U^J of one neighbour vector as a list of full (J+1)x(J+1) complex matrices
    indexed [ma][mb] (the oracle's recursion, snap_oracle.c u_and_du)."""
    lib = load()
    size = sum((J + 1) ** 2 for J in range(twojmax + 1))
    out = np.zeros(2 * size)
    lib.orc_ulist(int(twojmax), float(rfac0), float(rmin0), float(rcut), _d(np.asarray(rv, float)),
                  out.ctypes.data_as(pd))
    u = out[0::2] + 1j * out[1::2]
    mats, o = [], 0
    for J in range(twojmax + 1):
        m = u[o:o + (J + 1) ** 2].reshape(J + 1, J + 1)  # stored [mb][ma]
        mats.append(m.T.copy())
        o += (J + 1) ** 2
    return mats


def cg(j1, m1, j2, m2, J, M):
    """Clebsch-Gordan <j1 m1 j2 m2 | J M> of the oracle (arguments are 2j / 2m)."""
    return load().orc_cg(j1, m1, j2, m2, J, M)


def snap_fn(pot):
    """gradient closure for the oracle integrator."""
    return lambda q: snap(q, pot.box, pot)[1]
