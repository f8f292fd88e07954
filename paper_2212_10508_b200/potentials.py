"""Device potentials behind the reference's ``Potential`` protocol.

Mirrors /root/reference/pkg/src/paralangevin/potentials.py:
  Potential        potentials.py:39-59   energy(q) / gradient(q) on flat q
  Free/Harmonic/DoubleWell/LennardJonesCluster/Perturbed  potentials.py:62-214
  gradient_check   potentials.py:217-229
  PropagatorPair   potentials.py:290-312
plus the periodic many-body potentials the hot path needs (absent from the
reference): ``EAM`` (tabulated Finnis-Sinclair) and ``SNAP``.

Every evaluation runs in libparalangevin_b200 on the GPU.  ``energy`` and
``gradient`` keep the reference's single-vector signatures (host numpy in,
host numpy out); ``energies`` / ``gradients`` take a batch of systems and
accept device tensors, which is how the engines call them.
"""

from __future__ import annotations

import ctypes as C
import sys as _sys
from dataclasses import dataclass, field

import numpy as np

from . import _lib


class PotentialError(ValueError):
    """Invalid coordinates or parameters for a potential evaluation."""


class MinimizationError(RuntimeError):
    """Gradient descent failed to reach the requested tolerance."""


def _coeff(value, name: str):
    if np.isscalar(value):
        out = float(value)
        if not np.isfinite(out):
            raise ValueError(f"{name} must be finite")
        return out
    arr = np.array(value, dtype=float)
    if arr.ndim != 1 or arr.size == 0 or not np.isfinite(arr).all():
        raise ValueError(f"{name} must be a finite scalar or 1-d vector")
    arr.setflags(write=False)
    return arr


def _raise(err: _lib.CallError):
    if err.code in (_lib.PL_EARG, _lib.PL_EPOT):
        raise PotentialError(err.message) from None
    raise err


class Potential:
    """Base interface: device-evaluated energy and gradient on flat coordinates."""

    dimension: int | None = None

    # ---- device handle management
    def _create(self, ctx) -> C.c_void_p:  # pragma: no cover - abstract
        raise NotImplementedError

    def handle(self, ctx=None) -> C.c_void_p:
        ctx = ctx or _lib.context()
        cache = self.__dict__.setdefault("_handles", {})
        h = cache.get(ctx.device)
        if h is None:
            try:
                h = self._create(ctx)
            except _lib.CallError as err:
                _raise(err)
            cache[ctx.device] = h
        return h

    def __del__(self):
        try:
            if _sys.is_finalizing():
                return
            for h in self.__dict__.get("_handles", {}).values():
                if _lib._lib is not None and h:
                    _lib._lib.pl_pot_destroy(h)
        except Exception:
            pass

    def flops_per_eval(self) -> float:
        return float(_lib.load().pl_pot_flops(self.handle()))

    # ---- reference API
    def _check_q(self, q) -> np.ndarray:
        q = np.asarray(q, dtype=float)
        if q.ndim != 1:
            raise PotentialError(f"coordinates must be a 1-d vector, got shape {q.shape}")
        if self.dimension is not None and q.shape[0] != self.dimension:
            raise PotentialError(
                f"{type(self).__name__} expects dimension {self.dimension}, got {q.shape[0]}")
        return q

    def energy(self, q) -> float:
        q = self._check_q(q)
        return float(self.energies(q[None, :])[0])

    def gradient(self, q) -> np.ndarray:
        q = self._check_q(q)
        return self.gradients(q[None, :])[0]

    # ---- batched device API
    def evaluate(self, Q, energy=True, gradient=True, virial=False):
        """Batched evaluation; Q is (B, d) numpy or CUDA tensor. Returns torch tensors."""
        import torch
        ctx = _lib.context()
        dev = torch.device("cuda", ctx.device)
        Qt = torch.as_tensor(Q, dtype=torch.float64).to(dev).contiguous()
        if Qt.ndim != 2:
            raise PotentialError("batched coordinates must be (B, d)")
        B, d = Qt.shape
        if self.dimension is not None and d != self.dimension:
            raise PotentialError(
                f"{type(self).__name__} expects dimension {self.dimension}, got {d}")
        E = torch.empty(B, dtype=torch.float64, device=dev) if energy else None
        G = torch.empty((B, d), dtype=torch.float64, device=dev) if gradient else None
        V = torch.empty((B, 6), dtype=torch.float64, device=dev) if virial else None
        try:
            _lib.check(_lib.load().pl_compute(ctx.handle, self.handle(ctx), B, d, _lib.ptr(Qt),
                                              _lib.ptr(E), _lib.ptr(G), _lib.ptr(V)))
        except _lib.CallError as err:
            _raise(err)
        return E, G, V

    def energies(self, Q) -> np.ndarray:
        return self.evaluate(Q, True, False)[0].cpu().numpy()

    def gradients(self, Q) -> np.ndarray:
        return self.evaluate(Q, False, True)[1].cpu().numpy()


@dataclass(frozen=True, eq=False)
class Free(Potential):
    """V = 0."""

    def _create(self, ctx):
        h = C.c_void_p()
        _lib.check(_lib.load().pl_pot_free(ctx.handle, C.byref(h)))
        return h


@dataclass(frozen=True, eq=False)
class Harmonic(Potential):
    """V(q) = sum_i k_i q_i^2 / 2 (potentials.py:75-95)."""

    k: float | np.ndarray = 1.0

    def __post_init__(self) -> None:
        k = _coeff(self.k, "k")
        if np.any(np.asarray(k) <= 0.0):
            raise ValueError("k must be positive")
        object.__setattr__(self, "k", k)
        if isinstance(k, np.ndarray):
            object.__setattr__(self, "dimension", k.shape[0])

    def _create(self, ctx):
        h = C.c_void_p()
        k = np.ascontiguousarray(np.atleast_1d(np.asarray(self.k, dtype=float)))
        dim = self.dimension or 0
        _lib.check(_lib.load().pl_pot_harmonic(ctx.handle, dim, _lib.dptr(k), C.byref(h)))
        return h


@dataclass(frozen=True, eq=False)
class DoubleWell(Potential):
    """V(q) = sum_i a_i (q_i^2 - b_i)^2 (potentials.py:98-128)."""

    a: float | np.ndarray = 1.0
    b: float | np.ndarray = 1.0

    def __post_init__(self) -> None:
        a = _coeff(self.a, "a")
        b = _coeff(self.b, "b")
        if np.any(np.asarray(a) <= 0.0) or np.any(np.asarray(b) <= 0.0):
            raise ValueError("a and b must be positive")
        object.__setattr__(self, "a", a)
        object.__setattr__(self, "b", b)
        dims = {x.shape[0] for x in (a, b) if isinstance(x, np.ndarray)}
        if len(dims) > 1:
            raise ValueError("a and b have inconsistent dimensions")
        if dims:
            object.__setattr__(self, "dimension", dims.pop())

    def _create(self, ctx):
        h = C.c_void_p()
        dim = self.dimension or 0
        n = dim or 1
        a = np.ascontiguousarray(np.broadcast_to(np.asarray(self.a, dtype=float), (n,)))
        b = np.ascontiguousarray(np.broadcast_to(np.asarray(self.b, dtype=float), (n,)))
        _lib.check(_lib.load().pl_pot_double_well(ctx.handle, dim, _lib.dptr(a), _lib.dptr(b),
                                                  C.byref(h)))
        return h


@dataclass(frozen=True, eq=False)
class LennardJonesCluster(Potential):
    """All-pairs LJ cluster on atom-major flat coordinates (potentials.py:131-180)."""

    epsilon: float = 1.0
    sigma: float = 1.0
    n_atoms: int = 7
    space_dim: int = 2

    def __post_init__(self) -> None:
        if not (np.isfinite(self.epsilon) and self.epsilon > 0.0):
            raise ValueError("epsilon must be positive")
        if not (np.isfinite(self.sigma) and self.sigma > 0.0):
            raise ValueError("sigma must be positive")
        if self.n_atoms < 2:
            raise ValueError("need at least 2 atoms")
        if self.space_dim < 1:
            raise ValueError("space_dim must be >= 1")
        object.__setattr__(self, "dimension", self.n_atoms * self.space_dim)

    def _create(self, ctx):
        h = C.c_void_p()
        _lib.check(_lib.load().pl_pot_lj(ctx.handle, float(self.epsilon), float(self.sigma),
                                         int(self.n_atoms), int(self.space_dim), C.byref(h)))
        return h


@dataclass(frozen=True, eq=False)
class Perturbed(Potential):
    """V = V_base + lam * V_delta; lam == 0 is the base bit for bit (potentials.py:183-214)."""

    base: Potential
    delta: Potential
    lam: float = 0.0

    def __post_init__(self) -> None:
        if not np.isfinite(self.lam):
            raise ValueError("lam must be finite")
        dims = {p.dimension for p in (self.base, self.delta) if p.dimension is not None}
        if len(dims) > 1:
            raise ValueError("base and delta have incompatible dimensions")
        if dims:
            object.__setattr__(self, "dimension", dims.pop())

    def _create(self, ctx):
        h = C.c_void_p()
        _lib.check(_lib.load().pl_pot_perturbed(ctx.handle, self.base.handle(ctx),
                                                self.delta.handle(ctx), float(self.lam),
                                                C.byref(h)))
        return h


@dataclass(frozen=True, eq=False)
class EAM(Potential):
    """Tabulated EAM (Finnis-Sinclair form) in an orthorhombic periodic box.

    ``tables`` holds cubic-Hermite coefficient arrays ``rho`` / ``phi``
    (n_r x 4 on [0, rcut], spacing ``dr``) and ``F`` (n_rho x 4, spacing
    ``drho``); see :func:`paper_2212_10508_b200.tungsten.eam_tables`.
    """

    n_atoms: int
    box: tuple
    rcut: float
    dr: float
    rho: np.ndarray = field(repr=False)
    phi: np.ndarray = field(repr=False)
    drho: float = 0.0
    F: np.ndarray = field(repr=False, default=None)

    def __post_init__(self) -> None:
        object.__setattr__(self, "dimension", 3 * int(self.n_atoms))
        object.__setattr__(self, "box", tuple(float(x) for x in self.box))

    def _create(self, ctx):
        h = C.c_void_p()
        box = np.ascontiguousarray(self.box, dtype=float)
        rho = np.ascontiguousarray(self.rho, dtype=float)
        phi = np.ascontiguousarray(self.phi, dtype=float)
        F = np.ascontiguousarray(self.F, dtype=float)
        _lib.check(_lib.load().pl_pot_eam(
            ctx.handle, int(self.n_atoms), _lib.dptr(box), float(self.rcut), rho.shape[0],
            float(self.dr), _lib.dptr(rho), _lib.dptr(phi), F.shape[0], float(self.drho),
            _lib.dptr(F), C.byref(h)))
        return h


@dataclass(frozen=True, eq=False)
class SNAP(Potential):
    """Single-element SNAP: E_i = beta_0 + sum_k beta_k B_k(i) (fp64)."""

    n_atoms: int
    box: tuple
    beta: np.ndarray = field(repr=False)
    twojmax: int = 8
    rcut: float = 4.73
    rfac0: float = 0.99363
    rmin0: float = 0.0
    switchflag: int = 1
    wself: float = 1.0

    def __post_init__(self) -> None:
        object.__setattr__(self, "dimension", 3 * int(self.n_atoms))
        object.__setattr__(self, "box", tuple(float(x) for x in self.box))
        beta = np.array(self.beta, dtype=float)
        beta.setflags(write=False)
        object.__setattr__(self, "beta", beta)

    def _create(self, ctx):
        h = C.c_void_p()
        box = np.ascontiguousarray(self.box, dtype=float)
        beta = np.ascontiguousarray(self.beta, dtype=float)
        _lib.check(_lib.load().pl_pot_snap(
            ctx.handle, int(self.n_atoms), _lib.dptr(box), int(self.twojmax), float(self.rcut),
            float(self.rfac0), float(self.rmin0), int(self.switchflag), float(self.wself),
            _lib.dptr(beta), beta.shape[0], C.byref(h)))
        return h


def gradient_check(pot: Potential, q, h: float = 1e-6) -> float:
    """Largest gap between the gradient and central differences (potentials.py:217-229).

    All 2d displaced configurations are evaluated in one batched device call.
    """
    q = np.asarray(q, dtype=float)
    d = q.shape[0]
    grad = pot.gradient(q)
    Q = np.repeat(q[None, :], 2 * d, axis=0)
    idx = np.arange(d)
    Q[2 * idx, idx] += h
    Q[2 * idx + 1, idx] -= h
    E = pot.energies(Q)
    fd = (E[0::2] - E[1::2]) / (2.0 * h)
    return float(np.max(np.abs(fd - grad)))


def minimize_batch(pot: Potential, starts, tol: float = 1e-8, max_iter: int = 50_000):
    """B steepest descents with Armijo backtracking in one device pass (pl_minimize).

    The reference's ``_descend`` (potentials.py:231-266) per start, batched:
    returns ``(minima (B, d), status (B,), iterations (B,), energies (B,))``
    with status 0 converged, 1 line search stalled, 2 no convergence.
    """
    import torch
    X = np.atleast_2d(np.asarray(starts, dtype=float))
    B, d = X.shape
    if pot.dimension is not None and d != pot.dimension:
        raise PotentialError(f"{type(pot).__name__} expects dimension {pot.dimension}, got {d}")
    ctx = _lib.context()
    Xd = torch.from_numpy(np.array(X)).to(torch.device("cuda", ctx.device))
    status = np.zeros(B, dtype=np.int32)
    iters = np.zeros(B, dtype=np.int64)
    energy = np.zeros(B, dtype=float)
    try:
        _lib.check(_lib.load().pl_minimize(ctx.handle, pot.handle(ctx), B, d, _lib.ptr(Xd), float(tol),
                                           int(max_iter), status.ctypes.data_as(_lib.pi32),
                                           iters.ctypes.data_as(_lib.pi64), _lib.dptr(energy)))
    except _lib.CallError as err:
        _raise(err)
    return Xd.cpu().numpy(), status, iters, energy


def local_minima(pot: Potential, starts, tol: float = 1e-8, max_iter: int = 50_000) -> list:
    """Distinct minima in first-found order (potentials.py:268-287), all descents batched.

    Raises MinimizationError naming the first start (in order) whose descent
    stalls or does not converge, as the sequential reference would.
    """
    if tol <= 0.0:
        raise ValueError("tol must be positive")
    starts = [np.asarray(s, dtype=float) for s in starts]
    if not starts:
        return []
    X, status, _, _ = minimize_batch(pot, np.stack(starts), tol, max_iter)
    minima: list = []
    for i, x in enumerate(X):
        if status[i] == 1:
            raise MinimizationError(f"line search stalled while minimizing from start {starts[i].tolist()}")
        if status[i] == 2:
            raise MinimizationError(f"no convergence to |grad| <= {tol} within {max_iter} iterations "
                                    f"from start {starts[i].tolist()}")
        if all(np.linalg.norm(x - m) > tol for m in minima):
            minima.append(x)
    return minima


@dataclass(frozen=True)
class PropagatorPair:
    """Fine and coarse potentials with their configured per-window costs."""

    fine: Potential
    coarse: Potential
    cost_fine: float = 1.0
    cost_coarse: float = 1.0

    def __post_init__(self) -> None:
        if not (np.isfinite(self.cost_coarse) and self.cost_coarse > 0.0):
            raise ValueError("cost_coarse must be positive")
        if not (np.isfinite(self.cost_fine) and self.cost_fine >= self.cost_coarse):
            raise ValueError("cost_fine must be >= cost_coarse")
        dims = {p.dimension for p in (self.fine, self.coarse) if p.dimension is not None}
        if len(dims) > 1:
            raise ValueError("fine and coarse potentials have incompatible dimensions")
