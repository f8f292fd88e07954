"""Parareal engines with the fine stage batched on the GPU.

Mirrors /root/reference/pkg/src/paralangevin/parareal.py:
  PararealConfig / SlabAttempt / SlabRecord / PararealResult  parareal.py:65-192
  relative_error                                              parareal.py:201-225
  sequential_propagate                                        parareal.py:243-267
  parareal_classic(_engine)                                   parareal.py:315-363, 490-509
  parareal_adaptive(_engine)                                  parareal.py:366-475, 512-529

Device engine (used whenever the propagators are device window propagators,
i.e. always for ``parareal_classic`` / ``parareal_adaptive``):
  * noise for every window is generated once and stays in HBM (it is
    iteration-invariant);
  * the jump stage F(prev[m]) - C(prev[m]) is ONE batched
    ``pl_propagate_windows`` launch over all slab windows; C(prev[m]) is the
    coarse output cached by the previous sweep/bootstrap (bitwise the same
    value the reference recomputes, SURVEY.md finding 7);
  * the corrected sweep runs in ``pl_sweep`` on the device; only the running
    error crosses back to the host, once per node, to drive the slab logic.
The control flow below is a line-by-line restatement of the reference
engines, so slab records, iteration counts and error histories follow the
same decisions.  Engines given arbitrary Python callables (scripted
propagators) run the same control flow over those callables.
"""

from __future__ import annotations

import warnings
from dataclasses import dataclass
from typing import Callable, NamedTuple

import numpy as np

from . import _lib
from .distributed import sharded_fine, world
from .integrator import BlowUpError, TemperatureSchedule, WindowKernel
from .model import LangevinParams, NodeTrajectory, PhaseState
from .potentials import PropagatorPair
from .rng import NoisePlan

WindowPropagator = Callable[[PhaseState, int], PhaseState]


class DegenerateNormalizationError(ValueError):
    """The relative-error denominator vanished."""


class SlabCollapseError(RuntimeError):
    def __init__(self, message: str, slab_index: int, n_init: int):
        super().__init__(message)
        self.slab_index = slab_index
        self.n_init = n_init


@dataclass(frozen=True)
class PararealConfig:
    n_windows: int
    delta_conv: float
    delta_expl: float | None = None
    k_max: int | None = None

    def __post_init__(self) -> None:
        if not isinstance(self.n_windows, int) or self.n_windows < 1:
            raise ValueError(f"n_windows must be a positive integer, got {self.n_windows}")
        if not (np.isfinite(self.delta_conv) and self.delta_conv > 0.0):
            raise ValueError(f"delta_conv must be positive and finite, got {self.delta_conv}")
        if self.delta_expl is not None and not self.delta_expl > self.delta_conv:
            raise ValueError(
                f"delta_expl ({self.delta_expl}) must exceed delta_conv ({self.delta_conv})")
        if self.k_max is not None and (not isinstance(self.k_max, int) or self.k_max < 1):
            raise ValueError(f"k_max must be a positive integer, got {self.k_max}")

    @property
    def iteration_cap(self) -> int:
        return self.k_max if self.k_max is not None else self.n_windows + 1


class SlabAttempt(NamedTuple):
    n_final: int
    iterations: int


@dataclass(frozen=True)
class SlabRecord:
    slab_index: int
    n_init: int
    attempts: tuple
    n_final: int
    k_conv: int

    def __post_init__(self) -> None:
        attempts = tuple(SlabAttempt(int(a[0]), int(a[1])) for a in self.attempts)
        object.__setattr__(self, "attempts", attempts)
        if self.slab_index < 1:
            raise ValueError(f"slab_index must be >= 1, got {self.slab_index}")
        if not attempts:
            raise ValueError("a slab record needs at least one attempt")
        if not 0 <= self.n_init < self.n_final:
            raise ValueError(f"slab range [{self.n_init}, {self.n_final}] must be non-empty")
        for a, b in zip(attempts, attempts[1:]):
            if b.n_final > a.n_final:
                raise ValueError("attempt endpoints must be non-increasing")
        if attempts[-1].n_final != self.n_final:
            raise ValueError(f"last attempt ends at {attempts[-1].n_final}, slab at {self.n_final}")
        if any(a.iterations < 1 for a in attempts):
            raise ValueError("every attempt must count at least one iteration")
        if sum(a.iterations for a in attempts) != self.k_conv:
            raise ValueError("k_conv must equal the sum of attempt iterations")

    @property
    def width(self) -> int:
        return self.n_final - self.n_init


@dataclass(frozen=True)
class PararealResult:
    trajectory: NodeTrajectory
    slabs: tuple
    error_history: tuple
    converged: bool
    iterates: tuple | None = None

    def __post_init__(self) -> None:
        object.__setattr__(self, "slabs", tuple(self.slabs))
        object.__setattr__(self, "error_history",
                           tuple((int(s), int(k), float(e)) for s, k, e in self.error_history))
        if self.iterates is not None:
            object.__setattr__(self, "iterates", tuple(self.iterates))
        if not self.slabs:
            raise ValueError("a result needs at least one slab record")
        if self.slabs[0].n_init != 0:
            raise ValueError("the first slab must start at window 0")
        for i, slab in enumerate(self.slabs):
            if slab.slab_index != i + 1:
                raise ValueError("slab indices must run 1..n_slab in order")
        for a, b in zip(self.slabs, self.slabs[1:]):
            if b.n_init != a.n_final:
                raise ValueError(f"slabs must tile the window range: {a.n_final} != {b.n_init}")
        if self.converged and self.slabs[-1].n_final != self.trajectory.n_windows:
            raise ValueError("a converged result must cover every window")

    @property
    def n_slab(self) -> int:
        return len(self.slabs)

    @property
    def total_iterations(self) -> int:
        return sum(slab.k_conv for slab in self.slabs)


def _close_attempt(attempts, n_init, n_final, iterations):
    width = n_final - n_init
    if iterations > width + 1:
        warnings.warn(
            f"slab [{n_init}, {n_final}] needed {iterations} iterations, beyond the width + 1 = "
            f"{width + 1} exact-arithmetic bound; delta_conv may be below roundoff",
            RuntimeWarning, stacklevel=3)
    attempts.append(SlabAttempt(n_final=n_final, iterations=iterations))


def relative_error(a, b, n_init: int, n_final: int) -> float:
    """sum_n |b_n.q - a_n.q| / sum_n |a_n.q| over max(n_init,1)..n_final (host helper)."""
    if n_init < 0:
        raise ValueError(f"n_init must be >= 0, got {n_init}")
    if n_final < max(n_init, 1):
        raise ValueError(
            f"n_final must be >= max(n_init, 1), got n_init={n_init}, n_final={n_final}")
    if n_final >= len(a) or n_final >= len(b):
        raise IndexError(
            f"node {n_final} out of range for trajectories of {len(a)} and {len(b)} nodes")
    num = den = 0.0
    for n in range(max(n_init, 1), n_final + 1):
        num += float(np.linalg.norm(b[n].q - a[n].q))
        den += float(np.linalg.norm(a[n].q))
    if den == 0.0:
        raise DegenerateNormalizationError(
            f"all reference positions on nodes {max(n_init, 1)}..{n_final} are zero")
    return num / den


# ======================================================================
# device window propagator
class DevicePropagator:
    """``WindowPropagator`` backed by the GPU: (state, m) -> state, plus batch access."""

    def __init__(self, pot, params: LangevinParams, schedule: TemperatureSchedule, plan: NoisePlan,
                 dim: int):
        self.pot, self.params, self.schedule, self.plan = pot, params, schedule, plan
        self.kernel = WindowKernel(pot, params, schedule, dim)
        self.d = dim
        self._noise = None

    def noise_all(self):
        """(N, (L+1)*d) device noise of every planned window, generated once."""
        if self._noise is None:
            self._noise = self.kernel.noise(np.asarray(self.plan.window_seeds, dtype=np.uint64))
        return self._noise

    def share_noise(self, other: "DevicePropagator") -> None:
        if other.plan == self.plan and other.kernel.L == self.kernel.L and other.d == self.d:
            self._noise = other.noise_all()

    def __call__(self, state: PhaseState, m: int) -> PhaseState:
        import torch
        dev = self.kernel.device
        Q0 = torch.from_numpy(np.array(state.q)[None]).to(dev)
        P0 = torch.from_numpy(np.array(state.p)[None]).to(dev)
        Q1, P1, blow = self.kernel.run(Q0, P0, self.noise_all()[m:m + 1])
        b = int(blow.cpu()[0])
        if b:
            raise BlowUpError(
                f"state left the trusted range (|component| > 1e+12 or non-finite) at substep {b}",
                substep=b)
        return PhaseState(q=Q1[0].cpu().numpy(), p=P1[0].cpu().numpy())


def _window_propagator(pot, params, schedule, plan, dim) -> DevicePropagator:
    return DevicePropagator(pot, params, schedule, plan, dim)


def _attach_context(err: BlowUpError, window: int, iteration: int) -> None:
    if err.window is None:
        err.window = window
    if err.iteration is None:
        err.iteration = iteration


def _call(prop, state, m, iteration):
    try:
        return prop(state, m)
    except BlowUpError as err:
        _attach_context(err, window=m + 1, iteration=iteration)
        raise


class _FineCache:
    """Fine-window results keyed by their exact start state.

    Behind the parareal exactness front prev[m] stops changing bit for bit, so
    F(prev[m]) is the previous iteration's value: a row is re-propagated only
    when its start (q, p) differs in any bit from the cached input (the fine
    propagator is deterministic, so results are identical to recomputing).
    The reference recomputes every slab window each iteration
    (parareal.py:270-286); the gain model still charges them (accounting.py).
    Disable with PL_PARAREAL_NOCACHE=1.
    """

    def __init__(self, rows: int, d: int, device):
        import os

        import torch
        f64 = dict(dtype=torch.float64, device=device)
        self.inQ = torch.zeros((rows, d), **f64)
        self.inP = torch.zeros((rows, d), **f64)
        self.outQ = torch.zeros((rows, d), **f64)
        self.outP = torch.zeros((rows, d), **f64)
        self.valid = torch.zeros(rows, dtype=torch.bool, device=device)
        self.enabled = os.environ.get("PL_PARAREAL_NOCACHE", "0") in ("", "0")
        self.propagated = 0  # rows actually propagated (diagnostics)

    def run(self, rows, Qs, Ps, noise_of, run_fn):
        """rows: LongTensor of cache rows; Qs/Ps their start states; noise_of(pos)
        the noise rows of positions ``pos`` of ``rows``.  run_fn(Q, P, N) ->
        (FQ, FP, blow) propagates a (sub)batch.  Returns
        (FQ, FP, blow, positions) for all rows; blow/positions refer to the
        propagated subset (positions index into ``rows``)."""
        import torch
        if self.enabled:
            same = self.valid.index_select(0, rows)
            same &= (Qs.view(torch.int64) == self.inQ.index_select(0, rows).view(torch.int64)).all(dim=1)
            same &= (Ps.view(torch.int64) == self.inP.index_select(0, rows).view(torch.int64)).all(dim=1)
            pos = torch.nonzero(~same).squeeze(1)
        else:
            pos = torch.arange(rows.numel(), device=rows.device)
        blow = torch.zeros(0, dtype=torch.int32, device=rows.device)
        if pos.numel():
            sub = rows.index_select(0, pos)
            q0, p0 = Qs.index_select(0, pos), Ps.index_select(0, pos)
            FQ, FP, blow = run_fn(q0, p0, noise_of(pos).contiguous())
            self.inQ.index_copy_(0, sub, q0)
            self.inP.index_copy_(0, sub, p0)
            self.outQ.index_copy_(0, sub, FQ)
            self.outP.index_copy_(0, sub, FP)
            ok = (blow == 0)
            self.valid.index_copy_(0, sub, ok)
            self.propagated += int(pos.numel())
        return self.outQ.index_select(0, rows), self.outP.index_select(0, rows), blow, pos

    def fill(self, rows, q0, p0, FQ, FP, ok):
        """Store results computed elsewhere (speculative windows): ``ok`` (bool,
        per row) marks the rows whose propagation can be trusted."""
        self.inQ.index_copy_(0, rows, q0)
        self.inP.index_copy_(0, rows, p0)
        self.outQ.index_copy_(0, rows, FQ)
        self.outP.index_copy_(0, rows, FP)
        self.valid.index_copy_(0, rows, ok)


LAST_RUN_STATS: dict = {}  # diagnostics of the last single-run device engine (bench, tests)
_SWEEP_POOL = None           # one worker thread for blocking sweep calls (speculation)


def _spec_parts() -> int:
    """Speculative batches per sweep (PL_PARAREAL_SPEC_PARTS, default 2)."""
    import os
    try:
        return max(1, int(os.environ.get("PL_PARAREAL_SPEC_PARTS", "2")))
    except ValueError:
        return 2


def _sweep_pool():
    global _SWEEP_POOL
    if _SWEEP_POOL is None:
        from concurrent.futures import ThreadPoolExecutor
        _SWEEP_POOL = ThreadPoolExecutor(max_workers=1, thread_name_prefix="pl-sweep")
    return _SWEEP_POOL


def _spec_mode(fine, coarse, n: int, d: int) -> bool:
    """Speculative pipelining of the fine stage behind the sweep: PL_PARAREAL_SPEC=1
    turns it on (one rank, fine-window cache on, EAM coarse sweep on the cluster
    kernel, which publishes its progress).  Off by default: measured on one B200
    at the larger config it does not shorten the run (20.5 s plain; 20.9 s with 2
    speculative batches per sweep, 21.7 s with 4, 21.9 s with 8): the speculative
    batches run at lower efficiency than the full slab batch, the cluster sweep
    slows down next to them, and a batch of ~2000 launches fills the launch queue,
    so the host returns from it only near its end."""
    import os
    mode = os.environ.get("PL_PARAREAL_SPEC", "0")
    if mode != "1" or os.environ.get("PL_PARAREAL_NOCACHE", "0") not in ("", "0"):
        return False
    if world()[1] > 1 or getattr(fine.pot, "n_atoms", None) is None:
        return False
    ctx = _lib.context()
    return _lib.load().pl_sweep_path(coarse.pot.handle(ctx)) == 2  # progress comes from the cluster sweep


def _timed(key):
    """Accumulate the host wall time of a _DeviceRun method into self.t[key]."""
    import functools
    import time

    def deco(fn):
        @functools.wraps(fn)
        def wrap(self, *a, **kw):
            t0 = time.perf_counter()
            try:
                return fn(self, *a, **kw)
            finally:
                self.t[key] += time.perf_counter() - t0
        return wrap
    return deco


class _DeviceRun:
    """Device-resident trajectory + cached coarse outputs for one engine run."""

    def __init__(self, initial: PhaseState, fine: DevicePropagator, coarse: DevicePropagator, n: int):
        import torch
        self.fine, self.coarse, self.n, self.d = fine, coarse, n, initial.dim
        if fine.d != initial.dim or coarse.d != initial.dim:
            raise ValueError("propagator dimension does not match the initial state")
        if fine.plan.n_windows < n:
            raise ValueError(f"noise plan covers {fine.plan.n_windows} windows, need {n}")
        coarse.share_noise(fine)
        dev = fine.kernel.device
        d = self.d
        f64 = dict(dtype=torch.float64, device=dev)
        self.Q = torch.zeros((n + 1, d), **f64)
        self.P = torch.zeros((n + 1, d), **f64)
        self.Q[0] = torch.from_numpy(np.array(initial.q))
        self.P[0] = torch.from_numpy(np.array(initial.p))
        self.prevQ = torch.zeros((n + 1, d), **f64)
        self.baseQ = torch.zeros((n, d), **f64)
        self.baseP = torch.zeros((n, d), **f64)
        self.jumpQ = torch.zeros((n, d), **f64)
        self.jumpP = torch.zeros((n, d), **f64)
        self.hist = torch.zeros(n, **f64)
        self.noise_f = fine.noise_all()
        self.noise_c = coarse.noise_all()
        self.fcache = _FineCache(n, d, dev)
        self.spec = torch.cuda.Stream(device=dev) if _spec_mode(fine, coarse, n, d) else None
        self.spec_windows = 0  # speculative windows launched (diagnostics)
        self.t = {"bootstrap": 0.0, "jumps": 0.0, "sweep": 0.0, "speculate": 0.0}  # host wall seconds

    @_timed("bootstrap")
    def bootstrap(self, n_init: int) -> None:
        """cur[m+1] = C(cur[m]) for m = n_init..N-1 (parareal.py:404-405); caches base."""
        if self.spec is not None:  # speculative copies of the old nodes must be taken first
            import torch
            torch.cuda.current_stream(self.Q.device).wait_stream(self.spec)
        k = self.coarse.kernel
        lib, ctx = _lib.load(), _lib.context()
        out = np.zeros(1, dtype=np.int64)
        blow = np.zeros(1, dtype=np.int32)
        rc = lib.pl_bootstrap(
            ctx.handle, self.coarse.pot.handle(ctx), self.d, k.L, n_init, self.n, _lib.ptr(self.Q),
            _lib.ptr(self.P), _lib.ptr(self.baseQ), _lib.ptr(self.baseP), _lib.ptr(self.noise_c),
            _lib.dptr(k.amp), _lib.ptr(k.mass), k.dt, k.h, k.hg, out.ctypes.data_as(_lib.pi64),
            blow.ctypes.data_as(_lib.pi32))
        if rc == _lib.PL_EBLOWUP:
            m = int(out[0])
            raise BlowUpError(f"state left the trusted range at substep {int(blow[0])}",
                              substep=int(blow[0]), window=m + 1, iteration=0)
        _lib.check(rc)

    @_timed("jumps")
    def jumps(self, n_init: int, n_final: int, iteration: int) -> None:
        """jump[m] = F(prev[m]) - C(prev[m]) for all slab windows.

        One batched launch per rank: with several ranks (torch.distributed
        initialised) each propagates a contiguous block of windows and one
        all-gather of the endpoints gives every rank the full set
        (distributed.sharded_fine).
        """
        import torch
        W = n_final - n_init
        if self.spec is not None:  # speculative windows of the last sweep must have landed in the cache
            torch.cuda.current_stream(self.Q.device).wait_stream(self.spec)

        def run_fn(q0, p0, nz):
            def run_block(lo, hi):
                return self.fine.kernel.run(q0[lo:hi].contiguous(), p0[lo:hi].contiguous(), nz[lo:hi])
            return sharded_fine(run_block, 0, q0.shape[0])

        rows = torch.arange(n_init, n_final, device=self.Q.device)
        nz = self.noise_f[n_init:n_final]
        FQ, FP, blow, pos = self.fcache.run(rows, self.Q[n_init:n_final], self.P[n_init:n_final],
                                            lambda p_: nz.index_select(0, p_), run_fn)
        b = blow.cpu().numpy()
        bad = np.nonzero(b)[0]
        if bad.size:
            i = int(pos[int(bad[0])])
            raise BlowUpError(
                f"state left the trusted range (|component| > 1e+12 or non-finite) at substep {b[bad[0]]}",
                substep=int(b[bad[0]]), window=n_init + i + 1, iteration=iteration)
        lib, ctx = _lib.load(), _lib.context()
        n = W * self.d
        _lib.check(lib.pl_sub(ctx.handle, n, _lib.ptr(FQ), _lib.ptr(self.baseQ[n_init:n_final]),
                              _lib.ptr(self.jumpQ[n_init:n_final])))
        _lib.check(lib.pl_sub(ctx.handle, n, _lib.ptr(FP), _lib.ptr(self.baseP[n_init:n_final]),
                              _lib.ptr(self.jumpP[n_init:n_final])))

    def snapshot_prev(self, n_init: int, n_final: int) -> None:
        self.prevQ[n_init:n_final + 1].copy_(self.Q[n_init:n_final + 1])

    @_timed("speculate")
    def _speculate(self, lo: int, hi: int) -> None:
        """Fine windows lo..hi-1 of the NEXT iteration from nodes the running sweep
        has finalised, launched on the second stream (the sweep kernel keeps its
        SMs; these windows fill the others).  Results go to the fine-window cache
        keyed by their exact start state, so the next jumps() uses them only if
        it asks for the same start bit for bit: no result changes (wasted work if
        the slab converges or shrinks instead)."""
        import torch
        if hi <= lo:
            return
        lib = _lib.load()
        with torch.cuda.stream(self.spec):
            ctx = _lib.context()
            q0 = self.Q[lo:hi].clone()   # later sweeps may overwrite the nodes
            p0 = self.P[lo:hi].clone()
            _lib.check(lib.pl_ctx_set_spec(ctx.handle, 1))
            try:
                FQ, FP, blow = self.fine.kernel.run(q0, p0, self.noise_f[lo:hi])
                over = torch.zeros(1, dtype=torch.int32, device=self.Q.device)
                _lib.check(lib.pl_pot_overflow_async(ctx.handle, self.fine.pot.handle(ctx), _lib.ptr(over)))
            finally:
                _lib.check(lib.pl_ctx_set_spec(ctx.handle, 0))
            rows = torch.arange(lo, hi, device=self.Q.device)
            self.fcache.fill(rows, q0, p0, FQ, FP, (blow == 0) & (over == 0))
        _lib.context()  # rebind the library stream to the main stream
        self.spec_windows += hi - lo

    def _sweep_call(self, main_stream, n_init, n_final, include_m0, expl, state, out, blow, progress):
        """pl_sweep on the main stream; in the worker thread when speculating (own
        library context, so the main thread can launch on the second stream)."""
        import ctypes as C

        import torch
        k = self.coarse.kernel
        lib = _lib.load()
        with torch.cuda.stream(main_stream):
            ctx = _lib.context()
            if progress is not None:
                ptr = C.c_void_p()
                _lib.check(lib.pl_ctx_enable_progress(ctx.handle, C.byref(ptr)))
                cnt = C.c_int64.from_address(ptr.value)
                cnt.value = 0  # (the launch resets it too) never expose the last sweep's count
                progress.append(cnt)
            rc = lib.pl_sweep(
                ctx.handle, self.coarse.pot.handle(ctx), self.d, k.L, n_init, n_final,
                1 if include_m0 else 0, _lib.ptr(self.Q), _lib.ptr(self.P), _lib.ptr(self.prevQ),
                _lib.ptr(self.baseQ), _lib.ptr(self.baseP), _lib.ptr(self.jumpQ), _lib.ptr(self.jumpP),
                _lib.ptr(self.noise_c), _lib.dptr(k.amp), _lib.ptr(k.mass), k.dt, k.h, k.hg,
                float(expl), _lib.dptr(state), _lib.ptr(self.hist),
                out.ctypes.data_as(_lib.pi64), blow.ctypes.data_as(_lib.pi32))
            # the error text is per host thread: take it here
            return rc, (lib.pl_last_error().decode(errors="replace") if rc != _lib.PL_OK else "")

    @_timed("sweep")
    def sweep(self, n_init: int, n_final: int, include_m0: bool, expl: float, iteration: int,
              front: int | None = None):
        """Corrected sweep on the device; returns (deltas, den) for the nodes updated.

        With speculation on, the (blocking) sweep call runs in a worker thread and
        this thread follows the kernel's host-mapped progress counter: as windows
        finish, the next iteration's fine windows starting on their nodes are
        launched on the second stream (windows below ``front``, whose start nodes
        are frozen behind the exactness front, are cache hits and skipped).
        """
        import time

        import torch
        state = np.zeros(2)
        out = np.zeros(1, dtype=np.int64)
        blow = np.zeros(1, dtype=np.int32)
        main = torch.cuda.current_stream(self.Q.device)
        if self.spec is None:
            rc, msg = self._sweep_call(main, n_init, n_final, include_m0, expl, state, out, blow, None)
        else:
            progress = []
            fut = _sweep_pool().submit(self._sweep_call, main, n_init, n_final, include_m0, expl, state, out,
                                    blow, progress)
            lo = max(n_init + 1, front if front is not None else n_init + 1)
            batch = max(1, -(-(n_final - n_init) // _spec_parts()))
            while True:
                finished = fut.done()
                done = int(progress[0].value) if progress else 0
                # windows whose start node n_init + done is final: n_init+1 .. n_init+done
                hi = min(n_init + done + 1, n_final)
                if hi - lo >= batch:
                    self._speculate(lo, hi)
                    lo = hi
                if finished:
                    break
                time.sleep(0.0002)
            rc, msg = fut.result()
        if rc == _lib.PL_EBLOWUP:
            m = int(out[0])
            if blow[0]:
                raise BlowUpError(f"coarse window blew up at substep {int(blow[0])}",
                                  substep=int(blow[0]), window=m + 1, iteration=iteration)
            raise BlowUpError(f"corrected state is not finite at window {m + 1} "
                              f"(iteration {iteration})", window=m + 1, iteration=iteration)
        if rc != _lib.PL_OK:
            raise _lib.CallError(rc, msg)
        n_done = int(out[0])
        deltas = self.hist[:n_done].cpu().numpy()
        return deltas, state[1]

    def trajectory(self) -> NodeTrajectory:
        return NodeTrajectory.from_arrays(self.Q.cpu().numpy(), self.P.cpu().numpy())


def _is_device(fine, coarse) -> bool:
    return isinstance(fine, DevicePropagator) and isinstance(coarse, DevicePropagator)


# ======================================================================
# engines
def sequential_propagate(initial: PhaseState, n_windows: int, pot, params: LangevinParams,
                         schedule: TemperatureSchedule, plan: NoisePlan) -> NodeTrajectory:
    """Chain n_windows fine windows on the device; node n+1 uses seed n+1."""
    if n_windows < 0:
        raise ValueError(f"n_windows must be >= 0, got {n_windows}")
    if plan.n_windows < n_windows:
        raise ValueError(f"noise plan covers {plan.n_windows} windows, need {n_windows}")
    if n_windows == 0:
        return NodeTrajectory((initial,))
    import torch
    prop = _window_propagator(pot, params, schedule, plan, initial.dim)
    k = prop.kernel
    noise = k.noise(np.asarray(plan.window_seeds[:n_windows], dtype=np.uint64))
    d = initial.dim
    Q = torch.empty((n_windows + 1, d), dtype=torch.float64, device=k.device)
    P = torch.empty_like(Q)
    Q[0] = torch.from_numpy(np.array(initial.q))
    P[0] = torch.from_numpy(np.array(initial.p))
    blows = torch.zeros(n_windows, dtype=torch.int32, device=k.device)
    for m in range(n_windows):
        _, _, b = k.run(Q[m:m + 1], P[m:m + 1], noise[m:m + 1], Q[m + 1:m + 2], P[m + 1:m + 2])
        blows[m:m + 1].copy_(b)
    bl = blows.cpu().numpy()
    bad = np.nonzero(bl)[0]
    if bad.size:
        m = int(bad[0])
        raise BlowUpError(f"state left the trusted range at substep {bl[m]}", substep=int(bl[m]),
                          window=m + 1, iteration=0)
    return NodeTrajectory.from_arrays(Q.cpu().numpy(), P.cpu().numpy())


def _classic_device(initial, fine, coarse, config, record_iterates):
    n = config.n_windows
    run = _DeviceRun(initial, fine, coarse, n)
    run.bootstrap(0)
    iterates = [run.trajectory()] if record_iterates else None
    history = []
    k = 0
    delta = 2.0 * config.delta_conv
    while delta >= config.delta_conv:
        if k >= config.iteration_cap:
            break
        k += 1
        run.jumps(0, n, k)
        run.snapshot_prev(0, n)
        deltas, den = run.sweep(0, n, False, 0.0, k)
        if den == 0.0:
            raise DegenerateNormalizationError(f"all reference positions on nodes 1..{n} are zero")
        delta = float(deltas[-1])
        history.append((1, k, delta))
        if record_iterates:
            iterates.append(run.trajectory())
    attempts = []
    _close_attempt(attempts, 0, n, k)
    slab = SlabRecord(slab_index=1, n_init=0, attempts=tuple(attempts), n_final=n, k_conv=k)
    return PararealResult(trajectory=run.trajectory(), slabs=(slab,), error_history=tuple(history),
                          converged=delta < config.delta_conv,
                          iterates=tuple(iterates) if record_iterates else None)


def _adaptive_machine(n, conv, expl, cap):
    """Algorithm 2 (parareal.py:366-475) as a generator of device actions.

    Yields ('bootstrap', n_init) and ('iterate', n_init, n_final, include_m0,
    iteration); an 'iterate' is answered with (deltas, den) of the sweep.
    Returns (slabs, history, converged).  The single-run and the replica-batch
    engines drive this same machine, so both take the reference's decisions.
    """
    mid = 0.5 * (conv + expl)
    n_init = n_final = 0
    delta = mid
    n_slab = 0
    slabs, history, attempts = [], [], []
    k_in_slab = 0
    converged = True
    while n_final < n:
        if delta < expl:
            n_init, n_final = n_final, n
            yield ("bootstrap", n_init)
            n_slab += 1
            attempts = []
            k_in_slab = 0
        delta = mid
        k_attempt = 0
        aborted = False
        while conv <= delta <= expl:
            if k_attempt >= cap:
                aborted = True
                break
            deltas, den = yield ("iterate", n_init, n_final, n_init >= 1, k_in_slab + 1)
            k_attempt += 1
            k_in_slab += 1
            for dl in deltas:
                history.append((n_slab, k_in_slab, float(dl)))
                delta = float(dl)
            if den == 0.0:
                raise DegenerateNormalizationError(
                    f"all reference positions on nodes {max(n_init, 1)}..{n_init + len(deltas)} are zero")
            if delta > expl:
                m = n_init + len(deltas) - 1
                if m == n_init:
                    raise SlabCollapseError(
                        f"slab {n_slab} exploded at its first window {n_init + 1}; no shorter slab exists",
                        slab_index=n_slab, n_init=n_init)
                _close_attempt(attempts, n_init, n_final, k_attempt)
                n_final = m
        if aborted:
            _close_attempt(attempts, n_init, n_final, k_attempt)
            slabs.append(SlabRecord(n_slab, n_init, tuple(attempts), n_final,
                                    sum(a.iterations for a in attempts)))
            converged = False
            break
        if delta < conv:
            _close_attempt(attempts, n_init, n_final, k_attempt)
            slabs.append(SlabRecord(n_slab, n_init, tuple(attempts), n_final,
                                    sum(a.iterations for a in attempts)))
    return slabs, history, converged


def _drive_adaptive(machine, run):
    """Answer the machine's actions with ``run.bootstrap`` / ``run.iterate``."""
    reply = None
    try:
        while True:
            act = machine.send(reply)
            if act[0] == "bootstrap":
                run.bootstrap(act[1])
                reply = None
            else:
                reply = run.iterate(*act[1:])
    except StopIteration as stop:
        return stop.value


def _adaptive_device(initial, fine, coarse, config):
    n = config.n_windows
    run = _DeviceRun(initial, fine, coarse, n)
    expl = config.delta_expl

    class _Dev:
        bootstrap = staticmethod(run.bootstrap)

        @staticmethod
        def iterate(n_init, n_final, inc, it):
            run.jumps(n_init, n_final, it)
            run.snapshot_prev(n_init, n_final)
            # node n_init + j is bitwise frozen from iteration j of the slab on, so after
            # iteration `it` the windows starting below n_init + it are cache hits
            return run.sweep(n_init, n_final, inc, expl, it, front=n_init + it)

    machine = _adaptive_machine(n, config.delta_conv, expl, config.iteration_cap)
    slabs, history, converged = _drive_adaptive(machine, _Dev)
    LAST_RUN_STATS.update(fine_windows_propagated=run.fcache.propagated, speculative_windows=run.spec_windows,
                          speculation=run.spec is not None, host_s=dict(run.t))
    return PararealResult(trajectory=run.trajectory(), slabs=tuple(slabs),
                          error_history=tuple(history), converged=converged)


class _BatchRun:
    """R independent replicas (own initial state and noise plan) on one device."""

    def __init__(self, initials, fine_pot, coarse_pot, params, schedule, plans, n):
        import torch
        self.R, self.n = len(initials), n
        d = initials[0].dim
        self.d = d
        self.fk = WindowKernel(fine_pot, params, schedule, d)
        self.ck = WindowKernel(coarse_pot, params, schedule, d)
        self.coarse_pot = coarse_pot
        dev = self.fk.device
        f64 = dict(dtype=torch.float64, device=dev)
        R, L = self.R, self.fk.L
        self.Q = torch.zeros((R, n + 1, d), **f64)
        self.P = torch.zeros((R, n + 1, d), **f64)
        for r, st in enumerate(initials):
            self.Q[r, 0] = torch.from_numpy(np.array(st.q))
            self.P[r, 0] = torch.from_numpy(np.array(st.p))
        self.baseQ = torch.zeros((R, n, d), **f64)
        self.baseP = torch.zeros((R, n, d), **f64)
        self.jumpQ = torch.zeros((R, n, d), **f64)
        self.jumpP = torch.zeros((R, n, d), **f64)
        self.hist = torch.zeros((R, n), **f64)
        seeds = np.concatenate([np.asarray(p.window_seeds[:n], dtype=np.uint64) for p in plans])
        self.noise = self.fk.noise(seeds).reshape(R, n, (L + 1) * d)
        self.fcache = _FineCache(R * n, d, dev)

    def _batch_call(self, slots, mode, expl):
        import numpy as np_
        lib, ctx = _lib.load(), _lib.context()
        k = self.ck
        Ra = len(slots)
        ridx = np_.array([r for r, _, _, _ in slots], dtype=np_.int32)
        m0 = np_.array([a for _, a, _, _ in slots], dtype=np_.int64)
        m1 = np_.array([b for _, _, b, _ in slots], dtype=np_.int64)
        inc = np_.array([1 if c else 0 for _, _, _, c in slots], dtype=np_.int32)
        state = np_.zeros(2 * Ra)
        out4 = np_.zeros(4 * Ra, dtype=np_.int64)
        rc = lib.pl_sweep_batch(
            ctx.handle, self.coarse_pot.handle(ctx), self.d, k.L, self.n, Ra, ridx.ctypes.data_as(_lib.pi32),
            m0.ctypes.data_as(_lib.pi64), m1.ctypes.data_as(_lib.pi64), inc.ctypes.data_as(_lib.pi32), mode,
            _lib.ptr(self.Q), _lib.ptr(self.P), _lib.ptr(self.baseQ), _lib.ptr(self.baseP),
            _lib.ptr(self.jumpQ), _lib.ptr(self.jumpP), _lib.ptr(self.noise), _lib.dptr(k.amp),
            _lib.ptr(k.mass), k.dt, k.h, k.hg, float(expl), _lib.dptr(state),
            out4.ctypes.data_as(_lib.pi64), _lib.ptr(self.hist))
        _lib.check(rc)
        return state.reshape(Ra, 2), out4.reshape(Ra, 4)

    def bootstrap(self, items):
        """items: [(replica, n_init)]"""
        slots = [(r, a, self.n, False) for r, a in items]
        _, out4 = self._batch_call(slots, 1, 0.0)
        for (r, a), o in zip(items, out4):
            if o[3] == 1:
                raise BlowUpError(f"replica {r}: coarse bootstrap blew up at substep {int(o[2])}",
                                  substep=int(o[2]), window=int(o[1]) + 1, iteration=0)

    def iterate(self, items, expl):
        """items: [(replica, n_init, n_final, include_m0, iteration)] -> [(deltas, den)]"""
        import torch
        d, n = self.d, self.n
        rows_q = torch.tensor([r * (n + 1) + m for r, a, b, _, _ in items for m in range(a, b)],
                              dtype=torch.long, device=self.Q.device)
        rows_w = torch.tensor([r * n + m for r, a, b, _, _ in items for m in range(a, b)],
                              dtype=torch.long, device=self.Q.device)
        Qs = self.Q.view(-1, d).index_select(0, rows_q)
        Ps = self.P.view(-1, d).index_select(0, rows_q)
        Ns = self.noise.view(-1, self.noise.shape[-1])

        def run_fn(q0, p0, nz):
            def run_block(lo, hi):
                return self.fk.run(q0[lo:hi].contiguous(), p0[lo:hi].contiguous(), nz[lo:hi].contiguous())
            return sharded_fine(run_block, 0, q0.shape[0])

        FQ, FP, blow, pos = self.fcache.run(rows_w, Qs, Ps, lambda p_: Ns.index_select(0, rows_w.index_select(0, p_)),
                                            run_fn)
        b = blow.cpu().numpy()
        if b.any():
            i = int(np.nonzero(b)[0][0])
            raise BlowUpError(f"fine window blew up at substep {int(b[i])} (batch row {int(pos[i])})",
                              substep=int(b[i]))
        lib, ctx = _lib.load(), _lib.context()
        bq = self.baseQ.view(-1, d).index_select(0, rows_w)
        bp = self.baseP.view(-1, d).index_select(0, rows_w)
        jq = torch.empty_like(bq)
        jp = torch.empty_like(bp)
        _lib.check(lib.pl_sub(ctx.handle, jq.numel(), _lib.ptr(FQ), _lib.ptr(bq), _lib.ptr(jq)))
        _lib.check(lib.pl_sub(ctx.handle, jp.numel(), _lib.ptr(FP), _lib.ptr(bp), _lib.ptr(jp)))
        self.jumpQ.view(-1, d).index_copy_(0, rows_w, jq)
        self.jumpP.view(-1, d).index_copy_(0, rows_w, jp)
        slots = [(r, a, b, inc) for r, a, b, inc, _ in items]
        state, out4 = self._batch_call(slots, 0, expl)
        hist = self.hist.cpu().numpy()
        res = []
        for (r, a, b_, inc, it), st, o in zip(items, state, out4):
            if o[3] == 1:
                raise BlowUpError(f"replica {r}: coarse window blew up at substep {int(o[2])}",
                                  substep=int(o[2]), window=int(o[1]) + 1, iteration=it)
            if o[3] == 2:
                raise BlowUpError(f"replica {r}: corrected state is not finite at window {int(o[1]) + 1}",
                                  window=int(o[1]) + 1, iteration=it)
            res.append((hist[r, :int(o[0])].copy(), float(st[1])))  # hist[r, m - m0]
        return res

    def trajectory(self, r):
        return NodeTrajectory.from_arrays(self.Q[r].cpu().numpy(), self.P[r].cpu().numpy())


def parareal_adaptive_batch(initials, pair: PropagatorPair, params: LangevinParams,
                            schedule: TemperatureSchedule, plans, config: PararealConfig):
    """Adaptive parareal for many independent replicas at once (ensemble protocol).

    Replica r starts from ``initials[r]`` with noise plan ``plans[r]`` and runs
    exactly the reference algorithm (the same ``_adaptive_machine``); the
    device work of all replicas is batched: one bootstrap launch, one
    fine-stage launch (slices x replicas, sharded over ranks) and one sweep
    launch (one persistent CTA per replica) per round.  Returns one
    ``PararealResult`` per replica.
    """
    if config.delta_expl is None:
        raise ValueError("adaptive mode needs delta_expl in the configuration")
    n = config.n_windows
    for p in plans:
        _check_plan(p, n)
    run = _BatchRun(initials, pair.fine, pair.coarse, params, schedule, plans, n)
    machines = [_adaptive_machine(n, config.delta_conv, config.delta_expl, config.iteration_cap)
                for _ in initials]
    results = [None] * len(initials)
    pending = {}
    for r, mch in enumerate(machines):
        pending[r] = next(mch)
    while pending:
        boots = [(r, act[1]) for r, act in pending.items() if act[0] == "bootstrap"]
        replies = {}
        if boots:
            run.bootstrap(boots)
            for r, _ in boots:
                replies[r] = None
        else:
            its = [(r,) + act[1:] for r, act in pending.items()]
            for (r, *_), rep in zip(its, run.iterate(its, config.delta_expl)):
                replies[r] = rep
        for r, rep in replies.items():
            try:
                pending[r] = machines[r].send(rep)
            except StopIteration as stop:
                slabs, history, converged = stop.value
                results[r] = PararealResult(trajectory=run.trajectory(r), slabs=tuple(slabs),
                                            error_history=tuple(history), converged=converged)
                del pending[r]
    return results


# ---- generic control flow over arbitrary callables (scripted propagators)
def _accumulate(num, den, prev_state, cur_state):
    num += float(np.linalg.norm(cur_state.q - prev_state.q))
    den += float(np.linalg.norm(prev_state.q))
    return num, den


def _compute_jumps(fine, coarse, states, window_indices, iteration):
    out = []
    for m in window_indices:
        f = _call(fine, states[m], m, iteration)
        c = _call(coarse, states[m], m, iteration)
        out.append((f.q - c.q, f.p - c.p))
    return out


def _corrected(coarse, state, m, iteration, jump):
    base = _call(coarse, state, m, iteration)
    try:
        return PhaseState(q=base.q + jump[0], p=base.p + jump[1])
    except ValueError as err:
        raise BlowUpError(f"corrected state is not finite at window {m + 1} (iteration {iteration})",
                          window=m + 1, iteration=iteration) from err


class _HostRun:
    """The adaptive machine's actions for arbitrary callables (parareal.py:399-445):
    bootstrap by coarse windows, jump stage, corrected sweep truncated at the
    first node whose running error exceeds delta_expl."""

    def __init__(self, initial, fine, coarse, n, expl):
        self.fine, self.coarse, self.expl = fine, coarse, expl
        self.cur = [initial] + [None] * n

    def bootstrap(self, n_init):
        cur = self.cur
        for m in range(n_init, len(cur) - 1):
            cur[m + 1] = _call(self.coarse, cur[m], m, 0)

    def iterate(self, n_init, n_final, include_m0, iteration):
        cur = self.cur
        prev = list(cur)
        jumps = _compute_jumps(self.fine, self.coarse, prev, range(n_init, n_final), iteration)
        num = den = 0.0
        if include_m0:
            num, den = _accumulate(num, den, prev[n_init], cur[n_init])
        deltas = []
        for m in range(n_init, n_final):
            cur[m + 1] = _corrected(self.coarse, cur[m], m, iteration, jumps[m - n_init])
            num, den = _accumulate(num, den, prev[m + 1], cur[m + 1])
            if den == 0.0:  # the machine raises for nodes max(n_init, 1)..m+1
                deltas.append(float("nan"))
                return deltas, den
            deltas.append(num / den)
            if deltas[-1] > self.expl:
                break
        return deltas, den


def parareal_classic_engine(initial: PhaseState, fine: WindowPropagator, coarse: WindowPropagator,
                            config: PararealConfig, workers: int | None = None,
                            record_iterates: bool = False) -> PararealResult:
    """Classic parareal (Algorithm 1); device-resident when both propagators are device ones."""
    if _is_device(fine, coarse):
        return _classic_device(initial, fine, coarse, config, record_iterates)
    n = config.n_windows
    cur = [initial]
    for m in range(n):
        cur.append(_call(coarse, cur[m], m, 0))
    iterates = [NodeTrajectory(tuple(cur))] if record_iterates else None
    history = []
    k = 0
    delta = 2.0 * config.delta_conv
    while delta >= config.delta_conv:
        if k >= config.iteration_cap:
            break
        k += 1
        prev = list(cur)
        jumps = _compute_jumps(fine, coarse, prev, range(n), k)
        num = den = 0.0
        for m in range(n):
            cur[m + 1] = _corrected(coarse, cur[m], m, k, jumps[m])
            num, den = _accumulate(num, den, prev[m + 1], cur[m + 1])
        if den == 0.0:
            raise DegenerateNormalizationError(f"all reference positions on nodes 1..{n} are zero")
        delta = num / den
        history.append((1, k, delta))
        if record_iterates:
            iterates.append(NodeTrajectory(tuple(cur)))
    attempts = []
    _close_attempt(attempts, 0, n, k)
    slab = SlabRecord(slab_index=1, n_init=0, attempts=tuple(attempts), n_final=n, k_conv=k)
    return PararealResult(trajectory=NodeTrajectory(tuple(cur)), slabs=(slab,),
                          error_history=tuple(history), converged=delta < config.delta_conv,
                          iterates=tuple(iterates) if record_iterates else None)


def parareal_adaptive_engine(initial: PhaseState, fine: WindowPropagator, coarse: WindowPropagator,
                             config: PararealConfig, workers: int | None = None) -> PararealResult:
    """Adaptive slab-shortening parareal (Algorithm 2)."""
    if config.delta_expl is None:
        raise ValueError("adaptive mode needs delta_expl in the configuration")
    if _is_device(fine, coarse):
        return _adaptive_device(initial, fine, coarse, config)
    run = _HostRun(initial, fine, coarse, config.n_windows, config.delta_expl)
    machine = _adaptive_machine(config.n_windows, config.delta_conv, config.delta_expl, config.iteration_cap)
    slabs, history, converged = _drive_adaptive(machine, run)
    return PararealResult(trajectory=NodeTrajectory(tuple(run.cur)), slabs=tuple(slabs),
                          error_history=tuple(history), converged=converged)


def _check_plan(plan: NoisePlan, n_windows: int) -> None:
    if plan.n_windows < n_windows:
        raise ValueError(f"noise plan covers {plan.n_windows} windows, need {n_windows}")


def parareal_classic(initial: PhaseState, pair: PropagatorPair, params: LangevinParams,
                     schedule: TemperatureSchedule, plan: NoisePlan, config: PararealConfig,
                     workers: int | None = None, record_iterates: bool = False) -> PararealResult:
    _check_plan(plan, config.n_windows)
    return parareal_classic_engine(
        initial, _window_propagator(pair.fine, params, schedule, plan, initial.dim),
        _window_propagator(pair.coarse, params, schedule, plan, initial.dim), config,
        workers=workers, record_iterates=record_iterates)


def parareal_adaptive(initial: PhaseState, pair: PropagatorPair, params: LangevinParams,
                      schedule: TemperatureSchedule, plan: NoisePlan, config: PararealConfig,
                      workers: int | None = None) -> PararealResult:
    _check_plan(plan, config.n_windows)
    return parareal_adaptive_engine(
        initial, _window_propagator(pair.fine, params, schedule, plan, initial.dim),
        _window_propagator(pair.coarse, params, schedule, plan, initial.dim), config,
        workers=workers)
