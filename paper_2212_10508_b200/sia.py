"""SIA hop detection and residence statistics.

``sia_site_labels`` labels every node of one or many trajectories on the
device (``pl_sia_sites``: Wigner-Seitz occupancy of the perfect BCC lattice).
``residence_times`` and ``mean_ci`` restate the reference's post-processing
(analysis.py:114-174) so the ensemble statistics follow the same conventions:
run-length encoding with an optional hysteresis ``min_run``, the final run
censored, and a normal 95 % interval mean +- 1.96 s / sqrt(n).
"""

from __future__ import annotations

import math
from typing import NamedTuple

import numpy as np

from . import _lib


class ResidenceEvent(NamedTuple):
    basin: int
    duration: int
    censored: bool


class InsufficientDataError(ValueError):
    """Fewer than two complete residence events."""


def sia_site_labels(positions, n_cells: int, a: float) -> np.ndarray:
    """(T,) or (R, T) int labels for positions of shape (T, 3N) or (R, T, 3N)."""
    import torch
    ctx = _lib.context()
    Q = torch.as_tensor(positions, dtype=torch.float64).to(torch.device("cuda", ctx.device)).contiguous()
    shape = Q.shape[:-1]
    Qf = Q.reshape(-1, Q.shape[-1])
    out = torch.empty(Qf.shape[0], dtype=torch.int32, device=Qf.device)
    _lib.check(_lib.load().pl_sia_sites(ctx.handle, Qf.shape[0], Qf.shape[1] // 3, int(n_cells), float(a),
                                        _lib.ptr(Qf), _lib.ptr(out)))
    return out.cpu().numpy().reshape(shape)


def _debounce(labels: np.ndarray, min_run: int) -> np.ndarray:
    out = np.empty_like(labels)
    current = labels[0]
    i, n = 0, len(labels)
    while i < n:
        j = i
        while j < n and labels[j] == labels[i]:
            j += 1
        if i == 0 or j - i >= min_run:
            current = labels[i]
        out[i:j] = current
        i = j
    return out


def residence_times(labels, min_run: int = 1):
    """Run-length encoding of a label sequence; the last run is censored (analysis.py:114-156)."""
    if min_run < 1:
        raise ValueError(f"min_run must be >= 1, got {min_run}")
    labels = np.asarray(labels)
    if labels.size == 0:
        return []
    if labels.ndim != 1:
        raise ValueError("labels must form a one-dimensional sequence")
    if min_run > 1:
        labels = _debounce(labels, min_run)
    events, start = [], 0
    for i in range(1, len(labels)):
        if labels[i] != labels[start]:
            events.append(ResidenceEvent(int(labels[start]), i - start, False))
            start = i
    events.append(ResidenceEvent(int(labels[start]), len(labels) - start, True))
    return events


def mean_ci(durations):
    """Mean with normal 95 % interval (analysis.py:159-174)."""
    values = np.asarray(durations, dtype=float)
    if values.size < 2:
        raise InsufficientDataError(f"need at least 2 complete residence events, got {values.size}")
    if np.any(values <= 0):
        raise ValueError("residence durations must be positive")
    mean = float(np.mean(values))
    half = 1.96 * float(np.std(values, ddof=1)) / math.sqrt(values.size)
    return mean, mean - half, mean + half


class ResidenceStats(NamedTuple):
    """Residence-time summary of a pooled ensemble (analysis.py:177-226)."""

    mean: float
    ci_low: float
    ci_high: float
    n_events: int
    censored: int

    def as_dict(self) -> dict:
        return {"mean": self.mean, "ci_low": self.ci_low, "ci_high": self.ci_high,
                "n_events": self.n_events, "censored": self.censored}


class EnsembleComparison(NamedTuple):
    overlap: bool
    intervals: tuple


def residence_stats(events) -> ResidenceStats:
    """Censored events are counted but never enter the mean (analysis.py:213-229)."""
    complete = [e.duration for e in events if not e.censored]
    censored = sum(1 for e in events if e.censored)
    mean, lo, hi = mean_ci(complete)
    return ResidenceStats(mean, lo, hi, len(complete), censored)


def compare_ensembles(a: ResidenceStats, b: ResidenceStats) -> EnsembleComparison:
    """Do the two 95 % intervals intersect? (analysis.py:232-238)"""
    return EnsembleComparison(bool(a.ci_low <= b.ci_high and b.ci_low <= a.ci_high),
                              ((a.ci_low, a.ci_high), (b.ci_low, b.ci_high)))
