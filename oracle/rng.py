"""Oracle restatement of the reference noise generator (TEST INFRASTRUCTURE).

Follows /root/reference/pkg/src/paralangevin/rng.py:
  * SplitMix64 finalizer ........................ rng.py:31-45
  * per-window seed  mix(master ^ n*GOLDEN) ....... rng.py:57-78
  * j-th uniform  (mix(seed+(j+1)*GOLDEN)>>11)*2^-53  rng.py:81-84
  * Marsaglia polar, pairs in counter order, odd count drops the last y,
    scalar ``math.log`` path below 16 variates, numpy ``np.log`` above
    ............................................. rng.py:87-185
The stream is prefix-stable: the first ``count`` variates of the infinite
accepted-pair stream.  This module computes it chunk-wise instead of the
reference's oversample-and-retry loop; outputs are bitwise identical (pinned
by tests/golden/rng_golden.npz).
"""

from __future__ import annotations

import math

import numpy as np

MASK64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15
U53 = 2.0 ** -53
SCALAR_CUTOFF = 16


def mix(z: int) -> int:
    z &= MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def mix_u64(z: np.ndarray) -> np.ndarray:
    z = z ^ (z >> np.uint64(30))
    z = z * np.uint64(0xBF58476D1CE4E5B9)
    z = z ^ (z >> np.uint64(27))
    z = z * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def derive_seed(master: int, n: int) -> int:
    return mix(master ^ ((n * GOLDEN) & MASK64))


def derive_seeds(master: int, n_windows: int) -> np.ndarray:
    n = np.arange(1, n_windows + 1, dtype=np.uint64)
    return mix_u64(np.uint64(master) ^ (n * np.uint64(GOLDEN)))


def uniforms(seed: int, j0: int, n: int) -> np.ndarray:
    """Uniforms j0 .. j0+n-1 of the counter stream of ``seed``."""
    j = np.arange(j0 + 1, j0 + n + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = mix_u64(np.uint64(seed) + j * np.uint64(GOLDEN))
    return (z >> np.uint64(11)).astype(np.float64) * U53


def accepted_pairs(seed: int, pair0: int, npairs: int):
    """Candidate pairs pair0..pair0+npairs-1: (x, y, s, accept mask)."""
    u = uniforms(seed, 2 * pair0, 2 * npairs)
    x = 2.0 * u[0::2] - 1.0
    y = 2.0 * u[1::2] - 1.0
    s = x * x + y * y
    return x, y, s, (s > 0.0) & (s < 1.0)


def gaussian_stream(seed: int, count: int) -> np.ndarray:
    """``count`` N(0,1) variates, bitwise equal to rng.py:154-167."""
    if count == 0:
        return np.empty(0)
    out = np.empty(count + 1)
    filled = 0
    pair0 = 0
    scalar = count < SCALAR_CUTOFF
    while filled < count:
        need = (count - filled + 1) // 2
        npairs = need + (need >> 2) + 8
        x, y, s, acc = accepted_pairs(seed, pair0, npairs)
        pair0 += npairs
        xs, ys, ss = x[acc], y[acc], s[acc]
        if scalar:
            f = np.array([math.sqrt(-2.0 * math.log(v) / v) for v in ss])
        else:
            f = np.sqrt(-2.0 * np.log(ss) / ss)
        take = min(len(ss), need)
        inter = np.empty(2 * take)
        inter[0::2] = (xs * f)[:take] if take else inter[0::2]
        inter[1::2] = (ys * f)[:take] if take else inter[1::2]
        out[filled:filled + 2 * take] = inter
        filled += 2 * take
    return out[:count].copy()


def gaussian_streams(seeds, count: int) -> np.ndarray:
    seeds = np.asarray(seeds, dtype=np.uint64)
    return np.stack([gaussian_stream(int(s), count) for s in seeds]) if len(seeds) else np.empty((0, count))
