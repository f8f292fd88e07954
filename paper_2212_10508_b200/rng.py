"""Counter-based noise, API-compatible with the reference's rng module.

  derive_seed / derive_seeds   rng.py:57-78   SplitMix64(master ^ n*GOLDEN)
  gaussian_stream(s)           rng.py:154-185 Marsaglia polar on counter uniforms
  NoisePlan                    rng.py:188-223
Seeds are 64-bit integer bookkeeping done on the host (they are the plan,
not the hot path).  Gaussian streams are generated on the device by
``pl_gaussian_streams``; the host functions below copy results back for API
compatibility, while the engines keep the streams resident in HBM.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib

_MASK64 = (1 << 64) - 1
_GOLDEN = 0x9E3779B97F4A7C15


def _mix(z: int) -> int:
    z &= _MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK64
    return z ^ (z >> 31)


def _check_u64(value, name: str) -> int:
    if not isinstance(value, (int, np.integer)):
        raise TypeError(f"{name} must be an integer, got {type(value).__name__}")
    value = int(value)
    if not 0 <= value <= _MASK64:
        raise ValueError(f"{name} must be in [0, 2^64), got {value}")
    return value


def derive_seed(master_seed: int, n: int) -> int:
    master_seed = _check_u64(master_seed, "master_seed")
    if n < 1:
        raise ValueError(f"window index must be >= 1, got {n}")
    return _mix(master_seed ^ ((n * _GOLDEN) & _MASK64))


def derive_seeds(master_seed: int, n_windows: int) -> np.ndarray:
    master_seed = _check_u64(master_seed, "master_seed")
    if n_windows < 0:
        raise ValueError(f"n_windows must be >= 0, got {n_windows}")
    return np.array([derive_seed(master_seed, n) for n in range(1, n_windows + 1)],
                    dtype=np.uint64)


def device_streams(seeds, count: int, device=None):
    """Gaussian streams on the device: torch float64 tensor (len(seeds), count)."""
    import torch
    ctx = _lib.context(device)
    seeds = np.ascontiguousarray(np.asarray(seeds, dtype=np.uint64))
    dev = torch.device("cuda", ctx.device)
    out = torch.empty((seeds.shape[0], count), dtype=torch.float64, device=dev)
    if seeds.shape[0] == 0 or count == 0:
        return out
    d_seeds = torch.from_numpy(seeds.view(np.int64)).to(dev)
    for r0 in range(0, seeds.shape[0], 65535):
        r1 = min(r0 + 65535, seeds.shape[0])
        _lib.check(_lib.load().pl_gaussian_streams(
            ctx.handle, _lib.vp(d_seeds.data_ptr() + 8 * r0), r1 - r0, count,
            _lib.vp(out.data_ptr() + 8 * r0 * count)))
    return out


def gaussian_stream(seed: int, count: int) -> np.ndarray:
    seed = _check_u64(seed, "seed")
    if count < 0:
        raise ValueError(f"count must be >= 0, got {count}")
    if count == 0:
        return np.empty(0)
    return device_streams([seed], count)[0].cpu().numpy()


def gaussian_streams(seeds, count: int) -> np.ndarray:
    seeds = np.asarray(seeds, dtype=np.uint64)
    if seeds.ndim != 1:
        raise ValueError("seeds must be a 1-d array")
    if count < 0:
        raise ValueError(f"count must be >= 0, got {count}")
    if count == 0:
        return np.empty((seeds.shape[0], 0))
    return device_streams(seeds, count).cpu().numpy()


@dataclass(frozen=True)
class NoisePlan:
    """Master seed plus the derived per-window seeds of one run."""

    master_seed: int
    window_seeds: tuple

    def __post_init__(self) -> None:
        _check_u64(self.master_seed, "master_seed")
        expected = derive_seeds(self.master_seed, len(self.window_seeds))
        if not np.array_equal(np.asarray(self.window_seeds, dtype=np.uint64), expected):
            raise ValueError("window_seeds are not the seeds derived from master_seed")

    @classmethod
    def for_windows(cls, master_seed: int, n_windows: int) -> "NoisePlan":
        seeds = derive_seeds(master_seed, n_windows)
        return cls(master_seed=int(master_seed), window_seeds=tuple(int(s) for s in seeds))

    @property
    def n_windows(self) -> int:
        return len(self.window_seeds)

    def seed_for(self, n: int) -> int:
        if not 1 <= n <= len(self.window_seeds):
            raise IndexError(f"window {n} outside plan range 1..{len(self.window_seeds)}")
        return self.window_seeds[n - 1]
