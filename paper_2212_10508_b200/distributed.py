"""Slice sharding of the parareal fine stage over ranks.

Windows of a slab are independent within an iteration (parareal.py:270-286),
so rank r propagates a contiguous block of them and one all-gather of the
fine endpoints (q, p and the blow-up flags) gives every rank the full jump
set.  Every rank then runs the identical, bitwise-deterministic coarse sweep,
so no broadcast of corrected states is needed and all ranks take the same
slab decisions.  One process per GPU, ``torch.distributed`` (NCCL on GPUs,
gloo in the CPU tests).
"""

from __future__ import annotations


def world():
    """(rank, world_size) of the default process group, (0, 1) if none."""
    try:
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized():
            return dist.get_rank(), dist.get_world_size()
    except Exception:
        pass
    return 0, 1


def shard_bounds(n_init: int, n_final: int, world_size: int, rank: int):
    """Contiguous, balanced block [lo, hi) of windows n_init..n_final-1 for `rank`."""
    W = n_final - n_init
    base, extra = divmod(W, world_size)
    lo = n_init + rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


def gather_blocks(local, n_init: int, n_final: int, world_size: int, out=None):
    """All-gather per-rank blocks (rows = windows) into the (W, ...) full array.

    ``local`` is this rank's (hi - lo, ...) tensor; blocks are padded to the
    largest block so one ``all_gather_into_tensor`` moves everything.
    """
    import torch
    import torch.distributed as dist
    W = n_final - n_init
    sizes = [shard_bounds(n_init, n_final, world_size, r) for r in range(world_size)]
    bmax = max(hi - lo for lo, hi in sizes)
    tail = tuple(local.shape[1:])
    pad = torch.zeros((bmax,) + tail, dtype=local.dtype, device=local.device)
    pad[: local.shape[0]].copy_(local)
    buf = torch.empty((world_size * bmax,) + tail, dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(buf, pad)
    if out is None:
        out = torch.empty((W,) + tail, dtype=local.dtype, device=local.device)
    for r, (lo, hi) in enumerate(sizes):
        if hi > lo:
            out[lo - n_init: hi - n_init].copy_(buf[r * bmax: r * bmax + (hi - lo)])
    return out


def sharded_fine(run_block, n_init: int, n_final: int):
    """Fine stage over windows n_init..n_final-1 sharded across ranks.

    ``run_block(lo, hi) -> (FQ, FP, blow)`` propagates windows lo..hi-1 on this
    rank (torch tensors, rows = windows).  Returns the full (FQ, FP, blow) on
    every rank, rows in window order.
    """
    rank, ws = world()
    if ws == 1:
        return run_block(n_init, n_final)
    lo, hi = shard_bounds(n_init, n_final, ws, rank)
    FQ, FP, blow = run_block(lo, hi)
    return (gather_blocks(FQ, n_init, n_final, ws), gather_blocks(FP, n_init, n_final, ws),
            gather_blocks(blow, n_init, n_final, ws))
