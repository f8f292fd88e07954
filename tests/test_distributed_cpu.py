"""Multi-rank host logic of the sharded fine stage, on CPU with gloo (world size 2).

The device kernels cannot run here, so the per-rank block propagator is the
CPU oracle; what is tested is the sharding/all-gather path the GPU engine
uses (paper_2212_10508_b200.distributed), which must reproduce the
unsharded jump stage bit for bit.
"""

import os

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from paper_2212_10508_b200.distributed import shard_bounds


def test_shard_bounds_cover_exactly():
    for n_init, n_final in ((0, 16), (3, 10), (5, 6), (0, 1), (7, 7)):
        for ws in (1, 2, 3, 4, 8):
            got = []
            for r in range(ws):
                lo, hi = shard_bounds(n_init, n_final, ws, r)
                assert n_init <= lo <= hi <= n_final
                got.extend(range(lo, hi))
            assert got == list(range(n_init, n_final))


def _worker(rank, ws, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        from oracle import integrator as oint, rng as orng, toy
        from paper_2212_10508_b200.distributed import sharded_fine
        n, d, L = 11, 3, 4
        rs = np.random.default_rng(0)
        Q = rs.normal(size=(n, d))
        P = rs.normal(size=(n, d))
        seeds = orng.derive_seeds(9, n)
        g = toy.double_well(1.0, 1.0)

        def run_block(lo, hi):
            fq, fp = [], []
            for m in range(lo, hi):
                a, b = oint.propagate_window(Q[m], P[m], g, 0.5, 0.4, 0.05, L, oint.robust(L), int(seeds[m]))
                fq.append(a)
                fp.append(b)
            z = np.zeros((0, d))
            return (torch.from_numpy(np.array(fq) if fq else z), torch.from_numpy(np.array(fp) if fp else z),
                    torch.zeros(hi - lo, dtype=torch.int32))

        outs = []
        for n_init, n_final in ((0, n), (2, 9), (4, 5)):
            FQ, FP, blow = sharded_fine(run_block, n_init, n_final)
            outs.append((FQ.numpy().copy(), FP.numpy().copy(), blow.numpy().copy()))
        q.put((rank, outs))
    finally:
        dist.destroy_process_group()


def test_sharded_fine_gloo_world2_matches_serial():
    from oracle import integrator as oint, rng as orng, toy
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000)
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    n, d, L = 11, 3, 4
    rs = np.random.default_rng(0)
    Q = rs.normal(size=(n, d))
    P = rs.normal(size=(n, d))
    seeds = orng.derive_seeds(9, n)
    g = toy.double_well(1.0, 1.0)
    for k, (n_init, n_final) in enumerate(((0, n), (2, 9), (4, 5))):
        ref = [oint.propagate_window(Q[m], P[m], g, 0.5, 0.4, 0.05, L, oint.robust(L), int(seeds[m]))
               for m in range(n_init, n_final)]
        RQ = np.array([a for a, _ in ref])
        RP = np.array([b for _, b in ref])
        for rank in (0, 1):
            FQ, FP, blow = res[rank][k]
            assert FQ.tobytes() == RQ.tobytes() and FP.tobytes() == RP.tobytes()
            assert not blow.any()
