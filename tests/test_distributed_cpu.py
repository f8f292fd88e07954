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


# ---------------------------------------------------------------- engine at world size 2
_N, _L = 25, 1


def _engine_props():
    """Reference truncating trace (test_parareal.py:549-564): DoubleWell fine, Harmonic(0.3)
    coarse, gamma 0.5, inv_beta 0.4, dt 0.1, one substep, windows seeded by NoisePlan(11)."""
    from oracle import integrator as oint, rng as orng, toy
    import paper_2212_10508_b200 as pl
    seeds = orng.derive_seeds(11, _N)
    gf, gc = toy.double_well(1.0, 1.0), toy.harmonic(0.3)

    def mk(g):
        def prop(state, m):
            q, p = oint.propagate_window(state.q, state.p, g, 0.5, 0.4, 0.1, _L, oint.robust(_L), int(seeds[m]))
            return pl.PhaseState(q=q, p=p)
        return prop
    return mk(gf), mk(gc)


class _ShardedHostRun:
    """The machine's actions with the jump stage sharded over ranks (distributed.sharded_fine),
    every rank running the identical host sweep: the multi-GPU engine's structure with
    host propagators."""

    def __init__(self, initial, fine, coarse, n, expl):
        from paper_2212_10508_b200.parareal import _HostRun
        self.host = _HostRun(initial, fine, coarse, n, expl)
        self.fine, self.coarse, self.expl = fine, coarse, expl

    def bootstrap(self, n_init):
        self.host.bootstrap(n_init)

    def iterate(self, n_init, n_final, include_m0, iteration):
        import paper_2212_10508_b200 as pl
        from paper_2212_10508_b200.distributed import sharded_fine
        from paper_2212_10508_b200.parareal import _accumulate, _corrected
        cur = self.host.cur
        prev = list(cur)
        d = cur[0].dim

        def run_block(lo, hi):
            fq, fp = np.zeros((hi - lo, 2 * d)), np.zeros((hi - lo, 2 * d))
            for i, m in enumerate(range(lo, hi)):
                f, c = self.fine(prev[m], m), self.coarse(prev[m], m)
                fq[i, :d], fq[i, d:] = f.q, f.p
                fp[i, :d], fp[i, d:] = c.q, c.p
            return torch.from_numpy(fq), torch.from_numpy(fp), torch.zeros(hi - lo, dtype=torch.int32)

        F, C, _ = sharded_fine(run_block, n_init, n_final)
        F, C = F.numpy(), C.numpy()
        jumps = [(F[i, :d] - C[i, :d], F[i, d:] - C[i, d:]) for i in range(n_final - n_init)]
        num = den = 0.0
        if include_m0:
            num, den = _accumulate(num, den, prev[n_init], cur[n_init])
        deltas = []
        for m in range(n_init, n_final):
            cur[m + 1] = _corrected(self.coarse, cur[m], m, iteration, jumps[m - n_init])
            num, den = _accumulate(num, den, prev[m + 1], cur[m + 1])
            deltas.append(num / den)
            if deltas[-1] > self.expl:
                break
        return deltas, den


def _engine_worker(rank, ws, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        import paper_2212_10508_b200 as pl
        from paper_2212_10508_b200.parareal import _adaptive_machine, _drive_adaptive
        fine, coarse = _engine_props()
        init = pl.PhaseState(q=np.array([-1.2]), p=np.array([0.0]))
        run = _ShardedHostRun(init, fine, coarse, _N, 0.1)
        slabs, hist, conv = _drive_adaptive(_adaptive_machine(_N, 1e-9, 0.1, _N + 1), run)
        traj = np.array([s.q for s in run.host.cur] + [s.p for s in run.host.cur])
        q.put((rank, ([(s.slab_index, s.n_init, s.n_final, s.k_conv,
                        tuple((a.n_final, a.iterations) for a in s.attempts)) for s in slabs],
                       hist, conv, traj.tobytes())))
    finally:
        dist.destroy_process_group()


def test_adaptive_engine_gloo_world2_matches_single_rank():
    """Adaptive machine + sharded fine stage at world size 2 == the single-rank engine
    (slabs, attempts, error history, trajectory bit for bit), identical on both ranks."""
    import paper_2212_10508_b200 as pl
    from paper_2212_10508_b200.parareal import parareal_adaptive_engine
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29700 + (os.getpid() % 1000)
    procs = [ctx.Process(target=_engine_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    fine, coarse = _engine_props()
    init = pl.PhaseState(q=np.array([-1.2]), p=np.array([0.0]))
    ref = parareal_adaptive_engine(init, fine, coarse, pl.PararealConfig(_N, 1e-9, 0.1))
    assert ref.converged and ref.n_slab >= 2 and any(len(s.attempts) > 1 for s in ref.slabs)
    ref_slabs = [(s.slab_index, s.n_init, s.n_final, s.k_conv, tuple((a.n_final, a.iterations) for a in s.attempts))
                 for s in ref.slabs]
    ref_traj = np.array([s.q for s in ref.trajectory] + [s.p for s in ref.trajectory]).tobytes()
    assert res[0] == res[1]
    slabs, hist, conv, traj = res[0]
    assert slabs == ref_slabs
    assert tuple(hist) == ref.error_history
    assert conv and traj == ref_traj
