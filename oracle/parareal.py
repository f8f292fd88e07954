"""Oracle restatement of the parareal engines (TEST INFRASTRUCTURE).

Follows /root/reference/pkg/src/paralangevin/parareal.py:
  * error metric: running sums of ||cur.q-prev.q||_2 and ||prev.q||_2 per
    node, np.linalg.norm ............................ parareal.py:195-198
  * sequential fine chain, seed m+1 for window m .... parareal.py:243-267
  * jumps F(prev[m]) - C(prev[m]) ................... parareal.py:270-286
  * corrected value C(cur[m]) + jump ................ parareal.py:289-299
  * classic engine (Algorithm 1) .................... parareal.py:315-363
  * adaptive slab engine (Algorithm 2) .............. parareal.py:366-475
States are (q, p) tuples of fp64 arrays; propagators are ``f(state, m)``.
Returns plain dicts so the tests can compare against both the reference's
records and the product's ``PararealResult``.
"""

from __future__ import annotations

import numpy as np


class OracleSlabCollapse(RuntimeError):
    pass


def _acc(num, den, prev, cur):
    num += float(np.linalg.norm(cur[0] - prev[0]))
    den += float(np.linalg.norm(prev[0]))
    return num, den


def sequential(initial, fine, n_windows):
    states = [initial]
    for m in range(n_windows):
        states.append(fine(states[m], m))
    return states


def classic(initial, fine, coarse, n, conv, k_max=None):
    cap = k_max if k_max is not None else n + 1
    cur = [initial]
    for m in range(n):
        cur.append(coarse(cur[m], m))
    history = []
    k = 0
    delta = 2.0 * conv
    while delta >= conv:
        if k >= cap:
            break
        k += 1
        prev = list(cur)
        jumps = []
        for m in range(n):
            f = fine(prev[m], m)
            c = coarse(prev[m], m)
            jumps.append((f[0] - c[0], f[1] - c[1]))
        num = den = 0.0
        for m in range(n):
            base = coarse(cur[m], m)
            cur[m + 1] = (base[0] + jumps[m][0], base[1] + jumps[m][1])
            num, den = _acc(num, den, prev[m + 1], cur[m + 1])
        delta = num / den
        history.append((1, k, delta))
    return dict(trajectory=cur, slabs=[(1, 0, ((n, k),), n, k)], history=history,
                converged=delta < conv)


def adaptive(initial, fine, coarse, n, conv, expl, k_max=None):
    cap = k_max if k_max is not None else n + 1
    mid = 0.5 * (conv + expl)
    cur = [initial] + [None] * n
    n_init = n_final = 0
    delta = mid
    n_slab = 0
    slabs, history, attempts = [], [], []
    k_in_slab = 0
    converged = True
    while n_final < n:
        if delta < expl:
            n_init, n_final = n_final, n
            for m in range(n_init, n):
                cur[m + 1] = coarse(cur[m], m)
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
            prev = list(cur)
            jumps = []
            for m in range(n_init, n_final):
                f = fine(prev[m], m)
                c = coarse(prev[m], m)
                jumps.append((f[0] - c[0], f[1] - c[1]))
            k_attempt += 1
            k_in_slab += 1
            num = den = 0.0
            if n_init >= 1:
                num, den = _acc(num, den, prev[n_init], cur[n_init])
            for m in range(n_init, n_final):
                base = coarse(cur[m], m)
                j = jumps[m - n_init]
                cur[m + 1] = (base[0] + j[0], base[1] + j[1])
                num, den = _acc(num, den, prev[m + 1], cur[m + 1])
                delta = num / den
                history.append((n_slab, k_in_slab, delta))
                if delta > expl:
                    if m == n_init:
                        raise OracleSlabCollapse(f"slab {n_slab} collapsed at {n_init}")
                    attempts.append((n_final, k_attempt))
                    n_final = m
                    break
        if aborted or delta < conv:
            attempts.append((n_final, k_attempt))
            slabs.append((n_slab, n_init, tuple(attempts), n_final,
                          sum(a[1] for a in attempts)))
            if aborted:
                converged = False
                break
    return dict(trajectory=cur, slabs=slabs, history=history, converged=converged)
