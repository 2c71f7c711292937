"""Exact GED by brute force — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Independent of the C oracle (different language, no shared code, no levels, no
charging order).  It enumerates every partial injection f: V1 -> V2 u {DEL}
(the complete vertex-centric edit paths of PAPER.md:89-100; insertions are the
g2 vertices outside the image) and evaluates the order-free cost

    cost(f) = sum_{f(i)=DEL} vdel + sum_{f(i)=j} [l1(i) != l2(j)] vsub + vins (n2 - |img f|)
            + sum_{(a,b) in E1} ( f(a),f(b) != DEL and (f(a),f(b)) in E2
                                   ? [beta1(a,b) != beta2(f(a),f(b))] esub : edel )
            + sum_{(x,y) in E2} ( x,y in img f and (f^-1 x, f^-1 y) in E1 ? 0 : eins )

i.e. the definition d(g1,g2) = min over edit paths of the summed costs
 with the implied edge cases of PAPER.md:103-116.
Guard: n1, n2 <= 8 (130,922 injections for 7x7; 1,441,729 for 8x8).
"""
from __future__ import annotations

from functools import lru_cache

import numpy as np

DEL = -1


@lru_cache(maxsize=64)
def injections(n1: int, n2: int) -> np.ndarray:
    """All partial injections as an int64[W, n1] array (DEL = -1), enumerated in
    the vertex-branching tree's order (v_0 first; per vertex: DEL, then targets)."""
    if n1 > 8 or n2 > 8:
        raise ValueError("brute force guard: n1, n2 <= 8")
    cur = np.zeros((1, 0), np.int64)
    for _ in range(n1):
        parts = [np.concatenate([cur, np.full((cur.shape[0], 1), DEL)], 1)]
        for j in range(n2):
            ok = ~(cur == j).any(axis=1)
            parts.append(np.concatenate([cur[ok], np.full((int(ok.sum()), 1), j)], 1))
        cur = np.concatenate(parts, 0)
    cur.setflags(write=False)
    return cur


def _adj(g):
    n = int(g.n)
    has = np.zeros((n + 1, n + 1), bool)  # extra row/col n = "no vertex"
    lab = np.zeros((n + 1, n + 1), np.int64)
    e = np.asarray(g.edges, np.int64).reshape(-1, 2)
    el = np.zeros(e.shape[0], np.int64) if g.elabels is None else np.asarray(g.elabels, np.int64)
    if e.shape[0]:
        has[e[:, 0], e[:, 1]] = has[e[:, 1], e[:, 0]] = True
        lab[e[:, 0], e[:, 1]] = lab[e[:, 1], e[:, 0]] = el
    return has, lab, e, el


def costs_of(g1, g2, costs, F: np.ndarray) -> np.ndarray:
    """Order-free cost of each row of F (int64[W, n1])."""
    vsub, vdel, vins, esub, edel, eins = (int(x) for x in costs)
    n1, n2 = int(g1.n), int(g2.n)
    F = np.asarray(F, np.int64)
    if F.ndim == 1:
        F = F.reshape(1, n1)
    W = F.shape[0]
    vl1 = np.asarray(g1.vlabels, np.int64)
    vl2 = np.concatenate([np.asarray(g2.vlabels, np.int64), [0]])
    Fs = np.where(F < 0, n2, F)  # DEL -> sentinel index n2
    mapped = F >= 0
    total = np.zeros(W, np.int64)
    # vertex substitutions / deletions / insertions
    total += np.where(mapped, (vl1[None, :] != vl2[Fs]) * vsub, vdel).sum(axis=1)
    total += vins * (n2 - mapped.sum(axis=1))
    has1, _lab1, e1, el1 = _adj(g1)
    has2, lab2, e2, _el2 = _adj(g2)
    # g1 edges: substituted (esub if labels differ) or deleted
    for (a, b), l in zip(e1, el1):
        fa, fb = Fs[:, a], Fs[:, b]
        present = has2[fa, fb]
        total += np.where(present, (lab2[fa, fb] != l) * esub, edel)
    # g2 edges: matched by a g1 edge (already charged) or inserted
    inv = np.full((W, n2 + 1), n1, np.int64)
    rows = np.repeat(np.arange(W), n1)
    cols = Fs.reshape(-1)
    src = np.tile(np.arange(n1), W)
    ok = cols < n2
    inv[rows[ok], cols[ok]] = src[ok]
    for (x, y) in e2:
        ix, iy = inv[:, x], inv[:, y]
        matched = has1[ix, iy]
        total += np.where(matched, 0, eins)
    return total


def exact_ged(g1, g2, costs):
    """Returns (GED, all costs int64[W], injections int64[W, n1])."""
    F = injections(int(g1.n), int(g2.n))
    c = costs_of(g1, g2, costs, F)
    return int(c.min()), c, F


def width(n1: int, n2: int, level: int) -> int:
    """Number of partial injections of `level` source vertices into n2 targets."""
    from math import comb, perm
    return sum(comb(level, k) * perm(n2, k) for k in range(0, min(level, n2) + 1))
