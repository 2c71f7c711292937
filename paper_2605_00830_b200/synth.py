"""Seeded synthetic workloads for FAST-GED (arXiv 2605.00830).

This module holds the input generators shared by the tests, ``bench.py`` and
``__graft_entry__``.  It contains none of the method's arithmetic (no costs are
evaluated here, nothing is searched): it only draws graphs.  Both the CUDA path
and the CPU oracle receive the same arrays from here.

Workload recipes:

* Erdős–Rényi G(n, p) with uniform vertex labels — the paper's random graphs
  ("randomly generated with an average density of 0.4"; Table 1
  random pairs PAPER.md:301-328).
* AIDS-like / Mutagenicity-like labelled molecular graphs — shaped after the
  IAM datasets the paper uses: a degree-capped random
  tree plus a few ring closures, element-frequency vertex labels and bond-order
  edge labels.  The statistics are a recipe of this repo, not paper claims.

Randomness: numpy ``PCG64`` seeded from ``SeedSequence([seed, stream])``; every
draw is made in a fixed order, so a (config, seed) pair always yields the same
bytes.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

import numpy as np

__all__ = [
    "Graph", "COSTS", "rng_for", "er_graph", "molecule_graph", "path_graph", "cycle_graph",
    "complete_graph", "empty_graph", "complete_bipartite", "star_graph", "relabel",
    "config_workload", "Workload",
]

# Cost presets (vsub, vdel, vins, esub, edel, eins).
COSTS = {
    # PAPER.md:298 defaults = "Setting 1" of PAPER.md:577-578.
    "setting1": (2, 4, 4, 1, 2, 2),
    # PAPER.md:579-580.
    "setting2": (4, 12, 12, 1, 10, 10),
    # PAPER.md:707 "uniform GED costs (c_ins=c_del=2, c_sub=1)"; esub=1.
    "uniform": (1, 2, 2, 1, 2, 2),
    # BASELINE.json configs[0] "unit edit costs".
    "unit": (1, 1, 1, 1, 1, 1),
}


@dataclass
class Graph:
    """Simple undirected labelled graph G = (V, E, alpha, beta).

    ``vlabels``: int32[n]; ``edges``: int32[m, 2] with u < v; ``elabels``: int32[m]
    or None (every edge label 0).
    """

    n: int
    vlabels: np.ndarray
    edges: np.ndarray
    elabels: Optional[np.ndarray] = None

    @property
    def m(self) -> int:
        return int(self.edges.shape[0])

    def __post_init__(self):
        self.n = int(self.n)
        self.vlabels = np.ascontiguousarray(self.vlabels, dtype=np.int32).reshape(self.n)
        self.edges = np.ascontiguousarray(self.edges, dtype=np.int32).reshape(-1, 2)
        if self.elabels is not None:
            self.elabels = np.ascontiguousarray(self.elabels, dtype=np.int32).reshape(-1)


def rng_for(seed: int, *stream: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([int(seed)] + [int(s) for s in stream])))


# ---------------------------------------------------------------- named graphs
def _from_pairs(n: int, pairs: Sequence[Tuple[int, int]], vlabels=None, elabels=None) -> Graph:
    e = np.array(sorted((min(a, b), max(a, b)) for a, b in pairs), dtype=np.int32).reshape(-1, 2)
    vl = np.zeros(n, np.int32) if vlabels is None else np.asarray(vlabels, np.int32)
    return Graph(n, vl, e, None if elabels is None else np.asarray(elabels, np.int32))


def empty_graph(n: int) -> Graph:
    return _from_pairs(n, [])


def path_graph(n: int) -> Graph:
    return _from_pairs(n, [(i, i + 1) for i in range(n - 1)])


def cycle_graph(n: int) -> Graph:
    return _from_pairs(n, [(i, (i + 1) % n) for i in range(n)] if n >= 3 else [])


def complete_graph(n: int) -> Graph:
    return _from_pairs(n, [(i, j) for i in range(n) for j in range(i + 1, n)])


def complete_bipartite(a: int, b: int) -> Graph:
    return _from_pairs(a + b, [(i, a + j) for i in range(a) for j in range(b)])


def star_graph(leaves: int) -> Graph:
    return _from_pairs(leaves + 1, [(0, i) for i in range(1, leaves + 1)])


def relabel(g: Graph, vlabels=None, elabels=None) -> Graph:
    return Graph(g.n, g.vlabels if vlabels is None else vlabels, g.edges.copy(),
                 g.elabels if elabels is None else elabels)


def permute(g: Graph, perm: np.ndarray) -> Graph:
    """Isomorphic copy: vertex v of g becomes perm[v]."""
    perm = np.asarray(perm, np.int64)
    vl = np.empty(g.n, np.int32)
    vl[perm] = g.vlabels
    e = perm[g.edges.astype(np.int64)] if g.m else np.zeros((0, 2), np.int64)
    e = np.sort(e, axis=1)
    order = np.lexsort((e[:, 1], e[:, 0])) if g.m else np.zeros(0, np.int64)
    el = None if g.elabels is None else g.elabels[order]
    return Graph(g.n, vl, e[order], el)


# ------------------------------------------------------------------ generators
def er_graph(rng: np.random.Generator, n: int, p: float, n_vlabels: int = 1, n_elabels: int = 1) -> Graph:
    """G(n, p): each of the n(n-1)/2 pairs independently with probability p."""
    vl = rng.integers(0, n_vlabels, size=n, dtype=np.int32) if n_vlabels > 1 else np.zeros(n, np.int32)
    iu, ju = np.triu_indices(n, 1)
    keep = rng.random(iu.shape[0]) < p
    e = np.stack([iu[keep], ju[keep]], axis=1).astype(np.int32)
    el = rng.integers(0, n_elabels, size=e.shape[0], dtype=np.int32) if n_elabels > 1 else None
    return Graph(n, vl, e, el)


# Element frequencies (label id order) and bond-order frequencies.  Recipe of this repo.
_AIDS_V = np.array([0.62, 0.16, 0.11, 0.03] + [0.08 / 25] * 25)           # C O N S + 25 rare
_MUTA_V = np.array([0.45, 0.30, 0.12, 0.07, 0.02, 0.01, 0.01, 0.01] + [0.01 / 6] * 6)
_AIDS_E = np.array([0.75, 0.20, 0.05])
_MUTA_E = np.array([0.80, 0.17, 0.03])


def molecule_graph(rng: np.random.Generator, kind: str) -> Graph:
    """Degree-capped (<=4) random tree plus ring closures, labelled like a molecule.

    kind="aids": n ~ U{5..10}, rings ~ U{0..2}, 29 vertex labels.
    kind="muta": n = round(N(30, 6)) clipped to [16, 44], rings ~ U{0..3}, 14 labels.
    """
    if kind == "aids":
        n = int(rng.integers(5, 11)); rings = int(rng.integers(0, 3)); pv, pe = _AIDS_V, _AIDS_E
    elif kind == "muta":
        n = int(np.clip(np.rint(rng.normal(30.0, 6.0)), 16, 44)); rings = int(rng.integers(0, 4)); pv, pe = _MUTA_V, _MUTA_E
    else:
        raise ValueError(kind)
    deg = np.zeros(n, np.int32)
    pairs = []
    for t in range(1, n):
        cand = np.flatnonzero(deg[:t] < 4)
        a = int(cand[rng.integers(0, cand.shape[0])])
        pairs.append((a, t)); deg[a] += 1; deg[t] += 1
    adj = {(a, b) for a, b in pairs}
    for _ in range(rings):
        for _try in range(20):
            a, b = (int(x) for x in rng.integers(0, n, size=2))
            if a == b:
                continue
            a, b = min(a, b), max(a, b)
            if (a, b) in adj or deg[a] >= 4 or deg[b] >= 4:
                continue
            adj.add((a, b)); pairs.append((a, b)); deg[a] += 1; deg[b] += 1
            break
    vl = rng.choice(pv.shape[0], size=n, p=pv / pv.sum()).astype(np.int32)
    pairs.sort()
    el = (rng.choice(pe.shape[0], size=len(pairs), p=pe / pe.sum()) + 1).astype(np.int32)
    return Graph(n, vl, np.array(pairs, np.int32).reshape(-1, 2), el)


def two_class_molecules(n_per_class: int, seed: int = 13) -> Tuple[List[Graph], np.ndarray]:
    """A synthetic two-class corpus shaped like Mutagenicity (the IAM dataset itself is
    not available): class 0 = Mutagenicity-like molecules (``molecule_graph(.., "muta")``); class 1 = the
    same recipe with one or two nitro groups (an N bonded to two O, bond labels 2 and 1) attached to random
    carbons of degree < 4 -- the structural alert of mutagenic compounds.  Labels are the class of each
    graph; graphs alternate between the classes.  A recipe of this repo, not a paper claim."""
    r = rng_for(seed)
    graphs, labels = [], []
    C, O, N = 0, 2, 3  # label ids in _MUTA_V order (C, H, O, N, ...)
    for k in range(2 * n_per_class):
        cls = k % 2
        g = molecule_graph(r, "muta")
        if cls == 1:
            vl = list(g.vlabels.tolist())
            pairs = [tuple(e) for e in g.edges.tolist()]
            el = list(g.elabels.tolist())
            deg = np.zeros(g.n, np.int32)
            for a, b in pairs:
                deg[a] += 1; deg[b] += 1
            for _ in range(int(r.integers(1, 3))):
                cand = [v for v in range(len(vl)) if vl[v] == C and deg[v] < 4]
                if not cand:
                    break
                a = int(cand[int(r.integers(0, len(cand)))])
                nn = len(vl)
                vl += [N, O, O]
                pairs += [(a, nn), (nn, nn + 1), (nn, nn + 2)]
                el += [1, 2, 1]
                deg[a] += 1
                deg = np.concatenate([deg, [3, 1, 1]]).astype(np.int32)
            order = sorted(range(len(pairs)), key=lambda x: pairs[x])
            g = Graph(len(vl), np.array(vl, np.int32), np.array([pairs[x] for x in order], np.int32).reshape(-1, 2),
                      np.array([el[x] for x in order], np.int32))
        graphs.append(g)
        labels.append(cls)
    return graphs, np.array(labels, np.int32)


# ------------------------------------------------------------------- workloads
@dataclass
class Workload:
    """A batch of (g1, g2) pairs with one cost model and one K.

    ``graphs`` holds the distinct graphs; ``pair_a``/``pair_b`` index them, so the
    all-pairs workload (config 5) needs no copies.
    """

    name: str
    graphs: List[Graph]
    pair_a: np.ndarray
    pair_b: np.ndarray
    costs: Tuple[int, int, int, int, int, int]
    K: int

    @property
    def npairs(self) -> int:
        return int(self.pair_a.shape[0])

    def pair(self, k: int) -> Tuple[Graph, Graph]:
        return self.graphs[int(self.pair_a[k])], self.graphs[int(self.pair_b[k])]

    def subset(self, idx) -> "Workload":
        idx = np.asarray(idx, np.int64)
        return Workload(self.name + "[subset]", self.graphs, self.pair_a[idx], self.pair_b[idx], self.costs, self.K)


def _pairs_workload(name, pairs, costs, K) -> Workload:
    graphs = [g for ab in pairs for g in ab]
    a = np.arange(0, 2 * len(pairs), 2, dtype=np.int64)
    return Workload(name, graphs, a, a + 1, costs, K)


def config_workload(cfg: int, seed: Optional[int] = None, npairs: Optional[int] = None,
                    K: Optional[int] = None, variant: Optional[str] = None) -> Workload:
    """The five BASELINE.json configs as concrete seeded inputs.

    ``npairs`` truncates/extends the pair count (same recipe), ``K`` overrides K.
    """
    if cfg == 1:  # two unlabeled 6-vertex graphs, unit costs, K=16
        seed = 1 if seed is None else seed
        total = 1000 if npairs is None else npairs
        pairs = []
        for k in range(total):
            p = (0.2, 0.5, 0.8)[k % 3]
            r = rng_for(seed, k)
            pairs.append((er_graph(r, 6, p), er_graph(r, 6, p)))
        return _pairs_workload("cfg1-G(6,p)-unit-K16", pairs, COSTS["unit"], 16 if K is None else K)
    if cfg == 2:  # AIDS-like molecule pairs, K=100
        seed = 2 if seed is None else seed
        total = 10000 if npairs is None else npairs
        r = rng_for(seed)
        graphs = [molecule_graph(r, "aids") for _ in range(2 * total)]
        a = np.arange(0, 2 * total, 2, dtype=np.int64)
        return Workload("cfg2-aids-like-K100", graphs, a, a + 1, COSTS["setting1"], 100 if K is None else K)
    if cfg == 3:  # ER n in 30..70 x p in 0.1..0.5, 4 vertex labels, K=1000
        seed = 3 if seed is None else seed
        total = 10000 if npairs is None else npairs
        ns, ps = (30, 40, 50, 60, 70), (0.1, 0.2, 0.3, 0.4, 0.5)
        nvl = 1 if variant == "unlabeled" else 4
        pairs = []
        for k in range(total):
            cell = k % 25
            n, p = ns[cell // 5], ps[cell % 5]
            r = rng_for(seed, k)
            pairs.append((er_graph(r, n, p, nvl), er_graph(r, n, p, nvl)))
        return _pairs_workload("cfg3-ER-n30-70-K1000", pairs, COSTS["setting1"], 1000 if K is None else K)
    if cfg == 4:  # single large ER pairs
        seed = 4 if seed is None else seed
        runs = [(n, p, kk) for n in (200, 500) for p in (0.05, 0.2) for kk in (10_000, 100_000)]
        pairs, Ks = [], []
        for idx, (n, p, kk) in enumerate(runs):
            r = rng_for(seed, idx)
            pairs.append((er_graph(r, n, p, 4), er_graph(r, n, p, 4)))
            Ks.append(kk)
        w = _pairs_workload("cfg4-ER-large", pairs, COSTS["setting1"], 100_000 if K is None else K)
        w.run_K = Ks  # type: ignore[attr-defined]
        w.run_np = runs  # type: ignore[attr-defined]
        return w
    if cfg == 5:  # all unordered pairs of 2000 Mutagenicity-like graphs
        seed = 5 if seed is None else seed
        r = rng_for(seed)
        ng = 2000
        graphs = [molecule_graph(r, "muta") for _ in range(ng)]
        ia, ib = np.triu_indices(ng, 1)
        a, b = ia.astype(np.int64), ib.astype(np.int64)
        if npairs is not None:
            a, b = a[:npairs], b[:npairs]
        costs = COSTS["setting2"] if variant == "setting2" else COSTS["setting1"]
        return Workload("cfg5-muta-like-allpairs-K1000", graphs, a, b, costs, 1000 if K is None else K)
    raise ValueError(f"unknown config {cfg}")


def large_pair(n: int, p: float, seed: int = 4, nvl: int = 4) -> Tuple[Graph, Graph]:
    r = rng_for(seed, n, int(p * 1000))
    return er_graph(r, n, p, nvl), er_graph(r, n, p, nvl)
