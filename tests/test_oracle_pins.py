"""Pins for the CPU oracle (oracle/fastged_oracle.c) and the brute force (oracle/bruteforce.py).

Neither is trusted until pinned to something other than itself:
  * values SPEC.md prints for worked examples (tests/golden/spec_worked_examples.json),
  * closed forms and hand traces derived from PAPER.md:103-116 (tests/golden/derived_closed_forms.json),
  * counting identities of the vertex-branching tree (partial-injection widths),
  * the brute force (an order-free formula, another language) on every small pair,
  * invariants: upper bound, exactness at full width, identity,
    lower bound, symmetry, witness re-verification.
No GPU is used here.
"""
import json
import math
import os

import numpy as np
import pytest

from paper_2605_00830_b200 import synth
from paper_2605_00830_b200.synth import COSTS, Graph

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _g(d):
    return Graph(d["n"], d["vl"], np.array(d["e"], np.int32).reshape(-1, 2),
                 None if d["el"] is None else d["el"])


NAMED = {
    "path3": synth.path_graph(3), "k3": synth.complete_graph(3), "path6": synth.path_graph(6),
    "cycle6": synth.cycle_graph(6), "k33": synth.complete_bipartite(3, 3), "k6": synth.complete_graph(6),
    "empty6": synth.empty_graph(6),
}


# ------------------------------------------------------------------ SPEC examples
def _spec_cases():
    with open(os.path.join(GOLD, "spec_worked_examples.json")) as f:
        return json.load(f)["cases"]


@pytest.mark.parametrize("case", _spec_cases(), ids=lambda c: c["name"])
def test_spec_worked_examples(oracle_lib, case):
    from oracle import bruteforce
    g1, g2 = _g(case["g1"]), _g(case["g2"])
    r = oracle_lib.kbest(g1, g2, case["costs"], case["K"])
    assert r["cost"] == case["cost"], case["cite"]
    assert bruteforce.exact_ged(g1, g2, case["costs"])[0] == case["cost"], case["cite"]


def test_edge_label_substitution():
    """Edge in both graphs with different labels -> esub (P:256 'different weights', reading C2)."""
    from oracle import oracle, bruteforce
    g1 = Graph(2, [0, 0], [[0, 1]], [5])
    g2 = Graph(2, [0, 0], [[0, 1]], [7])
    for costs in (COSTS["setting1"], COSTS["setting2"]):
        assert oracle.kbest(g1, g2, costs, 1)["cost"] == costs[3]
        assert bruteforce.exact_ged(g1, g2, costs)[0] == costs[3]
    # with esub > edel + eins the edge is deleted and re-inserted instead
    costs = (1, 5, 5, 9, 2, 3)
    assert bruteforce.exact_ged(g1, g2, costs)[0] == min(9, 2 * 5 + 2 + 3)


# ------------------------------------------------------------------ closed forms
def _closed():
    with open(os.path.join(GOLD, "derived_closed_forms.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("case", _closed()["cases"], ids=lambda c: c["name"])
def test_closed_forms(oracle_lib, case):
    from oracle import bruteforce
    g1, g2 = NAMED[case["g1"]], NAMED[case["g2"]]
    assert bruteforce.exact_ged(g1, g2, case["costs"])[0] == case["ged"]
    # K >= final width 13,327 (6x6): K-Best is exhaustive and exact.
    assert oracle_lib.kbest(g1, g2, case["costs"], 16384)["cost"] == case["ged"]


@pytest.mark.parametrize("case", _closed()["hand_traces_K1"], ids=lambda c: c["name"])
def test_hand_traces_k1(oracle_lib, case):
    r = oracle_lib.kbest(NAMED[case["g1"]], NAMED[case["g2"]], case["costs"], 1)
    assert r["cost"] == case["cost"]
    assert r["mapping"].tolist() == case["mapping"]


def _k2_cases():
    with open(os.path.join(GOLD, "hand_traces_k2.json")) as f:
        return json.load(f)["cases"]


@pytest.mark.parametrize("case", _k2_cases(), ids=lambda c: c["name"])
def test_hand_traces_k2(oracle_lib, case):
    """K >= 2 hand traces that pin the two readings the K = 1 traces cannot see:
    C13 (survivors re-ordered by (p, j)) and C10 (last level ranked by PED, completion after)."""
    from oracle import bruteforce
    g1, g2 = _g(case["g1"]), _g(case["g2"])
    r = oracle_lib.kbest(g1, g2, case["costs"], case["K"], levels=True)
    assert r["cost"] == case["cost"], case["name"]
    assert r["mapping"].tolist() == case["mapping"], case["name"]
    assert [list(x) for x in r["levels"]] == case["levels"], case["name"]
    # the pinned value is an upper bound of the exact GED, and its witness re-verifies
    assert r["cost"] >= bruteforce.exact_ged(g1, g2, case["costs"])[0]
    assert int(bruteforce.costs_of(g1, g2, case["costs"], r["mapping"][None, :])[0]) == r["cost"]


@pytest.mark.parametrize("case", _k2_cases(), ids=lambda c: c["name"])
def test_variant_last_by_total_hand_traces(oracle_lib, case):
    """NEXT-4 variant (last level ranked by PED + completion): the hand-traced values."""
    g1, g2 = _g(case["g1"]), _g(case["g2"])
    r = oracle_lib.kbest(g1, g2, case["costs"], case["K"], flags=oracle_lib.LAST_BY_TOTAL)
    assert r["cost"] == case["variant_cost"] and r["mapping"].tolist() == case["variant_mapping"]


def test_variant_never_worse_and_exact_at_full_width(oracle_lib):
    """The variant keeps the same frontier up to the last level and then the K smallest totals, so its
    cost is <= the paper-literal cost for every K, >= the exact GED, and = exact once K covers the widths."""
    from oracle import bruteforce
    rng = synth.rng_for(4040)
    for k in range(150):
        n1, n2 = int(rng.integers(1, 7)), int(rng.integers(1, 7))
        g1 = synth.er_graph(rng, n1, (0.2, 0.5, 0.8)[k % 3], 2, 1 + k % 2)
        g2 = synth.er_graph(rng, n2, (0.2, 0.5, 0.8)[k % 3], 2, 1 + k % 2)
        c = (COSTS["unit"], COSTS["setting1"], ASYM)[k % 3]
        ged = bruteforce.exact_ged(g1, g2, c)[0]
        for K in (1, 2, 5, bruteforce.width(n1, n2, n1)):
            lit = oracle_lib.kbest(g1, g2, c, K)["cost"]
            var = oracle_lib.kbest(g1, g2, c, K, flags=oracle_lib.LAST_BY_TOTAL)
            assert ged <= var["cost"] <= lit
            assert oracle_lib.mapping_cost(g1, g2, c, var["mapping"]) == var["cost"]
            if K >= bruteforce.width(n1, n2, n1):
                assert var["cost"] == ged


def test_selection_examples(oracle_lib):
    """P5: the selection step keeps the k smallest unique keys."""
    sel = oracle_lib.select
    # [5,1,3,2,4], k=2 -> {1,2} (the values at indices 1 and 3)
    assert sel([5, 1, 3, 2, 4], [0] * 5, [0, 1, 2, 3, 4], 2).tolist() == [1, 3]
    # k >= size -> everything
    assert sel([5, 1, 3], [0] * 3, [0, 1, 2], 7).tolist() == [0, 1, 2]
    # equal PEDs: the smaller tag wins ([1,1,1] with tags 0,1,2, k=2 -> {0,1})
    assert sel([1, 1, 1], [0, 0, 0], [0, 1, 2], 2).tolist() == [0, 1]
    # ties broken by parent before child (C12)
    assert sel([3, 3, 3, 1], [2, 0, 1, 9], [0, 5, 4, 0], 3).tolist() == [1, 2, 3]
    assert sel([], [], [], 3).tolist() == []


def test_selection_equals_full_sort(oracle_lib):
    """P5: quickselect and a full sort by (PED, p, j) pick the same set (keys are unique), on
    random pools shaped like a level (few distinct PEDs, many ties, every k)."""
    rng = synth.rng_for(515)
    for trial in range(300):
        n = int(rng.integers(1, 400))
        npar = int(rng.integers(1, 40))
        p = rng.integers(0, npar, size=n)
        j = rng.permutation(n).astype(np.int32)  # unique (p, j) keys
        ped = rng.integers(0, int(rng.integers(1, 12)), size=n)
        k = int(rng.integers(0, n + 3))
        order = np.lexsort((j, p, ped))
        want = np.sort(order[:min(k, n)])
        got = oracle_lib.select(ped, p, j, k)
        assert np.array_equal(got, want), (trial, n, k)


def test_empty_graph_closed_forms(oracle_lib):
    """n1 = 0 -> vins*n2 + eins*m2; n2 = 0 -> vdel*n1 + edel*m1 (C16)."""
    c = COSTS["setting1"]
    g = synth.cycle_graph(5)
    e = synth.empty_graph(0)
    r = oracle_lib.kbest(e, g, c, 3)
    assert r["cost"] == c[2] * 5 + c[5] * 5 and r["mapping"].size == 0
    r = oracle_lib.kbest(g, e, c, 3)
    assert r["cost"] == c[1] * 5 + c[4] * 5 and r["mapping"].tolist() == [-1] * 5


# ------------------------------------------------------------------ brute force pins
def test_injection_counts():
    """W(i) = sum_k C(i,k) P(n2,k): 13,327 for 6x6, 130,922 for 7x7."""
    from oracle import bruteforce
    assert bruteforce.injections(6, 6).shape[0] == 13327
    assert bruteforce.injections(7, 7).shape[0] == 130922
    for n1 in range(0, 5):
        for n2 in range(0, 5):
            F = bruteforce.injections(n1, n2)
            assert F.shape[0] == bruteforce.width(n1, n2, n1)
            # every row is injective on its non-deleted entries
            for row in F:
                m = row[row >= 0]
                assert len(set(m.tolist())) == m.size


def test_bruteforce_symmetry():
    """Exact GED is symmetric when vdel = vins and edel = eins."""
    from oracle import bruteforce
    rng = synth.rng_for(99)
    for k in range(60):
        n1, n2 = int(rng.integers(0, 6)), int(rng.integers(0, 6))
        g1 = synth.er_graph(rng, n1, 0.5, 2, 2)
        g2 = synth.er_graph(rng, n2, 0.5, 2, 2)
        for costs in (COSTS["unit"], COSTS["uniform"], (3, 5, 5, 2, 4, 4)):
            assert bruteforce.exact_ged(g1, g2, costs)[0] == bruteforce.exact_ged(g2, g1, costs)[0]


def test_bruteforce_isomorphic_zero():
    from oracle import bruteforce
    rng = synth.rng_for(7)
    for k in range(20):
        g = synth.er_graph(rng, 6, 0.5, 3, 2)
        h = synth.permute(g, rng.permutation(6))
        assert bruteforce.exact_ged(g, h, COSTS["setting1"])[0] == 0


# ------------------------------------------------------------------ oracle vs brute force
def _lower_bound(g1, g2, c):
    vsub, vdel, vins, esub, edel, eins = c
    return (max(0, g1.n - g2.n) * vdel + max(0, g2.n - g1.n) * vins
            + max(0, g1.m - g2.m) * edel + max(0, g2.m - g1.m) * eins)


ASYM = (3, 5, 7, 2, 4, 6)  # every cost distinct: catches swapped cost terms


@pytest.mark.parametrize("costs", ["unit", "setting1", "setting2", "asym"])
def test_oracle_vs_bruteforce_small(oracle_lib, costs):
    """K-Best >= exact for every K; = exact once K covers the widths; LB holds;
    the witness re-verifies with the order-free formula."""
    from oracle import bruteforce
    c = ASYM if costs == "asym" else COSTS[costs]
    rng = synth.rng_for(2024, len(costs))
    for k in range(120):
        n1, n2 = int(rng.integers(0, 7)), int(rng.integers(0, 7))
        p = (0.2, 0.5, 0.8)[k % 3]
        nl = 1 + k % 3
        g1 = synth.er_graph(rng, n1, p, nl, 1 + (k % 2))
        g2 = synth.er_graph(rng, n2, p, nl, 1 + (k % 2))
        ged, allc, F = bruteforce.exact_ged(g1, g2, c)
        full = bruteforce.width(n1, n2, n1)
        lb = _lower_bound(g1, g2, c)
        assert ged >= lb
        for K in (1, 2, 16, full):
            r = oracle_lib.kbest(g1, g2, c, K)
            assert r["cost"] >= ged
            # the returned mapping is one of the injections and its order-free cost is the cost
            assert int(bruteforce.costs_of(g1, g2, c, r["mapping"][None, :])[0]) == r["cost"]
            assert oracle_lib.mapping_cost(g1, g2, c, r["mapping"]) == r["cost"]
            if K >= full:
                assert r["cost"] == ged


def test_oracle_identity_mapping(oracle_lib):
    """GED_K(G,G) = 0 with the identity mapping for every K >= 1 (O.3 P4)."""
    rng = synth.rng_for(11)
    for k in range(40):
        n = int(rng.integers(1, 25))
        g = synth.er_graph(rng, n, float(rng.random()), 3, 2)
        for K in (1, 3, 50):
            r = oracle_lib.kbest(g, g, COSTS["setting1"], K)
            assert r["cost"] == 0
            assert r["mapping"].tolist() == list(range(n))


def test_oracle_tree_counts_exhaustive(oracle_lib):
    """With K >= every width nothing is pruned: children = sum_{i=1..n1} W(i),
    parents = sum_{i=0..n1-1} W(i) (each child is a distinct partial injection)."""
    from oracle import bruteforce
    rng = synth.rng_for(5)
    for n1, n2 in [(1, 1), (2, 3), (3, 2), (4, 4), (5, 3), (3, 5)]:
        g1 = synth.er_graph(rng, n1, 0.5, 2)
        g2 = synth.er_graph(rng, n2, 0.5, 2)
        r = oracle_lib.kbest(g1, g2, COSTS["setting1"], 10 ** 6, levels=True)
        assert r["children"] == sum(bruteforce.width(n1, n2, i) for i in range(1, n1 + 1))
        assert r["parents"] == sum(bruteforce.width(n1, n2, i) for i in range(0, n1))
        for i, (front, cand, thr) in enumerate(r["levels"]):
            assert front == bruteforce.width(n1, n2, i) and cand == bruteforce.width(n1, n2, i + 1) and thr == -1


def test_oracle_frontier_bound_and_counts(oracle_lib):
    """Frontier <= K every level; candidates = sum over parents of (n2 - s + 1)."""
    rng = synth.rng_for(6)
    g1 = synth.er_graph(rng, 9, 0.4, 3)
    g2 = synth.er_graph(rng, 10, 0.4, 3)
    K = 37
    r = oracle_lib.kbest(g1, g2, COSTS["setting1"], K, levels=True)
    for i, (front, cand, thr) in enumerate(r["levels"]):
        assert front <= K
        assert front <= cand <= front * (g2.n + 1)
        if cand > K:
            assert thr >= 0
        if i + 1 < len(r["levels"]):
            assert r["levels"][i + 1][0] == min(K, cand)


def test_oracle_deterministic_batch(oracle_lib):
    """Identical results regardless of thread count."""
    w = synth.config_workload(3, npairs=6, K=20)
    pairs = [w.pair(k) for k in range(w.npairs)]
    a = oracle_lib.kbest_batch(pairs, w.costs, w.K, nthreads=1)
    b = oracle_lib.kbest_batch(pairs, w.costs, w.K, nthreads=4)
    assert np.array_equal(a[0], b[0]) and all(np.array_equal(x, y) for x, y in zip(a[1], b[1]))
    for k, (g1, g2) in enumerate(pairs):
        r = oracle_lib.kbest(g1, g2, w.costs, w.K)
        assert r["cost"] == a[0][k] and np.array_equal(r["mapping"], a[1][k]) and r["children"] == a[2][k]


def test_oracle_rejects_bad_input(oracle_lib):
    from oracle.oracle import OracleError
    g = synth.path_graph(3)
    loop = Graph(2, [0, 0], [[1, 1]])
    dup = Graph(3, [0, 0, 0], [[0, 1], [1, 0]])
    oob = Graph(2, [0, 0], [[0, 2]])
    for bad in (loop, dup, oob):
        with pytest.raises(OracleError) as e:
            oracle_lib.kbest(bad, g, COSTS["unit"], 2)
        assert e.value.code == 2
    with pytest.raises(OracleError):
        oracle_lib.kbest(g, g, COSTS["unit"], 0)
    with pytest.raises(OracleError):
        oracle_lib.kbest(g, g, (1, -1, 1, 1, 1, 1), 2)


# ------------------------------------------------------------------ NEXT-4: approximate top-K
def _lex_first_k(n1, n2, K):
    """The lexicographically first K complete nodes of the vertex-branching tree in its canonical child
    order (free targets ascending, deletion last; readings C5, C13), from the brute force's enumeration."""
    from oracle import bruteforce
    F = bruteforce.injections(n1, n2)
    if n1 == 0:
        return F
    key = np.where(F == bruteforce.DEL, n2, F)
    order = np.lexsort(key.T[::-1])  # column 0 most significant
    return F[order[:K]]


def test_approx_topk_one_bin_is_lexicographic_first_k(oracle_lib):
    """With one bin for every PED (2^15 wide) the keys all tie, so every level keeps its first K children in
    (p, j) order; the survivors are then the lexicographically first K complete mappings (each parent has a
    deletion child, so the first K children of a level come from its first K parents), and the result is the
    order-free cost minimum over them, first position on ties -- the brute force's enumeration and formula."""
    from oracle import bruteforce
    rng = synth.rng_for(5151)
    differs = 0
    for k in range(120):
        n1, n2 = int(rng.integers(1, 6)), int(rng.integers(1, 6))
        g1 = synth.er_graph(rng, n1, (0.2, 0.5, 0.8)[k % 3], 2, 1 + k % 2)
        g2 = synth.er_graph(rng, n2, (0.2, 0.5, 0.8)[k % 3], 2, 1 + k % 2)
        c = (COSTS["unit"], COSTS["setting1"], ASYM)[k % 3]
        for K in (1, 3, 20):
            first = _lex_first_k(n1, n2, K)
            cst = bruteforce.costs_of(g1, g2, c, first)
            b = int(np.argmin(cst))
            r = oracle_lib.kbest(g1, g2, c, K, flags=oracle_lib.APPROX(15))
            assert r["cost"] == int(cst[b]), (k, K)
            assert r["mapping"].tolist() == first[b].tolist(), (k, K)
            differs += r["cost"] != oracle_lib.kbest(g1, g2, c, K)["cost"]
    assert differs > 0  # the pin separates the variant from the exact selection


def test_approx_topk_bounds(oracle_lib):
    """Any bin width: shift 0 is the exact selection; the cost is >= the exact GED, the witness re-verifies,
    and once K covers every level's width (nothing is dropped) the cost is the exact GED."""
    from oracle import bruteforce
    rng = synth.rng_for(5252)
    for k in range(100):
        n1, n2 = int(rng.integers(1, 7)), int(rng.integers(1, 7))
        g1 = synth.er_graph(rng, n1, (0.2, 0.5, 0.8)[k % 3], 3, 1 + k % 2)
        g2 = synth.er_graph(rng, n2, (0.2, 0.5, 0.8)[k % 3], 3, 1 + k % 2)
        c = (COSTS["unit"], COSTS["setting1"], ASYM)[k % 3]
        ged = bruteforce.exact_ged(g1, g2, c)[0]
        full = bruteforce.width(n1, n2, n1)
        for K in (1, 4, full):
            ex = oracle_lib.kbest(g1, g2, c, K)
            z = oracle_lib.kbest(g1, g2, c, K, flags=oracle_lib.APPROX(0))
            assert z["cost"] == ex["cost"] and z["mapping"].tolist() == ex["mapping"].tolist()
            for s in (1, 2, 3):
                r = oracle_lib.kbest(g1, g2, c, K, flags=oracle_lib.APPROX(s))
                assert r["cost"] >= ged
                assert oracle_lib.mapping_cost(g1, g2, c, r["mapping"]) == r["cost"]
                if K >= full:
                    assert r["cost"] == ged
