"""Pins for the exact DFS branch-and-bound oracle (og_exact).

It extends the exactness checks of the K-Best path beyond the brute force's 7 vertices (Table-1
protocol).  Pinned against: the brute force over all partial injections (another
language, an order-free cost), SPEC's printed values, the admissible root bound, symmetry under
symmetric costs, and independence from its incumbent.  No GPU."""
import numpy as np
import pytest

from paper_2605_00830_b200 import synth
from paper_2605_00830_b200.synth import COSTS

ASYM = (3, 5, 7, 2, 4, 6)


@pytest.mark.parametrize("costs", ["unit", "setting1", "setting2", "asym"])
def test_exact_equals_bruteforce(oracle_lib, costs):
    from oracle import bruteforce
    c = ASYM if costs == "asym" else COSTS[costs]
    rng = synth.rng_for(333, len(costs))
    for k in range(100):
        n1, n2 = int(rng.integers(0, 7)), int(rng.integers(0, 7))
        g1 = synth.er_graph(rng, n1, (0.2, 0.5, 0.8)[k % 3], 1 + k % 3, 1 + k % 2)
        g2 = synth.er_graph(rng, n2, (0.2, 0.5, 0.8)[k % 3], 1 + k % 3, 1 + k % 2)
        e = oracle_lib.exact(g1, g2, c)
        assert e["optimal"]
        assert e["cost"] == bruteforce.exact_ged(g1, g2, c)[0]
        assert int(bruteforce.costs_of(g1, g2, c, e["mapping"][None, :])[0]) == e["cost"]


def test_exact_spec_examples(oracle_lib):
    """exact(g, g) = 0 with the identity; exact(triangle, P3) = 2; exact(K1 C, K1 N) = 2."""
    s1 = COSTS["setting1"]
    rng = synth.rng_for(9)
    g = synth.er_graph(rng, 9, 0.4, 3, 2)
    e = oracle_lib.exact(g, g, s1)
    assert e["cost"] == 0 and e["mapping"].tolist() == list(range(9))
    assert oracle_lib.exact(synth.complete_graph(3), synth.path_graph(3), s1)["cost"] == 2
    k1c, k1n = synth.relabel(synth.empty_graph(1), [0]), synth.relabel(synth.empty_graph(1), [1])
    assert oracle_lib.exact(k1c, k1n, s1)["cost"] == 2


def test_root_lower_bound_example(oracle_lib):
    """the root bound of K1 vs triangle is 2*4 + 3*2 = 14, which is also the exact distance."""
    assert oracle_lib.exact(synth.empty_graph(1), synth.complete_graph(3), COSTS["setting1"])["cost"] == 14


def test_exact_beyond_bruteforce(oracle_lib):
    """8-10 vertices: exact <= K-Best for every K, = K-Best at a K covering the widths (n = 8: W(8) for
    8x8 = 1,441,729 leaves), symmetric under symmetric costs, independent of the incumbent's K."""
    rng = synth.rng_for(808)
    for k in range(12):
        n = 8 + k % 3
        g1 = synth.er_graph(rng, n, (0.2, 0.5, 0.8)[k % 3], 3)
        g2 = synth.er_graph(rng, n, (0.2, 0.5, 0.8)[k % 3], 3)
        c = COSTS["uniform"] if k % 2 else COSTS["setting2"]  # both symmetric (vdel = vins, edel = eins)
        e = oracle_lib.exact(g1, g2, c)
        assert e["optimal"]
        for K in (1, 50, 2000):
            assert e["cost"] <= oracle_lib.kbest(g1, g2, c, K)["cost"]
        assert oracle_lib.exact(g2, g1, c)["cost"] == e["cost"]
        assert oracle_lib.exact(g1, g2, c, K0=300)["cost"] == e["cost"]
        if n == 8:
            assert oracle_lib.kbest(g1, g2, c, 1_441_729)["cost"] == e["cost"]


def test_exact_budget(oracle_lib):
    """With the expansion budget exhausted the best path found is returned, flagged non-optimal."""
    rng = synth.rng_for(1)
    g1, g2 = synth.er_graph(rng, 10, 0.5, 2), synth.er_graph(rng, 10, 0.5, 2)
    e = oracle_lib.exact(g1, g2, COSTS["setting1"], K0=1, node_limit=3)
    assert not e["optimal"]
    assert e["cost"] <= oracle_lib.kbest(g1, g2, COSTS["setting1"], 1)["cost"]
    assert oracle_lib.mapping_cost(g1, g2, COSTS["setting1"], e["mapping"]) == e["cost"]


def test_exact_batch_matches_single(oracle_lib):
    rng = synth.rng_for(77)
    pairs = [(synth.er_graph(rng, 7, 0.4, 3), synth.er_graph(rng, 8, 0.4, 3)) for _ in range(10)]
    c, m, nodes, opt = oracle_lib.exact_batch(pairs, COSTS["setting1"], nthreads=4)
    for k, (g1, g2) in enumerate(pairs):
        e = oracle_lib.exact(g1, g2, COSTS["setting1"])
        assert opt[k] and c[k] == e["cost"] and np.array_equal(m[k], e["mapping"])
