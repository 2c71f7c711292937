"""Edit-path materialisation and application.

libfastged's host functions against the plain oracle (oracle/editpath.py), element by element, and
against what the definitions fix: the operation costs sum to the order-free path cost of the mapping
(O.4, another formula), prefix 0 is g1, the full path reproduces g2 under the returned origin, and SPEC's
printed examples.  No GPU: the mappings come from the CPU oracle's K-Best search."""
import numpy as np
import pytest

from paper_2605_00830_b200 import synth
from paper_2605_00830_b200.synth import COSTS, Graph


@pytest.fixture(scope="module")
def fgb():
    from paper_2605_00830_b200 import binding, build
    build.build()
    binding.lib()
    return binding


def test_spec_examples(fgb):
    from oracle import editpath as oe
    P2, K1 = synth.path_graph(2), synth.empty_graph(1)
    ops, cost = fgb.edit_path(P2, K1, COSTS["setting1"], [0, -1])
    assert cost == 6  # Sub v0->u0 (0) + Del v1 (4) + implied edel (2)
    assert [o[0] for o in ops] == ["vsub", "vdel", "edel"]
    g, org = fgb.apply_edit_path(P2, K1, [0, -1], 2)  # single vertex, zero edges
    assert g.n == 1 and g.m == 0 and fgb.graphs_equal_under_mapping(g, K1, org)
    g0, org0 = fgb.apply_edit_path(P2, K1, [0, -1], 0)  # prefix 0 = g1
    assert g0.n == 2 and g0.m == 1 and org0.tolist() == [-1, -2]
    c, n = Graph(1, [0], np.zeros((0, 2))), Graph(1, [1], np.zeros((0, 2)))
    assert fgb.graphs_equal_under_mapping(c, c, [0]) and not fgb.graphs_equal_under_mapping(c, n, [0])
    assert not fgb.graphs_equal_under_mapping(synth.complete_graph(3), synth.path_graph(3), [0, 1, 2])
    assert oe.edit_path(P2, K1, COSTS["setting1"], [0, -1]) == (ops, cost)


def test_against_oracle_on_kbest_mappings(fgb, oracle_lib):
    from oracle import editpath as oe
    rng = synth.rng_for(2121)
    for k in range(60):
        n1, n2 = int(rng.integers(0, 12)), int(rng.integers(0, 12))
        g1 = synth.er_graph(rng, n1, 0.4, 3, 1 + k % 3)
        g2 = synth.er_graph(rng, n2, 0.4, 3, 1 + k % 3)
        costs = (COSTS["setting1"], COSTS["unit"], (3, 5, 7, 2, 4, 6))[k % 3]
        r = oracle_lib.kbest(g1, g2, costs, 20)
        m = r["mapping"]
        ops, cost = fgb.edit_path(g1, g2, costs, m)
        assert (ops, cost) == oe.edit_path(g1, g2, costs, m)
        assert cost == r["cost"] == oracle_lib.mapping_cost(g1, g2, costs, m)  # the order-free cost (O.4)
        nins = n2 - int((m >= 0).sum())
        for t in range(0, n1 + nins + 1):
            g, org = fgb.apply_edit_path(g1, g2, m, t)
            n, vl, edges, origin = oe.apply_edit_path(g1, g2, m, t)
            assert g.n == n and g.vlabels.tolist() == vl and org.tolist() == origin
            assert sorted((int(a), int(b), int(l)) for (a, b), l in zip(g.edges.tolist(), g.elabels.tolist())) == edges
        assert (org >= 0).all() and fgb.graphs_equal_under_mapping(g, g2, org)  # full path gives g2
        assert oe.graphs_equal_under_mapping(g, g2, org)


def test_invalid_mapping_rejected(fgb):
    g = synth.path_graph(3)
    for bad in ([0, 0, 1], [0, 5, 1]):
        with pytest.raises(fgb.FastGedError) as e:
            fgb.edit_path(g, g, COSTS["unit"], bad)
        assert e.value.code == fgb.ERR_INPUT
    with pytest.raises(fgb.FastGedError):
        fgb.apply_edit_path(g, g, [0, 1, 2], 9)
