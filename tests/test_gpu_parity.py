"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by element.

All arithmetic is integer, so the bar is bit-exact: same GED, same mapping (the same edit path
under the (PED, parent, child) tie rule), same number of children evaluated, same per-level
frontier sizes and thresholds.  Inputs are the seeded synthetic workloads of DESIGN.md §5.
"""
import os

import numpy as np
import pytest

from paper_2605_00830_b200 import synth
from paper_2605_00830_b200.synth import COSTS, Graph

pytestmark = pytest.mark.gpu

NCPU = os.cpu_count() or 1


@pytest.fixture(scope="module")
def fg():
    from paper_2605_00830_b200 import binding, build
    build.build()
    return binding


@pytest.fixture(scope="module")
def handle(fg):
    h = fg.Handle(0)
    yield h
    h.close()


@pytest.fixture(scope="module")
def oracle():
    from oracle import oracle as o
    o.build()
    return o


def gpu_batch(fg, h, pairs, costs, K):
    graphs = [g for ab in pairs for g in ab]
    packed = fg.PackedGraphs(graphs)
    a = np.arange(0, 2 * len(pairs), 2)
    c, m, offs, ch = h.solve_batch(packed, a, a + 1, costs, K)
    return c, [m[offs[k]:offs[k + 1]] for k in range(len(pairs))], ch


def assert_batch_parity(fg, h, oracle, pairs, costs, K, label=""):
    gc, gm, gch = gpu_batch(fg, h, pairs, costs, K)
    oc, om, och = oracle.kbest_batch(pairs, costs, K, nthreads=NCPU)
    bad = [k for k in range(len(pairs)) if gc[k] != oc[k] or not np.array_equal(gm[k], om[k]) or gch[k] != och[k]]
    assert not bad, f"{label}: {len(bad)} of {len(pairs)} pairs differ, first {bad[:5]}: " \
                    f"gpu {gc[bad[0]]} {gm[bad[0]].tolist()} {gch[bad[0]]} / oracle {oc[bad[0]]} {om[bad[0]].tolist()} {och[bad[0]]}"
    return gc


# ------------------------------------------------------------------ configs
def test_config1_all_pairs(fg, handle, oracle):
    """configs[0]: 1000 unlabeled G(6,p) pairs, unit costs, K=16 — every pair."""
    w = synth.config_workload(1)
    pairs = [w.pair(k) for k in range(w.npairs)]
    assert_batch_parity(fg, handle, oracle, pairs, w.costs, w.K, "cfg1")


def test_config1_exact_at_full_width(fg, handle):
    """K=16384 >= 13,327 = final width of 6x6: the GPU result equals brute-force exact GED."""
    from oracle import bruteforce
    w = synth.config_workload(1, npairs=150)
    pairs = [w.pair(k) for k in range(w.npairs)]
    gc, gm, _ = gpu_batch(fg, handle, pairs, w.costs, 16384)
    for k, (g1, g2) in enumerate(pairs):
        assert gc[k] == bruteforce.exact_ged(g1, g2, w.costs)[0]
        assert int(bruteforce.costs_of(g1, g2, w.costs, gm[k][None, :])[0]) == gc[k]


def test_config2_aids_like(fg, handle, oracle):
    """configs[1]: 10k AIDS-like labelled molecule pairs, K=100 — every pair."""
    w = synth.config_workload(2)
    pairs = [w.pair(k) for k in range(w.npairs)]
    assert_batch_parity(fg, handle, oracle, pairs, w.costs, w.K, "cfg2")


def test_mixed_groups_one_batch(fg, handle, oracle):
    """One batch holding every kernel variant at once — unlabelled ER pairs of word widths 1..4 and
    labelled molecule pairs — so the word-width/label groups run concurrently on their own streams
    and scratch slices; also repeated through the pipelined (>= 4096 pairs) path."""
    w3 = synth.config_workload(3, npairs=50, K=200)
    w2 = synth.config_workload(2, npairs=50)
    big = [synth.large_pair(n, 0.1, seed=n)[0:2] for n in (100, 120)]  # n2 in (96, 128]: W = 4
    pairs = [w3.pair(k) for k in range(w3.npairs)] + [w2.pair(k) for k in range(w2.npairs)] + big
    order = np.random.default_rng(7).permutation(len(pairs))
    pairs = [pairs[k] for k in order]
    assert_batch_parity(fg, handle, oracle, pairs, w3.costs, 200, "mixed")
    st = handle.stats()
    assert st["kernel_launches"] >= 5
    many = pairs * (4100 // len(pairs) + 1)
    gc, gm, gch = gpu_batch(fg, handle, many, w3.costs, 200)
    base, bm, bch = gpu_batch(fg, handle, pairs, w3.costs, 200)
    for k in range(len(many)):
        r = k % len(pairs)
        assert gc[k] == base[r] and np.array_equal(gm[k], bm[r]) and gch[k] == bch[r], k


def test_config3_er_grid_sampled(fg, handle, oracle):
    """configs[2]: ER n=30..70, p=.1-.5, K=1000 — 100 pairs covering all 25 (n, p) cells, run in the
    same batched launch configuration bench.py times."""
    w = synth.config_workload(3, npairs=100)
    pairs = [w.pair(k) for k in range(w.npairs)]
    assert_batch_parity(fg, handle, oracle, pairs, w.costs, w.K, "cfg3")


def _golden(name):
    f = os.path.join(os.path.dirname(__file__), "golden", name)
    if not os.path.exists(f):
        pytest.fail(f"{f} missing: run scripts/make_golden.py (oracle results at full size)")
    return np.load(f)


def assert_golden(z, gc, gm, goffs, gch, label):
    """GPU results of the pairs z['idx'] against the oracle's stored results, element by element."""
    idx, oc, om, oo, och = z["idx"], z["cost"], z["map"], z["offs"], z["children"]
    bad = [x for x in range(idx.shape[0])
           if gc[idx[x]] != oc[x] or gch[idx[x]] != och[x]
           or not np.array_equal(gm[goffs[idx[x]]:goffs[idx[x] + 1]], om[oo[x]:oo[x + 1]])]
    assert not bad, f"{label}: {len(bad)} of {idx.shape[0]} pairs differ from the oracle, first pair {idx[bad[0]]}"
    return idx.shape[0]


def test_config3_full_batch_vs_golden(fg, handle):
    """configs[2], the bench workload: all 10,000 pairs in the launch configuration bench.py times,
    bit-exact against the oracle's results for every pair (tests/golden/oracle_cfg3.npz)."""
    w = synth.config_workload(3)
    packed = fg.PackedGraphs(w.graphs)
    gc, gm, offs, gch = handle.solve_batch(packed, w.pair_a, w.pair_b, w.costs, w.K)
    assert assert_golden(_golden("oracle_cfg3.npz"), gc, gm, offs, gch, "cfg3") == 10_000
    # the device-resident path bench.py times gives the same results
    b = handle.upload(packed, w.pair_a, w.pair_b)
    b.run(w.costs, w.K)
    r = b.download()
    b.free()
    assert np.array_equal(r[0], gc) and np.array_equal(r[1], gm)


@pytest.mark.parametrize("setting", ["s1", "s2"])
def test_config5_allpairs_vs_golden(fg, handle, setting):
    """configs[4]: the full 1,999,000-pair all-pairs batch in one call (Setting 1 and Setting 2);
    every 100th pair (19,990) bit-exact against the oracle (tests/golden/oracle_cfg5_*.npz)."""
    w = synth.config_workload(5, variant=None if setting == "s1" else "setting2")
    packed = fg.PackedGraphs(w.graphs)
    gc, gm, offs, gch = handle.solve_batch(packed, w.pair_a, w.pair_b, w.costs, w.K)
    assert gc.shape[0] == 1_999_000 and (gc >= 0).all()
    assert assert_golden(_golden(f"oracle_cfg5_{setting}.npz"), gc, gm, offs, gch, f"cfg5-{setting}") == 19_990


def test_batched_frontier_beyond_65535(fg, handle, oracle):
    """K = 70,000 on small pairs: the frontier capacity exceeds 65,535, so the batched kernel keeps
    its work arrays in global scratch and decodes survivor positions by binary search over the parent
    offsets (batch_kernel.cuh decode, Kc > 65535 branch)."""
    rng = synth.rng_for(70)
    pairs = []
    for k in range(6):
        n1, n2 = int(rng.integers(6, 9)), int(rng.integers(9, 14))
        pairs.append((synth.er_graph(rng, n1, 0.4, 3), synth.er_graph(rng, n2, 0.4, 3)))
    assert_batch_parity(fg, handle, oracle, pairs, COSTS["setting1"], 70_000, "K=70000")


def test_oversize_pairs_routed_inside_a_batch(fg, handle, oracle):
    """Pairs beyond the batched limits (n2 in {150, 300}) inside one fastged_solve_batch call are solved
    by the whole-GPU kernel and land in the same outputs; the rest of the batch is unaffected."""
    small = [synth.config_workload(3, npairs=6, K=300).pair(k) for k in range(6)]
    big = [synth.large_pair(150, 0.1, seed=3), synth.large_pair(300, 0.05, seed=5)]
    pairs = [small[0], big[0], small[1], small[2], big[1], small[3]]
    assert_batch_parity(fg, handle, oracle, pairs, COSTS["setting1"], 300, "mixed sizes")


def test_frontier_2_24_with_128_targets(fg, handle, oracle):
    """K = 2^24 with n2 = 128: the batched plan's 32-bit offsets would wrap (Kc * csmax
    > 2^31), so the pair must go to the whole-GPU kernel, inside a batch too; the result equals the
    oracle's (2.7e8 candidates at the last level, 2^24 kept)."""
    rng = synth.rng_for(24)
    g1 = synth.er_graph(rng, 4, 0.5, 2)
    g2 = synth.er_graph(rng, 128, 0.02, 2)
    K = 1 << 24
    o = oracle.kbest(g1, g2, COSTS["setting1"], K)
    r = handle.solve_pair(g1, g2, COSTS["setting1"], K)
    assert r["cost"] == o["cost"] and np.array_equal(r["mapping"], o["mapping"]) and r["children"] == o["children"]
    small = (synth.path_graph(3), synth.cycle_graph(4))
    gc, gm, gch = gpu_batch(fg, handle, [(g1, g2), small], COSTS["setting1"], K)
    assert gc[0] == o["cost"] and np.array_equal(gm[0], o["mapping"])
    assert gc[1] == oracle.kbest(*small, COSTS["setting1"], K)["cost"]


# ------------------------------------------------------------------ per-level parity
@pytest.mark.parametrize("flags", [0, 2], ids=["window253", "window2"])
def test_per_level_trace(fg, oracle, flags):
    """Frontier size, candidates and threshold PED of every level equal the oracle's."""
    h = fg.Handle(0, flags=flags)
    rng = synth.rng_for(77)
    for k in range(12):
        n1, n2 = int(rng.integers(5, 40)), int(rng.integers(5, 40))
        g1 = synth.er_graph(rng, n1, 0.3, 3)
        g2 = synth.er_graph(rng, n2, 0.3, 3)
        K = int(rng.integers(1, 300))
        r = h.solve_pair(g1, g2, COSTS["setting1"], K, levels=True)
        o = oracle.kbest(g1, g2, COSTS["setting1"], K, levels=True)
        assert r["levels"] == [tuple(x) for x in o["levels"]]
        assert r["cost"] == o["cost"] and np.array_equal(r["mapping"], o["mapping"])
        assert r["children"] == o["children"] and r["parents"] == o["parents"]
    h.close()


# ------------------------------------------------------------------ method variant (NEXT-4)
@pytest.mark.parametrize("shift", [1, 3])
@pytest.mark.parametrize("window", [0, 2], ids=["window253", "window2"])
def test_variant_approx_topk_matches_oracle(fg, oracle, shift, window):
    """FASTGED_FLAG_APPROX (approximate top-K: PED bins of 2^shift) on the whole-GPU kernel against the
    oracle's variant, bit-exact: cost, mapping, children and per-level records (the threshold is the K-th
    smallest key's bin) for single pairs, a batch (every pair routed to the whole-GPU kernel) and 2 virtual
    ranks of the sharded mode."""
    flags = fg.FLAG_APPROX(shift) | (fg.FLAG_DEBUG_WINDOW if window else 0)
    h = fg.Handle(0, flags=flags)
    hs = fg.Handle(0, world_size=2, flags=flags | fg.FLAG_VIRTUAL_SHARDS)
    rng = synth.rng_for(71, shift, window)
    pairs = []
    for k in range(8):
        n1, n2 = int(rng.integers(3, 60)), int(rng.integers(3, 60))
        pairs.append((synth.er_graph(rng, n1, (0.1, 0.3)[k % 2], 4, 1 + k % 2), synth.er_graph(rng, n2, (0.1, 0.3)[k % 2], 4, 1 + k % 2)))
    for k, (g1, g2) in enumerate(pairs):
        K = int(rng.integers(1, 2000))
        o = oracle.kbest(g1, g2, COSTS["setting1"], K, levels=True, flags=oracle.APPROX(shift))
        for hh in (h, hs):
            r = hh.solve_pair(g1, g2, COSTS["setting1"], K, levels=True)
            assert r["cost"] == o["cost"] and np.array_equal(r["mapping"], o["mapping"]), (k, K)
            assert r["children"] == o["children"] and r["levels"] == [tuple(x) for x in o["levels"]], (k, K)
    g1, g2 = synth.large_pair(300, 0.05, seed=12)
    o = oracle.kbest(g1, g2, COSTS["setting1"], 3000, flags=oracle.APPROX(shift))
    r = h.solve_pair(g1, g2, COSTS["setting1"], 3000)
    assert r["cost"] == o["cost"] and np.array_equal(r["mapping"], o["mapping"])
    gc, gm, gch = gpu_batch(fg, h, pairs, COSTS["setting2"], 200)
    oc, om, och = oracle.kbest_batch(pairs, COSTS["setting2"], 200, flags=oracle.APPROX(shift))
    for k in range(len(pairs)):
        assert gc[k] == oc[k] and np.array_equal(gm[k], om[k]) and gch[k] == och[k], k
    h.close()
    hs.close()


@pytest.mark.parametrize("window", [0, 2], ids=["window127", "window2"])
def test_variant_last_by_total_matches_oracle(fg, oracle, window):
    """FASTGED_FLAG_LAST_BY_TOTAL (last level ranked by PED + completion, the alternative to reading C10)
    against the oracle's variant, bit-exact, on ER, labelled molecule and n1 != n2 pairs, through the batched,
    whole-GPU and sharded kernels; combined with the approximate top-K flag it is refused."""
    flags = fg.FLAG_LAST_BY_TOTAL | (fg.FLAG_DEBUG_WINDOW if window else 0)
    h = fg.Handle(0, flags=flags)
    w3 = synth.config_workload(3, npairs=50, K=300)
    w2 = synth.config_workload(2, npairs=200)
    rng = synth.rng_for(61)
    odd = [(synth.er_graph(rng, int(rng.integers(2, 30)), 0.3, 3), synth.er_graph(rng, int(rng.integers(2, 60)), 0.2, 3))
           for _ in range(30)]
    for pairs, costs, K in (([w3.pair(k) for k in range(w3.npairs)], w3.costs, w3.K),
                            ([w2.pair(k) for k in range(w2.npairs)], w2.costs, w2.K),
                            (odd, COSTS["setting2"], 40)):
        gc, gm, gch = gpu_batch(fg, h, pairs, costs, K)
        oc, om, och = oracle.kbest_batch(pairs, costs, K, flags=oracle.LAST_BY_TOTAL)
        lc, _, _ = oracle.kbest_batch(pairs, costs, K)
        for k in range(len(pairs)):
            assert gc[k] == oc[k] and np.array_equal(gm[k], om[k]) and gch[k] == och[k], k
            assert gc[k] <= lc[k]
    # the whole-GPU kernel (n2 > 128, or forced) and 2 virtual ranks of the sharded kernel rank the last level the same way
    hs = fg.Handle(0, world_size=2, flags=flags | fg.FLAG_VIRTUAL_SHARDS)
    hf = fg.Handle(0, flags=flags | fg.FLAG_FORCE_LARGE)
    rng2 = synth.rng_for(62, window)
    cases = [synth.large_pair(150, 0.1, seed=3), synth.large_pair(140, 0.05, seed=4)] + \
            [(synth.er_graph(rng2, int(rng2.integers(1, 40)), 0.3, 3, 1 + x % 2),
              synth.er_graph(rng2, int(rng2.integers(1, 60)), 0.3, 3, 1 + x % 2)) for x in range(10)]
    for x, (g1, g2) in enumerate(cases):
        K = 100 if x < 2 else int(rng2.integers(1, 500))
        o = oracle.kbest(g1, g2, COSTS["setting1"], K, levels=True, flags=oracle.LAST_BY_TOTAL)
        for hh in (h, hs, hf):
            r = hh.solve_pair(g1, g2, COSTS["setting1"], K, levels=True)
            assert r["cost"] == o["cost"] and np.array_equal(r["mapping"], o["mapping"]), (x, K)
            assert r["children"] == o["children"] and r["levels"] == [tuple(v) for v in o["levels"]], (x, K)
    with pytest.raises(fg.FastGedError) as e:
        fg.Handle(0, flags=flags | fg.FLAG_APPROX(2)).solve_pair(*cases[0], COSTS["setting1"], 100)
    assert e.value.code == fg.ERR_ARG
    h.close()
    hs.close()
    hf.close()


# ------------------------------------------------------------------ KNN_GED (NEXT-3)
def test_knn_ged_matrix_matches_oracle(fg, handle, oracle):
    """The test -> train GED matrix of the KNN_GED protocol (uniform costs) from one
    batched GPU call equals the oracle's matrix element by element, so the classification is the same."""
    from paper_2605_00830_b200 import knn
    graphs, y = synth.two_class_molecules(15, seed=5)
    tr, te = knn.split_70_30(len(graphs), seed=1)
    D = knn.ged_matrix(handle, fg.PackedGraphs(graphs), te, tr, COSTS["uniform"], 1000)
    pairs = [(graphs[a], graphs[b]) for a in te for b in tr]
    oc, _, _ = oracle.kbest_batch(pairs, COSTS["uniform"], 1000, nthreads=NCPU)
    assert np.array_equal(D.reshape(-1), oc)
    acc, pred, te2, _ = knn.knn_ged(handle, graphs, y, COSTS["uniform"], K=1000, k=1, seed=1)
    assert np.array_equal(te2, te) and np.array_equal(pred, knn.knn_predict(oc.reshape(D.shape), y[tr], 1))


def test_allpairs_checkpointed_matches_one_batch(fg, handle, tmp_path):
    """The checkpointed all-pairs driver (chunks written atomically, resumed after an interruption) gives
    the same costs and mappings as one fastged_solve_batch over all pairs."""
    from paper_2605_00830_b200 import allpairs
    w = synth.config_workload(5)
    graphs = w.graphs[:30]  # 435 unordered pairs
    assert allpairs.all_pairs(handle, graphs, w.costs, 200, str(tmp_path), chunk=100, keep_mappings=True, max_chunks=2) is None
    ia, ib, cost, ch, maps, offs = allpairs.all_pairs(handle, graphs, w.costs, 200, str(tmp_path), chunk=100, keep_mappings=True)
    c2, m2, o2, ch2 = handle.solve_batch(fg.PackedGraphs(graphs), ia, ib, w.costs, 200)
    assert np.array_equal(cost, c2) and np.array_equal(ch, ch2) and np.array_equal(maps.astype(np.int32), m2)


def test_random_torture(fg, handle, oracle):
    """Random sizes (n1, n2 in 0..90: every word width, n1 != n2), densities, vertex-label counts, 1..5 edge
    labels (more than 3 routes a pair to the whole-GPU path inside the batch), random costs including zeros
    and K from 1 to 5000 -- one batch per K against the oracle, element by element."""
    rng = synth.rng_for(9090)
    for K in (1, 2, 3, 7, 50, 500, 5000):
        pairs = []
        for k in range(40):
            nmax = 90 if K <= 500 else 40
            n1, n2 = int(rng.integers(0, nmax)), int(rng.integers(0, nmax))
            p = float(rng.random())
            nv, ne = int(rng.integers(1, 6)), int(rng.integers(1, 6))
            pairs.append((synth.er_graph(rng, n1, p, nv, ne), synth.er_graph(rng, n2, p, nv, ne)))
        costs = tuple(int(x) for x in rng.integers(0, 7, size=6))
        assert_batch_parity(fg, handle, oracle, pairs, costs, K, f"torture K={K} costs={costs}")


def test_package_entry_points(fg, oracle):
    """paper_2605_00830_b200.ged / ged_batch (convenience wrappers over the C ABI) give the oracle's results."""
    import paper_2605_00830_b200 as pkg
    w = synth.config_workload(2, npairs=20)
    pairs = [w.pair(k) for k in range(w.npairs)]
    c, maps = pkg.ged_batch(pairs, w.costs, K=w.K)
    oc, om, _ = oracle.kbest_batch(pairs, w.costs, w.K)
    assert np.array_equal(c, oc) and all(np.array_equal(x, y) for x, y in zip(maps, om))
    r = pkg.ged(*pairs[0], w.costs, K=w.K)
    assert r["cost"] == oc[0] and np.array_equal(r["mapping"], om[0])


# ------------------------------------------------------------------ edge cases
def test_edge_cases(fg, handle, oracle):
    rng = synth.rng_for(31)
    cases = []
    E = synth.empty_graph
    cases += [(E(0), E(0)), (E(0), synth.cycle_graph(5)), (synth.cycle_graph(5), E(0)), (E(3), E(4)),
              (synth.complete_graph(7), E(1))]
    # W boundaries and the deletion slot past the lanes (n2 = 32 W)
    for n2 in (1, 31, 32, 33, 63, 64, 65, 95, 96, 97, 127, 128):
        cases.append((synth.er_graph(rng, 20, 0.3, 2), synth.er_graph(rng, n2, 0.3, 2)))
    # many more source vertices than targets (deletions forced)
    cases.append((synth.er_graph(rng, 40, 0.2, 2), synth.er_graph(rng, 5, 0.5, 2)))
    # labelled edges with mismatches; g1 labels absent from g2
    g1 = synth.er_graph(rng, 15, 0.4, 3, 3)
    g2 = synth.er_graph(rng, 16, 0.4, 3, 2)
    cases.append((g1, g2))
    cases.append((Graph(g1.n, g1.vlabels, g1.edges, np.full(g1.m, 9, np.int32)), g2))
    for K in (1, 2, 7, 100, 5000):
        for costs in (COSTS["setting1"], (3, 5, 7, 2, 4, 6), COSTS["unit"], (0, 0, 0, 0, 0, 0)):
            assert_batch_parity(fg, handle, oracle, cases, costs, K, f"edge K={K} {costs}")


def test_identity_any_size(fg, handle):
    """GED_K(G, G) = 0 with the identity mapping for every K (O.3 P4)."""
    rng = synth.rng_for(3)
    pairs = []
    for k in range(40):
        g = synth.er_graph(rng, int(rng.integers(1, 129)), float(rng.random()), 4, 1 + k % 3)
        pairs.append((g, g))
    for K in (1, 64, 1000):
        gc, gm, _ = gpu_batch(fg, handle, pairs, COSTS["setting1"], K)
        assert (gc == 0).all()
        for k, (g, _) in enumerate(pairs):
            assert gm[k].tolist() == list(range(g.n))


# ------------------------------------------------------------------ whole-GPU (large) path
def test_large_path_small_pairs_forced(fg, oracle):
    """The whole-GPU cooperative kernel on small pairs (forced) agrees with the oracle."""
    h = fg.Handle(0, flags=fg.FLAG_FORCE_LARGE)
    hw = fg.Handle(0, flags=fg.FLAG_FORCE_LARGE | fg.FLAG_DEBUG_WINDOW)
    rng = synth.rng_for(41)
    for k in range(16):
        n1, n2 = int(rng.integers(0, 60)), int(rng.integers(0, 60))
        g1 = synth.er_graph(rng, n1, 0.3, 3, 1 + k % 2)
        g2 = synth.er_graph(rng, n2, 0.3, 3, 1 + k % 2)
        K = int(rng.integers(1, 2000))
        o = oracle.kbest(g1, g2, COSTS["setting1"], K, levels=True)
        for hh in (h, hw):
            r = hh.solve_pair(g1, g2, COSTS["setting1"], K, levels=True)
            assert r["cost"] == o["cost"] and np.array_equal(r["mapping"], o["mapping"]), k
            assert r["levels"] == [tuple(x) for x in o["levels"]]
    h.close()
    hw.close()


@pytest.mark.parametrize("n,p,K", [(150, 0.2, 2000), (260, 0.05, 1000), (300, 0.1, 500), (300, 0.92, 48)])
def test_large_pairs(fg, handle, oracle, n, p, K):
    """n2 > 128 (uint8 and uint16 lambda rows; p=0.92 gives g2 degrees > 255, i.e. uint16 counters) against the oracle."""
    g1, g2 = synth.large_pair(n, p, seed=9)
    r = handle.solve_pair(g1, g2, COSTS["setting1"], K, levels=True)
    o = oracle.kbest(g1, g2, COSTS["setting1"], K, levels=True)
    assert r["cost"] == o["cost"] and np.array_equal(r["mapping"], o["mapping"])
    assert r["children"] == o["children"]
    assert r["levels"] == [tuple(x) for x in o["levels"]]


def _cfg4_golden():
    import json
    f = os.path.join(os.path.dirname(__file__), "golden", "oracle_cfg4.json")
    return json.load(open(f))["runs"] if os.path.exists(f) else {}


@pytest.mark.parametrize("idx", range(8), ids=lambda k: "({},{},{})".format(*synth.config_workload(4).run_np[k]))
def test_config4_corners_vs_golden(fg, handle, idx):
    """configs[3]: every single-pair corner n in {200, 500} x p in {0.05, 0.2} x K in {1e4, 1e5}
    (the bench pair is (500, 0.05, 1e5)) bit-exact against the oracle's stored result: cost, mapping,
    children evaluated and every level's (N_i, c_i, threshold) (tests/golden/oracle_cfg4.json)."""
    runs = _cfg4_golden()
    if str(idx) not in runs:
        pytest.fail("tests/golden/oracle_cfg4.json lacks this corner: run scripts/make_golden.py cfg4")
    o = runs[str(idx)]
    w = synth.config_workload(4)
    g1, g2 = w.pair(idx)
    r = handle.solve_pair(g1, g2, w.costs, o["K"], levels=True)
    assert r["cost"] == o["cost"] and r["mapping"].tolist() == o["mapping"]
    assert r["children"] == o["children"] and r["parents"] == o["parents"]
    assert [list(x) for x in r["levels"]] == o["levels"]


def test_config4_n500_witness(fg, handle):
    """configs[3] bench pair (n=500, p=0.05, K=1e5): the returned mapping is injective and its
    order-free cost (O.4) equals the returned cost.  (No monotonicity in K is asserted: per-pair
    monotonicity is not guaranteed, SPEC S:247 / SURVEY C25.)"""
    from oracle import oracle as o
    w = synth.config_workload(4)
    g1, g2 = w.pair(5)  # (500, 0.05, 1e5)
    r = handle.solve_pair(g1, g2, w.costs, 100_000)
    m = r["mapping"]
    used = m[m >= 0]
    assert len(set(used.tolist())) == used.size and (used < g2.n).all()
    assert o.mapping_cost(g1, g2, w.costs, m) == r["cost"]


# ------------------------------------------------------------------ errors
def test_error_paths(fg, handle):
    g = synth.path_graph(4)
    for bad in (Graph(2, [0, 0], [[1, 1]]), Graph(3, [0, 0, 0], [[0, 1], [1, 0]]), Graph(2, [0, 0], [[0, 5]])):
        with pytest.raises(fg.FastGedError) as e:
            handle.solve_pair(bad, g, COSTS["unit"], 4)
        assert e.value.code == fg.ERR_INPUT
    with pytest.raises(fg.FastGedError) as e:
        handle.solve_pair(g, g, COSTS["unit"], 0)
    assert e.value.code == fg.ERR_ARG
    with pytest.raises(fg.FastGedError) as e:
        handle.solve_pair(g, g, (1, -1, 1, 1, 1, 1), 4)
    assert e.value.code == fg.ERR_ARG
    with pytest.raises(fg.FastGedError) as e:
        handle.solve_pair(g, g, (2 ** 30, 2 ** 30, 1, 1, 1, 1), 4)
    assert e.value.code == fg.ERR_OVERFLOW
    big = synth.er_graph(synth.rng_for(1), 1100, 0.01)
    with pytest.raises(fg.FastGedError) as e:
        handle.solve_pair(g, big, COSTS["unit"], 4)
    assert e.value.code == fg.ERR_CAPACITY
    # a bad pair inside a batch names its index
    with pytest.raises(fg.FastGedError) as e:
        gpu_batch(fg, handle, [(g, g), (g, Graph(2, [0, 0], [[1, 1]]))], COSTS["unit"], 4)
    assert "pair 1" in str(e.value)


def test_device_resident_split_matches_solve_batch(fg, handle):
    w = synth.config_workload(3, npairs=64)
    packed = fg.PackedGraphs(w.graphs)
    a = handle.solve_batch(packed, w.pair_a, w.pair_b, w.costs, w.K)
    b = handle.upload(packed, w.pair_a, w.pair_b)
    b.run(w.costs, w.K)
    r1 = b.download()
    b.run(w.costs, w.K)  # re-run on the resident batch
    r2 = b.download()
    b.free()
    for x, y in ((a, r1), (a, r2)):
        assert np.array_equal(x[0], y[0]) and np.array_equal(x[1], y[1]) and np.array_equal(x[3], y[3])


def test_pipelined_solve_batch(fg, handle):
    """solve_batch splits >= 4096 pairs into pipelined chunks of doubling size (512, 1024, 2048, 1416
    here): same results as one resident batch,
    and a bad pair in the second chunk is reported with its global index."""
    w = synth.config_workload(2, npairs=5000)
    packed = fg.PackedGraphs(w.graphs)
    a = handle.solve_batch(packed, w.pair_a, w.pair_b, w.costs, w.K)
    st = handle.stats()
    assert st["children_evaluated"] == int(np.sum(a[3])) and st["kernel_launches"] >= 2
    b = handle.upload(packed, w.pair_a, w.pair_b)
    b.run(w.costs, w.K)
    r = b.download()
    b.free()
    assert np.array_equal(a[0], r[0]) and np.array_equal(a[1], r[1]) and np.array_equal(a[2], r[2])
    assert np.array_equal(a[3], r[3])
    g = synth.path_graph(4)
    pairs = [(g, g)] * 4999 + [(g, Graph(2, [0, 0], [[1, 1]]))]
    with pytest.raises(fg.FastGedError) as e:
        gpu_batch(fg, handle, pairs, COSTS["unit"], 4)
    assert "pair 4999" in str(e.value)


def test_determinism_repeat(fg, handle):
    w = synth.config_workload(3, npairs=50, variant="unlabeled")
    packed = fg.PackedGraphs(w.graphs)
    r = [handle.solve_batch(packed, w.pair_a, w.pair_b, w.costs, 300) for _ in range(3)]
    for x in r[1:]:
        assert np.array_equal(x[0], r[0][0]) and np.array_equal(x[1], r[0][1])


# ------------------------------------------------------------------ sharded single pair (§8 a6)
@pytest.mark.parametrize("G", [1, 2, 3, 4, 8])
def test_sharded_virtual_matches_oracle(fg, oracle, G):
    """The frontier split over G virtual ranks (CTA groups of one grid, the in-kernel exchange) gives the oracle's
    cost, mapping, children count and per-level records for every G (bit-identical)."""
    flags = fg.FLAG_VIRTUAL_SHARDS
    hs = fg.Handle(0, world_size=G, flags=flags)
    hw = fg.Handle(0, world_size=G, flags=flags | fg.FLAG_DEBUG_WINDOW)
    rng = synth.rng_for(53, G)
    for k in range(6):
        n1, n2 = int(rng.integers(3, 45)), int(rng.integers(3, 45))
        g1 = synth.er_graph(rng, n1, 0.3, 3, 1 + k % 2)
        g2 = synth.er_graph(rng, n2, 0.3, 3, 1 + k % 2)
        K = int(rng.integers(1, 600))
        o = oracle.kbest(g1, g2, COSTS["setting1"], K, levels=True)
        for h in (hs, hw):
            r = h.solve_pair(g1, g2, COSTS["setting1"], K, levels=True)
            assert r["cost"] == o["cost"] and np.array_equal(r["mapping"], o["mapping"]), (G, k)
            assert r["children"] == o["children"] and r["levels"] == [tuple(x) for x in o["levels"]]
    hs.close()
    hw.close()


def test_sharded_virtual_large_pair(fg, handle):
    """A config-4-style pair (n2 > 254, uint16 lambda): 4 virtual shards == the single-GPU path."""
    g1, g2 = synth.large_pair(300, 0.05, seed=11)
    ref = handle.solve_pair(g1, g2, COSTS["setting1"], 2000, levels=True)
    h = fg.Handle(0, world_size=4, flags=fg.FLAG_VIRTUAL_SHARDS)
    r = h.solve_pair(g1, g2, COSTS["setting1"], 2000, levels=True)
    h.close()
    assert r["cost"] == ref["cost"] and np.array_equal(r["mapping"], ref["mapping"]) and r["levels"] == ref["levels"]


def test_work_routing_single_wide_pair(fg, oracle):
    """A single pair with wide levels runs on the whole-GPU kernel (its phase clocks are set), a narrow one on
    the batched kernel; both give the oracle's result (prefers_whole_gpu)."""
    rng = synth.rng_for(808)
    g1, g2 = synth.er_graph(rng, 20, 0.4, 4), synth.er_graph(rng, 20, 0.4, 4)
    h = fg.Handle(0)
    for K, whole in ((1000, False), (200_000, True)):
        r = h.solve_pair(g1, g2, COSTS["setting1"], K)
        st = h.stats()
        assert (sum(st["phase_ms"]) > 0) == whole, (K, st["phase_ms"])
        o = oracle.kbest(g1, g2, COSTS["setting1"], K)
        assert r["cost"] == o["cost"] and np.array_equal(r["mapping"], o["mapping"]) and r["children"] == o["children"]
    h.close()


def test_whole_gpu_and_sharded_degenerate_pairs(fg, oracle):
    """Empty and one-vertex graphs through the whole-GPU kernel and 3 virtual ranks of the sharded kernel (most
    ranks then own empty slices of the one-node levels): the oracle's cost and mapping (readings C16, C5)."""
    hl = fg.Handle(0, flags=fg.FLAG_FORCE_LARGE)
    hs = fg.Handle(0, world_size=3, flags=fg.FLAG_VIRTUAL_SHARDS)
    rng = synth.rng_for(909)
    for n1, n2 in ((0, 0), (0, 5), (5, 0), (1, 1), (1, 7), (7, 1), (2, 2)):
        g1, g2 = synth.er_graph(rng, n1, 0.5, 2), synth.er_graph(rng, n2, 0.5, 2)
        for K in (1, 3, 100):
            o = oracle.kbest(g1, g2, COSTS["setting1"], K)
            for h in (hl, hs):
                r = h.solve_pair(g1, g2, COSTS["setting1"], K)
                assert r["cost"] == o["cost"] and np.array_equal(r["mapping"], o["mapping"]), (n1, n2, K)
    hl.close()
    hs.close()
