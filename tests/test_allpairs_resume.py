"""Checkpoint / resume of the all-pairs driver (paper_2605_00830_b200/allpairs.py).  The per-chunk solver
here is the CPU oracle standing in for binding.Handle (the GPU parity tests check the real path)."""
import numpy as np
import pytest

from paper_2605_00830_b200 import allpairs, synth


class OracleSolver:
    def __init__(self, graphs):
        self.graphs = graphs
        self.calls = 0

    def solve_batch(self, packed, a, b, costs, K):
        from oracle import oracle
        self.calls += 1
        pairs = [(self.graphs[int(x)], self.graphs[int(y)]) for x, y in zip(a, b)]
        c, maps, ch = oracle.kbest_batch(pairs, costs, K, nthreads=2)
        offs = np.concatenate([[0], np.cumsum([m.shape[0] for m in maps])]).astype(np.int64)
        return c, np.concatenate(maps + [np.zeros(0, np.int32)]), offs, ch


def test_resume_after_interruption(tmp_path, oracle_lib):
    graphs = [synth.molecule_graph(synth.rng_for(8, k), "aids") for k in range(12)]  # 66 pairs
    costs = synth.COSTS["setting1"]
    s1 = OracleSolver(graphs)
    assert allpairs.all_pairs(s1, graphs, costs, 20, str(tmp_path), chunk=10, keep_mappings=True, max_chunks=3) is None
    assert s1.calls == 3 and len(list(tmp_path.glob("chunk_*.npz"))) == 3
    s2 = OracleSolver(graphs)
    ia, ib, cost, ch, maps, offs = allpairs.all_pairs(s2, graphs, costs, 20, str(tmp_path), chunk=10, keep_mappings=True)
    assert s2.calls == 4  # only the 4 missing chunks of 7
    ref_c, ref_m, ref_ch = oracle_lib.kbest_batch([(graphs[a], graphs[b]) for a, b in zip(ia, ib)], costs, 20)
    assert np.array_equal(cost, ref_c) and np.array_equal(ch, ref_ch)
    assert all(np.array_equal(maps[offs[k]:offs[k + 1]], ref_m[k]) for k in range(len(ia)))
    s3 = OracleSolver(graphs)  # everything on disk: nothing recomputed
    allpairs.all_pairs(s3, graphs, costs, 20, str(tmp_path), chunk=10, keep_mappings=True)
    assert s3.calls == 0


def test_refuses_a_different_run(tmp_path):
    graphs = [synth.molecule_graph(synth.rng_for(8, k), "aids") for k in range(5)]
    allpairs.all_pairs(OracleSolver(graphs), graphs, synth.COSTS["setting1"], 20, str(tmp_path), chunk=4)
    with pytest.raises(ValueError):
        allpairs.all_pairs(OracleSolver(graphs), graphs, synth.COSTS["setting1"], 21, str(tmp_path), chunk=4)
