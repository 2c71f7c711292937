"""KNN_GED host logic: split, nearest-neighbour vote and the
synthetic two-class corpus.  The GED matrix itself comes from the GPU path (tests/test_gpu_parity.py)."""
import numpy as np

from paper_2605_00830_b200 import knn, synth


def test_split_70_30():
    tr, te = knn.split_70_30(2000, seed=0)
    assert tr.shape[0] == 1400 and te.shape[0] == 600
    assert np.array_equal(np.sort(np.concatenate([tr, te])), np.arange(2000))
    tr2, te2 = knn.split_70_30(2000, seed=0)
    assert np.array_equal(tr, tr2) and np.array_equal(te, te2)


def test_knn_vote_and_ties():
    y = np.array([0, 1, 1, 0])
    D = np.array([[3, 1, 2, 9],    # nearest = col 1 -> class 1
                  [0, 5, 5, 0],    # tie at 0 between cols 0 and 3 -> smaller index (col 0) -> 0
                  [4, 2, 2, 1]])   # nearest = col 3 -> 0
    assert knn.knn_predict(D, y, 1).tolist() == [1, 0, 0]
    # k = 3: row 0 -> {1, 2, 0}: classes 1, 1, 0 -> 1; row 2 -> {3, 1, 2} -> 0, 1, 1 -> 1
    assert knn.knn_predict(D, y, 3).tolist()[0] == 1 and knn.knn_predict(D, y, 3).tolist()[2] == 1
    # k = 2 class tie: row 0 -> {1 (cls 1), 2 (cls 1)} = 1; row 2 -> {3 (cls 0), 1 (cls 1)}: tie -> nearest (0)
    assert knn.knn_predict(D, y, 2).tolist()[2] == 0


def test_two_class_corpus():
    g, y = synth.two_class_molecules(40, seed=3)
    assert len(g) == 80 and (y == np.arange(80) % 2).all()
    N, O = 3, 2
    def has_nitro(h):
        nb = {v: [] for v in range(h.n)}
        for a, b in h.edges.tolist():
            nb[a].append(b); nb[b].append(a)
        return any(h.vlabels[v] == N and sum(h.vlabels[u] == O for u in nb[v]) >= 2 for v in range(h.n))
    assert all(has_nitro(h) for h, c in zip(g, y) if c == 1)
    g2, y2 = synth.two_class_molecules(40, seed=3)
    assert all(np.array_equal(a.edges, b.edges) and np.array_equal(a.vlabels, b.vlabels) for a, b in zip(g, g2))
    for h in g:  # simple graphs, edges sorted u < v
        e = h.edges
        assert (e[:, 0] < e[:, 1]).all() and len({tuple(x) for x in e.tolist()}) == h.m
