"""KNN_GED graph classification on top of the batched K-Best path.

PAPER.md:701-707: the graphs are split 70 % / 30 % into training and test sets and each test graph takes
the class of its nearest training graph in GED (k = 1), with uniform costs (c_ins = c_del = 2, c_sub = 1;
reading C24).  Reading of this repo: the test graph is the source g1 and the training graph the target g2
(GED_K is direction-dependent, C18).  Every GED of the test x train matrix is one pair of a single
``fastged_solve_batch`` call on the GPU; only the nearest-neighbour vote runs on the host.
"""
from __future__ import annotations

from typing import Sequence, Tuple

import numpy as np


def split_70_30(n: int, seed: int = 0) -> Tuple[np.ndarray, np.ndarray]:
    """Deterministic 70 / 30 split of n graphs."""
    perm = np.random.Generator(np.random.PCG64(seed)).permutation(n)
    ntr = int(round(0.7 * n))
    return np.sort(perm[:ntr]), np.sort(perm[ntr:])


def ged_matrix(solver, packed, src_idx: Sequence[int], dst_idx: Sequence[int], costs, K: int) -> np.ndarray:
    """D[a, b] = GED_K(graph src_idx[a] -> graph dst_idx[b]) from one batched GPU call."""
    src = np.asarray(src_idx, np.int64)
    dst = np.asarray(dst_idx, np.int64)
    pa = np.repeat(src, dst.shape[0])
    pb = np.tile(dst, src.shape[0])
    c, _, _, _ = solver.solve_batch(packed, pa, pb, costs, K)
    return c.reshape(src.shape[0], dst.shape[0])


def knn_predict(D: np.ndarray, train_labels: np.ndarray, k: int = 1) -> np.ndarray:
    """Class of each row's k nearest columns by majority vote; ties between distances are broken by the
    smaller training index, ties between classes by the class of the nearest of the tied classes."""
    order = np.lexsort((np.broadcast_to(np.arange(D.shape[1]), D.shape), D), axis=1)[:, :k]
    out = np.empty(D.shape[0], np.int32)
    for r in range(D.shape[0]):
        nb = train_labels[order[r]]
        counts = np.bincount(nb)
        best = np.flatnonzero(counts == counts.max())
        out[r] = next(int(x) for x in nb if x in best)  # nearest among the tied classes
    return out


def knn_ged(solver, graphs, labels, costs, K: int = 1000, k: int = 1, seed: int = 0):
    """The paper's protocol end to end: split, GPU GED matrix (test -> train), k-NN vote.  Returns
    (accuracy, predictions, test indices, distance matrix)."""
    from .binding import PackedGraphs
    labels = np.asarray(labels)
    tr, te = split_70_30(len(graphs), seed)
    D = ged_matrix(solver, PackedGraphs(graphs), te, tr, costs, K)
    pred = knn_predict(D, labels[tr], k)
    return float((pred == labels[te]).mean()), pred, te, D
