#!/usr/bin/env python3
"""KNN_GED protocol on the synthetic two-class corpus.

2 x 1000 Mutagenicity-like graphs (class 1 carries nitro groups; synth.two_class_molecules), 70/30 split,
uniform costs (c_ins = c_del = 2, c_sub = 1; C24), K = 1000: every test -> train GED on the GPU in one
batched call (600 x 1400 = 840,000 pairs), then k-NN for k = 1, 3, 5.  Baseline for context: the same vote
over the |n1 - n2| + |m1 - m2| size distance (no GED).  The paper reports 75 % at k = 1 on the real dataset.

    python scripts/knn_protocol.py [out.json]
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_00830_b200 import binding, build, knn, synth  # noqa: E402


def main(out):
    build.build()
    graphs, y = synth.two_class_molecules(1000, seed=13)
    tr, te = knn.split_70_30(len(graphs), seed=0)
    h = binding.Handle(0, flags=binding.FLAG_TIMING)
    t0 = time.time()
    D = knn.ged_matrix(h, binding.PackedGraphs(graphs), te, tr, synth.COSTS["uniform"], 1000)
    dt = time.time() - t0
    st = h.stats()
    res = {"protocol": "KNN_GED (PAPER.md:701-707) on synth.two_class_molecules(1000, seed=13): 70/30 split, "
                       "uniform costs 1,2,2,1,2,2, K=1000, test graph = source g1",
           "pairs": int(D.size), "solve_batch_s": round(dt, 3), "device_ms": st["device_ms"],
           "pairs_per_s_e2e": D.size / dt, "accuracy": {}, "size_baseline_accuracy": {}}
    sz = np.array([[abs(graphs[a].n - graphs[b].n) + abs(graphs[a].m - graphs[b].m) for b in tr] for a in te])
    for k in (1, 3, 5):
        res["accuracy"][str(k)] = float((knn.knn_predict(D, y[tr], k) == y[te]).mean())
        res["size_baseline_accuracy"][str(k)] = float((knn.knn_predict(sz, y[tr], k) == y[te]).mean())
    print(json.dumps(res))
    json.dump(res, open(out, "w"), indent=1)
    h.close()


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/knn_protocol.json")
