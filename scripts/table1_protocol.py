#!/usr/bin/env python3
"""Synthetic Table-1 protocol and K-sweep (fig:increas-k,
PAPER.md:576-584; NEXT-4).

Per density d in {0.1, 0.3, 0.5, 0.7, 0.9}: 100 pairs of 10-vertex Erdos-Renyi graphs with 4 vertex labels
(the paper does not state its labels; this is our recipe), Setting-1 costs.  The K-Best search runs on
the GPU through fastged_solve_batch at K = 700,000 (P:298's default); the optimum comes from the exact
branch-and-bound oracle (oracle/og_exact, CPU, every host core).  Reported per density: mean GED_K, mean
exact GED, deviation % (mean over pairs of (GED_K - GED) / GED), optimal count -- Table 1's rows.  The
K-sweep repeats the GPU search at K in {1, 10, 100, 1e3, 1e4, 1e5, 7e5} and reports mean GED_K / GED.

    python scripts/table1_protocol.py [out.json]
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle  # noqa: E402  (the optimum only: the exact oracle)
from paper_2605_00830_b200 import binding, build, synth  # noqa: E402


def main(out):
    build.build()
    oracle.build()
    costs = synth.COSTS["setting1"]
    h = binding.Handle(0, flags=binding.FLAG_TIMING)
    res = {"protocol": "Table 1 (PAPER.md:301-328) on synthetic 10-vertex ER pairs, 4 vertex labels, Setting 1; "
                       "GED_K from the GPU path, optimum from the exact B&B oracle", "densities": {}, "k_sweep": {}}
    Ks = [1, 10, 100, 1000, 10_000, 100_000, 700_000]
    allpairs, allexact = [], []
    for d in (0.1, 0.3, 0.5, 0.7, 0.9):
        rng = synth.rng_for(11, int(d * 10))
        pairs = [(synth.er_graph(rng, 10, d, 4), synth.er_graph(rng, 10, d, 4)) for _ in range(100)]
        t0 = time.time()
        ex, _, nodes, opt = oracle.exact_batch(pairs, costs)
        t_exact = time.time() - t0
        graphs = [g for ab in pairs for g in ab]
        packed = binding.PackedGraphs(graphs)
        a = np.arange(0, 200, 2)
        t0 = time.time()
        gc, gm, offs, gch = h.solve_batch(packed, a, a + 1, costs, 700_000)
        t_gpu = time.time() - t0
        assert (gc >= ex).all(), "a K-Best cost below the exact optimum"
        for k, (g1, g2) in enumerate(pairs):  # the witness re-verifies
            assert oracle.mapping_cost(g1, g2, costs, gm[offs[k]:offs[k + 1]]) == gc[k]
        dev = np.where(ex > 0, (gc - ex) / np.maximum(ex, 1), 0.0)
        res["densities"][str(d)] = {
            "pairs": 100, "mean_ged_K700k": float(gc.mean()), "mean_exact": float(ex.mean()),
            "deviation_pct": float(100 * dev.mean()), "optimal": int((gc == ex).sum()),
            "exact_all_proven": bool(opt.all()), "exact_nodes_mean": float(nodes.mean()),
            "gpu_solve_batch_s": round(t_gpu, 3), "gpu_device_ms": h.stats()["device_ms"],
            "oracle_exact_s": round(t_exact, 2), "children_per_pair_mean": float(gch.mean())}
        print(d, res["densities"][str(d)], flush=True)
        allpairs += pairs
        allexact.append(ex)
    ex = np.concatenate(allexact)
    graphs = [g for ab in allpairs for g in ab]
    packed = binding.PackedGraphs(graphs)
    a = np.arange(0, 2 * len(allpairs), 2)
    for K in Ks:
        gc, _, _, _ = h.solve_batch(packed, a, a + 1, costs, K)
        res["k_sweep"][str(K)] = {"mean_ged_over_exact": float((gc / np.maximum(ex, 1)).mean()),
                                  "optimal_pct": float(100 * (gc == ex).mean()), "mean_ged": float(gc.mean()),
                                  "device_ms": h.stats()["device_ms"]}
        print("K", K, res["k_sweep"][str(K)], flush=True)
    h.close()
    json.dump(res, open(out, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/table1_protocol.json")
