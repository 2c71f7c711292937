#!/usr/bin/env python3
"""Approximate top-K versus the exact selection, on the GPU path.

PAPER.md:288 suggests approximate top-k selection when the top-K step becomes the bottleneck at extreme K.
FASTGED_FLAG_APPROX(s) ranks children by PED bins of 2^s (position order inside a bin).  Measured here:
  * the whole-GPU kernel on the eight config-4 corners (K = 1e4 / 1e5): device time and the time of the
    selection phases (T + B + C1) for s = 0 (exact) .. 4, and the resulting GED upper bound;
  * quality on 200 synthetic Table-1 pairs (10-vertex ER, 4 labels, Setting 1, densities 0.3 / 0.7) at
    K = 1000: mean GED_K / exact GED (exact from the B&B oracle) and optimal count, per s.

    python scripts/approx_protocol.py [out.json]
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle  # noqa: E402  (the optimum only: the exact oracle)
from paper_2605_00830_b200 import binding, build, synth  # noqa: E402

SHIFTS = (0, 1, 2, 3, 4)


def main(out):
    build.build()
    oracle.build()
    res = {"protocol": "approximate top-K (PED bins of 2^s) vs exact (s = 0) on the GPU path", "config4": [], "table1_k1000": {}}
    w = synth.config_workload(4)
    for idx in range(w.npairs):
        g1, g2 = w.pair(idx)
        row = {"pair": list(w.run_np[idx]), "K": int(w.run_K[idx])}
        for s in SHIFTS:
            h = binding.Handle(0, flags=binding.FLAG_APPROX(s))
            h.solve_pair(g1, g2, w.costs, w.run_K[idx])  # warm
            r = h.solve_pair(g1, g2, w.costs, w.run_K[idx])
            st = h.stats()
            row[f"s{s}"] = {"cost": int(r["cost"]), "device_ms": round(st["device_ms"], 2),
                            "select_ms": round(sum(st["phase_ms"][1:3]), 2), "phase_ms": [round(x, 2) for x in st["phase_ms"]]}
            h.close()
        print(row, flush=True)
        res["config4"].append(row)
    costs = synth.COSTS["setting1"]
    pairs = []
    for d in (0.3, 0.7):
        rng = synth.rng_for(11, int(d * 10))
        pairs += [(synth.er_graph(rng, 10, d, 4), synth.er_graph(rng, 10, d, 4)) for _ in range(100)]
    ex, _, _, opt = oracle.exact_batch(pairs, costs)
    graphs = [g for ab in pairs for g in ab]
    packed = binding.PackedGraphs(graphs)
    a = np.arange(0, 2 * len(pairs), 2)
    for s in SHIFTS:
        h = binding.Handle(0, flags=binding.FLAG_APPROX(s))
        gc, _, _, _ = h.solve_batch(packed, a, a + 1, costs, 1000)
        h.close()
        assert (gc >= ex).all()
        res["table1_k1000"][f"s{s}"] = {"pairs": len(pairs), "mean_ratio": float((gc / np.maximum(ex, 1)).mean()),
                                        "optimal": int((gc == ex).sum()), "exact_proven": bool(opt.all())}
        print(s, res["table1_k1000"][f"s{s}"], flush=True)
    json.dump(res, open(out, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "approx_protocol.json"))
