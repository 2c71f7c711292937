#!/usr/bin/env python3
"""Randomised parity stress of every search path against the oracle (bit-exact cost, mapping, children):
random ER / labelled pairs (n1, n2 in 1..48, densities 0.05..0.6, 1..4 vertex labels, 1..3 edge labels),
random integer costs (0..9 each), random K (1..3000), through the batched kernel (one batch), the whole-GPU
kernel (FASTGED_FLAG_FORCE_LARGE, with and without the 2-wide debug window), 3 virtual ranks of the sharded
kernel, the approximate top-K variant (s = 2) and the last-level-by-total variant on the whole-GPU kernel (each
against the oracle's variant).

    python scripts/stress_parity.py [npairs] [out.json]
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle  # noqa: E402
from paper_2605_00830_b200 import binding, build, synth  # noqa: E402


def main(npairs, out):
    build.build()
    oracle.build()
    rng = np.random.default_rng(20261018)
    pairs, Ks, costs = [], [], []
    for _ in range(npairs):
        n1, n2 = int(rng.integers(1, 49)), int(rng.integers(1, 49))
        p = float(rng.choice([0.05, 0.15, 0.3, 0.6]))
        nvl, nel = int(rng.integers(1, 5)), int(rng.integers(1, 4))
        pairs.append((synth.er_graph(rng, n1, p, nvl, nel), synth.er_graph(rng, n2, p, nvl, nel)))
        Ks.append(int(rng.integers(1, 3001)))
        costs.append(tuple(int(x) for x in rng.integers(0, 10, size=6)))
    res = {"pairs": npairs, "paths": {}}
    handles = {"whole_gpu": binding.Handle(0, flags=binding.FLAG_FORCE_LARGE),
               "whole_gpu_window2": binding.Handle(0, flags=binding.FLAG_FORCE_LARGE | binding.FLAG_DEBUG_WINDOW),
               "sharded_3_virtual": binding.Handle(0, world_size=3, flags=binding.FLAG_VIRTUAL_SHARDS),
               "approx_s2": binding.Handle(0, flags=binding.FLAG_APPROX(2)),
               "last_by_total_whole_gpu": binding.Handle(0, flags=binding.FLAG_FORCE_LARGE | binding.FLAG_LAST_BY_TOTAL)}
    bad = {k: [] for k in handles}
    bad["batched"] = []
    for k, ((g1, g2), K, c) in enumerate(zip(pairs, Ks, costs)):
        o = oracle.kbest(g1, g2, c, K)
        for name, h in handles.items():
            if name in ("approx_s2", "last_by_total_whole_gpu"):
                oa = oracle.kbest(g1, g2, c, K, flags=oracle.APPROX(2) if name == "approx_s2" else oracle.LAST_BY_TOTAL)
                r = h.solve_pair(g1, g2, c, K)
                ok = r["cost"] == oa["cost"] and np.array_equal(r["mapping"], oa["mapping"]) and r["children"] == oa["children"]
            else:
                r = h.solve_pair(g1, g2, c, K)
                ok = r["cost"] == o["cost"] and np.array_equal(r["mapping"], o["mapping"]) and r["children"] == o["children"]
            if not ok:
                bad[name].append(k)
    # the batched kernel: the whole set as one batch per cost model and K (the batch API takes one of each)
    hb = binding.Handle(0)
    for K in (50, 700):
        for c in ((1, 1, 1, 1, 1, 1), (2, 4, 4, 1, 2, 2), (3, 1, 7, 2, 5, 0)):
            packed = binding.PackedGraphs([g for ab in pairs for g in ab])
            a = np.arange(0, 2 * npairs, 2)
            gc, gm, offs, gch = hb.solve_batch(packed, a, a + 1, c, K)
            oc, om, och = oracle.kbest_batch(pairs, c, K)
            for k in range(npairs):
                if gc[k] != oc[k] or not np.array_equal(gm[offs[k]:offs[k + 1]], om[k]) or gch[k] != och[k]:
                    bad["batched"].append((K, c, k))
    for name, b in bad.items():
        res["paths"][name] = {"mismatches": len(b), "first": [list(x) if isinstance(x, tuple) else x for x in b[:5]]}
    print(json.dumps(res), flush=True)
    json.dump(res, open(out, "w"), indent=1)
    return 0 if all(len(b) == 0 for b in bad.values()) else 1


if __name__ == "__main__":
    sys.exit(main(int(sys.argv[1]) if len(sys.argv) > 1 else 400,
                  sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "gpurun_out", "stress_parity.json")))
