"""Small mixed workload (labelled/unlabelled, narrow/wide frontiers, window 2 and normal) for sanitizer runs."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2605_00830_b200 import binding, synth
from oracle import oracle
for flags in (0, binding.FLAG_DEBUG_WINDOW):
    h = binding.Handle(0, flags=flags)
    for cfg, kw in ((3, dict(npairs=6, K=300)), (2, dict(npairs=30)), (5, dict(npairs=4, K=300))):
        w = synth.config_workload(cfg, **kw)
        packed = binding.PackedGraphs(w.graphs)
        gc, gm, offs, _ = h.solve_batch(packed, w.pair_a, w.pair_b, w.costs, w.K)
        oc, om, _ = oracle.kbest_batch([w.pair(k) for k in range(w.npairs)], w.costs, w.K)
        ok = all(gc[k] == oc[k] and np.array_equal(gm[offs[k]:offs[k+1]], om[k]) for k in range(w.npairs))
        print(w.name, flags, "parity", ok, flush=True)
    g1, g2 = synth.large_pair(150, 0.1, seed=2)  # whole-GPU cooperative path
    r = h.solve_pair(g1, g2, synth.COSTS["setting1"], 500)
    o = oracle.kbest(g1, g2, synth.COSTS["setting1"], 500)
    print("large n=150", flags, "parity", r["cost"] == o["cost"] and np.array_equal(r["mapping"], o["mapping"]), flush=True)
    h.close()
