import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_00830_b200 import binding, synth
from oracle import oracle
h = binding.Handle(0, flags=binding.FLAG_DEBUG_WINDOW)
rng = synth.rng_for(77)
for k in range(12):
    n1, n2 = int(rng.integers(5, 40)), int(rng.integers(5, 40))
    g1 = synth.er_graph(rng, n1, 0.3, 3); g2 = synth.er_graph(rng, n2, 0.3, 3)
    K = int(rng.integers(1, 300))
    print(k, n1, n2, K, flush=True)
    r = h.solve_pair(g1, g2, synth.COSTS["setting1"], K, levels=True)
    o = oracle.kbest(g1, g2, synth.COSTS["setting1"], K, levels=True)
    print(r["cost"], o["cost"], r["levels"] == [tuple(x) for x in o["levels"]], flush=True)
