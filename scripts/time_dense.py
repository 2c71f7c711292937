"""Whole-GPU kernel on dense and sparse large pairs (n = 500 / 950, density 0.05 / 0.4, K = 5000): device time
and the phase split (A+T, B, C1) -- the cB popcount path dominates A on dense g2."""
import sys, os
sys.path.insert(0, os.getcwd())
from paper_2605_00830_b200 import binding, synth, build
build.build()
for n, p, K in ((950, 0.4, 5000), (500, 0.4, 5000), (950, 0.05, 5000)):
    r2 = synth.rng_for(607, n)
    a, b = synth.er_graph(r2, n, p, 4), synth.er_graph(r2, n, p, 4)
    h = binding.Handle(0)
    h.solve_pair(a, b, synth.COSTS["setting1"], K)
    r = h.solve_pair(a, b, synth.COSTS["setting1"], K)
    st = h.stats()
    print(n, p, K, "device", round(st["device_ms"], 1), "phases", [round(x, 1) for x in st["phase_ms"]], "children", r["children"], flush=True)
