import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_00830_b200 import binding, synth, build
build.build()
w = synth.config_workload(4)
idx = int(sys.argv[1]) if len(sys.argv) > 1 else 0
g1, g2 = w.pair(idx)
h = binding.Handle(0)
r = h.solve_pair(g1, g2, w.costs, w.run_K[idx])
print(w.run_np[idx], r["cost"], h.stats()["device_ms"])
