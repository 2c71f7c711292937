"""Per-level records (N_i, c_i, threshold) of one cfg4 corner through the library FASTGED_LIB points at
(debugging aid: compare two builds level by level)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_00830_b200 import binding, synth
w = synth.config_workload(4)
idx = int(sys.argv[1]) if len(sys.argv) > 1 else 0
g1, g2 = w.pair(idx)
h = binding.Handle(0)
r = h.solve_pair(g1, g2, w.costs, w.run_K[idx], levels=True)
json.dump({"cost": int(r["cost"]), "levels": [list(map(int, x)) for x in r["levels"]]}, open(sys.argv[2], "w"))
