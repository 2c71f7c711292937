"""One batched launch set on a config-5 slice (Mutagenicity-like all-pairs, K=1000) for ncu captures."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_00830_b200 import binding, synth, build
npairs = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
build.build()
w = synth.config_workload(5, npairs=npairs)
packed = binding.PackedGraphs(w.graphs)
h = binding.Handle(0, flags=binding.FLAG_TIMING)
b = h.upload(packed, w.pair_a, w.pair_b)
b.run(w.costs, w.K)
b.download()
print("cfg5 slice", npairs, "device ms", h.stats()["device_ms"])
