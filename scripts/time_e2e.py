"""e2e (fastged_solve_batch with host buffers) of the cfg3 and cfg5-slice batches, best of 5."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_00830_b200 import binding, synth, build
build.build()
h = binding.Handle(0, flags=binding.FLAG_TIMING)
for cfg, kw in ((3, {}), (5, {"npairs": 200_000})):
    w = synth.config_workload(cfg, **kw)
    packed = binding.PackedGraphs(w.graphs)
    h.solve_batch(packed, w.pair_a, w.pair_b, w.costs, w.K)
    best = 1e9
    for _ in range(5):
        t0 = time.perf_counter(); h.solve_batch(packed, w.pair_a, w.pair_b, w.costs, w.K); best = min(best, time.perf_counter() - t0)
    print(os.environ.get("FASTGED_PIPE_DIV", "16"), os.environ.get("FASTGED_PIPE_GROWTH", "2"), f"cfg{cfg}", f"e2e {w.npairs / best:.0f} pairs/s ({1e3 * best:.1f} ms)", flush=True)
