"""Sharded single-pair mode (virtual shards on one GPU) vs the whole-GPU kernel on cfg4 corners."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_00830_b200 import binding, synth, build
build.build()
w = synth.config_workload(4)
for idx in (0, 4, 5):
    g1, g2 = w.pair(idx)
    K = w.run_K[idx]
    h = binding.Handle(0)
    r = h.solve_pair(g1, g2, w.costs, K)
    t_large = h.stats()["device_ms"]
    h.close()
    for G in (1, 2, 4):
        hs = binding.Handle(0, world_size=G, flags=binding.FLAG_VIRTUAL_SHARDS)
        t0 = time.perf_counter()
        rs = hs.solve_pair(g1, g2, w.costs, K)
        wall = time.perf_counter() - t0
        print(w.run_np[idx], f"G={G}", "cost", rs["cost"], "same" if rs["cost"] == r["cost"] and (rs["mapping"] == r["mapping"]).all() else "DIFF",
              f"sharded device {hs.stats()['device_ms']:.1f} ms wall {1e3 * wall:.1f} ms vs whole-GPU kernel {t_large:.1f} ms", flush=True)
        hs.close()
