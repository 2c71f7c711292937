"""Time the whole-GPU (cooperative) path on the config-4 corners."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_00830_b200 import binding, synth, build
build.build()
w = synth.config_workload(4)
h = binding.Handle(0, flags=binding.FLAG_TIMING)
sel = [int(x) for x in sys.argv[1:]] or range(8)
for idx in sel:
    g1, g2 = w.pair(idx)
    n, p, K = w.run_np[idx]
    for rep in range(2):
        t0 = time.perf_counter()
        r = h.solve_pair(g1, g2, w.costs, K)
        t1 = time.perf_counter()
    st = h.stats()
    print(f"n={n} p={p} K={K}: cost={r['cost']} wall={1e3*(t1-t0):.1f} ms device={st['device_ms']:.1f} ms "
          f"children={r['children']:.3e} nodes/s={r['children']/(st['device_ms']/1e3):.3e} alg_bytes={st['alg_bytes']:.3e} "
          f"GB/s={st['alg_bytes']/(st['device_ms']/1e3)/1e9:.1f} phases(A,B,C1,C2,fin)ms={[round(x, 1) for x in st['phase_ms']]} hist_frac={st['hist_children']/max(1,r['children']):.3f}", flush=True)
