"""Device throughput of the batched kernel on configs 1, 2, 3 and a config-5 slice."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_00830_b200 import binding, synth, build
build.build()
h = binding.Handle(0, flags=binding.FLAG_TIMING)
for cfg, kw in ((1, {}), (2, {}), (3, {}), (5, {"npairs": 50_000}), (5, {"npairs": 50_000, "variant": "setting2"})):
    w = synth.config_workload(cfg, **kw)
    packed = binding.PackedGraphs(w.graphs)
    b = h.upload(packed, w.pair_a, w.pair_b)
    for rep in range(2):
        b.run(w.costs, w.K); out = b.download()
    st = h.stats()
    t0 = time.perf_counter(); r = h.solve_batch(packed, w.pair_a, w.pair_b, w.costs, w.K); t1 = time.perf_counter()
    print(f"{w.name} {kw}: pairs={w.npairs} device={st['device_ms']:.2f} ms -> {w.npairs/st['device_ms']*1e3:.0f} pairs/s, "
          f"{st['children_evaluated']/st['device_ms']*1e3:.3e} nodes/s; e2e {w.npairs/(t1-t0):.0f} pairs/s; launches {st['kernel_launches']}", flush=True)
    b.free()
