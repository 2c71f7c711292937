"""Run one batched K-Best launch set on a config-3 subset (for ncu captures and host timing)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2605_00830_b200 import binding, synth, build

npairs = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
K = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
build.build()
w = synth.config_workload(3, npairs=npairs, K=K)
packed = binding.PackedGraphs(w.graphs)
h = binding.Handle(0, flags=binding.FLAG_TIMING)
for r in range(reps):
    t0 = time.perf_counter()
    b = h.upload(packed, w.pair_a, w.pair_b)
    t1 = time.perf_counter()
    b.run(w.costs, w.K)
    t2 = time.perf_counter()
    out = b.download()
    t3 = time.perf_counter()
    st = h.stats()
    t4 = time.perf_counter()
    r2 = h.solve_batch(packed, w.pair_a, w.pair_b, w.costs, w.K)
    t5 = time.perf_counter()
    print(f"upload {1e3*(t1-t0):.1f} ms  run(enqueue) {1e3*(t2-t1):.1f} ms  download(sync) {1e3*(t3-t2):.1f} ms  "
          f"solve_batch {1e3*(t5-t4):.1f} ms  device {st['device_ms']:.2f} ms  kernels {st['branch_ms']:.2f} ms "
          f"launches {st['kernel_launches']} children {st['children_evaluated']:.3e} alg_bytes {st['alg_bytes']:.3e}")
    b.free()
