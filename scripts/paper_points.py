#!/usr/bin/env python3
"""The paper's own single-pair timings (context -- other hardware) re-measured on this B200.

* fig:cpu-gpu: search time of one pair of 20-vertex graphs vs K = 1e3 .. 1.2e6 (A100: 0.035 s
  at K = 1e3, 0.473 s at K = 7e5).  Our recipe: ER G(20, 0.4), 4 vertex labels, Setting-1 integer costs (the paper
  states neither density nor labels).
* fig:scal-size: search time vs graph size n = 50 .. 950, random graphs of density 0.4, K = 5000
  (A100: 0.428 s at n = 500, 1.0 s at n = 950).
Each point: fastged_solve_pair through the default size routing and through the whole-GPU kernel
(FASTGED_FLAG_FORCE_LARGE); device time (CUDA events) and wall time of the call; the two costs must agree.

    python scripts/paper_points.py [out.json]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_00830_b200 import binding, build, synth  # noqa: E402

PAPER_K = {1000: 0.035, 100_000: 0.12, 200_000: 0.175, 500_000: 0.355, 700_000: 0.473, 1_000_000: 0.65, 1_200_000: 0.78}
PAPER_N = {300: 0.256, 500: 0.428, 700: 0.672, 950: 1.0}


def point(g1, g2, K, costs):
    row = {}
    for name, flags in (("default", 0), ("whole_gpu", binding.FLAG_FORCE_LARGE)):
        h = binding.Handle(0, flags=flags)
        h.solve_pair(g1, g2, costs, K)  # warm (allocations)
        t0 = time.perf_counter()
        r = h.solve_pair(g1, g2, costs, K)
        wall = time.perf_counter() - t0
        row[name] = {"cost": int(r["cost"]), "device_ms": round(h.stats()["device_ms"], 3), "wall_ms": round(1e3 * wall, 3),
                     "children": int(r["children"])}
        h.close()
    assert row["default"]["cost"] == row["whole_gpu"]["cost"]
    return row


def main(out):
    build.build()
    costs = synth.COSTS["setting1"]
    res = {"source": __doc__.strip().split("\n\n")[0], "fig_cpu_gpu": [], "fig_scal_size": []}
    rng = synth.rng_for(606)
    g1, g2 = synth.er_graph(rng, 20, 0.4, 4), synth.er_graph(rng, 20, 0.4, 4)
    for K, a100 in PAPER_K.items():
        row = {"n": 20, "K": K, "paper_a100_s": a100, **point(g1, g2, K, costs)}
        print(row, flush=True)
        res["fig_cpu_gpu"].append(row)
    for n in (50, 100, 300, 500, 700, 950):
        r2 = synth.rng_for(607, n)
        a, b = synth.er_graph(r2, n, 0.4, 4), synth.er_graph(r2, n, 0.4, 4)
        row = {"n": n, "K": 5000, "paper_a100_s": PAPER_N.get(n), **point(a, b, 5000, costs)}
        print(row, flush=True)
        res["fig_scal_size"].append(row)
    json.dump(res, open(out, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "paper_points.json"))
