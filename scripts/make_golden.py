#!/usr/bin/env python3
"""Write the oracle's results for the BASELINE configs into tests/golden/ (test fixtures).

Calls ONLY oracle/ (the CPU oracle, OpenMP over pairs or over parents) on the seeded inputs of
paper_2605_00830_b200/synth.py, so every stored value comes from the oracle and none from the CUDA
path.  The GPU parity tests (tests/test_gpu_parity.py) compare the CUDA path element by element
with these files at the full sizes the bench runs, which the oracle cannot redo inside a test.

    python scripts/make_golden.py cfg3 cfg5 cfg4     # (cfg4: the eight single-pair corners)

Files (costs int64, children int64, mappings int16 concatenated in pair order, -1 = deleted):
  tests/golden/oracle_cfg3.npz        all 10,000 pairs of configs[2] (K=1000, Setting 1)
  tests/golden/oracle_cfg5_s1.npz     every 100th pair of the 1,999,000 of configs[4], Setting 1
  tests/golden/oracle_cfg5_s2.npz     the same pairs, Setting 2 (C23)
  tests/golden/oracle_cfg4.json       the eight configs[3] corners (cost, children, mapping, levels)
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle  # noqa: E402
from paper_2605_00830_b200 import synth  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")


def oracle_sha() -> str:
    with open(oracle.SRC_PATH, "rb") as f:
        return hashlib.sha256(f.read()).hexdigest()[:16]


def batch_golden(w, idx, path, note):
    pairs = [w.pair(int(k)) for k in idx]
    t0 = time.time()
    costs, maps, children = oracle.kbest_batch(pairs, w.costs, w.K)
    dt = time.time() - t0
    offs = np.zeros(len(pairs) + 1, np.int64)
    offs[1:] = np.cumsum([m.shape[0] for m in maps])
    flat = np.concatenate(maps).astype(np.int16) if maps else np.zeros(0, np.int16)
    meta = {"note": note, "K": int(w.K), "costs": list(w.costs), "oracle_sha256_16": oracle_sha(),
            "seconds": round(dt, 1), "threads": oracle.max_threads(), "npairs": len(pairs)}
    np.savez_compressed(path, idx=np.asarray(idx, np.int64), cost=costs, children=children, map=flat, offs=offs,
                        meta=json.dumps(meta))
    print(f"{path}: {len(pairs)} pairs in {dt:.0f} s", flush=True)


def main(what):
    oracle.build()
    if "cfg3" in what:
        w = synth.config_workload(3)
        batch_golden(w, np.arange(w.npairs), os.path.join(GOLD, "oracle_cfg3.npz"),
                     "configs[2]: all 10,000 ER pairs (synth.config_workload(3)), K=1000, Setting 1")
    if "cfg5" in what:
        for variant, name in ((None, "s1"), ("setting2", "s2")):
            w = synth.config_workload(5, variant=variant)
            idx = np.arange(0, w.npairs, 100)
            batch_golden(w, idx, os.path.join(GOLD, f"oracle_cfg5_{name}.npz"),
                         f"configs[4]: every 100th of the 1,999,000 all-pairs (synth.config_workload(5, variant={variant!r})), K=1000")
    if "cfg4" in what:
        w = synth.config_workload(4)
        path = os.path.join(GOLD, "oracle_cfg4.json")
        out = json.load(open(path)) if os.path.exists(path) else {"runs": {}}
        out["note"] = ("configs[3]: the eight single-pair corners of synth.config_workload(4) "
                       "(n, p, K), Setting 1; levels = (N_i, c_i, threshold PED or -1)")
        # cheapest first, so partial files are useful
        order = sorted(range(len(w.run_np)), key=lambda k: w.run_np[k][0] ** 3 * w.run_np[k][2])
        for idx in order:
            key = str(idx)
            if key in out["runs"] and out["runs"][key].get("oracle_sha256_16") == oracle_sha():
                continue
            g1, g2 = w.pair(idx)
            n, p, K = w.run_np[idx]
            t0 = time.time()
            r = oracle.kbest(g1, g2, w.costs, K, levels=True)
            out["runs"][key] = {"n": n, "p": p, "K": K, "cost": r["cost"], "children": r["children"],
                                "parents": r["parents"], "mapping": r["mapping"].tolist(),
                                "levels": [list(map(int, x)) for x in r["levels"]],
                                "seconds": round(time.time() - t0, 1), "threads": oracle.max_threads(),
                                "oracle_sha256_16": oracle_sha()}
            with open(path, "w") as f:
                json.dump(out, f)
            print(f"cfg4 run {idx} {w.run_np[idx]}: cost {r['cost']} in {time.time() - t0:.0f} s", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["cfg3", "cfg5", "cfg4"])
