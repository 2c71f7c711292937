#!/usr/bin/env python3
"""FAST-GED K-Best hot path benchmark (BASELINE.json metric: GED pairs/sec and expanded tree
nodes/sec at K=1000, 1/2/4/8 B200).

Workload: BASELINE configs[2] — 10,000 Erdős–Rényi pairs per GPU, n = 30..70,
p = 0.1..0.5 (400 pairs per (n, p) cell), 4 vertex labels, Setting-1 costs, K = 1000.
One step = one K-Best search of every pair of the batch (all levels: branch, rank, update,
finalize).  Multi-GPU: every rank is given the same canonical batch of
10,000 x N pairs, pair r is solved by rank r mod N (weak scaling, no data-path collective), and the
end-to-end number includes gathering every cost and mapping to rank 0.  --workload cfg5 runs the
1,999,000-pair all-pairs batch (strong scaling), cfg4 one large pair (frontier sharded).

  python bench.py [--steps K] [--warmup W] [--impl ours|reference] [--workload cfg3|cfg2|cfg5|cfg4]
  python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 ... bench.py --gpus N ...
  (--gpus N must equal WORLD_SIZE: a bare `--gpus 8` exits with an error instead of measuring 1 GPU)

Prints one JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "GED pairs/sec and expanded tree nodes/sec at K=1000, 1/2/4/8 B200"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--npairs", type=int, default=None,
                    help="cfg3/cfg2: pairs per GPU (default 10,000); cfg5: first N pairs of the all-pairs batch (default all)")
    ap.add_argument("--variant", choices=["setting2"], default=None, help="cfg5: Setting-2 costs (C23)")
    ap.add_argument("--K", type=int, default=None, help="override K (default: the config's K)")
    ap.add_argument("--workload", choices=["cfg3", "cfg2", "cfg5", "cfg4"], default="cfg3",
                    help="cfg3 (default, the BASELINE metric's K=1000 batch), cfg2/cfg5 batches, "
                         "cfg4 = one large pair (n=500, p=0.05, K=1e5; frontier sharded over the ranks)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="target CPU time of the oracle sample")
    return ap.parse_args()


def dist_env():
    rank, local_rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    # test hook (tests/test_bench_multirank.py): FASTGED_BENCH_SHARE_GPU=1 puts every rank on cuda:0 with the
    # gloo backend, so the N > 1 code path (sharding, gather, max over ranks) runs on a one-GPU box; the
    # numbers of such a run are not a measurement of N GPUs
    if os.environ.get("FASTGED_BENCH_SHARE_GPU") == "1":
        local_rank = 0
    return rank, local_rank, world


WORKLOADS = {
    "cfg3": (3, "cfg3: ER pairs n=30..70 x p=0.1..0.5 (4 vertex labels, unlabelled edges), Setting-1 costs, K=1000"),
    "cfg2": (2, "cfg2: AIDS-like labelled molecule pairs (n=5..10), Setting-1 costs, K=100"),
    "cfg5": (5, "cfg5: all-pairs slice of 2000 Mutagenicity-like labelled graphs (n~30), Setting-1 costs, K=1000"),
}
ARGS = None


def workload_name(w) -> str:
    return WORKLOADS[ARGS.workload][1] if ARGS else WORKLOADS["cfg3"][1]


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        rows = [r for r in self.rows if len(r) >= 9]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[5 + k].lower() == "active"})
        loaded = [s for s in sm if s > 0.5 * (max(sm) if sm else 1)]
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# ------------------------------------------------------------------ oracle (CPU baseline / reference arm)
def oracle_sample(w, seconds: float, gpu=None):
    """Time the oracle, as it stands, on host cores over a bounded sample of the workload:
    whole chunks of consecutive pairs (every (n, p) cell equally) until `seconds` of wall time.
    gpu = (costs, flat mappings, offsets) of the GPU run: the oracle's results for the sampled pairs
    are compared with it element by element (bit-exact cost and mapping)."""
    from oracle import oracle
    oracle.build()
    cores = oracle.max_threads()
    chunk = 25 * max(1, (cores + 24) // 25)
    done, nodes, t0, bad = 0, 0, time.perf_counter(), 0
    while done < w.npairs:
        idx = range(done, min(w.npairs, done + chunk))
        pairs = [w.pair(k) for k in idx]
        oc, om, ch = oracle.kbest_batch(pairs, w.costs, w.K, nthreads=cores)
        if gpu is not None:
            gc, gm, go = gpu
            for x, k in enumerate(idx):
                if gc[k] != oc[x] or not np.array_equal(gm[go[k]:go[k + 1]], om[x]):
                    bad += 1
        done += len(pairs)
        nodes += int(ch.sum())
        if time.perf_counter() - t0 >= seconds:
            break
    dt = time.perf_counter() - t0
    par = {"checked": done, "mismatches": bad, "against": "the oracle run timed here"} if gpu is not None else None
    return {"pairs": done, "seconds": dt, "pairs_per_s": done / dt, "nodes_per_s": nodes / dt, "cores": cores,
            "parity": par}


# ------------------------------------------------------------------ our arm
def canonical_workload(world: int):
    """The one batch every rank is given (§8(e)): pair r is solved by rank r mod world.
    cfg3/cfg2: npairs x world pairs of the config recipe (weak scaling: pairs per GPU fixed; at N=1
    exactly BASELINE configs[1]/[2]).  cfg5: the all-pairs batch (1,999,000 pairs, or the first
    --npairs of them), fixed total (strong scaling)."""
    from paper_2605_00830_b200 import synth
    cfg = WORKLOADS[ARGS.workload][0]
    if cfg == 5:
        w = synth.config_workload(5, K=ARGS.K, variant=ARGS.variant)
        if ARGS.npairs:
            w = w.subset(np.arange(min(ARGS.npairs, w.npairs)))
        return w, "strong"
    per = ARGS.npairs or 10_000
    return synth.config_workload(cfg, npairs=per * world, K=ARGS.K), "weak"


def golden_parity(w, world, res):
    """Compare rank 0's gathered results with the oracle's stored results (tests/golden, written by
    scripts/make_golden.py from oracle/ only) where the canonical batch has them."""
    path = {"cfg3": "oracle_cfg3.npz", "cfg5": "oracle_cfg5_s2.npz" if ARGS.variant == "setting2" else "oracle_cfg5_s1.npz"}.get(ARGS.workload)
    if path is None or res is None or (ARGS.K not in (None, 1000)):
        return None
    f = os.path.join(ROOT, "tests", "golden", path)
    if not os.path.exists(f):
        return None
    z = np.load(f)
    gidx, gc, gm, go = z["idx"], z["cost"], z["map"], z["offs"]
    keep = gidx < w.npairs
    c, m, offs = res
    bad = 0
    for x in np.flatnonzero(keep):
        k = int(gidx[x])
        if c[k] != gc[x] or not np.array_equal(m[offs[k]:offs[k + 1]], gm[go[x]:go[x + 1]]):
            bad += 1
    return {"checked": int(keep.sum()), "mismatches": bad, "against": f"tests/golden/{path} (oracle results, bit-exact cost + mapping)"}


def run_ours(args, rank, local_rank, world):
    import torch
    import torch.distributed as dist

    from paper_2605_00830_b200 import binding, build
    from paper_2605_00830_b200 import dist as fdist

    build.build()
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    # a dedicated (non-default) stream: the library launches on it and the CUDA events time it
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    assert stream.cuda_stream != 0
    w, scaling = canonical_workload(world)
    packed = binding.PackedGraphs(w.graphs)
    idx = fdist.shard_pairs(w.npairs, rank, world)  # pair r -> rank r mod world
    mine_a, mine_b = w.pair_a[idx], w.pair_b[idx]
    h = binding.Handle(local_rank, stream=stream.cuda_stream, flags=binding.FLAG_TIMING)
    batch = h.upload(packed, mine_a, mine_b)  # this rank's pairs resident in HBM before timing
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device=dev)  # > 126 MB L2

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        batch.run(w.costs, w.K)
    torch.cuda.synchronize(dev)
    ref = batch.download()

    # ---- device-resident timed region: K steps, L2 flushed between steps (outside the events)
    clocks = ClockSampler(local_rank)
    clocks.start()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    branch_ms, branch_launches, launches, alg_bytes, children, parents, lib_ms, alg_ops = 0.0, 0, 0, 0, 0, 0, 0.0, 0
    barrier()
    torch.cuda.synchronize(dev)
    wall0 = time.perf_counter()
    for s in range(args.steps):
        flush.fill_(s)
        ev[s][0].record(stream)
        batch.run(w.costs, w.K)
        ev[s][1].record(stream)
        out = batch.download()  # per-step result read (also fills per-launch kernel timings)
        st = h.stats()
        branch_ms += st["branch_ms"]
        lib_ms += st["device_ms"]
        branch_launches += st["branch_launches"]
        launches += st["kernel_launches"]
        alg_bytes += st["alg_bytes"]
        alg_ops += st["alg_ops"]
        children += st["children_evaluated"]
        parents += st["parents_expanded"]
    torch.cuda.synchronize(dev)
    barrier()
    wall = time.perf_counter() - wall0
    clk = clocks.stop()
    dev_ms = sum(a.elapsed_time(b) for a, b in ev)
    # the library's own events (same stream) must agree with ours: guards against timing the wrong stream
    assert abs(dev_ms - lib_ms) <= 0.25 * max(dev_ms, lib_ms) + 0.5, (dev_ms, lib_ms)
    assert np.array_equal(out[0], ref[0]) and np.array_equal(out[1], ref[1]), "results changed between steps"

    # ---- end to end through the public API with host buffers: every rank solves its shard of the
    # canonical batch (H2D, search, D2H inside fastged_solve_batch) and rank 0 gathers every cost
    # and mapping (§8(e): "wall time is the slowest rank's, including the final gather")
    e2e_t = []
    h2d = d2h = 0
    fdist_group = None
    if world > 1:
        res = fdist.solve_batch_sharded(h, packed, w.pair_a, w.pair_b, w.costs, w.K)  # untimed: staging allocs
    else:
        h.solve_batch(packed, mine_a, mine_b, w.costs, w.K)
    for s in range(max(1, args.steps)):
        flush.fill_(s)
        torch.cuda.synchronize(dev)
        barrier()
        t0 = time.perf_counter()
        if world > 1:
            res = fdist.solve_batch_sharded(h, packed, w.pair_a, w.pair_b, w.costs, w.K, group=fdist_group)
        else:
            c_, m_, o_, _ = h.solve_batch(packed, mine_a, mine_b, w.costs, w.K)
            res = (c_, m_, o_)
        e2e_t.append(time.perf_counter() - t0)
        st = h.stats()
        h2d, d2h = st["h2d_bytes"], st["d2h_bytes"]
    if world == 1:
        assert np.array_equal(res[0], ref[0]), "e2e results differ from the device-resident run"
    else:
        mine_ok = res is None or all(res[0][int(k)] == ref[0][x] for x, k in enumerate(idx))
        assert mine_ok, "gathered results differ from the device-resident run"

    # ---- max over ranks
    red = "cpu" if os.environ.get("FASTGED_BENCH_SHARE_GPU") == "1" else dev  # (gloo reduces host tensors)
    vals = torch.tensor([dev_ms, sum(e2e_t), wall], dtype=torch.float64, device=red)  # (e2e: the K timed steps)
    if world > 1:
        dist.all_reduce(vals, op=dist.ReduceOp.MAX)
    dev_ms_max, e2e_max, wall_max = (float(x) for x in vals.tolist())
    tot = torch.tensor([children, parents, alg_bytes, alg_ops], dtype=torch.float64, device=red)
    if world > 1:
        dist.all_reduce(tot)
    pairs_total = w.npairs * args.steps
    value = pairs_total / (dev_ms_max / 1e3)
    nodes_per_s = float(tot[0]) / (dev_ms_max / 1e3)

    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    alu = int_peak(sms, peaks)
    # the word-width groups' launches overlap (fork/join): the kernel time of a step is the union of
    # their intervals, i.e. the step's device time (CUDA events on the launching stream around the run)
    kern_s = min(branch_ms, dev_ms) / args.steps / 1e3
    achieved = (alg_ops / args.steps) / kern_s / 1e9 if branch_ms > 0 else None
    hbm_ach = (alg_bytes / args.steps) / kern_s / 1e9 if branch_ms > 0 else None
    traffic = None
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "ncu_summary.json")))
        # DRAM bytes of all batched launches of one step (ncu --set full of the same workload), the unit of
        # roofline.achieved (algorithmic ops or bytes per step over the step's kernel time)
        traffic = (prof.get("bench_kernel_dram_bytes_per_step") or {}).get(args.workload)
    except Exception:
        pass
    line = {
        "metric": METRIC,
        "value": value,
        "unit": "pairs/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": dev_ms_max / args.steps,
        "higher_is_better": True,
        "scaling": scaling,
        "vs_baseline": None,
        "dtype": "int32",
        "data": "synthetic (seeded generators, DESIGN.md §5)",
        "tree_nodes_per_s": nodes_per_s,
        "parents_per_s": float(tot[1]) / (dev_ms_max / 1e3),
        "config": {
            "workload": workload_name(w),
            "pairs_total": w.npairs,
            "pairs_per_gpu": len(idx),
            "K": w.K,
            "costs": list(w.costs),
            "parallelism": f"one canonical batch, pair r -> GPU r mod {world}; no data-path collective; "
                           f"e2e gathers every cost and mapping to rank 0",
            "l2": "256 MiB buffer written between timed steps (outside the CUDA-event region)",
        },
        "roofline": {
            "bound": "alu",
            "kernel": "kbest_batch_kernel (branch+rank+update, all levels; one launch per word-width group)",
            "achieved": achieved,
            "peak": alu["peak"],
            "peak_source": alu["source"],
            "unit": "Gop/s",
            "frac": (achieved / alu["peak"]) if achieved else None,
            "traffic": traffic,
            "alg_ops_per_step": alg_ops / args.steps,
            "launches_per_step": branch_launches / args.steps,
            "hbm_view": {"alg_bytes_per_step": alg_bytes / args.steps, "achieved_gbs": hbm_ach, "peak_gbs": hbm_peak,
                         "frac": (hbm_ach / hbm_peak) if hbm_ach else None,
                         "note": "frontier bytes each level touches (SURVEY §8(d) D.4), rank 0's GPU"},
        },
        "e2e": {
            "value": pairs_total / e2e_max if e2e_max > 0 else None,
            "unit": "pairs/s",
            "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h,
            "includes": "validation, packing, H2D, search, D2H" + (", gather of all results to rank 0" if world > 1 else ""),
        },
        "gpu_launches": launches,
        "clocks": clk,
        "wall_s": wall_max,
        "timing_crosscheck": {"torch_events_ms": dev_ms, "library_events_ms": lib_ms},
    }
    if rank == 0:
        line["parity"] = {"golden": golden_parity(w, world, res)}
        if not args.no_cpu_baseline:
            cb = oracle_sample(w, args.cpu_seconds, gpu=res)
            line["cpu_baseline"] = {"value": cb["pairs_per_s"], "unit": "pairs/s", "cores": cb["cores"], "kind": "oracle",
                                    "sample": f"first {cb['pairs']} pairs of the same canonical batch, {cb['seconds']:.1f} s "
                                              f"on rank 0's host cores", "tree_nodes_per_s": cb["nodes_per_s"]}
            line["parity"]["oracle_live"] = cb["parity"]
    batch.free()
    h.close()
    return line


def int_peak(sms, peaks):
    """Integer lane-op peak for the 'alu' roofline: the MEASURED microbenchmark
    (scripts/micro/int_peak.cu -> profiles/int_peak.json) if present, else derived."""
    try:
        m = json.load(open(os.path.join(ROOT, "profiles", "int_peak.json")))
        return {"peak": float(m["mix_gops"]), "source": f"measured: {m['source']}"}
    except Exception:
        clk = float(peaks.get("sm_max_mhz", 1965.0))
        return {"peak": sms * 128 * clk * 1e6 / 1e9,
                "source": f"derived: {sms} SMs x 128 int lanes/clk x {clk:.0f} MHz (no measured int peak found)"}


def run_pair(args, rank, local_rank, world):
    """cfg4: one large pair per step (n=500, p=0.05, K=1e5); N>1: frontier sharded over the ranks."""
    import torch
    import torch.distributed as dist

    from paper_2605_00830_b200 import binding, build, synth
    from paper_2605_00830_b200 import dist as fdist

    build.build()
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    w = synth.config_workload(4)
    idx = 5  # (500, 0.05, 1e5)
    g1, g2 = w.pair(idx)
    K = args.K or w.run_K[idx]
    h = fdist.sharded_handle(local_rank) if world > 1 else binding.Handle(local_rank)
    for _ in range(args.warmup):
        r = h.solve_pair(g1, g2, w.costs, K)
    clocks = ClockSampler(local_rank)
    clocks.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    dev_ms, kern_ms, wall = 0.0, 0.0, time.perf_counter()
    for _ in range(args.steps):
        r2 = h.solve_pair(g1, g2, w.costs, K)
        st2 = h.stats()
        dev_ms += st2["device_ms"]
        kern_ms += st2["branch_ms"]  # CUDA events around the cooperative kernel, on its stream
        assert r2["cost"] == r["cost"]
    torch.cuda.synchronize(dev)
    wall = time.perf_counter() - wall
    clk = clocks.stop()
    red = "cpu" if os.environ.get("FASTGED_BENCH_SHARE_GPU") == "1" else dev
    vals = torch.tensor([dev_ms, wall], dtype=torch.float64, device=red)
    if world > 1:
        dist.all_reduce(vals, op=dist.ReduceOp.MAX)
    dev_ms, wall = (float(x) for x in vals.tolist())
    st = h.stats()
    h.close()
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    traffic = None
    try:
        traffic = json.load(open(os.path.join(ROOT, "profiles", "ncu_summary.json"))).get("large_kernel_dram_bytes_per_launch")
    except Exception:
        pass
    parity = None
    try:  # the oracle's stored result for this corner (tests/golden, written by scripts/make_golden.py)
        gold = json.load(open(os.path.join(ROOT, "tests", "golden", "oracle_cfg4.json")))["runs"].get(str(idx))
        if gold is not None and int(gold["K"]) == int(K):
            parity = {"checked": 1, "mismatches": int(not (r["cost"] == gold["cost"] and r["mapping"].tolist() == gold["mapping"]
                                                           and r["children"] == gold["children"])),
                      "against": "tests/golden/oracle_cfg4.json (oracle cost, mapping, children)"}
    except Exception:
        pass
    kern_s = kern_ms / args.steps / 1e3
    ach = st["alg_bytes"] / kern_s / 1e9 if (world == 1 and kern_s > 0) else None
    roof = {"bound": "hbm", "kernel": "kbest_large_kernel (all levels of the pair in one cooperative launch)",
            "achieved": ach, "peak": hbm_peak,
            "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "B200_PROFILING.md fallback",
            "unit": "GB/s", "frac": (ach / hbm_peak) if ach else None, "traffic": traffic,
            "alg_bytes_per_launch": st["alg_bytes"],
            "note": "algorithmic bytes = SURVEY §8(d) D.4 per level (parent PED + lambda rows read, child rows written); "
                    "traffic = ncu dram read+write of the same launch (counters, used masks and candidate lists on top)"}
    return {
        "metric": METRIC, "value": args.steps / (dev_ms / 1e3), "unit": "pairs/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dev_ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "int32", "data": "synthetic (seeded ER pair, DESIGN.md §5)",
        "tree_nodes_per_s": r["children"] / (dev_ms / args.steps / 1e3),
        "config": {"workload": f"cfg4: single ER pair n=500 p=0.05, 4 vertex labels, Setting-1 costs, K={K}",
                   "parallelism": f"frontier sharded by parent over {world} GPU(s)" if world > 1 else "1 GPU (cooperative kernel)",
                   "cost": r["cost"]},
        "e2e": {"value": args.steps / wall, "unit": "pairs/s", "h2d_bytes_per_step": st["h2d_bytes"],
                "d2h_bytes_per_step": st["d2h_bytes"]},
        "roofline": roof,
        "parity": {"golden": parity},
        "gpu_launches": st["kernel_launches"] * args.steps,
        "clocks": clk,
    }


def run_reference(args, rank, world):
    """Reference arm: the CPU oracle, as it stands, on the host cores (rank 0 only)."""
    if rank != 0:
        return None
    w, scaling = canonical_workload(world)
    per = []
    total_pairs = 0
    nodes = 0
    cores = None
    for s in range(args.warmup + args.steps):
        cb = oracle_sample(w, args.cpu_seconds / max(1, args.steps))
        if s >= args.warmup:
            per.append(cb["seconds"])
            total_pairs += cb["pairs"]
            nodes += cb["nodes_per_s"] * cb["seconds"]
        cores = cb["cores"]
    secs = sum(per)
    value = total_pairs / secs
    return {
        "impl": "reference",
        "metric": METRIC,
        "value": value,
        "unit": "pairs/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": 1e3 * secs / args.steps,
        "higher_is_better": True,
        "scaling": scaling,
        "vs_baseline": None,
        "dtype": "int64",
        "data": "synthetic (seeded ER graphs, DESIGN.md §5)",
        "tree_nodes_per_s": nodes / secs,
        "config": {"workload": workload_name(w), "pairs_total": w.npairs, "K": w.K, "costs": list(w.costs)},
        "cpu_baseline": {"value": value, "unit": "pairs/s", "cores": cores, "kind": "oracle",
                         "sample": f"each step: consecutive pairs of the workload for ~{args.cpu_seconds / max(1, args.steps):.1f} s"},
        "e2e": {"value": value, "unit": "pairs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }


def main():
    global ARGS
    args = parse()
    ARGS = args
    rank, local_rank, world = dist_env()
    if world != args.gpus:
        # the driver launches N>1 under torchrun (one rank per GPU); a bare `--gpus N` would silently
        # measure one GPU, so refuse instead
        sys.stderr.write(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; for N>1 launch one rank per GPU:\n"
                         f"  python -m torch.distributed.run --nnodes=1 --nproc-per-node {args.gpus} "
                         f"--master-addr 127.0.0.1 --master-port 29511 bench.py --gpus {args.gpus} ...\n")
        sys.exit(2)
    if args.impl == "reference":
        if args.workload == "cfg4":
            if rank == 0:
                print(json.dumps({"impl": "reference", "unavailable": "cfg4 oracle run exceeds the bench time budget"}))
            return
        line = run_reference(args, rank, world)
        if line is not None:
            print(json.dumps(line), flush=True)
        return
    import torch
    if not torch.cuda.is_available() or torch.cuda.device_count() <= local_rank:
        sys.stderr.write(f"bench.py: rank {rank} needs cuda:{local_rank} but torch sees "
                         f"{torch.cuda.device_count() if torch.cuda.is_available() else 0} CUDA device(s); "
                         "this benchmark has no CPU path\n")
        sys.exit(3)
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        if os.environ.get("FASTGED_BENCH_SHARE_GPU") == "1":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    line = run_pair(args, rank, local_rank, world) if args.workload == "cfg4" else run_ours(args, rank, local_rank, world)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
