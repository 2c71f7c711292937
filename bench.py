#!/usr/bin/env python3
"""FAST-GED K-Best hot path benchmark (BASELINE.json metric: GED pairs/sec and expanded tree
nodes/sec at K=1000, 1/2/4/8 B200).

Workload: BASELINE configs[2] — 10,000 Erdős–Rényi pairs per GPU, n = 30..70,
p = 0.1..0.5 (400 pairs per (n, p) cell), 4 vertex labels, Setting-1 costs, K = 1000.
One step = one K-Best search of every pair of the batch (all levels: branch, rank, update,
finalize).  Multi-GPU: weak scaling, every rank searches its own 10,000 pairs, no data-path
collective (pairs are independent).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...

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
    ap.add_argument("--npairs", type=int, default=10_000, help="pairs per GPU")
    ap.add_argument("--K", type=int, default=None, help="override K (default: the config's K)")
    ap.add_argument("--workload", choices=["cfg3", "cfg2", "cfg5", "cfg4"], default="cfg3",
                    help="cfg3 (default, the BASELINE metric's K=1000 batch), cfg2/cfg5 batches, "
                         "cfg4 = one large pair (n=500, p=0.05, K=1e5; frontier sharded over the ranks)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="target CPU time of the oracle sample")
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))


WORKLOADS = {
    "cfg3": (3, "cfg3: ER pairs n=30..70 x p=0.1..0.5 (4 vertex labels, unlabelled edges), Setting-1 costs, K=1000"),
    "cfg2": (2, "cfg2: AIDS-like labelled molecule pairs (n=5..10), Setting-1 costs, K=100"),
    "cfg5": (5, "cfg5: all-pairs slice of 2000 Mutagenicity-like labelled graphs (n~30), Setting-1 costs, K=1000"),
}
ARGS = None


def workload(rank: int, npairs: int, K):
    from paper_2605_00830_b200 import synth
    cfg = WORKLOADS[ARGS.workload][0] if ARGS else 3
    # rank 0 = the canonical inputs; other ranks draw their own pairs (weak scaling)
    if cfg == 5:  # a contiguous slice of the 1,999,000 all-pairs per rank
        w = synth.config_workload(5, K=K)
        sl = np.arange(rank * npairs, (rank + 1) * npairs) % w.npairs
        return w.subset(sl)
    return synth.config_workload(cfg, seed=cfg + 1000 * rank, npairs=npairs, K=K)


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
def oracle_sample(w, seconds: float):
    """Time the oracle, as it stands, on host cores over a bounded sample of the workload:
    whole chunks of consecutive pairs (every (n, p) cell equally) until `seconds` of wall time."""
    from oracle import oracle
    oracle.build()
    cores = oracle.max_threads()
    chunk = 25 * max(1, (cores + 24) // 25)
    done, nodes, t0 = 0, 0, time.perf_counter()
    while done < w.npairs:
        idx = range(done, min(w.npairs, done + chunk))
        pairs = [w.pair(k) for k in idx]
        _, _, ch = oracle.kbest_batch(pairs, w.costs, w.K, nthreads=cores)
        done += len(pairs)
        nodes += int(ch.sum())
        if time.perf_counter() - t0 >= seconds:
            break
    dt = time.perf_counter() - t0
    return {"pairs": done, "seconds": dt, "pairs_per_s": done / dt, "nodes_per_s": nodes / dt, "cores": cores}


# ------------------------------------------------------------------ our arm
def run_ours(args, rank, local_rank, world):
    import torch
    import torch.distributed as dist

    from paper_2605_00830_b200 import binding, build

    build.build()
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    # a dedicated (non-default) stream: the library launches on it and the CUDA events time it
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    assert stream.cuda_stream != 0
    w = workload(rank, args.npairs, args.K)
    packed = binding.PackedGraphs(w.graphs)
    h = binding.Handle(local_rank, stream=stream.cuda_stream, flags=binding.FLAG_TIMING)
    batch = h.upload(packed, w.pair_a, w.pair_b)  # inputs resident in HBM before timing
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

    # ---- end-to-end through the public API with host buffers (H2D + search + D2H each step)
    e2e_t = []
    h2d = d2h = 0
    # one untimed call: the handle allocates its per-chunk pinned staging on first use
    h.solve_batch(packed, w.pair_a, w.pair_b, w.costs, w.K)
    for s in range(max(1, args.steps)):
        flush.fill_(s)
        torch.cuda.synchronize(dev)
        barrier()
        t0 = time.perf_counter()
        r = h.solve_batch(packed, w.pair_a, w.pair_b, w.costs, w.K)
        torch.cuda.synchronize(dev)
        e2e_t.append(time.perf_counter() - t0)
        st = h.stats()
        h2d, d2h = st["h2d_bytes"], st["d2h_bytes"]
    assert np.array_equal(r[0], ref[0]), "e2e results differ from the device-resident run"

    # ---- max over ranks
    vals = torch.tensor([dev_ms, sum(e2e_t), wall], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(vals, op=dist.ReduceOp.MAX)
    dev_ms_max, e2e_max, wall_max = (float(x) for x in vals.tolist())
    tot = torch.tensor([children, parents], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tot)
    pairs_total = args.npairs * world * args.steps
    value = pairs_total / (dev_ms_max / 1e3)
    nodes_per_s = float(tot[0]) / (dev_ms_max / 1e3)

    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    clk_mhz = float(peaks.get("sm_max_mhz", 1965.0))
    # integer lane-op peak: 4 SMSPs x (16 ALU-pipe + 16 FMA-pipe lanes) per clock per SM
    alu_peak = sms * 128 * clk_mhz * 1e6 / 1e9  # Gop/s
    # the word-width groups' launches overlap (fork/join): the kernel time of a step is the union of
    # their intervals, i.e. the step's device time (CUDA events on the launching stream around the run)
    kern_s = min(branch_ms, dev_ms_max) / args.steps / 1e3
    achieved = (alg_ops / args.steps) / kern_s / 1e9 if branch_ms > 0 else None
    hbm_ach = (alg_bytes / args.steps) / kern_s / 1e9 if branch_ms > 0 else None
    traffic = None
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "ncu_summary.json")))
        if args.workload == "cfg3":  # the ncu capture is of the cfg3 bench workload
            traffic = prof.get("bench_kernel_dram_bytes_per_launch")
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
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "int32",
        "data": "synthetic (seeded ER graphs, DESIGN.md §5)",
        "tree_nodes_per_s": nodes_per_s,
        "parents_per_s": float(tot[1]) / (dev_ms_max / 1e3),
        "config": {
            "workload": workload_name(w),
            "pairs_per_gpu": args.npairs,
            "K": w.K,
            "costs": list(w.costs),
            "parallelism": f"pairs strided over {world} GPU(s), no data-path collective",
            "l2": "256 MiB buffer written between timed steps (outside the CUDA-event region)",
        },
        "roofline": {
            "bound": "alu",
            "kernel": "kbest_batch_kernel (branch+rank+update, all levels; one launch per word-width group)",
            "achieved": achieved,
            "peak": alu_peak,
            "peak_source": f"derived: {sms} SMs x 128 int lanes/clk x {clk_mhz:.0f} MHz (MEASURED_PEAKS sm_max_mhz)",
            "unit": "Gop/s",
            "frac": (achieved / alu_peak) if achieved else None,
            "traffic": traffic,
            "alg_ops_per_step": alg_ops / args.steps,
            "launches_per_step": branch_launches / args.steps,
            "hbm_view": {"alg_bytes_per_step": alg_bytes / args.steps, "achieved_gbs": hbm_ach, "peak_gbs": hbm_peak,
                         "frac": (hbm_ach / hbm_peak) if hbm_ach else None,
                         "note": "frontier bytes each level touches (SURVEY §8(d) D.4); they stay in L2/SMEM"},
        },
        "e2e": {
            "value": pairs_total / e2e_max if e2e_max > 0 else None,
            "unit": "pairs/s",
            "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h,
        },
        "gpu_launches": launches,
        "clocks": clk,
        "wall_s": wall_max,
        "timing_crosscheck": {"torch_events_ms": dev_ms, "library_events_ms": lib_ms},
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cb = oracle_sample(w, args.cpu_seconds)
        line["cpu_baseline"] = {"value": cb["pairs_per_s"], "unit": "pairs/s", "cores": cb["cores"], "kind": "oracle",
                                "sample": f"first {cb['pairs']} pairs of the same workload (all 25 (n,p) cells), "
                                          f"{cb['seconds']:.1f} s", "tree_nodes_per_s": cb["nodes_per_s"]}
    batch.free()
    h.close()
    return line


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
    vals = torch.tensor([dev_ms, wall], dtype=torch.float64, device=dev)
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
    kern_s = kern_ms / args.steps / 1e3
    ach = st["alg_bytes"] / kern_s / 1e9 if (world == 1 and kern_s > 0) else None
    roof = {"bound": "hbm", "kernel": "kbest_large_kernel (all levels of the pair in one cooperative launch)",
            "achieved": ach, "peak": hbm_peak,
            "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "B200_PROFILING.md fallback",
            "unit": "GB/s", "frac": (ach / hbm_peak) if ach else None, "traffic": traffic,
            "alg_bytes_per_launch": st["alg_bytes"],
            "note": "algorithmic bytes = SURVEY §8(d) D.4 per level (parent PED + lambda rows read, child rows written); "
                    "traffic = ncu dram read+write of the same launch (counters, used masks and rank codes on top)"}
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
        "gpu_launches": st["kernel_launches"] * args.steps,
        "clocks": clk,
    }


def run_reference(args, rank, world):
    """Reference arm: the CPU oracle, as it stands, on the host cores (rank 0 only)."""
    if rank != 0:
        return None
    w = workload(0, args.npairs, args.K)
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
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "int64",
        "data": "synthetic (seeded ER graphs, DESIGN.md §5)",
        "tree_nodes_per_s": nodes / secs,
        "config": {"workload": workload_name(w), "pairs_per_gpu": args.npairs, "K": w.K, "costs": list(w.costs)},
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
    if args.impl == "reference":
        if args.workload == "cfg4":
            if rank == 0:
                print(json.dumps({"impl": "reference", "unavailable": "cfg4 oracle run exceeds the bench time budget"}))
            return
        line = run_reference(args, rank, world)
        if line is not None:
            print(json.dumps(line), flush=True)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    line = run_pair(args, rank, local_rank, world) if args.workload == "cfg4" else run_ours(args, rank, local_rank, world)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
