"""Summarise gpurun_out/ evidence into profiles/ (launch list, ncu full metrics, hotspots, bench lines).

    python scripts/make_profiles.py r2      (after scripts/gpu_round.sh)
"""
import collections, csv, json, math, os, shutil, subprocess, sys
R = sys.argv[1] if len(sys.argv) > 1 else "r1"
REP = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out"   # where the .ncu-rep files are
OUT = sys.argv[3] if len(sys.argv) > 3 else "profiles"     # where the summaries go
os.makedirs(OUT, exist_ok=True)
rows = [r for r in csv.reader(open("gpurun_out/launches.csv")) if len(r) > 10]
hdr = rows[0]; ik = hdr.index("Kernel Name"); iv = hdr.index("Metric Value")
agg = collections.defaultdict(list)
for r in rows[1:]:
    agg[r[ik]].append(float(r[iv].replace(",", "")))
tot = sum(sum(v) for v in agg.values())
lines = ["# ncu launch list of `python bench.py --steps 2 --warmup 3 --no-cpu-baseline` (gpu__time_duration.sum, --clock-control none)",
         "# cold-cache, serialised replay: compare SHARES, not absolutes", "share   launches  mean_us  kernel"]
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    lines.append(f"{sum(v)/tot*100:6.2f}%  {len(v):3d}  {sum(v)/len(v)/1e3:10.1f}  {k}")
open(f"{OUT}/{R}_launches_bench.txt", "w").write("\n".join(lines) + "\n")
out = subprocess.run(["ncu", "-i", f"{REP}/prof_bench.ncu-rep", "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines())); hdr = r[0]; units = r[1]
want = ['Kernel Name', 'gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'smsp__inst_executed.sum',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active', 'sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'launch__registers_per_thread', 'launch__shared_mem_per_block_dynamic', 'launch__grid_size']
idx = {h: i for i, h in enumerate(hdr)}
recs = [{w: row[idx[w]] for w in want if w in idx} for row in r[2:]]
for x in recs:
    x["units"] = {w: units[idx[w]] for w in want if w in idx}
json.dump(recs, open(f"{OUT}/{R}_ncu_full_batch.json", "w"), indent=1)
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
dram = []
for x in recs:
    try:
        v = (float(x['dram__bytes_read.sum']) + float(x['dram__bytes_write.sum'])) * scale.get(x["units"]['dram__bytes_read.sum'], 1)
        dram.append(None if math.isnan(v) else v)
    except Exception:
        dram.append(None)
valid = [d for d in dram if d is not None]
summary = {"source": "ncu --set full --clock-control none -k regex:kbest_batch -c 3 python scripts/prof_batch.py 10000 1000 1 (the bench workload)",
           "kernels": [x['Kernel Name'] for x in recs], "dram_bytes_per_launch": dram,
           # DRAM bytes per launch of the batched kernels, keyed by bench workload (bench.py roofline.traffic)
           "bench_kernel_dram_bytes_per_launch": {"cfg3": (sum(valid) / len(valid)) if valid else None},
           # all batched launches of one step (the word-width groups run concurrently): bench.py roofline.traffic
           "bench_kernel_dram_bytes_per_step": {"cfg3": sum(valid) if valid else None}}
if os.path.exists(f"{REP}/prof_cfg5.ncu-rep"):
    o5 = subprocess.run(["ncu", "-i", f"{REP}/prof_cfg5.ncu-rep", "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r5 = list(csv.reader(o5.splitlines())); h5 = r5[0]; u5 = r5[1]
    vals = []
    for row in r5[2:]:
        i1, i2 = h5.index("dram__bytes_read.sum"), h5.index("dram__bytes_write.sum")
        vals.append((float(row[i1]) + float(row[i2])) * scale.get(u5[i1], 1))
    summary["bench_kernel_dram_bytes_per_launch"]["cfg5"] = sum(vals) / len(vals) if vals else None
    summary["bench_kernel_dram_bytes_per_step"]["cfg5"] = sum(vals) if vals else None
    summary["cfg5_source"] = "ncu --set full --clock-control none -k regex:kbest_batch -c 2 python scripts/prof_cfg5.py 20000"
if os.path.exists(f"{REP}/prof_large5.ncu-rep"):  # cfg4 bench launch (n=500 p=0.05 K=1e5)
    o2 = subprocess.run(["ncu", "-i", f"{REP}/prof_large5.ncu-rep", "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r2 = list(csv.reader(o2.splitlines())); h2 = r2[0]; u2 = r2[1]
    def val(k):
        i = h2.index(k); return float(r2[2][i].replace(",", "")) * scale.get(u2[i], 1)
    summary["large_kernel_dram_bytes_per_launch"] = val("dram__bytes_read.sum") + val("dram__bytes_write.sum")
    summary["large_source"] = "ncu --set full --clock-control none -k regex:kbest_large -c 1 python scripts/prof_large.py 5"
json.dump(summary, open(f"{OUT}/ncu_summary.json", "w"), indent=1)
subprocess.run(f"python scripts/ncu_lines.py {REP}/prof_bench.ncu-rep 'kbest_batch_kernel<(int)2' 30 "
               f"paper_2605_00830_b200/csrc/batch_kernel.cuh > {OUT}/{R}_ncu_source_hotspots_w2.txt", shell=True)
if os.path.exists(f"{REP}/prof_large5.ncu-rep"):
    subprocess.run(f"python scripts/ncu_stalls.py {REP}/prof_large5.ncu-rep kbest_large 30 > {OUT}/{R}_ncu_large_stalls.txt", shell=True)
for f in ("bench.json", "bench_cfg5.json", "bench_cfg2.json", "bench_cfg4.json", "bench_ref.json", "time_large.txt", "nvsmi.txt",
          "smoke.log", "pytest_gpu.log"):
    if os.path.exists(f"gpurun_out/{f}"):
        shutil.copy(f"gpurun_out/{f}", f"{OUT}/{R}_{f}")
print(open(f"{OUT}/{R}_launches_bench.txt").read()); print(json.dumps(summary, indent=1))
