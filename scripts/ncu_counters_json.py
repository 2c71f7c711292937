"""gpurun_out/ncu_counters_cfg{3,5,4}.csv (scripts/gpu_r2_evidence.sh) -> profiles/<round>_ncu_counters.json."""
import csv, json, sys
R = sys.argv[1] if len(sys.argv) > 1 else "r2"
out = {"source": "ncu --metrics <L2/atomic/shared/pipe counters> --clock-control none (scripts/gpu_r2_evidence.sh): cfg3 = the "
                  "bench batch (10k ER pairs, K=1000), cfg5 = 20k all-pairs slice, cfg4 = the n=500 p=0.05 K=1e5 pair",
       "kernels": []}
for wl in ("cfg3", "cfg5", "cfg4"):
    rows = [r for r in csv.reader(open(f"gpurun_out/ncu_counters_{wl}.csv")) if len(r) > 10]
    hdr = rows[0]
    ik, im, iu, iv, iid = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value", "ID"))
    recs = {}
    for r in rows[1:]:
        rec = recs.setdefault(r[iid], {"workload": wl, "kernel": r[ik]})
        name = r[im] + (f" [{r[iu]}]" if r[iu] else "")
        try:
            rec[name] = float(r[iv].replace(",", ""))
        except ValueError:
            rec[name] = r[iv]
    out["kernels"] += list(recs.values())
json.dump(out, open(f"profiles/{R}_ncu_counters.json", "w"), indent=1)
print(len(out["kernels"]), "kernels")
