"""Aggregate an ncu '--page source --print-source cuda,sass' CSV by CUDA source line.
usage: python scripts/ncu_lines.py report.ncu-rep [kernel-substring] [top]"""
import csv, subprocess, sys, collections
rep = sys.argv[1]; ksub = sys.argv[2] if len(sys.argv) > 2 else ""; top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
func = None; hdr = None; cur = None; fpath = ""
agg = collections.defaultdict(lambda: [0, 0, ""])
for r in rows:
    if not r: continue
    if r[0] == "File Path": fpath = r[1].split("/")[-1]; continue
    if r[0] == "Function Name": func = r[1]; continue
    if r[0] == "Line No": hdr = r; ix_inst = hdr.index("Instructions Executed"); ix_samp = hdr.index("Warp Stall Sampling (All Samples)"); continue
    if r[0] == "File Path" or hdr is None: continue
    if ksub and (func is None or ksub not in func): continue
    if r[0] != "":
        cur = (func, fpath, int(r[0])); agg[cur][2] = r[1][:90]; continue
    try:
        agg[cur][0] += int(float(r[ix_inst])); agg[cur][1] += int(float(r[ix_samp]))
    except Exception:
        pass
tot_i = sum(v[0] for v in agg.values()) or 1; tot_s = sum(v[1] for v in agg.values()) or 1
print(f"total warp-instructions {tot_i:.3e}, stall samples {tot_s}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{100*v[1]/tot_s:5.1f}% samp {100*v[0]/tot_i:5.1f}% inst  {k[1][:14]}:{k[2]:4d}  {v[2]}")

# phase totals: source lines grouped by the "// ---------------- <phase>" markers of the kernel file
if len(sys.argv) > 4:
    src = open(sys.argv[4]).read().splitlines()
    marks = [(n + 1, l.strip().strip("/- ").split(":")[0][:40]) for n, l in enumerate(src) if "// ----------------" in l]
    ph = collections.defaultdict(lambda: [0, 0])
    for k, v in agg.items():
        name = "pre"
        for ln, nm in marks:
            if k[2] >= ln: name = nm
        if k[1] != sys.argv[4].split("/")[-1]: name = "other files (" + k[1][:20] + ")"
        elif k[2] < 200: name = "helpers(<200)"
        ph[name][0] += v[0]; ph[name][1] += v[1]
    for nm, v in sorted(ph.items(), key=lambda kv: -kv[1][1]):
        print(f"PHASE {nm:42s} samp {100*v[1]/tot_s:5.1f}%  inst {100*v[0]/tot_i:5.1f}%")
