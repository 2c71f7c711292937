"""Per-source-line stall reasons and shared-memory excess wavefronts from an ncu report.
usage: python scripts/ncu_stalls.py report.ncu-rep kernel-substring [top]"""
import csv, subprocess, sys, collections
rep, ksub = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
func = fpath = hdr = None
cur = None
agg = collections.defaultdict(lambda: collections.Counter())
txt = {}
tot = collections.Counter()
for r in rows:
    if not r: continue
    if r[0] == "File Path": fpath = r[1]; continue
    if r[0] == "Function Name": func = r[1]; continue
    if r[0] == "Line No": hdr = r; continue
    if ksub not in (func or ""): continue
    if r[0] != "":
        cur = (fpath.split("/")[-1], int(r[0])); txt[cur] = r[1][:80]; continue
    for i, h in enumerate(hdr):
        if h.startswith("stall_") and "Not Issued" not in h or h in ("L1 Wavefronts Shared Excessive", "Instructions Executed", "L1 Wavefronts Shared"):
            try:
                v = float(r[i]); agg[cur][h] += v; tot[h] += v
            except Exception: pass
S = sum(v for h, v in tot.items() if h.startswith("stall_"))
print("kernel stall mix:", ", ".join(f"{h[6:]} {100*v/S:.1f}%" for h, v in tot.most_common() if h.startswith("stall_") and v / S > 0.01))
print(f"shared wavefronts {tot['L1 Wavefronts Shared']:.3e}, excessive {tot['L1 Wavefronts Shared Excessive']:.3e}")
print("top lines by excessive shared wavefronts:")
for k, c in sorted(agg.items(), key=lambda kv: -kv[1]["L1 Wavefronts Shared Excessive"])[:12]:
    print(f"  {c['L1 Wavefronts Shared Excessive']:.2e} / {c['L1 Wavefronts Shared']:.2e}  {k[0]}:{k[1]} {txt[k]}")
print("top lines by stall samples:")
for k, c in sorted(agg.items(), key=lambda kv: -sum(v for h, v in kv[1].items() if h.startswith("stall_")))[:top]:
    s = sum(v for h, v in c.items() if h.startswith("stall_"))
    mix = ", ".join(f"{h[6:]} {100*v/s:.0f}" for h, v in c.most_common(3) if h.startswith("stall_"))
    print(f"  {100*s/S:5.1f}%  {k[0]}:{k[1]:4d} [{mix}] {txt[k]}")
