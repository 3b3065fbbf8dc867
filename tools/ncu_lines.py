"""Aggregate warp-stall samples and executed instructions per CUDA source line of an .ncu-rep
(compiled with -lineinfo): python tools/ncu_lines.py rep [n]"""
import csv, subprocess, sys
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
key = 1 if len(sys.argv) > 3 and sys.argv[3] in ("ins", "bank") else 0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = None
agg = {}
fname = "?"
for r in rows:
    if len(r) == 2 and r[0] in ("File Name", "File Path"):
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No" or (r and r[0] == "#"):
        hdr = r
        ix = {}
        for i, k in enumerate(hdr):
            ix.setdefault(k, i)
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    try:
        ln = int(r[0])
    except ValueError:
        continue
    s = float(r[ix.get("Warp Stall Sampling (All Samples)", 0)] or 0) if "Warp Stall Sampling (All Samples)" in ix else 0
    ins = float(r[ix["Instructions Executed"]] or 0) if "Instructions Executed" in ix else 0
    if len(sys.argv) > 3 and sys.argv[3] == "bank":
        ins = float(r[ix["L1 Wavefronts Shared Excessive"]] or 0) if "L1 Wavefronts Shared Excessive" in ix else 0
    src = r[1]
    a = agg.setdefault((fname, ln), [0.0, 0.0, src])
    a[0] += s
    a[1] += ins
tot_s = sum(v[0] for v in agg.values()) or 1
tot_i = sum(v[1] for v in agg.values()) or 1
print(f"samples {tot_s:.0f} instructions {tot_i:.3e}")
for (f, ln), (s, i, src) in sorted(agg.items(), key=lambda kv: -kv[1][key])[:n]:
    print(f"{100*s/tot_s:5.1f}% smp {100*i/tot_i:5.1f}% ins  {f}:{ln}  {src.strip()[:80]}")
