"""Print the hottest SASS lines (warp-stall samples) of an .ncu-rep: python tools/ncu_hot.py rep [n]"""
import csv, subprocess, sys
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
ix = {k: i for i, k in enumerate(hdr)}
body = [r for r in rows[2:] if len(r) == len(hdr)]
tot = sum(float(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in body)
print(f"total samples {tot:.0f}, instructions {len(body)}")
for i, r in enumerate(body):
    r.append(i)
body.sort(key=lambda r: -float(r[ix["Warp Stall Sampling (All Samples)"]] or 0))
for r in body[:n]:
    s = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    print(f"{100*s/tot:5.1f}% #{r[-1]:5d} {r[ix['Source']].strip()[:90]}")
