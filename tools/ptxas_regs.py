"""Registers / spills per kernel from an nvcc -Xptxas -v log: python tools/ptxas_regs.py LOG [substr...]"""
import re, subprocess, sys
log = open(sys.argv[1]).read().splitlines()
pats = sys.argv[2:] or [""]
cur = None
rows = {}
for ln in log:
    m = re.search(r"Compiling entry function '(\S+)'", ln)
    if m:
        cur = m.group(1)
        rows[cur] = {}
        continue
    if cur is None:
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", ln)
    if m:
        rows[cur]["spill"] = f"{m.group(1)}/{m.group(2)}"
    m = re.search(r"Used (\d+) registers", ln)
    if m:
        rows[cur]["regs"] = int(m.group(1))
names = dict(zip(rows, subprocess.run(["c++filt"], input="\n".join(rows), capture_output=True, text=True).stdout.split("\n")))
for k, v in rows.items():
    n = names.get(k, k)
    if any(p in n for p in pats):
        print(f"{v.get('regs', '?'):>4} regs  spill {v.get('spill', '?'):>7}  {n[:110]}")
