"""Time the unmodified reference (baseline/_ref) on the GPU arm's full workload (3D Sedov Q3-Q2
23^3, 1.03M velocity dofs) for a few steps on this host: the reference point behind the
bench's 12^3 CPU sample.  python tools/ref_fullsize.py [--n 23] [--steps 2] [--threads T]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=23)
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--threads", type=int, default=8)
a = ap.parse_args()
out = {}
for th in sorted({1, a.threads}):
    V, times, kind = bench.cpu_reference_run(3, a.n, a.steps, 1, 0.05, th)
    out[f"threads_{th}"] = {"Mdof_per_s": V * len(times) / sum(times) / 1e6, "s_per_step": sum(times) / len(times),
                            "V": V, "kind": kind}
print(json.dumps({"workload": f"3D Sedov Q3-Q2 {a.n}^3 ({out[f'threads_{a.threads}']['V']} velocity dofs), CFL 0.05, "
                              f"{a.steps} steps after 1 warm-up", "cpu": bench.cpu_model(), "cores": os.cpu_count(),
                  "runs": out}))
