"""Timing of the TMOP device operators (meshopt.py:335-486) at the Lagrange bench size:
3D Q3 (23^3 elements, 1.03M position dofs), a 0.1 h random interior perturbation,
ideal-uniform targets, gamma = 1.  CUDA events around each C-ABI call (device
buffers resident, the launch + deterministic scatter + limiting pieces included), L2
flushed before every call.  Prints one JSON line.

    python tools/bench_tmop.py [--n 23] [--p 3] [--reps 20]
"""

import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=23)
    ap.add_argument("--p", type=int, default=3)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--cpu-n", type=int, default=8, help="CPU reference sample: elements per direction (0: skip)")
    args = ap.parse_args()
    from paper_2112_07075_b200 import _lib, meshopt
    from paper_2112_07075_b200._device import to_dev
    from paper_2112_07075_b200.fespace import cartesian_mesh
    from paper_2112_07075_b200.tensor_basis import gauss_legendre

    d, p, n = 3, args.p, args.n
    mesh = cartesian_mesh(d, (1.0,) * d, (n,) * d, p)
    quad = gauss_legendre(p + 2)
    rng = np.random.default_rng(1)
    obj = meshopt.TMOPObjective(mesh, quad, meshopt.build_targets(mesh, quad), gamma=1.0)
    free = obj.free_interior_mask()
    h = 1.0 / (n * p)
    x = mesh.coords + np.where(free, 0.1 * h * rng.uniform(-1, 1, mesh.coords.shape), 0.0)
    dx = np.where(free, rng.standard_normal(x.shape), 0.0)
    X, DX = to_dev(x), to_dev(dx)
    out = torch.empty_like(X)
    lib, hh = obj._ctx.lib, obj._h
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    mu, lim, ok = _lib.C.c_double(), _lib.C.c_double(), _lib.C.c_int()
    calls = {
        "objective": lambda: lib.hx_tmop_terms(hh, _lib.ptr(X), 1, _lib.C.byref(mu), _lib.C.byref(lim),
                                               _lib.C.byref(ok)),
        "gradient": lambda: lib.hx_tmop_gradient(hh, _lib.ptr(X), _lib.ptr(out)),
        "hessian_action": lambda: lib.hx_tmop_hessian_action(hh, _lib.ptr(X), _lib.ptr(DX), _lib.ptr(out)),
        "hessian_diagonal": lambda: lib.hx_tmop_hessian_diagonal(hh, _lib.ptr(X), _lib.ptr(out)),
    }
    V = d * mesh.num_nodes
    ne, nq, nl = mesh.num_elements, quad.n ** d, (p + 1) ** d
    # algorithmic bytes of the Hessian action: x and dx gathered (16 V), W^-1 and w detW
    # read (8 (d^2 + 1) NE nq), the E-vector written and read back by the node pass
    # (2 * 8 d NE nl), the result written (8 V); + the limiting pieces (r / dx field 16 V,
    # their E-vector 16 d NE nl, combine 24 V)
    alg_ha = 16 * V + 8 * (d * d + 1) * ne * nq + 16 * d * ne * nl + 8 * V + 16 * V + 16 * d * ne * nl + 24 * V
    res = {}
    stream = torch.cuda.current_stream()
    for name, fn in calls.items():
        for _ in range(3):
            assert fn() == 0, name
        torch.cuda.synchronize()
        tot = 0.0
        for _ in range(args.reps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            assert fn() == 0, name
            e1.record(stream)
            e1.synchronize()
            tot += e0.elapsed_time(e1)
        res[name] = {"ms": tot / args.reps, "Mdof_per_s": V / (tot / args.reps / 1e3) / 1e6}
    # the reference's own CPU path (baseline/_ref, unmodified) beside it, on an n^3 sample
    cpu = None
    ref_dir = os.path.join(ROOT, "baseline", "_ref")
    if args.cpu_n > 0 and os.path.isdir(os.path.join(ref_dir, "ale_minihydro")):
        import time

        sys.path.insert(0, ref_dir)
        from ale_minihydro import fespace as rf
        from ale_minihydro import meshopt as rm
        from ale_minihydro import tensor_basis as rt

        cn = args.cpu_n
        rmesh = rf.cartesian_mesh(d, (1.0,) * d, (cn,) * d, p)
        rquad = rt.gauss_legendre(p + 2)
        robj = rm.TMOPObjective(rmesh, rquad, rm.build_targets(rmesh, rquad), gamma=1.0)
        rfree = robj.free_interior_mask()
        rh = 1.0 / (cn * p)
        rx = rmesh.coords + np.where(rfree, 0.1 * rh * rng.uniform(-1, 1, rmesh.coords.shape), 0.0)
        rdx = np.where(rfree, rng.standard_normal(rx.shape), 0.0)
        cpu = {"sample": f"3D Q{p} {cn}^3 elements ({d * rmesh.num_nodes} position dofs), baseline/_ref "
                         f"ale_minihydro.meshopt (unmodified), {os.cpu_count()} host cores available"}
        Vc = d * rmesh.num_nodes
        for name, fn in (("gradient", lambda: robj.gradient(rx)),
                         ("hessian_action", lambda: robj.hessian_action(rx, rdx))):
            fn()
            t0 = time.perf_counter()
            for _ in range(2):
                fn()
            ms = 1e3 * (time.perf_counter() - t0) / 2
            cpu[name] = {"ms": ms, "Mdof_per_s": Vc / (ms / 1e3) / 1e6}
    pk = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    ha_gbs = alg_ha / (res["hessian_action"]["ms"] / 1e3) / 1e9
    print(json.dumps({"workload": f"TMOP 3D Q{p} {n}^3 elements ({V} position dofs), 0.1h perturbation, ideal-uniform "
                                  f"targets, gamma {obj.gamma:.4g}", "calls": res,
                      "hessian_action_roofline": {"alg_bytes": alg_ha, "achieved_gbs": ha_gbs, "peak_gbs": pk,
                                                  "frac": ha_gbs / pk},
                      "cpu_reference": cpu,
                      "note": "CUDA events around each C-ABI call (kernel + scatter + limiting pieces; "
                              "objective includes its host read-back), L2 flushed before each call"}))


if __name__ == "__main__":
    main()
