"""Split the host-buffer step (hx_step_host) into H2D / step / D2H with CUDA events."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2112_07075_b200 import _lib, problems  # noqa: E402
from paper_2112_07075_b200.fespace import cartesian_mesh  # noqa: E402
from paper_2112_07075_b200.hydro import LagrangeHydro, MaterialModel, StepControls, ViscosityModel, box_velocity_bc  # noqa: E402
from paper_2112_07075_b200.tensor_basis import gauss_legendre  # noqa: E402

d, p, n = 3, 3, 23
mesh = cartesian_mesh(d, (1.0,) * d, (n,) * d, p)
hy = LagrangeHydro(mesh, gauss_legendre(p + 2), MaterialModel(1.4), ViscosityModel(0.5, 2.0),
                   bc_mask=box_velocity_bc(mesh))
st = hy.initial_state(*problems.sedov(d, (1.0,) * d, (n,) * d))
ctl = StepControls(cfl=0.05, dt_max=1.0, t_final=1e9)
dev = hy.to_device(st)
for _ in range(3):
    dev, _ = hy.step(dev, ctl)
hst = hy.to_host(dev)
nx, nv, ne = hst.x.size, hst.v.size, hst.e.size
arena = torch.empty(nx + nv + ne, dtype=torch.float64).pin_memory()
hx, hv, he = arena[:nx].view(hst.x.shape), arena[nx:nx + nv].view(hst.v.shape), arena[nx + nv:].view(hst.e.shape)
hx.copy_(torch.from_numpy(hst.x)); hv.copy_(torch.from_numpy(hst.v)); he.copy_(torch.from_numpy(hst.e))
lib, h = hy._ctx.lib, hy._ctx.h
prm = hy._params(ctl)
info = _lib.StepInfo()
t = hst.t
for i in range(8):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    hy._ctx.sync_stream()
    rc = lib.hx_step_host(h, _lib.C.byref(prm), float(t), hx.data_ptr(), hv.data_ptr(), he.data_ptr(), _lib.C.byref(info))
    t1 = time.perf_counter()
    t = info.t_new
    print(f"hx_step_host {1e3 * (t1 - t0):.3f} ms rc={rc}")
# components with torch copies and the resident step
dx = torch.empty_like(dev.x); dv = torch.empty_like(dev.v); de = torch.empty_like(dev.e)
s = torch.cuda.current_stream()
for i in range(5):
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    torch.cuda.synchronize()
    evs[0].record(s)
    dx.copy_(hx, non_blocking=True); dv.copy_(hv, non_blocking=True); de.copy_(he, non_blocking=True)
    evs[1].record(s)
    dev.x, dev.v, dev.e = dx, dv, de
    dev2, _ = hy.step(dev, ctl)
    evs[2].record(s)
    hx.copy_(dev2.x, non_blocking=True); hv.copy_(dev2.v, non_blocking=True); he.copy_(dev2.e, non_blocking=True)
    evs[3].record(s)
    evs[3].synchronize()
    print("h2d %.3f step %.3f d2h %.3f ms" % (evs[0].elapsed_time(evs[1]), evs[1].elapsed_time(evs[2]),
                                            evs[2].elapsed_time(evs[3])))
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
for mode in ("flush", "noflush"):
    tt = []
    for i in range(8):
        if mode == "flush":
            flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        hy._ctx.sync_stream()
        rc = lib.hx_step_host(h, _lib.C.byref(prm), float(t), hx.data_ptr(), hv.data_ptr(), he.data_ptr(),
                              _lib.C.byref(info))
        tt.append(1e3 * (time.perf_counter() - t0))
        t = info.t_new
    print(mode, " ".join(f"{x:.3f}" for x in tt))
