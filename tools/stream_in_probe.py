"""hx_step_host timing per HX_STREAM_IN slab count (bench workload: 3D Sedov Q3-Q2 23^3),
plus the bare H2D of the state and the device-resident step, for the e2e overlap study."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2112_07075_b200 import _lib, problems  # noqa: E402
from paper_2112_07075_b200.fespace import cartesian_mesh  # noqa: E402
from paper_2112_07075_b200.hydro import (LagrangeHydro, MaterialModel, StepControls, ViscosityModel,  # noqa: E402
                                         box_velocity_bc)
from paper_2112_07075_b200.tensor_basis import gauss_legendre  # noqa: E402

n = int(os.environ.get("N", "23"))
mesh = cartesian_mesh(3, (1.0,) * 3, (n,) * 3, 3)
hy = LagrangeHydro(mesh, gauss_legendre(5), MaterialModel(1.4), ViscosityModel(0.5, 2.0), bc_mask=box_velocity_bc(mesh))
st = hy.initial_state(*problems.sedov(3, (1.0,) * 3, (n,) * 3))
ctl = StepControls(cfl=0.05, dt_max=1.0, t_final=10.0)
nx, nv, ne = st.x.size, st.v.size, st.e.size
arena = torch.empty(nx + nv + ne, dtype=torch.float64).pin_memory()
init = torch.cat([torch.from_numpy(np.ascontiguousarray(a)).reshape(-1) for a in (st.x, st.v, st.e)])
lib, h = hy._ctx.lib, hy._ctx.h
prm = hy._params(ctl)
info = _lib.StepInfo()
dbuf = torch.empty_like(arena, device="cuda")
# bare H2D
for _ in range(3):
    dbuf.copy_(arena, non_blocking=True)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    dbuf.copy_(arena, non_blocking=True)
torch.cuda.synchronize()
print(f"bare H2D {8 * arena.numel() / 1e6:.1f} MB: {(time.perf_counter() - t0) / 10 * 1e3:.3f} ms", flush=True)


def run(tag, steps=10):
    arena.copy_(init)
    t = st.t
    ts = []
    for k in range(3 + steps):
        if k == 3 + steps // 2:
            arena.copy_(init)
            t = st.t
        hy._ctx.sync_stream()
        t0 = time.perf_counter()
        rc = lib.hx_step_host(h, _lib.C.byref(prm), float(t), arena[:nx].data_ptr(), arena[nx:nx + nv].data_ptr(),
                              arena[nx + nv:].data_ptr(), _lib.C.byref(info))
        dt = time.perf_counter() - t0
        assert rc == 0, rc
        t = info.t_new
        if k >= 3:
            ts.append(dt)
    print(f"{tag}: hx_step_host {np.median(ts) * 1e3:.3f} ms median, {np.mean(ts) * 1e3:.3f} mean", flush=True)
    return float(np.median(ts))


res = {}
for rnd in range(int(os.environ.get("ROUNDS", "1"))):  # configurations interleaved per round
    for s in os.environ.get("SLABS", "0 3 3u 4 4u 2 6").split():  # 'u': equal layer counts
        os.environ["HX_STREAM_UNIFORM"] = "1" if s.endswith("u") else "0"
        os.environ["HX_STREAM_IN"] = s.rstrip("u")
        res.setdefault(s, []).append(run(f"slabs={s}"))
for s, v in res.items():
    print(f"summary slabs={s}: median over rounds {np.median(v) * 1e3:.3f} ms, min {min(v) * 1e3:.3f}", flush=True)
# device-resident step
dev = hy.to_device(st)
for _ in range(3):
    d2, _ = hy.step(dev, ctl)
torch.cuda.synchronize()
ts = []
for _ in range(10):
    t0 = time.perf_counter()
    d2, _ = hy.step(dev, ctl)
    torch.cuda.synchronize()
    ts.append(time.perf_counter() - t0)
print(f"device step: {np.median(ts) * 1e3:.3f} ms median", flush=True)
