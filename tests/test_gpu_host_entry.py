"""The C-ABI host-buffer entry hx_step_host (INTEGRATION.md route B, bench.py's e2e): H2D, the
step graph (whose x' and e' are read back while stage 2 still runs), D2H.  Its states must be
bit-identical to the device-resident step on the same inputs, step after step, and a failed
step must leave the caller's host arrays as they were."""

import ctypes as C

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _setup(n=4, p=3):
    from paper_2112_07075_b200 import problems
    from paper_2112_07075_b200.fespace import cartesian_mesh
    from paper_2112_07075_b200.hydro import LagrangeHydro, MaterialModel, ViscosityModel, box_velocity_bc
    from paper_2112_07075_b200.tensor_basis import gauss_legendre

    d = 3
    mesh = cartesian_mesh(d, (1.0,) * d, (n,) * d, p)
    hy = LagrangeHydro(mesh, gauss_legendre(p + 2), MaterialModel(1.4), ViscosityModel(0.5, 2.0),
                       bc_mask=box_velocity_bc(mesh))
    st = hy.initial_state(*problems.sedov(d, (1.0,) * d, (n,) * d))
    return hy, st


def _host_arena(st):
    nx, nv, ne = st.x.size, st.v.size, st.e.size
    arena = torch.empty(nx + nv + ne, dtype=torch.float64).pin_memory()
    arena[:nx] = torch.from_numpy(st.x.reshape(-1))
    arena[nx:nx + nv] = torch.from_numpy(st.v.reshape(-1))
    arena[nx + nv:] = torch.from_numpy(st.e.reshape(-1))
    return arena, (nx, nv, ne)


def test_host_entry_matches_device_steps():
    from paper_2112_07075_b200 import _lib
    from paper_2112_07075_b200.hydro import StepControls

    hy, st = _setup()
    ctl = StepControls(cfl=0.02, dt_max=1.0, t_final=10.0)
    arena, (nx, nv, ne) = _host_arena(st)
    lib, h = hy._ctx.lib, hy._ctx.h
    prm = hy._params(ctl)
    info = _lib.StepInfo()
    dev = hy.to_device(st)
    t = st.t
    for _ in range(6):  # the first step runs plain launches, the rest the captured graph
        hy._ctx.sync_stream()
        rc = lib.hx_step_host(h, C.byref(prm), float(t), arena[:nx].data_ptr(), arena[nx:nx + nv].data_ptr(),
                              arena[nx + nv:].data_ptr(), C.byref(info))
        assert rc == 0
        t = info.t_new
        dev, dinfo = hy.step(dev, ctl)
        ref = hy.to_host(dev)
        assert np.array_equal(arena[:nx].numpy(), ref.x.reshape(-1))
        assert np.array_equal(arena[nx:nx + nv].numpy(), ref.v.reshape(-1))
        assert np.array_equal(arena[nx + nv:].numpy(), ref.e.reshape(-1))
        assert info.dt == dinfo["dt"]


def test_host_entry_failed_step_leaves_state():
    from paper_2112_07075_b200 import _lib
    from paper_2112_07075_b200.hydro import StepControls

    hy, st = _setup()
    ok = StepControls(cfl=0.02, dt_max=1.0, t_final=10.0)
    arena, (nx, nv, ne) = _host_arena(st)
    lib, h = hy._ctx.lib, hy._ctx.h
    info = _lib.StepInfo()
    t = st.t
    for _ in range(3):  # warm the graph path
        hy._ctx.sync_stream()
        assert lib.hx_step_host(h, C.byref(hy._params(ok)), float(t), arena[:nx].data_ptr(),
                                arena[nx:nx + nv].data_ptr(), arena[nx + nv:].data_ptr(), C.byref(info)) == 0
        t = info.t_new
    before = arena.clone()
    bad = StepControls(cfl=0.02, dt_max=1.0, t_final=10.0, dt_min=1.0)  # every dt underflows
    for _ in range(2):  # new parameters: plain launches, then the graph for them
        hy._ctx.sync_stream()
        rc = lib.hx_step_host(h, C.byref(hy._params(bad)), float(t), arena[:nx].data_ptr(),
                              arena[nx:nx + nv].data_ptr(), arena[nx + nv:].data_ptr(), C.byref(info))
        assert rc == _lib.HX_EUNDERFLOW
        assert torch.equal(arena, before)


@pytest.mark.parametrize("slabs,pinned", [("0", True), ("1", True), ("3", True), ("64", True), ("3", False)])
def test_streamed_inputs_match_device_steps(slabs, pinned, monkeypatch):
    """hx_step_host streams x, v, e in z-slabs while the stage-1 rates kernel runs (each pass
    waits for its slab's flag): every slab count, including one slab per element layer and the
    single up-front copy (0), gives states bit-identical to the device-resident step."""
    from paper_2112_07075_b200 import _lib
    from paper_2112_07075_b200.hydro import StepControls

    monkeypatch.setenv("HX_STREAM_IN", slabs)
    hy, st = _setup(n=7, p=3)
    ctl = StepControls(cfl=0.02, dt_max=1.0, t_final=10.0)
    arena, (nx, nv, ne) = _host_arena(st)
    if not pinned:  # pageable host memory (staged copies)
        arena = torch.from_numpy(arena.numpy().copy())
    lib, h = hy._ctx.lib, hy._ctx.h
    prm = hy._params(ctl)
    info = _lib.StepInfo()
    dev = hy.to_device(st)
    t = st.t
    for _ in range(4):
        hy._ctx.sync_stream()
        rc = lib.hx_step_host(h, C.byref(prm), float(t), arena[:nx].data_ptr(), arena[nx:nx + nv].data_ptr(),
                              arena[nx + nv:].data_ptr(), C.byref(info))
        assert rc == 0
        t = info.t_new
        dev, dinfo = hy.step(dev, ctl)
        ref = hy.to_host(dev)
        assert np.array_equal(arena[:nx].numpy(), ref.x.reshape(-1))
        assert np.array_equal(arena[nx:nx + nv].numpy(), ref.v.reshape(-1))
        assert np.array_equal(arena[nx + nv:].numpy(), ref.e.reshape(-1))
        assert info.dt == dinfo["dt"]
