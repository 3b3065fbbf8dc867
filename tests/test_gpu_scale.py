"""GPU parity at production size: the multi-pass paths of the persistent kernels.

k_mass_brick walks more than one pass per CTA only when NE > 7,400 and k_rates_pc runs
296 CTAs x 2 elements per pass, so the golden fixtures (<= 256 elements) never leave the
first pass.  These tests cover those paths three ways:
  * one rates() and one fused step() on a 21^3 Q3 brick (NE = 9,261) of a deformed mesh
    with a nontrivial state, against the CPU oracle computed here on the host;
  * the existing small-fixture parity tests re-run with HX_GRID_CAP=2 and 3, which caps
    every persistent grid so that each CTA takes several passes;
  * the bench workload itself (23^3 Sedov Q3-Q2, CFL 0.05) against the REAL reference's
    run of it (tests/golden/scale_sedov23_q3.npz, make_golden_scale.py): the 20-step
    window bench.py times, and the horizon (TimestepUnderflow at step 42).
Per-entry checks use conftest.entry_err: |a - b| <= 1e-10 (|b| + 1e-4 max|b|).
"""

import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT, entry_err, golden, rel

pytestmark = pytest.mark.gpu


def _deformed_case(n, p=3, layout="brick"):
    """A 3D Q{p} brick with curved interior nodes, smooth velocity, and an energy field
    that is negative at some points (the clamp path), plus the oracle on the same arrays."""
    from oracle import pa_oracle as O
    from paper_2112_07075_b200.fespace import HighOrderMesh, cartesian_mesh
    from paper_2112_07075_b200.hydro import LagrangeHydro, MaterialModel, ViscosityModel, box_velocity_bc
    from paper_2112_07075_b200.tensor_basis import gauss_legendre

    d = 3
    base = cartesian_mesh(d, (1.0,) * d, (n,) * d, p)
    mask = box_velocity_bc(base)
    X = base.coords.copy()
    h = 1.0 / (n * p)
    interior = np.all((X > 1e-12) & (X < 1 - 1e-12), axis=1)
    bump = np.sin(np.pi * X[:, [1, 2, 0]]) * np.sin(2 * np.pi * X[:, [2, 0, 1]])
    X[interior] += 0.2 * h * bump[interior]
    mesh = HighOrderMesh(d, p, base.node_dofmap, X)

    def rho0(xq):
        return 1.0 + 0.3 * np.sin(2 * np.pi * xq[0]) * np.cos(np.pi * xq[1])

    def v0(x):
        s = np.pi * x
        return np.stack([np.sin(s[:, 0]) * np.cos(s[:, 1]) * np.sin(2 * s[:, 2]),
                         -np.cos(s[:, 0]) * np.sin(s[:, 1]) * np.sin(s[:, 2]),
                         0.5 * np.sin(2 * s[:, 0]) * np.sin(s[:, 2])], axis=1)

    def e0(pts):
        return 0.2 + np.cos(3 * np.pi * pts[0]) * np.cos(2 * np.pi * pts[1]) * np.sin(np.pi * pts[2])

    hy = LagrangeHydro(mesh, gauss_legendre(p + 2), MaterialModel(1.4), ViscosityModel(0.5, 2.0), bc_mask=mask)
    assert hy._ctx.layout() == layout
    st = hy.initial_state(rho0, v0, e0)
    oh = O.Hydro(d, p, mesh.node_dofmap, mesh.coords, 1.4, 0.5, 2.0, bc_mask=mask)
    ost = dict(x=np.array(st.x), v=np.array(st.v), e=np.array(st.e), qdata0=np.array(st.qdata0), t=0.0)
    oh.begin_phase(ost)
    return hy, st, oh, ost


@pytest.mark.parametrize("layout", ["brick", "csr"])
def test_rates_production_size(layout, monkeypatch):
    if layout == "csr":
        monkeypatch.setenv("HX_BRICK", "0")
    hy, st, oh, ost = _deformed_case(21, layout=layout)
    assert hy.mesh.num_elements == 9261 > 7400
    r = hy.rates(hy.to_device(st))
    ro = oh.rates(ost)
    dv, de = r.dv.cpu().numpy(), r.de.cpu().numpy()
    assert ro["clamped"] > 0 and r.clamped == ro["clamped"]
    assert r.min_h_over_speed == pytest.approx(ro["ratio"], rel=1e-13)
    assert hy.last_cg_iterations == oh.last_cg_iters
    assert rel(dv, ro["dv"]) < 1e-10
    assert rel(de, ro["de"]) < 1e-11
    # per entry: |a - b| <= 1e-10 (|b| + 1e-4 max|b|)
    assert entry_err(dv, ro["dv"], floor=1e-4) < 1e-10
    assert entry_err(de, ro["de"], floor=1e-4) < 1e-10


def test_fused_step_production_size():
    from paper_2112_07075_b200.hydro import StepControls

    hy, st, oh, ost = _deformed_case(21)
    ctl = StepControls(cfl=0.1, dt_max=1.0, t_final=10.0)
    new, info = hy.step(hy.to_device(st), ctl)
    new = hy.to_host(new)
    dt = oh.timestep_estimate(ost, 0.1, dt_max=1.0, t_final=10.0)
    c0 = oh.clamps
    onew, _ = oh.rk2_step(ost, dt)
    assert info["dt"] == pytest.approx(dt, rel=1e-13)
    for k in ("x", "v", "e"):
        a, b = getattr(new, k), onew[k]
        assert rel(a, b) < 1e-10, k
        assert entry_err(a, b, floor=1e-4) < 1e-10, k
    assert hy.clamp_warnings == oh.clamps  # timestep_estimate + both stages, as the reference counts
    assert oh.clamps > c0


@pytest.mark.parametrize("cap", [2, 3])
def test_small_fixtures_with_capped_grids(cap):
    """The golden-fixture parity tests with every persistent grid capped at `cap` CTAs, so
    every persistent kernel (mass, rates, node, validity, M_e^-1 setup) runs multi-pass."""
    env = dict(os.environ, HX_GRID_CAP=str(cap))
    sel = "test_mass_pa or test_hydro_point_data_and_rates or (test_nstep_run_matches_reference and sedov3d)"
    cmd = [sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
           os.path.join(ROOT, "tests", "test_gpu_parity.py"), "-k", sel]
    out = subprocess.run(cmd, env=env, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-2000:]
    assert " passed" in out.stdout and " failed" not in out.stdout


def test_bench_window_and_horizon_match_reference():
    """bench.py's workload (23^3 Sedov Q3-Q2, CFL 0.05) against the reference's own run:
    the 20-step window it times, then on to the reference's TimestepUnderflow."""
    from paper_2112_07075_b200 import problems
    from paper_2112_07075_b200.fespace import cartesian_mesh
    from paper_2112_07075_b200.hydro import (LagrangeHydro, MaterialModel, StepControls, TimestepUnderflow,
                                             ViscosityModel, box_velocity_bc)
    from paper_2112_07075_b200.tensor_basis import gauss_legendre

    z = golden("scale_sedov23_q3")
    zp = golden("scale_sedov23_q3_pert")
    n, p, d, W = int(z["n"]), int(z["p"]), 3, int(z["window"])
    mesh = cartesian_mesh(d, (1.0,) * d, (n,) * d, p)
    hy = LagrangeHydro(mesh, gauss_legendre(p + 2), MaterialModel(1.4), ViscosityModel(0.5, 2.0),
                       bc_mask=box_velocity_bc(mesh))
    st = hy.to_device(hy.initial_state(*problems.sedov(d, (1.0,) * d, (n,) * d)))
    ctl = StepControls(cfl=float(z["cfl"]), dt_max=1.0, t_final=1e9)
    dts, clamps, energies = [], [], [hy.total_energy(st)]
    for _ in range(W):
        c0 = hy.clamp_warnings
        st, info = hy.step(st, ctl)
        dts.append(info["dt"])
        clamps.append(hy.clamp_warnings - c0)
        energies.append(hy.total_energy(st))
    # the reference's own sensitivity to a 1e-15 perturbation of e0 over the window
    floor = max(rel(zp["dts"][:W], z["dts"][:W]), rel(zp["x_sub"], z["x_sub"]), rel(zp["v_sub"], z["v_sub"]),
                rel(zp["e_sub"], z["e_sub"]))
    tol = max(1e-10, 100 * floor)
    assert tol <= 1e-8
    assert rel(dts, z["dts"][:W]) < tol
    assert np.array_equal(np.array(clamps), z["clamps"][:W])
    assert rel(energies, z["energies"]) < tol
    h = hy.to_host(st)
    s = int(z["stride"])
    for k in ("x", "v", "e"):
        a = getattr(h, k).reshape(-1)
        assert rel(a[::s], z[k + "_sub"]) < tol, k
        assert np.linalg.norm(a) == pytest.approx(float(z[k + "_norm"]), rel=tol), k
    assert h.t == pytest.approx(float(z["t_window"]), rel=1e-12)
    # the horizon: dt collapses after step ~26 and the reference underflows at step 42
    step = W
    with pytest.raises(TimestepUnderflow) as exc:
        while step < 80:
            st, info = hy.step(st, ctl)
            step += 1
    assert abs((step + 1) - int(z["underflow_step"])) <= 1
    t_fail = float(str(exc.value).rsplit("t = ", 1)[1])
    assert t_fail == pytest.approx(float(z["underflow_t"]), rel=1e-5)
