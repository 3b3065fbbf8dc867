"""GPU parity: the sm_100a path through the C-ABI against golden vectors from the
real reference (tests/golden, made by make_golden.py) and the CPU oracle.

Tolerances: restriction (gather/scatter on identical inputs) bit-exact;
single operator applies 1e-13 relative (fp64, different summation order than
numpy/OpenBLAS); CG solutions 1e-10 with the same iteration count; N-step
states and energies 1e-10 relative (BASELINE.json north star), on configs whose
reference noise floor (1e-15 input perturbation) is below 1.2e-11.

Every norm-wise check is paired with a per-entry one (conftest.close): each entry within
100 tol of the reference relative to |b_i| + 1e-8 max|b| for single operator applies
(1e-6 max|b| for the D tables), and within 100 tol relative to |b_i| + 1e-2 max|b| for the
N-step states (every entry within 1e-10 max|b| absolute, entries above 1% of the maximum
within 1e-8 relative).  There the far-field velocities are many decades below the maximum;
measured on B200 (HX_ENTRY_LOG): up to 8e-12 max|v| absolute in the 3D Sedov runs, the
level of their reference noise floor (1.1e-11), which a norm-wise check alone would not
show.
"""

import numpy as np
import pytest

from conftest import close, golden, rel

pytestmark = pytest.mark.gpu

CASES = [(d, p) for d in (2, 3) for p in (1, 2, 3, 4)]


def _mesh_from(g, d, p):
    from paper_2112_07075_b200.fespace import HighOrderMesh

    return HighOrderMesh(d, p, g["dofmap"], g["coords"].copy())


@pytest.mark.parametrize("d,p", CASES)
def test_restriction_bitwise(d, p):
    from paper_2112_07075_b200.fespace import FiniteElementSpace

    g = golden(f"ops_{d}d_p{p}")
    mesh = _mesh_from(g, d, p)
    h1 = FiniteElementSpace(mesh, "H1")
    assert np.array_equal(h1.gather(g["gather_in"]), g["gather_out"])
    assert np.array_equal(h1.scatter_add(g["scatter_in"]), g["scatter_out"])
    assert np.array_equal(h1.scatter_add(g["scatter1_in"]), g["scatter1_out"])
    l2 = FiniteElementSpace(mesh, "L2", order=max(p - 1, 0))
    v = np.random.default_rng(1).normal(size=l2.ndof)
    e = l2.gather(v)
    assert np.array_equal(l2.scatter_add(e), v + 0.0)


@pytest.mark.parametrize("d,p", CASES)
def test_geometry(d, p):
    from paper_2112_07075_b200.fespace import compute_geometric_factors
    from paper_2112_07075_b200.tensor_basis import gauss_legendre

    g = golden(f"ops_{d}d_p{p}")
    geom = compute_geometric_factors(_mesh_from(g, d, p), gauss_legendre(p + 2))
    close(geom.jac, g["jac"], 1e-14, tag="geom.jac")
    close(geom.detj, g["detj"], 1e-14, tag="geom.detj")
    close(geom.jinv, g["jinv"], 1e-14, tag="geom.jinv")
    close(geom.wdetj, g["wdetj"], 1e-14, tag="geom.wdetj")
@pytest.mark.parametrize("brick", [True, False], ids=["brick", "csr"])
@pytest.mark.parametrize("d,p", CASES)
def test_mass_pa(d, p, brick, monkeypatch):
    """PA mass apply / diagonal / device CG; `csr` forces the generic (index-array) CG
    path on structured meshes, `brick` lets 3D p>=2 take the structured-brick kernels."""
    if not brick:
        monkeypatch.setenv("HX_BRICK", "0")
    from paper_2112_07075_b200.fespace import FiniteElementSpace, compute_geometric_factors
    from paper_2112_07075_b200.operators import MassPA, cg_solve
    from paper_2112_07075_b200.tensor_basis import gauss_legendre

    g = golden(f"ops_{d}d_p{p}")
    mesh = _mesh_from(g, d, p)
    geom = compute_geometric_factors(mesh, gauss_legendre(p + 2))
    m = MassPA(FiniteElementSpace(mesh, "H1"), geom, coeff=g["mass_coeff"])
    close(m.D, g["mass_D"], 1e-15, tag="m.D")
    close(m.apply(g["mass_u1"]), g["mass_y1"], 1e-13, tag="m.apply(g['mass_u1'])")
    close(m.apply(g["mass_u3"]), g["mass_y3"], 1e-13, tag="m.apply(g['mass_u3'])")
    close(m.diagonal(), g["mass_diag"], 1e-13, tag="m.diagonal()")
    x, it = cg_solve(m.apply, g["cg_b"], precond_diag=m.diagonal(), rel_tol=1e-8, max_iter=500)
    assert it == int(g["cg_iters"])
    close(x, g["cg_x"], 1e-10, tag="x")
@pytest.mark.parametrize("d,p", CASES)
def test_force_pa(d, p):
    from paper_2112_07075_b200.fespace import FiniteElementSpace, compute_geometric_factors
    from paper_2112_07075_b200.operators import ForcePA
    from paper_2112_07075_b200.tensor_basis import gauss_legendre

    g = golden(f"ops_{d}d_p{p}")
    mesh = _mesh_from(g, d, p)
    geom = compute_geometric_factors(mesh, gauss_legendre(p + 2))
    kin = FiniteElementSpace(mesh, "H1", vdim=d)
    thermo = FiniteElementSpace(mesh, "L2", order=max(p - 1, 0))
    f = ForcePA(kin, thermo, geom, g["force_sigma"])
    close(f.D, g["force_D"], 1e-14, floor=1e-6, tag="f.D")
    close(f.apply(g["force_e"]), g["force_Fe"], 1e-13, tag="f.apply(g['force_e'])")
    close(f.apply(np.ones(thermo.ndof)), g["force_F1"], 1e-13, tag="f.apply(np.ones(thermo.ndof))")
    close(f.apply_transpose(g["force_v"]), g["force_Ftv"], 1e-13, tag="f.apply_transpose(g['force_v'])")
    # adjointness (test_operators.py:195-203)
    e, v = g["force_e"], g["force_v"]
    assert np.vdot(f.apply(e), v) == pytest.approx(np.vdot(e, f.apply_transpose(v)), rel=1e-12)


def _hydro_from(g, d, p):
    from paper_2112_07075_b200.hydro import LagrangeHydro, MaterialModel, ViscosityModel
    from paper_2112_07075_b200.tensor_basis import gauss_legendre

    mesh = _mesh_from(g, d, p)
    return LagrangeHydro(mesh, gauss_legendre(p + 2), MaterialModel(1.4), ViscosityModel(0.5, 2.0),
                         bc_mask=g["bc_mask"])


@pytest.mark.parametrize("d,p", CASES)
def test_hydro_point_data_and_rates(d, p):
    from paper_2112_07075_b200.fespace import compute_geometric_factors
    from paper_2112_07075_b200.hydro import HydroState

    g = golden(f"ops_{d}d_p{p}")
    hy = _hydro_from(g, d, p)
    st = HydroState(g["st_x"], g["st_v"], g["st_e"], g["st_qdata0"], 0.0)
    hy.begin_phase(st)
    close(hy.mass_pa.D, g["mass_D_phase"], 1e-15, tag="hy.mass_pa.D")
    close(hy._mass_diag, g["mdiag"], 1e-13, tag="hy._mass_diag")
    close(hy._m_e_inv, g["minv"], 1e-11, tag="hy._m_e_inv")
    geom = compute_geometric_factors(hy.mesh, hy.quad, x=st.x)
    sig, ratio = hy.stress_qdata(st, geom)
    close(sig, g["stress_sigma"], 1e-13, tag="sig")
    assert ratio == pytest.approx(float(g["stress_ratio"]), rel=1e-13)
    assert hy.clamp_warnings == int(g["stress_clamps"])
    r = hy.rates(st)
    close(r.dv, g["rates_dv"], 1e-10, tag="r.dv")
    close(r.de, g["rates_de"], 1e-11, tag="r.de")
    assert r.min_h_over_speed == pytest.approx(float(g["rates_ratio"]), rel=1e-13)
    assert r.clamped == int(g["rates_clamped"])
    close(hy.solve_energy(g["esolve_rhs"]), g["esolve_out"], 1e-11, tag="hy.solve_energy(g['esolve_rhs'])")
    assert hy.kinetic_energy(st) == pytest.approx(float(g["ke"]), rel=1e-12)
    assert hy.internal_energy(st) == pytest.approx(float(g["ie"]), rel=1e-13)
    assert hy.total_mass(st) == pytest.approx(float(g["mass_total"]), rel=1e-15)
    new, info = hy.rk2_step(st, 1e-3)
    assert info["dt"] == 1e-3
    close(new.x, g["step_x"], 1e-12, tag="new.x")
    close(new.v, g["step_v"], 1e-10, tag="new.v")
    close(new.e, g["step_e"], 1e-11, tag="new.e")
RUNS = ["sedov2d_q2", "sedov3d_q3", "sedov3d_q2", "triple3d_q3", "tgv3d_q4"]


def _problem(z):
    from paper_2112_07075_b200 import problems

    d = int(z["dim"])
    prob = str(z["problem"])
    if prob == "sedov":
        return problems.sedov(d, tuple(z["extents"]), tuple(int(c) for c in z["counts"]))
    if prob == "tgv":
        return problems.taylor_green(d, float(z["gamma"]))
    return problems.triple_point(d, float(z["gamma"]))


@pytest.mark.parametrize("brick", [True, False], ids=["brick", "csr"])
@pytest.mark.parametrize("name", RUNS)
@pytest.mark.parametrize("fused", [False, True])
def test_nstep_run_matches_reference(name, fused, brick, monkeypatch):
    """N Lagrange steps (timestep_estimate + rk2_step) vs the reference's final state."""
    if not brick:
        monkeypatch.setenv("HX_BRICK", "0")
    from paper_2112_07075_b200.fespace import cartesian_mesh
    from paper_2112_07075_b200.hydro import (LagrangeHydro, MaterialModel, StepControls, ViscosityModel,
                                             box_velocity_bc)
    from paper_2112_07075_b200.tensor_basis import gauss_legendre

    z = golden("run_" + name)
    d, p = int(z["dim"]), int(z["p"])
    assert float(z["noise_floor"]) < 1.2e-11
    mesh = cartesian_mesh(d, tuple(z["extents"]), tuple(int(c) for c in z["counts"]), p)
    hy = LagrangeHydro(mesh, gauss_legendre(p + 2), MaterialModel(float(z["gamma"])),
                       ViscosityModel(float(z["q1"]), float(z["q2"])), bc_mask=box_velocity_bc(mesh))
    assert hy._ctx.layout() == ("brick" if (brick and d == 3 and p >= 2) else "csr")
    rho0, v0, e0 = _problem(z)
    st = hy.initial_state(rho0, v0, e0)
    ctl = StepControls(cfl=float(z["cfl"]), dt_max=1.0, t_final=10.0)
    energies = [hy.total_energy(st)]
    dts = []
    if fused:
        st = hy.to_device(st)
    for _ in range(int(z["nsteps"])):
        if fused:
            st, info = hy.step(st, ctl)
        else:
            dt = hy.timestep_estimate(st, ctl)
            st, info = hy.rk2_step(st, dt)
        dts.append(info["dt"])
        energies.append(hy.total_energy(st))
    st = hy.to_host(st)
    tol = 1e-10
    close(st.x, z["x"], tol, floor=1e-2, entry_tol=100 * tol, tag="st.x")
    close(st.v, z["v"], tol, floor=1e-2, entry_tol=100 * tol, tag="st.v")
    close(st.e, z["e"], tol, floor=1e-2, entry_tol=100 * tol, tag="st.e")
    close(dts, z["dts"], tol, floor=1e-2, entry_tol=100 * tol, tag="dts")
    assert abs(energies[-1] - float(z["energies"][-1])) <= tol * abs(float(z["energies"][-1]))
    assert st.t == pytest.approx(float(z["t"]), rel=1e-12)
    assert hy.clamp_warnings == int(z["clamps"])


@pytest.mark.parametrize("d,p", CASES)
def test_remap_operators(d, p):
    """DiffusionPA / ConvectionPA (operators.py:143-236) vs the reference's fixtures."""
    from paper_2112_07075_b200.fespace import FiniteElementSpace, compute_geometric_factors
    from paper_2112_07075_b200.operators import ConvectionPA, DiffusionPA
    from paper_2112_07075_b200.tensor_basis import gauss_legendre

    g = golden(f"remap_{d}d_p{p}")
    mesh = _mesh_from(g, d, p)
    geom = compute_geometric_factors(mesh, gauss_legendre(p + 2))
    h1 = FiniteElementSpace(mesh, "H1")
    dif = DiffusionPA(h1, geom, nu=g["nu"])
    close(dif.D, g["diff_D"], 1e-14, floor=1e-6, tag="dif.D")
    assert dif.stored_values == g["diff_D"].size
    close(dif.apply(g["diff_x"]), g["diff_y"], 1e-13, tag="dif.apply(g['diff_x'])")
    dif1 = DiffusionPA(h1, geom)
    close(dif1.D, g["diff1_D"], 1e-14, floor=1e-6, tag="dif1.D")
    close(dif1.apply(g["diff_x"]), g["diff1_y"], 1e-13, tag="dif1.apply(g['diff_x'])")
    con = ConvectionPA(h1, geom, g["conv_u"])
    close(con.D, g["conv_D"], 1e-14, floor=1e-6, tag="con.D")
    close(con.apply(g["diff_x"]), g["conv_y"], 1e-13, tag="con.apply(g['diff_x'])")
    with pytest.raises(ValueError):
        dif.apply(np.zeros(h1.ndof + 1))


@pytest.mark.parametrize("fused", [False, True])
def test_multimaterial_triple_point_matches_oracle(fused):
    """Multi-material extension (per-element gamma, hx_set_material): the Laghos triple point
    with gamma = (1.5, 1.4, 1.5) by region, 6 steps at CFL 0.02, against the oracle with the
    same per-element gamma (noise floor 1.1e-15).  The reference has one gamma per run, so this
    parity is against the oracle restatement only."""
    from oracle import pa_oracle as O
    from paper_2112_07075_b200 import problems
    from paper_2112_07075_b200.fespace import cartesian_mesh
    from paper_2112_07075_b200.hydro import (LagrangeHydro, MaterialModel, StepControls, ViscosityModel,
                                             box_velocity_bc)
    from paper_2112_07075_b200.tensor_basis import gauss_legendre

    d, p, counts, ext = 3, 3, (7, 6, 1), (7.0, 3.0, 1.5)
    r0, v0, e0, ge = problems.triple_point_multi(d, counts, ext)
    assert set(np.unique(ge)) == {1.4, 1.5}
    mesh = cartesian_mesh(d, ext, counts, p)
    hy = LagrangeHydro(mesh, gauss_legendre(p + 2), MaterialModel(ge), ViscosityModel(0.5, 2.0),
                       bc_mask=box_velocity_bc(mesh))
    st = hy.initial_state(r0, v0, e0)
    ctl = StepControls(cfl=0.02, dt_max=1.0, t_final=10.0)
    oh = O.Hydro(d, p, mesh.node_dofmap, mesh.coords, ge, 0.5, 2.0, bc_mask=O.box_mask(mesh.coords))
    ost = oh.initial_state(r0, v0, e0)
    close(st.e, ost["e"], 1e-15, tag="st.e")
    if fused:
        st = hy.to_device(st)
    for _ in range(6):
        if fused:
            st, info = hy.step(st, ctl)
        else:
            dt = hy.timestep_estimate(st, ctl)
            st, info = hy.rk2_step(st, dt)
        odt = oh.timestep_estimate(ost, 0.02, dt_max=1.0, t_final=10.0)
        ost, _ = oh.rk2_step(ost, odt)
        assert abs(info["dt"] - odt) <= 1e-12 * odt
    st = hy.to_host(st)
    for k in ("x", "v", "e"):
        close(getattr(st, k), ost[k], 1e-10, floor=1e-3, entry_tol=1e-9, tag=k)
    # the single-gamma run differs: the per-element gamma is really used
    hy1 = LagrangeHydro(mesh, gauss_legendre(p + 2), MaterialModel(1.5), ViscosityModel(0.5, 2.0),
                        bc_mask=box_velocity_bc(mesh))
    s1 = hy1.initial_state(r0, v0, e0)
    s1, _ = hy1.rk2_step(s1, hy1.timestep_estimate(s1, ctl))
    o1 = O.Hydro(d, p, mesh.node_dofmap, mesh.coords, ge, 0.5, 2.0, bc_mask=O.box_mask(mesh.coords))
    so = o1.initial_state(r0, v0, e0)
    so, _ = o1.rk2_step(so, o1.timestep_estimate(so, 0.02, dt_max=1.0, t_final=10.0))
    assert rel(s1.v, so["v"]) > 1e-6
