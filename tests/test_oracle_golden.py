"""Pin the CPU oracle against golden vectors produced by the real reference.

CPU-only (`-m "not gpu"`).  The fixtures come from tests/golden/make_golden.py,
which imports /root/reference/pkg/src in the build container.
"""

import numpy as np
import pytest

from conftest import golden, rel
from oracle import pa_oracle as O


def test_basis_tables_bitwise():
    g = golden("basis")
    for p in range(1, 5):
        pts, w = O.gauss_legendre(p + 2)
        assert np.array_equal(pts, g[f"qpts_{p}"]) and np.array_equal(w, g[f"qw_{p}"])
        assert np.array_equal(O.gauss_lobatto(p), g[f"lob_{p}"])
        B, G = O.basis_tables(O.gauss_lobatto(p), pts)
        assert np.array_equal(B, g[f"B_{p}"]) and np.array_equal(G, g[f"G_{p}"])
        Bt, Gt = O.basis_tables(O.l2_nodes(p - 1), pts)
        assert np.array_equal(Bt, g[f"Bt_{p}"]) and np.array_equal(Gt, g[f"Gt_{p}"])
    for n in range(1, 9):
        pts, w = O.gauss_legendre(n)
        assert np.array_equal(pts, g[f"gl_pts_{n}"]) and np.array_equal(w, g[f"gl_w_{n}"])


def test_cartesian_restriction_indices_bitwise():
    g = golden("mesh")
    i = 0
    while f"dofmap_{i}" in g:
        case = g[f"case_{i}"]
        d, p = int(case[0]), int(case[1])
        counts = tuple(int(c) for c in case[2 : 2 + d])
        dofmap, coords = O.box_mesh(d, (1.0,) * d, counts, p)
        assert np.array_equal(dofmap, g[f"dofmap_{i}"])
        assert np.array_equal(coords, g[f"coords_{i}"])
        i += 1
    assert i >= 5


CASES = [(d, p) for d in (2, 3) for p in (1, 2, 3, 4)]


@pytest.mark.parametrize("d,p", CASES)
def test_operator_fixtures(d, p):
    g = golden(f"ops_{d}d_p{p}")
    dofmap, x = g["dofmap"], g["coords"]
    nn = x.shape[0]
    qpts, qw = O.gauss_legendre(p + 2)
    jac, det, jinv, wdetj = O.geometry(dofmap, x, p, qpts, qw, d)
    assert rel(jac, g["jac"]) < 1e-14 and rel(det, g["detj"]) < 1e-14
    assert rel(jinv, g["jinv"]) < 1e-14 and rel(wdetj, g["wdetj"]) < 1e-14
    # restriction: bit-exact
    assert np.array_equal(O.gather(dofmap, g["gather_in"]), g["gather_out"])
    assert np.array_equal(O.scatter_add(dofmap, g["scatter_in"], nn), g["scatter_out"])
    assert np.array_equal(O.scatter_add(dofmap, g["scatter1_in"], nn), g["scatter1_out"])
    # mass
    B, G = O.basis_tables(O.gauss_lobatto(p), qpts)
    D = wdetj * g["mass_coeff"]
    assert rel(D, g["mass_D"]) < 1e-15
    assert rel(O.mass_apply(dofmap, D, B, g["mass_u1"], d), g["mass_y1"]) < 1e-14
    assert rel(O.mass_apply(dofmap, D, B, g["mass_u3"], d), g["mass_y3"]) < 1e-14
    assert rel(O.mass_diag(dofmap, D, B, nn, d), g["mass_diag"]) < 1e-14
    # force
    Bt, _ = O.basis_tables(O.l2_nodes(p - 1), qpts)
    DF = O.force_D(g["force_sigma"], jinv, wdetj)
    assert rel(DF, g["force_D"]) < 1e-14
    assert rel(O.force_apply(dofmap, nn, DF, B, G, Bt, g["force_e"], d), g["force_Fe"]) < 1e-13
    assert rel(O.force_apply_t(dofmap, DF, B, G, Bt, g["force_v"], d), g["force_Ftv"]) < 1e-13
    # cg
    xs, it = O.cg(lambda u: O.mass_apply(dofmap, D, B, u, d), g["cg_b"],
                  O.mass_diag(dofmap, D, B, nn, d), 1e-8, 500)
    assert it == int(g["cg_iters"])
    assert rel(xs, g["cg_x"]) < 1e-12
    # hydro level
    hy = O.Hydro(d, p, dofmap, x, 1.4, 0.5, 2.0, bc_mask=g["bc_mask"])
    st = dict(x=g["st_x"], v=g["st_v"], e=g["st_e"], qdata0=g["st_qdata0"], t=0.0)
    hy.begin_phase(st)
    assert rel(hy.Dm, g["mass_D_phase"]) < 1e-15
    assert rel(hy.mdiag, g["mdiag"]) < 1e-14
    assert rel(hy.Minv, g["minv"]) < 1e-12
    sig, ratio = hy.stress(st, (jac, det, jinv, wdetj))
    assert rel(sig, g["stress_sigma"]) < 1e-13
    assert ratio == pytest.approx(float(g["stress_ratio"]), rel=1e-14)
    assert hy.clamps == int(g["stress_clamps"])
    r = hy.rates(st)
    assert rel(r["dv"], g["rates_dv"]) < 1e-12
    assert rel(r["de"], g["rates_de"]) < 1e-12
    assert r["ratio"] == pytest.approx(float(g["rates_ratio"]), rel=1e-14)
    assert rel(hy.solve_energy(g["esolve_rhs"]), g["esolve_out"]) < 1e-13
    assert hy.kinetic_energy(st) == pytest.approx(float(g["ke"]), rel=1e-13)
    assert hy.internal_energy(st) == pytest.approx(float(g["ie"]), rel=1e-13)
    assert hy.total_mass(st) == pytest.approx(float(g["mass_total"]), rel=1e-15)
    new, info = hy.rk2_step(st, 1e-3)
    assert rel(new["x"], g["step_x"]) < 1e-13
    assert rel(new["v"], g["step_v"]) < 1e-11
    assert rel(new["e"], g["step_e"]) < 1e-12


def problem_fns(z):
    d = int(z["dim"])
    prob = str(z["problem"])
    if prob == "sedov":
        return O.sedov_fns(d, tuple(z["extents"]), tuple(z["counts"]))
    if prob == "tgv":
        return O.taylor_green_fns(d, float(z["gamma"]))
    return O.triple_point_fns(d, float(z["gamma"]))


def run_oracle(z, nsteps=None):
    d, p = int(z["dim"]), int(z["p"])
    ext, counts = tuple(z["extents"]), tuple(int(c) for c in z["counts"])
    dofmap, coords = O.box_mesh(d, ext, counts, p)
    hy = O.Hydro(d, p, dofmap, coords, float(z["gamma"]), float(z["q1"]), float(z["q2"]),
                 bc_mask=O.box_mask(coords))
    rho0, v0, e0 = problem_fns(z)
    st = hy.initial_state(rho0, v0, e0)
    energies = [hy.total_energy(st)]
    dts = []
    for _ in range(int(z["nsteps"]) if nsteps is None else nsteps):
        dt = hy.timestep_estimate(st, float(z["cfl"]), dt_max=1.0, t_final=10.0)
        st, info = hy.rk2_step(st, dt)
        dts.append(info["dt"])
        energies.append(hy.total_energy(st))
    return hy, st, np.array(dts), np.array(energies)


@pytest.mark.parametrize("name", ["sedov2d_q2", "triple3d_q3", "tgv3d_q4"])
def test_oracle_runs_match_reference(name):
    z = golden("run_" + name)
    hy, st, dts, energies = run_oracle(z)
    tol = 1e-10
    assert rel(st["x"], z["x"]) < tol
    assert rel(st["v"], z["v"]) < tol
    assert rel(st["e"], z["e"]) < tol
    assert rel(dts, z["dts"]) < tol
    assert abs(energies[-1] - z["energies"][-1]) < tol * abs(z["energies"][-1])
    assert hy.clamps == int(z["clamps"])


@pytest.mark.parametrize("d,p", CASES)
def test_remap_operator_fixtures(d, p):
    """DiffusionPA / ConvectionPA (operators.py:143-236): oracle restatement vs the reference."""
    g = golden(f"remap_{d}d_p{p}")
    dofmap, x = g["dofmap"], g["coords"]
    qpts, qw = O.gauss_legendre(p + 2)
    _, _, jinv, wdetj = O.geometry(dofmap, x, p, qpts, qw, d)
    assert rel(jinv, g["jinv"]) < 1e-14 and rel(wdetj, g["wdetj"]) < 1e-14
    B, G = O.basis_tables(O.gauss_lobatto(p), qpts)
    D = O.diffusion_D(jinv, wdetj, g["nu"])
    assert rel(D, g["diff_D"]) < 1e-14
    assert rel(O.diffusion_apply(dofmap, D, B, G, g["diff_x"], d), g["diff_y"]) < 1e-13
    D1 = O.diffusion_D(jinv, wdetj)
    assert rel(D1, g["diff1_D"]) < 1e-14
    assert rel(O.diffusion_apply(dofmap, D1, B, G, g["diff_x"], d), g["diff1_y"]) < 1e-13
    Dc = O.convection_D(jinv, g["conv_u"], wdetj)
    assert rel(Dc, g["conv_D"]) < 1e-14
    assert rel(O.convection_apply(dofmap, Dc, B, G, g["diff_x"], d), g["conv_y"]) < 1e-13
