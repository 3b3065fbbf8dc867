"""Known-answer properties of the reference test-suite, checked on the B200
path: the same physical/algebraic statements and tolerances as the reference's
test_hydro.py, test_operators.py and test_fespace.py, written against this package's
drop-in API (every operator below runs in libb200hydro.so).  Where the reference test is
2D only, a 3D case is added (the 3D kernels are the hot path)."""

import numpy as np
import pytest

from conftest import rel

pytestmark = pytest.mark.gpu

GAMMA = 1.4


def _hydro(dim=2, counts=(4, 4), order=2, q1=0.5, q2=2.0, extents=None, tol=1e-14, gamma=GAMMA):
    from paper_2112_07075_b200.fespace import cartesian_mesh
    from paper_2112_07075_b200.hydro import LagrangeHydro, MaterialModel, ViscosityModel, box_velocity_bc
    from paper_2112_07075_b200.tensor_basis import gauss_legendre

    extents = (1.0,) * dim if extents is None else extents
    mesh = cartesian_mesh(dim, extents, counts, order)
    return LagrangeHydro(mesh, gauss_legendre(order + 2), MaterialModel(gamma), ViscosityModel(q1, q2),
                         bc_mask=box_velocity_bc(mesh), momentum_rel_tol=tol)


def _uniform(hy, rho=1.0, e=1.0, vfn=None):
    return hy.initial_state(lambda xq: np.full(xq.shape[1:], rho),
                            (lambda x: np.zeros_like(x)) if vfn is None else vfn,
                            lambda pts: np.full(pts.shape[1:], e))


def _vortex(dim):
    def v(x):
        s = np.pi * x
        out = np.zeros_like(x)
        out[:, 0] = 0.1 * np.sin(s[:, 0]) * np.cos(s[:, 1])
        out[:, 1] = -0.1 * np.cos(s[:, 0]) * np.sin(s[:, 1])
        return out
    return v


DIMS = [(2, (4, 4)), (3, (3, 3, 2))]


# ---- hydro (test_hydro.py) ------------------------------------------------------------


@pytest.mark.parametrize("dim,counts", DIMS)
def test_uniform_pressure_sealed_box_is_in_equilibrium(dim, counts):
    hy = _hydro(dim, counts, order=3)
    r = hy.rates(_uniform(hy, rho=1.0, e=2.0))
    assert np.abs(np.asarray(r.dv)).max() < 1e-10
    assert np.abs(np.asarray(r.de)).max() < 1e-12


@pytest.mark.parametrize("dim,counts", DIMS)
def test_zero_stress_zero_acceleration(dim, counts):
    hy = _hydro(dim, counts)
    r = hy.rates(_uniform(hy, e=0.0))
    assert np.abs(np.asarray(r.dv)).max() < 1e-14


def test_sod_jump_accelerates_toward_low_pressure():
    hy = _hydro(2, (8, 2), extents=(1.0, 0.25), q1=0.0, q2=0.0)

    def e0(pts):
        left = pts[0] < 0.5
        return np.where(left, 1.0, 0.1) / ((GAMMA - 1.0) * np.where(left, 1.0, 0.125))

    st = hy.initial_state(lambda xq: np.where(xq[0] < 0.5, 1.0, 0.125), lambda x: np.zeros_like(x), e0)
    r = hy.rates(st)
    near = np.abs(hy.mesh.coords[:, 0] - 0.5) < 0.13
    dv = np.asarray(r.dv)
    assert dv[near, 0].mean() > 0.0 and np.abs(dv[near, 0]).max() > 1e-2


@pytest.mark.parametrize("dim,counts", DIMS)
def test_energy_rhs_zero_velocity(dim, counts):
    hy = _hydro(dim, counts)
    r = hy.rates(_uniform(hy, e=1.0))
    assert np.abs(np.asarray(r.de)).max() < 1e-13


@pytest.mark.parametrize("dim,counts", DIMS)
def test_energy_rhs_linear_in_velocity(dim, counts):
    from paper_2112_07075_b200.fespace import compute_geometric_factors
    from paper_2112_07075_b200.operators import ForcePA

    hy = _hydro(dim, counts)

    def vfn(x):
        out = np.zeros_like(x)
        out[:, 0], out[:, 1] = 0.05 * x[:, 1], -0.05 * x[:, 0]
        return out

    st = _uniform(hy, vfn=vfn)
    geom = compute_geometric_factors(hy.mesh, hy.quad, x=st.x)
    sigma, _ = hy.stress_qdata(st, geom)
    f = ForcePA(hy.kin, hy.thermo, geom, sigma)
    de1 = np.asarray(hy.solve_energy(f.apply_transpose(st.v)))
    de2 = np.asarray(hy.solve_energy(f.apply_transpose(2.0 * st.v)))
    assert np.allclose(de2, 2.0 * de1, rtol=1e-12)


@pytest.mark.parametrize("dim,counts", [(2, (6, 6)), (3, (3, 3, 3))])
def test_semi_discrete_energy_balance_per_stage(dim, counts):
    """d/dt (v'Mv/2 + 1'M_E e) = -(F1).v + v.(F1) = 0 at every stage (force pairing)."""
    from paper_2112_07075_b200.fespace import compute_geometric_factors
    from paper_2112_07075_b200.operators import ForcePA

    # 3D runs inviscid: the vortex is divergence-free, so the viscosity switch (div v < 0,
    # hydro.py:301) acts on rounding noise, and the fused rates kernel and the separate
    # stress_qdata path evaluate div v with different (equally valid) roundings
    hy = _hydro(dim, counts, q1=0.5 if dim == 2 else 0.0, q2=2.0 if dim == 2 else 0.0)
    st = hy.initial_state(lambda xq: 1.0 + 0.1 * xq[0], _vortex(dim), lambda pts: 1.0 + 0.2 * pts[1])
    r = hy.rates(st, momentum_rel_tol=1e-15)
    dke = float(np.vdot(st.v, np.asarray(hy.mass_pa.apply(r.dv))))
    geom = compute_geometric_factors(hy.mesh, hy.quad, x=st.x)
    sigma, _ = hy.stress_qdata(st, geom)
    f = ForcePA(hy.kin, hy.thermo, geom, sigma)
    die = float(np.sum(np.asarray(f.apply_transpose(st.v))))
    assert abs(dke + die) <= 1e-12 * hy.total_energy(st)


def test_timestep_uniform_sound_speed():
    from paper_2112_07075_b200.hydro import StepControls

    hy = _hydro(2, (4, 4), order=1)
    dt = hy.timestep_estimate(_uniform(hy, 1.0, 1.0), StepControls(cfl=0.4, dt_max=10.0, t_final=10.0))
    assert dt == pytest.approx(0.4 * (0.25 / 2.0) / np.sqrt(GAMMA * (GAMMA - 1.0)), rel=1e-12)


@pytest.mark.parametrize("dim,c1,c2", [(2, (4, 4), (8, 8)), (3, (2, 2, 2), (4, 4, 4))])
def test_timestep_halves_with_resolution(dim, c1, c2):
    from paper_2112_07075_b200.hydro import StepControls

    ctl = StepControls(cfl=0.5, dt_max=10.0, t_final=10.0)
    a, b = _hydro(dim, c1), _hydro(dim, c2)
    assert b.timestep_estimate(_uniform(b), ctl) == pytest.approx(a.timestep_estimate(_uniform(a), ctl) / 2,
                                                                  rel=1e-12)


def test_timestep_underflow_aborts_and_invalid_controls():
    from paper_2112_07075_b200.hydro import MaterialModel, StepControls, TimestepUnderflow, ViscosityModel

    hy = _hydro()
    with pytest.raises(TimestepUnderflow):
        hy.timestep_estimate(_uniform(hy), StepControls(cfl=0.5, dt_min=1e3, dt_max=1e4, t_final=1e5))
    with pytest.raises(ValueError):
        StepControls(cfl=0.0)
    with pytest.raises(ValueError):
        StepControls(dt_min=1.0, dt_max=0.5)
    with pytest.raises(ValueError):
        MaterialModel(1.0)
    with pytest.raises(ValueError):
        ViscosityModel(-0.1, 0.0)


@pytest.mark.parametrize("dim,counts", DIMS)
def test_rk2_static_state_unchanged(dim, counts):
    hy = _hydro(dim, counts)
    st = _uniform(hy, 1.0, 1.0)
    new, _ = hy.rk2_step(st, 1e-3)
    assert np.allclose(new.x, st.x, atol=1e-15)
    assert np.allclose(new.v, st.v, atol=1e-13)
    assert np.allclose(new.e, st.e, atol=1e-14)


@pytest.mark.parametrize("dim,counts", DIMS)
@pytest.mark.parametrize("fused", [False, True])
def test_rk2_mass_bitwise_constant(dim, counts, fused):
    hy = _hydro(dim, counts)
    st = _uniform(hy, vfn=_vortex(dim))
    m0 = hy.total_mass(st)
    if fused:
        from paper_2112_07075_b200.hydro import StepControls

        d = hy.to_device(st)
        for _ in range(5):
            d, _ = hy.step(d, StepControls(cfl=0.1, dt_max=2e-3, t_final=10.0))
        st = hy.to_host(d)
    else:
        for _ in range(5):
            st, _ = hy.rk2_step(st, 2e-3)
    assert hy.total_mass(st) == m0


@pytest.mark.parametrize("dim,counts", [(2, (4, 4)), (3, (3, 3, 3))])
@pytest.mark.parametrize("graph", [False, True])
def test_rk2_rejects_and_halves_on_inversion(dim, counts, graph):
    """A velocity that inverts elements in one step: the step is rejected and retried with
    dt/2 until the new geometry is valid (hydro.py:375-405).  `graph`: the context is warmed
    first, so the step runs as the captured CUDA graph whose failed validity check hands over
    to the device retry driver."""
    from paper_2112_07075_b200.fespace import compute_geometric_factors

    hy = _hydro(dim, counts, q1=0.0, q2=0.0)
    st = _uniform(hy, e=0.0, vfn=lambda x: -10.0 * (x - 0.5))
    st.v = -10.0 * (st.x - 0.5)  # ignore the wall mask for this stress test
    if graph:
        hy.rk2_step(st, 1e-6)  # first step of a context runs plain launches
    new, info = hy.rk2_step(st, 0.2)
    assert info["dt"] < 0.2
    compute_geometric_factors(hy.mesh, hy.quad, x=new.x)  # valid geometry


# ---- operators (test_operators.py) --------------------------------------------------


def _perturbed(dim, counts, p, seed, amount=0.15):
    from paper_2112_07075_b200.fespace import cartesian_mesh

    mesh = cartesian_mesh(dim, (1.0,) * dim, counts, p)
    rng = np.random.default_rng(seed)
    inner = np.setdiff1d(np.arange(mesh.num_nodes), mesh.boundary_nodes())
    mesh.coords[inner] += amount / (max(counts) * p) * rng.uniform(-1, 1, size=(len(inner), dim))
    return mesh


OPS = [(2, (3, 2), 2), (3, (2, 2, 2), 3)]


@pytest.mark.parametrize("dim,counts,p", OPS)
def test_mass_symmetry_positivity_linearity(dim, counts, p):
    from paper_2112_07075_b200.fespace import FiniteElementSpace, compute_geometric_factors
    from paper_2112_07075_b200.operators import MassPA
    from paper_2112_07075_b200.tensor_basis import gauss_legendre

    mesh = _perturbed(dim, counts, p, 7)
    geom = compute_geometric_factors(mesh, gauss_legendre(p + 2))
    h1 = FiniteElementSpace(mesh, "H1")
    m = MassPA(h1, geom)
    assert m.stored_values == mesh.num_elements * (p + 2) ** dim
    rng = np.random.default_rng(3)
    u, w = rng.normal(size=h1.ndof), rng.normal(size=h1.ndof)
    mu, mw = np.asarray(m.apply(u)), np.asarray(m.apply(w))
    assert abs(np.dot(w, mu) - np.dot(u, mw)) <= 1e-12 * abs(np.dot(u, mu))
    assert np.dot(u, mu) > 0.0
    assert np.abs(np.asarray(m.apply(np.zeros(h1.ndof)))).max() == 0.0
    m2 = MassPA(h1, geom, coeff=2.0 * np.ones_like(np.asarray(geom.wdetj)))
    assert rel(m2.apply(u), 2.0 * mu) < 1e-14
    # total mass: 1' M 1 = sum of w detJ
    assert np.sum(np.asarray(m.apply(np.ones(h1.ndof)))) == pytest.approx(float(np.sum(np.asarray(geom.wdetj))),
                                                                          rel=1e-13)


@pytest.mark.parametrize("dim,counts,p", OPS)
def test_force_adjoint_and_uniform_pressure(dim, counts, p):
    from paper_2112_07075_b200.fespace import FiniteElementSpace, compute_geometric_factors
    from paper_2112_07075_b200.operators import ForcePA
    from paper_2112_07075_b200.tensor_basis import gauss_legendre

    mesh = _perturbed(dim, counts, p, 11)
    geom = compute_geometric_factors(mesh, gauss_legendre(p + 2))
    kin = FiniteElementSpace(mesh, "H1", vdim=dim)
    th = FiniteElementSpace(mesh, "L2", order=p - 1)
    rng = np.random.default_rng(5)
    nq = (p + 2) ** dim
    sig = rng.normal(size=(dim, dim, nq, mesh.num_elements))
    f = ForcePA(kin, th, geom, sig)
    e, v = rng.normal(size=th.ndof), rng.normal(size=(kin.ndof, dim))
    lhs = float(np.sum(np.asarray(f.apply(e)) * v))
    rhs = float(np.dot(np.asarray(f.apply_transpose(v)), e))
    assert abs(lhs - rhs) <= 1e-12 * max(abs(lhs), 1.0)
    # uniform pressure self-equilibrates: the total force sums to zero componentwise
    # (the reference's statement; interior nodes do not vanish individually in 3D, where the
    # reference's _det_inv returns J^-T -- reproduced here, fespace.py:280-302)
    sp = np.zeros_like(sig)
    for a in range(dim):
        sp[a, a] = -3.0
    f1 = np.asarray(ForcePA(kin, th, geom, sp).apply(np.ones(th.ndof)))
    assert np.abs(f1.sum(axis=0)).max() < 1e-11 * max(np.abs(f1).sum(), 1.0)
    assert np.abs(np.asarray(ForcePA(kin, th, geom, np.zeros_like(sig)).apply(e))).max() == 0.0


@pytest.mark.parametrize("dim,counts,p", OPS)
def test_cg_properties(dim, counts, p):
    from paper_2112_07075_b200.fespace import FiniteElementSpace, compute_geometric_factors
    from paper_2112_07075_b200.operators import CGError, MassPA, cg_solve
    from paper_2112_07075_b200.tensor_basis import gauss_legendre

    mesh = _perturbed(dim, counts, p, 13)
    geom = compute_geometric_factors(mesh, gauss_legendre(p + 2))
    h1 = FiniteElementSpace(mesh, "H1")
    m = MassPA(h1, geom)
    x, it = cg_solve(m.apply, np.zeros(h1.ndof), precond_diag=m.diagonal())
    assert it == 0 and np.abs(np.asarray(x)).max() == 0.0
    b = np.random.default_rng(1).normal(size=h1.ndof)
    x, it = cg_solve(m.apply, b, precond_diag=m.diagonal(), rel_tol=1e-12, max_iter=500)
    assert rel(m.apply(x), b) < 1e-10 and it > 0
    with pytest.raises(CGError) as err:
        cg_solve(m.apply, b, precond_diag=m.diagonal(), rel_tol=1e-14, max_iter=2)
    assert len(err.value.residuals) == 3


@pytest.mark.parametrize("dim,counts,p", OPS)
def test_diffusion_nullspace_convection_constants(dim, counts, p):
    from paper_2112_07075_b200.fespace import FiniteElementSpace, compute_geometric_factors
    from paper_2112_07075_b200.operators import ConvectionPA, DiffusionPA
    from paper_2112_07075_b200.tensor_basis import gauss_legendre

    mesh = _perturbed(dim, counts, p, 17)
    geom = compute_geometric_factors(mesh, gauss_legendre(p + 2))
    h1 = FiniteElementSpace(mesh, "H1")
    one = np.ones(h1.ndof)
    k = DiffusionPA(h1, geom)
    assert np.abs(np.asarray(k.apply(one))).max() < 1e-12
    rng = np.random.default_rng(2)
    u, w = rng.normal(size=h1.ndof), rng.normal(size=h1.ndof)
    assert abs(np.dot(w, np.asarray(k.apply(u))) - np.dot(u, np.asarray(k.apply(w)))) < 1e-11
    nq = (p + 2) ** dim
    c = ConvectionPA(h1, geom, rng.normal(size=(dim, nq, mesh.num_elements)))
    assert np.abs(np.asarray(c.apply(one))).max() < 1e-12
    c0 = ConvectionPA(h1, geom, np.zeros((dim, nq, mesh.num_elements)))
    assert np.abs(np.asarray(c0.apply(u))).max() == 0.0


# ---- fespace (test_fespace.py) -------------------------------------------------------


@pytest.mark.parametrize("dim,counts,p", [(2, (3, 2), 2), (3, (2, 3, 2), 2), (3, (2, 2, 2), 3)])
def test_gather_scatter_adjoint_and_multiplicity(dim, counts, p):
    from paper_2112_07075_b200.fespace import FiniteElementSpace, cartesian_mesh

    h1 = FiniteElementSpace(cartesian_mesh(dim, (1.0,) * dim, counts, p), "H1")
    rng = np.random.default_rng(4)
    L = rng.normal(size=h1.ndof)
    E = rng.normal(size=(h1.nloc, h1.mesh.num_elements))
    assert abs(np.sum(np.asarray(h1.gather(L)) * E) - np.dot(L, np.asarray(h1.scatter_add(E)))) < 1e-11
    mult = np.asarray(h1.scatter_add(np.ones((h1.nloc, h1.mesh.num_elements))))
    assert mult.min() == 1.0 and mult.max() == 2.0**dim


@pytest.mark.parametrize("dim", [2, 3])
def test_inverted_element_reported(dim):
    from paper_2112_07075_b200.fespace import InvertedElementError, cartesian_mesh, compute_geometric_factors
    from paper_2112_07075_b200.tensor_basis import gauss_legendre

    mesh = cartesian_mesh(dim, (1.0,) * dim, (2,) * dim, 1)
    x = mesh.coords.copy()
    far = int(np.argmax(x.sum(axis=1)))  # the (1, 1[, 1]) corner, only in the last element
    x[far] = -1.0
    with pytest.raises(InvertedElementError) as err:
        compute_geometric_factors(mesh, gauss_legendre(3), x=x)
    assert err.value.element == mesh.num_elements - 1
    assert "<= 0" in str(err.value)


@pytest.mark.parametrize("order", [2, 3])
def test_timestep_estimate_reports_first_inverted_point(order):
    """timestep_estimate on an inverted mesh raises InvertedElementError naming the same first
    (q-major) point as compute_geometric_factors (hydro.py:364-367 -> fespace.py:340-344), and
    otherwise returns the ratio the reference pair (geometry + stress_qdata) gives -- the fused
    3D ratio launch (hx_timestep_ratio) against the device geometry + stress kernels."""
    from paper_2112_07075_b200.fespace import InvertedElementError, compute_geometric_factors
    from paper_2112_07075_b200.hydro import StepControls

    hy = _hydro(3, (3, 3, 2), order=order)
    st = _uniform(hy, e=1.0, vfn=_vortex(3))
    hy.begin_phase(st)
    ctl = StepControls(cfl=0.3, dt_max=1.0, t_final=10.0)
    dt = hy.timestep_estimate(st, ctl)
    _, ratio = hy.stress_qdata(st, compute_geometric_factors(hy.mesh, hy.quad, x=st.x))
    ref_dt = min(ctl.cfl * ratio, ctl.dt_max, ctl.t_final - st.t)
    assert abs(dt - ref_dt) <= 1e-14 * ref_dt  # (cbrt vs the stress kernel's h: an ulp at most)
    bad = st.x.copy()
    dm = hy.mesh.node_dofmap
    e0 = 7
    bad[dm[-1, e0]] = bad[dm[0, e0]] - 0.01  # fold the element's last corner past its first
    with pytest.raises(InvertedElementError) as ref:
        compute_geometric_factors(hy.mesh, hy.quad, x=bad)
    st.x = bad
    with pytest.raises(InvertedElementError) as got:
        hy.timestep_estimate(st, ctl)
    assert (got.value.element, got.value.point) == (ref.value.element, ref.value.point)
