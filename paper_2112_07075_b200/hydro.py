"""Single-material Lagrangian hydrodynamics phase on the B200.

Drop-in for `ale_minihydro.hydro` (hydro.py:40-432).  Same classes, names,
constructor signatures, return types and array layouts; the work runs in
libb200hydro.so:

  rates            -> hx_rates: one fused sm_100a kernel per element (geometry,
                      EOS, artificial viscosity, CFL ratio, F.1, F^T v, M_e^{-1})
                      + the device Jacobi PCG with the wall mask
  timestep_estimate-> hx_stress (fused geometry + stress kernel, ratio reduced on device)
  rk2_step         -> hx_rk2_step (midpoint RK2 with the reject-and-halve retries)
  step             -> hx_step: timestep_estimate + rk2_step with one host sync,
                      stage-1 rates reused for the CFL estimate (identical values)

Initial-condition sampling (`quad_points_physical`, `_sample_l2`) evaluates the
user's Python callables, so it stays on the host, as in the reference; it is
phase setup, not the time-step path.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._device import DeviceContext, empty, is_torch, like, to_dev
from .fespace import FiniteElementSpace, HighOrderMesh, InvertedElementError, compute_geometric_factors
from .kernel_exec import SEQ, ExecPlace
from .operators import CGError, MassPA

__all__ = [
    "MaterialModel",
    "ViscosityModel",
    "StepControls",
    "HydroState",
    "LagrangeHydro",
    "advance_positions",
    "box_velocity_bc",
    "TimestepUnderflow",
]


@dataclass(frozen=True, eq=False)
class MaterialModel:
    """Ideal gas p = (gamma - 1) rho e (hydro.py:40-48).

    Extension (not in the reference, which has one gamma): `gamma` may be an array of one
    adiabatic index per element (multi-material, e.g. the triple point); the device kernels
    then read gamma per element (hx_set_material)."""

    gamma: float = 5.0 / 3.0

    def __post_init__(self):
        if np.any(np.asarray(self.gamma, dtype=float) <= 1.0):
            raise ValueError("adiabatic index must exceed 1")

    @property
    def per_element(self) -> bool:
        return np.ndim(self.gamma) > 0


@dataclass(frozen=True)
class ViscosityModel:
    """Tensor artificial viscosity mu = rho h (q1 c_s + q2 h |div v|) under compression (hydro.py:51-65)."""

    q1: float = 0.5
    q2: float = 2.0

    def __post_init__(self):
        if self.q1 < 0 or self.q2 < 0:
            raise ValueError("viscosity coefficients must be nonnegative")


@dataclass(frozen=True)
class StepControls:
    cfl: float = 0.5
    dt_min: float = 1e-12
    dt_max: float = 1.0
    t_final: float = 1.0

    def __post_init__(self):
        if not 0.0 < self.cfl <= 1.0:
            raise ValueError("cfl must lie in (0, 1]")
        if not 0.0 < self.dt_min <= self.dt_max:
            raise ValueError("need 0 < dt_min <= dt_max")


class TimestepUnderflow(RuntimeError):
    pass


@dataclass
class HydroState:
    """x, v (NN, d) H1 fields; e (NE*nt) L2 field; qdata0 = rho0*detJ0 (nq, NE) (hydro.py:86-98).

    Arrays may be numpy (host, reference semantics) or CUDA tensors (resident)."""

    x: object
    v: object
    e: object
    qdata0: object
    t: float = 0.0

    def copy(self) -> "HydroState":
        cp = (lambda a: a.clone()) if is_torch(self.x) else (lambda a: a.copy())
        return HydroState(cp(self.x), cp(self.v), cp(self.e), self.qdata0, self.t)


@dataclass
class _Rates:
    dx: object
    dv: object
    de: object
    min_h_over_speed: float
    clamped: int


def advance_positions(x, dt, velocity_fn, t: float = 0.0):
    """One midpoint step of dx/dt = w(x, t) for prescribed mesh motion (hydro.py:110-115)."""
    k1 = velocity_fn(x, t)
    xm = x + (0.5 * dt) * k1
    k2 = velocity_fn(xm, t + 0.5 * dt)
    return x + dt * k2


def box_velocity_bc(mesh: HighOrderMesh, extents=None, tol: float = 1e-10) -> np.ndarray:
    """Sealed-box mask: normal velocity held at zero on axis-aligned walls (hydro.py:118-131)."""
    d = mesh.dim
    lo = mesh.coords.min(axis=0)
    hi = mesh.coords.max(axis=0) if extents is None else np.asarray(extents, dtype=float)
    mask = np.zeros((mesh.num_nodes, d), dtype=bool)
    for a in range(d):
        scale = max(hi[a] - lo[a], 1.0)
        on_wall = (np.abs(mesh.coords[:, a] - lo[a]) < tol * scale) | (
            np.abs(mesh.coords[:, a] - hi[a]) < tol * scale)
        mask[on_wall, a] = True
    return mask


def _interp_host(B, t, d):
    # setup-only host interpolation of nodal element tensors (tensor_interp semantics)
    for a in range(d):
        t = np.moveaxis(np.tensordot(B, t, axes=(1, a)), 0, a)
    return np.ascontiguousarray(t)


class LagrangeHydro:
    """One Lagrange phase on a fixed topology (hydro.py:134-423)."""

    def __init__(
        self,
        mesh: HighOrderMesh,
        quad,
        material: MaterialModel,
        viscosity: ViscosityModel = ViscosityModel(),
        thermo_order: int | None = None,
        bc_mask=None,
        place: ExecPlace = SEQ,
        pool=None,
        momentum_rel_tol: float = 1e-8,
    ):
        self.mesh = mesh
        self.quad = quad
        self.material = material
        self.viscosity = viscosity
        self.place = place
        self.pool = pool  # accepted for compatibility: device workspaces are preallocated per context
        self.momentum_rel_tol = momentum_rel_tol
        d = mesh.dim
        self.kin = FiniteElementSpace(mesh, "H1", vdim=d)
        t_order = max(mesh.order - 1, 0) if thermo_order is None else thermo_order
        if t_order != max(mesh.order - 1, 0):
            raise ValueError("the B200 kernels pair kinematic order p with thermodynamic order p-1")
        self.thermo = FiniteElementSpace(mesh, "L2", order=t_order)
        self.bc_mask = np.zeros((mesh.num_nodes, d), dtype=bool) if bc_mask is None else bc_mask
        self.ones_thermo = np.ones(self.thermo.ndof)
        self.clamp_warnings = 0
        self.mass_pa: MassPA | None = None
        self._m_e_inv = None
        self._mass_diag = None
        # a private device context: the phase data (mass qdata, M_e^{-1}, mask) live in it
        self._ctx = DeviceContext(mesh, quad)
        self._mask_dev = to_dev(np.asarray(self.bc_mask), torch.uint8)
        self._phase_ready = False
        if material.per_element:
            g = np.asarray(material.gamma, dtype=float).reshape(-1)
            if g.shape != (mesh.num_elements,):
                raise ValueError(f"per-element gamma must have {mesh.num_elements} entries")
            self._gamma_dev = to_dev(g)
            self._ctx.sync_stream()
            self._ctx.check(self._ctx.lib.hx_set_material(self._ctx.h, _lib.ptr(self._gamma_dev)), "MaterialModel")

    # -- helpers ----------------------------------------------------------------

    def _params(self, controls: StepControls | None = None, rel_tol=None, max_retries=5):
        c = controls or StepControls()
        g0 = float(np.asarray(self.material.gamma, dtype=float).reshape(-1)[0])
        return _lib.Params(g0, float(self.viscosity.q1), float(self.viscosity.q2),
                           float(self.momentum_rel_tol if rel_tol is None else rel_tol), 2000, int(max_retries),
                           float(c.cfl), float(c.dt_min), float(c.dt_max), float(c.t_final))

    def _call(self, fn, *args):
        self._ctx.sync_stream()
        return fn(self._ctx.h, *args)

    # -- phase setup (hydro.py:176-232) -------------------------------------------

    def quad_points_physical(self, x):
        """Physical coordinates of all quadrature points, (d, nq, NE) (hydro.py:176-187)."""
        d = self.mesh.dim
        xh = x.cpu().numpy() if is_torch(x) else np.asarray(x)
        basis = self.kin.basis(self.quad)
        xe = self.kin.e_tensor(xh[self.mesh.node_dofmap], extra=(d,))
        nq = self.quad.n**d
        out = np.empty((d, nq, self.mesh.num_elements))
        for a in range(d):
            out[a] = _interp_host(basis.B, np.ascontiguousarray(xe[..., a, :]), d).reshape(nq, -1)
        return out

    def initial_state(self, rho0_fn, v0_fn, e0_fn) -> HydroState:
        """Sample the initial condition and freeze the per-point mass data (hydro.py:189-202)."""
        x = self.mesh.coords.copy()
        geom0 = compute_geometric_factors(self.mesh, self.quad, x=x)
        xq = self.quad_points_physical(x)
        qdata0 = rho0_fn(xq) * geom0.detj
        v = np.where(self.bc_mask, 0.0, v0_fn(x))
        e = self._sample_l2(e0_fn, x)
        state = HydroState(x=x, v=v, e=e, qdata0=qdata0, t=0.0)
        self.begin_phase(state)
        return state

    def _sample_l2(self, fn, x):
        """Interpolate fn at the thermodynamic nodes of each element (hydro.py:204-218)."""
        from .tensor_basis import eval_basis

        d = self.mesh.dim

        class _Pts:  # a bare point set used where a rule is expected (hydro.py:426-432)
            def __init__(self, pts):
                self.points = np.asarray(pts, dtype=float)
                self.weights = np.zeros_like(self.points)
                self.n = len(self.points)

        Bn = eval_basis(self.mesh.lobatto_nodes, _Pts(self.thermo.nodes1d)).B
        xe = self.kin.e_tensor(np.asarray(x)[self.mesh.node_dofmap], extra=(d,))
        cols = [_interp_host(Bn, np.ascontiguousarray(xe[..., a, :]), d).reshape(self.thermo.nloc, -1)
                for a in range(d)]
        vals = fn(np.stack(cols, axis=0))
        return self.thermo.scatter_add(np.asarray(vals, dtype=float))

    def begin_phase(self, state: HydroState):
        """Mass qdata (wdetj/detj)*qdata0, its diagonal and M_e^{-1} per element (hydro.py:220-232)."""
        d, nq, ne = self.mesh.dim, self.quad.n**self.mesh.dim, self.mesh.num_elements
        X, Q0 = to_dev(state.x), to_dev(state.qdata0)
        Dm = empty((nq, ne))
        diag = empty((self.mesh.num_nodes,))
        nt = self.thermo.nloc
        minv = empty((ne, nt, nt))
        rc = self._call(self._ctx.lib.hx_phase_begin, _lib.ptr(X), _lib.ptr(Q0), _lib.ptr(self._mask_dev),
                        _lib.ptr(Dm), _lib.ptr(diag), _lib.ptr(minv))
        if rc == _lib.HX_EINVERTED:
            compute_geometric_factors(self.mesh, self.quad, x=state.x)  # raises with the offender
        self._ctx.check(rc, "begin_phase")
        geom0 = compute_geometric_factors(self.mesh, self.quad, x=X)
        self.mass_pa = MassPA(self.kin, geom0, qdata=like(Dm, state.x), place=self.place)
        self._mass_diag = like(diag, state.x)
        self._m_e_inv = like(minv, state.x)
        self._phase_ready = True
        d = d  # noqa

    # -- point data ----------------------------------------------------------------

    def density_at_points(self, state: HydroState, geom=None):
        """rho = qdata0 / detJ at every point (hydro.py:236-240)."""
        if geom is None:
            geom = compute_geometric_factors(self.mesh, self.quad, x=state.x)
        return state.qdata0 / geom.detj

    def _weights_tensor(self) -> np.ndarray:
        w = self.quad.weights
        wq = w
        for _ in range(self.mesh.dim - 1):
            wq = np.multiply.outer(wq, w)
        return wq.reshape(-1)

    def total_mass(self, state: HydroState) -> float:
        """sum w_q qdata0 -- independent of the positions (hydro.py:242-245)."""
        q0 = state.qdata0.cpu().numpy() if is_torch(state.qdata0) else state.qdata0
        return float(np.sum(self._weights_tensor()[:, None] * q0))

    def stress_qdata(self, state: HydroState, geom):
        """Total stress sigma = -pI + sigma_visc and min h/(c_s+|v|) (hydro.py:254-315).

        The kernel recomputes the geometry from the positions `geom` was built on."""
        d, nq, ne = self.mesh.dim, self.quad.n**self.mesh.dim, self.mesh.num_elements
        xg = geom.x if getattr(geom, "x", None) is not None else state.x
        X, V, E, Q0 = to_dev(xg), to_dev(state.v), to_dev(state.e), to_dev(state.qdata0)
        sig = empty((d, d, nq, ne))
        ratio = C.c_double()
        clamps = C.c_int64()
        inv = _lib.Inverted()
        prm = self._params()
        rc = self._call(self._ctx.lib.hx_stress, C.byref(prm), _lib.ptr(X), _lib.ptr(V), _lib.ptr(E), _lib.ptr(Q0),
                        _lib.ptr(sig), C.byref(ratio), C.byref(clamps), C.byref(inv))
        if rc == _lib.HX_EINVERTED:
            raise InvertedElementError(int(inv.element), int(inv.point), float("nan"))
        self._ctx.check(rc, "stress_qdata")
        self.clamp_warnings += int(clamps.value)
        return like(sig, state.v), float(ratio.value)

    # -- semi-discrete right-hand side (hydro.py:319-360) -----------------------------

    def _solve_momentum(self, rhs_v, rel_tol=None):
        mask = self.bc_mask
        rhs = np.where(mask, 0.0, rhs_v) if not is_torch(rhs_v) else torch.where(
            self._mask_dev.bool(), torch.zeros((), dtype=rhs_v.dtype, device=rhs_v.device), rhs_v)
        md = to_dev(self._mass_diag)
        diag = torch.where(self._mask_dev.bool(), torch.ones((), dtype=md.dtype, device=md.device),
                           md[:, None].expand(-1, self.mesh.dim))
        x, _ = self.mass_pa.solve(rhs, diag, self._mask_dev,
                                  self.momentum_rel_tol if rel_tol is None else rel_tol, 2000)
        return x

    def solve_energy(self, rhs_e):
        """de = M_e^{-1} rhs per element (hydro.py:339-344)."""
        R = to_dev(rhs_e)
        out = empty((self.thermo.ndof,))
        self._ctx.check(self._call(self._ctx.lib.hx_energy_solve, _lib.ptr(R), _lib.ptr(out)), "solve_energy")
        return like(out, rhs_e)

    def _raise(self, info, where):
        if info.code == _lib.HX_EINVERTED:
            raise InvertedElementError(int(info.inv.element), int(info.inv.point), float("nan"))
        if info.code == _lib.HX_ECG_MAXITER:
            raise CGError("CG did not converge in 2000 iterations", [])
        if info.code == _lib.HX_ECG_BREAKDOWN:
            raise CGError("CG breakdown: p^T A p <= 0", [])
        if info.code == _lib.HX_EUNDERFLOW:
            raise TimestepUnderflow(where)
        if info.code != _lib.HX_OK:
            self._ctx.check(info.code, where)

    def rates(self, state: HydroState, momentum_rel_tol=None) -> _Rates:
        """dx = v, dv = M^{-1}(-F.1) (masked), de = M_e^{-1} F^T v (hydro.py:346-360)."""
        X, V, E = to_dev(state.x), to_dev(state.v), to_dev(state.e)
        dv = empty(tuple(X.shape))
        de = empty(tuple(E.shape))
        info = _lib.StepInfo()
        prm = self._params(rel_tol=momentum_rel_tol)
        rc = self._call(self._ctx.lib.hx_rates, C.byref(prm), _lib.ptr(X), _lib.ptr(V), _lib.ptr(E), _lib.ptr(dv),
                        _lib.ptr(de), C.byref(info))
        if rc not in (_lib.HX_OK,) and info.code == 0:
            self._ctx.check(rc, "rates")
        self._raise(info, "rates")
        self.clamp_warnings += int(info.clamped)
        self.last_cg_iterations = int(info.cg_iterations[0])  # diagnostics (not in the reference)
        dx = state.v.clone() if is_torch(state.v) else state.v.copy()
        return _Rates(dx=dx, dv=like(dv, state.v), de=like(de, state.e),
                      min_h_over_speed=float(info.min_h_over_speed), clamped=int(info.clamped))

    # -- stepping (hydro.py:364-405) ---------------------------------------------------

    def timestep_estimate(self, state: HydroState, controls: StepControls) -> float:
        """dt = min(cfl * min h/(c_s+|v|), dt_max, t_final - t) (hydro.py:364-373).

        3D p >= 2: one fused device launch (hx_timestep_ratio) with the semantics of the
        reference's compute_geometric_factors + stress_qdata pair (same first inverted
        point, same clamp count, same ratio); otherwise those two calls."""
        if self.mesh.dim == 3 and self.mesh.order >= 2 and self._phase_ready:
            X, V, E = to_dev(state.x), to_dev(state.v), to_dev(state.e)
            ratio = C.c_double()
            clamps = C.c_int64()
            inv = _lib.Inverted()
            rc = self._call(self._ctx.lib.hx_timestep_ratio, C.byref(self._params()), _lib.ptr(X), _lib.ptr(V),
                            _lib.ptr(E), C.byref(ratio), C.byref(clamps), C.byref(inv))
            if rc == _lib.HX_EINVERTED:
                raise InvertedElementError(int(inv.element), int(inv.point), float("nan"))
            self._ctx.check(rc, "timestep_estimate")
            self.clamp_warnings += int(clamps.value)
            min_ratio = float(ratio.value)
        else:
            geom = compute_geometric_factors(self.mesh, self.quad, x=state.x)
            _, min_ratio = self.stress_qdata(state, geom)
        dt = controls.cfl * min_ratio
        dt = min(dt, controls.dt_max, controls.t_final - state.t)
        if dt < controls.dt_min:
            raise TimestepUnderflow(
                f"dt = {dt:.3e} fell below dt_min = {controls.dt_min:.3e} at t = {state.t:.6e}")
        return dt

    def _new_state(self, state, Xo, Vo, Eo, t_new):
        return HydroState(x=like(Xo, state.x), v=like(Vo, state.v), e=like(Eo, state.e),
                          qdata0=state.qdata0, t=t_new)

    def rk2_step(self, state: HydroState, dt: float, max_retries: int = 5):
        """Midpoint step; on an inverted element retry at half dt, up to max_retries (hydro.py:375-405)."""
        X, V, E = to_dev(state.x), to_dev(state.v), to_dev(state.e)
        Xo, Vo, Eo = torch.empty_like(X), torch.empty_like(V), torch.empty_like(E)
        info = _lib.StepInfo()
        prm = self._params(max_retries=max_retries)
        rc = self._call(self._ctx.lib.hx_rk2_step, C.byref(prm), float(state.t), float(dt), _lib.ptr(X),
                        _lib.ptr(V), _lib.ptr(E), _lib.ptr(Xo), _lib.ptr(Vo), _lib.ptr(Eo), C.byref(info))
        if rc != _lib.HX_OK and info.code == _lib.HX_OK:
            self._ctx.check(rc, "rk2_step")  # failed before the step info was written
        if info.code == _lib.HX_EUNDERFLOW:
            self.clamp_warnings += int(info.clamped)
            raise TimestepUnderflow(f"step rejected {max_retries + 1} times from dt = {dt:.3e}")
        self._raise(info, "rk2_step")
        self.clamp_warnings += int(info.clamped)
        new = self._new_state(state, Xo, Vo, Eo, state.t + info.dt)
        return new, {"dt": float(info.dt), "min_h_over_speed": float(info.min_h_over_speed),
                     "cg_iterations": (int(info.cg_iterations[0]), int(info.cg_iterations[1])),
                     "retries": int(info.retries)}

    def step(self, state: HydroState, controls: StepControls, max_retries: int = 5, out=None):
        """timestep_estimate + rk2_step in one device call (hx_step).

        Identical results to calling the two separately: the CFL estimate is the
        stage-1 ratio of the same state.  `out` may supply three preallocated CUDA
        tensors for the new x, v, e (ping-pong buffers for a resident time loop)."""
        X, V, E = to_dev(state.x), to_dev(state.v), to_dev(state.e)
        if out is None:
            Xo, Vo, Eo = torch.empty_like(X), torch.empty_like(V), torch.empty_like(E)
        else:
            Xo, Vo, Eo = out
        info = _lib.StepInfo()
        prm = self._params(controls, max_retries=max_retries)
        rc = self._call(self._ctx.lib.hx_step, C.byref(prm), float(state.t), _lib.ptr(X), _lib.ptr(V),
                        _lib.ptr(E), _lib.ptr(Xo), _lib.ptr(Vo), _lib.ptr(Eo), C.byref(info))
        if rc != _lib.HX_OK and info.code == _lib.HX_OK:
            self._ctx.check(rc, "step")  # failed before the step info was written
        if info.code == _lib.HX_EUNDERFLOW:
            self.clamp_warnings += int(info.clamped)
            if info.failed_stage == 0 and info.retries == 0:
                raise TimestepUnderflow(
                    f"dt = {info.dt:.3e} fell below dt_min = {controls.dt_min:.3e} at t = {state.t:.6e}")
            raise TimestepUnderflow(f"step rejected {max_retries + 1} times")
        self._raise(info, "step")
        self.clamp_warnings += int(info.clamped)
        new = self._new_state(state, Xo, Vo, Eo, float(info.t_new))
        return new, {"dt": float(info.dt), "min_h_over_speed": float(info.min_h_over_speed),
                     "cg_iterations": (int(info.cg_iterations[0]), int(info.cg_iterations[1])),
                     "retries": int(info.retries)}

    # -- diagnostics (hydro.py:409-423) ----------------------------------------------

    def _energies(self, state):
        V, E, Q0 = to_dev(state.v), to_dev(state.e), to_dev(state.qdata0)
        ke, ie = C.c_double(), C.c_double()
        self._ctx.check(self._call(self._ctx.lib.hx_energies, _lib.ptr(V), _lib.ptr(E), _lib.ptr(Q0),
                                   C.byref(ke), C.byref(ie)), "energies")
        return float(ke.value), float(ie.value)

    def kinetic_energy(self, state: HydroState) -> float:
        return self._energies(state)[0]

    def internal_energy(self, state: HydroState) -> float:
        return self._energies(state)[1]

    def total_energy(self, state: HydroState) -> float:
        ke, ie = self._energies(state)
        return ke + ie

    # -- residency helpers -------------------------------------------------------------

    def to_device(self, state: HydroState) -> HydroState:
        """Copy a host state to CUDA tensors (later steps stay resident)."""
        return HydroState(to_dev(state.x), to_dev(state.v), to_dev(state.e), to_dev(state.qdata0), state.t)

    @staticmethod
    def to_host(state: HydroState) -> HydroState:
        h = (lambda a: a.cpu().numpy() if is_torch(a) else a)
        return HydroState(h(state.x), h(state.v), h(state.e), h(state.qdata0), state.t)
