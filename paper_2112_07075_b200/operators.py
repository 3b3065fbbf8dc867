"""Partial-assembly operators and the Jacobi-PCG solver on the B200.

Drop-in for `ale_minihydro.operators` on the Lagrange path: `MassPA`
(operators.py:84-140), `ForcePA` (operators.py:239-324), `cg_solve`
(operators.py:333-366) and `CGError` (operators.py:327-330).  The operator
applies run in libb200hydro.so (sum-factorised sm_100a kernels with the
deterministic restriction); `cg_solve` on a `MassPA.apply` runs entirely on the
device with the stop test evaluated there (`hx_mass_cg`).

`DiffusionPA` / `ConvectionPA` (operators.py:143-236) belong to the remap phase,
not the Lagrange hot path; they run on the same contraction machinery (SURVEY.md
section 8f, "next").  The `.assemble()` full-assembly oracles are not provided: the
test suite checks against the CPU oracle in `oracle/` and the reference's fixtures.
"""

from __future__ import annotations

import ctypes as C
import weakref

import numpy as np
import torch

from . import _lib
from ._device import context_for, empty, like, to_dev
from .kernel_exec import SEQ, ExecPlace

__all__ = ["MassPA", "ForcePA", "DiffusionPA", "ConvectionPA", "cg_solve", "CGError", "ELEMENT_BLOCK"]

ELEMENT_BLOCK = 32  # reference team block (operators.py:39); informational on the device


class CGError(RuntimeError):
    """CG breakdown or non-convergence; carries the residual history (operators.py:327-330)."""

    def __init__(self, message: str, residuals):
        super().__init__(message)
        self.residuals = residuals


class MassPA:
    """Mass operator; D holds w_q * coeff_q * detJ_q per point per element (operators.py:84-95)."""

    def __init__(self, space, geom, coeff=None, qdata=None, place: ExecPlace = SEQ):
        self.space = space
        self.geom = geom
        self.place = place
        self.basis = space.basis(geom.quad)
        self.d = space.mesh.dim
        self.q1d = geom.quad.n
        self.ne = space.mesh.num_elements
        if qdata is not None:
            self.D = qdata.clone() if isinstance(qdata, torch.Tensor) else np.array(qdata, dtype=float)
        else:
            w = geom.wdetj
            self.D = w.clone() if isinstance(w, torch.Tensor) else w.copy()
            if coeff is not None:
                self.D = self.D * coeff
        self.stored_values = int(np.prod(tuple(self.D.shape)))  # NE * Q1D^d exactly
        self._ctx = context_for(space.mesh, geom.quad)
        h = C.c_void_p()
        Dd = to_dev(self.D)
        self._ctx.sync_stream()
        self._ctx.check(self._ctx.lib.hx_mass_create(self._ctx.h, _lib.ptr(Dd), C.byref(h)), "MassPA")
        self._h = h
        self._fin = weakref.finalize(self, self._ctx.lib.hx_mass_destroy, h)

    def apply(self, x):
        """y = G^T B^T D B G x per component (operators.py:97-115)."""
        nc = 1 if x.ndim == 1 else int(x.shape[1])
        if x.shape[0] != self.space.ndof or nc > 3:
            raise ValueError(f"vector of shape {tuple(x.shape)} does not match {self.space.ndof} dofs")
        X = to_dev(x)
        Y = empty(tuple(x.shape))
        self._ctx.sync_stream()
        self._ctx.check(self._ctx.lib.hx_mass_apply(self._h, _lib.ptr(X), nc, _lib.ptr(Y)), "MassPA.apply")
        return like(Y, x)

    def diagonal(self):
        """Matrix-free diagonal via squared-basis contractions (operators.py:117-124)."""
        out = empty((self.space.ndof,))
        self._ctx.sync_stream()
        self._ctx.check(self._ctx.lib.hx_mass_diagonal(self._h, _lib.ptr(out)), "MassPA.diagonal")
        return like(out, self.D)

    def solve(self, b, precond_diag=None, bc_mask=None, rel_tol=1e-8, max_iter=1000):
        """Device Jacobi PCG on this operator (cg_solve + the wall mask of _solve_momentum)."""
        flat = b.reshape(-1) if b.ndim > 1 else b
        nc = 1 if b.ndim == 1 else int(b.shape[1])
        B = to_dev(b)
        Xo = empty(tuple(b.shape))
        Pd = None if precond_diag is None else to_dev(precond_diag)
        Mk = None if bc_mask is None else to_dev(bc_mask, torch.uint8)
        hist = empty((max_iter + 1,))
        info = _lib.CGInfo()
        self._ctx.sync_stream()
        rc = self._ctx.lib.hx_mass_cg(self._h, _lib.ptr(B), nc, _lib.ptr(Mk), _lib.ptr(Pd), float(rel_tol),
                                      int(max_iter), _lib.ptr(Xo), _lib.ptr(hist), C.byref(info))
        if rc in (_lib.HX_ECG_BREAKDOWN, _lib.HX_ECG_MAXITER):
            res = [float(r) for r in hist[: info.n_residuals].cpu()]
            if rc == _lib.HX_ECG_MAXITER:
                raise CGError(f"CG did not converge in {max_iter} iterations", res)
            raise CGError("CG breakdown: p^T A p <= 0", res)
        self._ctx.check(rc, "MassPA CG")
        del flat
        return like(Xo, b), int(info.iterations)

    def assemble(self):
        raise NotImplementedError("full assembly is a CPU test oracle; see oracle/pa_oracle.py")


class _ScalarPA:
    """Common part of the scalar H1 PA operators of the remap phase (operators.py:143-236)."""

    def _finish(self, space, geom, place, h, Dout, ref_like):
        self.space, self.geom, self.place = space, geom, place
        self.basis = space.basis(geom.quad)
        self.d = space.mesh.dim
        self.q1d = geom.quad.n
        self.ne = space.mesh.num_elements
        self._h = h
        self._fin = weakref.finalize(self, self._ctx.lib.hx_op_destroy, h)
        self.D = like(Dout, ref_like)
        self.stored_values = int(np.prod(tuple(Dout.shape)))

    def _qshape(self):
        return (self.q1d,) * self.d

    def apply(self, x):
        if tuple(x.shape) != (self.space.ndof,):
            raise ValueError(f"vector of shape {tuple(x.shape)} does not match {self.space.ndof} dofs")
        X = to_dev(x)
        Y = empty((self.space.ndof,))
        self._ctx.sync_stream()
        self._ctx.check(self._ctx.lib.hx_op_apply(self._h, _lib.ptr(X), _lib.ptr(Y)), type(self).__name__)
        return like(Y, x)

    def assemble(self):
        raise NotImplementedError("full assembly is a CPU test oracle; see oracle/pa_oracle.py")


class DiffusionPA(_ScalarPA):
    """Stiffness operator; D holds w detJ J^{-1} nu J^{-T} per point (operators.py:143-168)."""

    def __init__(self, space, geom, nu=None, place: ExecPlace = SEQ):
        self._ctx = context_for(space.mesh, geom.quad)
        d, nq, ne = space.mesh.dim, geom.quad.n**space.mesh.dim, space.mesh.num_elements
        Ji, W = to_dev(geom.jinv), to_dev(geom.wdetj)
        Nu = None if nu is None else to_dev(nu)
        Dout = empty((d, d, nq, ne))
        h = C.c_void_p()
        self._ctx.sync_stream()
        self._ctx.check(self._ctx.lib.hx_diffusion_create(self._ctx.h, _lib.ptr(Ji), _lib.ptr(W), _lib.ptr(Nu),
                                                          _lib.ptr(Dout), C.byref(h)), "DiffusionPA")
        self._finish(space, geom, place, h, Dout, geom.wdetj)


class ConvectionPA(_ScalarPA):
    """(K w)_i = integral phi_i (u . grad w); D holds w detJ J^{-1} u per point (operators.py:188-214)."""

    def __init__(self, space, geom, u_points, place: ExecPlace = SEQ):
        self._ctx = context_for(space.mesh, geom.quad)
        d, nq, ne = space.mesh.dim, geom.quad.n**space.mesh.dim, space.mesh.num_elements
        if tuple(u_points.shape) != (d, nq, ne):
            raise ValueError(f"u_points must have shape {(d, nq, ne)}")
        Ji, W, U = to_dev(geom.jinv), to_dev(geom.wdetj), to_dev(u_points)
        Dout = empty((d, nq, ne))
        h = C.c_void_p()
        self._ctx.sync_stream()
        self._ctx.check(self._ctx.lib.hx_convection_create(self._ctx.h, _lib.ptr(Ji), _lib.ptr(U), _lib.ptr(W),
                                                           _lib.ptr(Dout), C.byref(h)), "ConvectionPA")
        self._finish(space, geom, place, h, Dout, geom.wdetj)


class ForcePA:
    """Rectangular force operator H1^d x L2 (operators.py:239-300).

    apply(e): (F e)_{a,i} = sum_q D[a,l,q] dphi_i/dxi_l(q) psi(q);
    apply_transpose is its exact adjoint.  D = w detJ sigma jinv^T (operators.py:258).
    """

    def __init__(self, kin_space, thermo_space, geom, stress_points, place: ExecPlace = SEQ):
        self.kin = kin_space
        self.thermo = thermo_space
        self.geom = geom
        self.place = place
        self.d = kin_space.mesh.dim
        self.ne = kin_space.mesh.num_elements
        self.q1d = geom.quad.n
        self.kin_basis = kin_space.basis(geom.quad)
        self.thermo_basis = thermo_space.basis(geom.quad)
        if thermo_space.order != max(kin_space.order - 1, 0):
            raise ValueError("the B200 force kernels pair H1 order p with L2 order p-1")
        self._ctx = context_for(kin_space.mesh, geom.quad)
        d, nq = self.d, geom.quad.n**self.d
        S = to_dev(stress_points)
        Ji, W = to_dev(geom.jinv), to_dev(geom.wdetj)
        Dout = empty((d, d, nq, self.ne))
        h = C.c_void_p()
        self._ctx.sync_stream()
        self._ctx.check(self._ctx.lib.hx_force_create(self._ctx.h, _lib.ptr(S), _lib.ptr(Ji), _lib.ptr(W),
                                                      _lib.ptr(Dout), C.byref(h)), "ForcePA")
        self._h = h
        self._fin = weakref.finalize(self, self._ctx.lib.hx_force_destroy, h)
        self.D = like(Dout, stress_points)
        self.stored_values = int(np.prod(tuple(Dout.shape)))

    def _qshape(self):
        return (self.q1d,) * self.d

    def apply(self, e_field):
        """L2 scalar -> H1 vector (the momentum right-hand side is -apply(ones))."""
        if e_field.shape[0] != self.thermo.ndof:
            raise ValueError("thermodynamic vector size mismatch")
        E = to_dev(e_field)
        Y = empty((self.kin.ndof, self.d))
        self._ctx.sync_stream()
        self._ctx.check(self._ctx.lib.hx_force_apply(self._h, _lib.ptr(E), _lib.ptr(Y)), "ForcePA.apply")
        return like(Y, e_field)

    def apply_transpose(self, v):
        """H1 vector -> L2 scalar: (F^T v)_j = sum_q (sigma : grad v) psi_j w detJ."""
        if tuple(v.shape) != (self.kin.ndof, self.d):
            raise ValueError("velocity field shape mismatch")
        V = to_dev(v)
        Y = empty((self.thermo.ndof,))
        self._ctx.sync_stream()
        self._ctx.check(self._ctx.lib.hx_force_apply_t(self._h, _lib.ptr(V), _lib.ptr(Y)),
                        "ForcePA.apply_transpose")
        return like(Y, v)

    def assemble(self):
        raise NotImplementedError("full assembly is a CPU test oracle; see oracle/pa_oracle.py")


def cg_solve(apply_op, b, precond_diag=None, rel_tol: float = 1e-8, max_iter: int = 1000):
    """Jacobi-preconditioned CG, x0 = 0, stop at sqrt(r.z) <= rel_tol*sqrt(r0.z0) (operators.py:333-366).

    When `apply_op` is `MassPA.apply` the whole solve runs on the device
    (`hx_mass_cg`).  Any other operator is driven from the host with device
    vectors (the same recurrence, one host sync per iteration).
    """
    owner = getattr(apply_op, "__self__", None)
    if isinstance(owner, MassPA) and getattr(apply_op, "__func__", None) is MassPA.apply:
        b_arr = b if isinstance(b, torch.Tensor) else np.asarray(b, dtype=float)
        if b_arr.shape[0] == owner.space.ndof:
            return owner.solve(b_arr, precond_diag, None, rel_tol, max_iter)
    bt = to_dev(b)
    x = torch.zeros_like(bt)
    if not bool(torch.any(bt != 0)):
        return like(x, b), 0
    inv_diag = None if precond_diag is None else 1.0 / to_dev(precond_diag)
    r = bt.clone()
    z = r if inv_diag is None else inv_diag * r
    p = z.clone()
    rz = float(torch.dot(r.reshape(-1), z.reshape(-1)))
    norm0 = float(np.sqrt(rz))
    residuals = [norm0]
    for it in range(1, max_iter + 1):
        Ap = to_dev(apply_op(like(p, b)))
        pAp = float(torch.dot(p.reshape(-1), Ap.reshape(-1)))
        if pAp <= 0.0:
            raise CGError(f"CG breakdown: p^T A p = {pAp:.3e} <= 0", residuals)
        alpha = rz / pAp
        x += alpha * p
        r -= alpha * Ap
        z = r if inv_diag is None else inv_diag * r
        rz_new = float(torch.dot(r.reshape(-1), z.reshape(-1)))
        residuals.append(float(np.sqrt(max(rz_new, 0.0))))
        if residuals[-1] <= rel_tol * norm0:
            return like(x, b), it
        p = z + (rz_new / rz) * p
        rz = rz_new
    raise CGError(f"CG did not converge in {max_iter} iterations", residuals)
