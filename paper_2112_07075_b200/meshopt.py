"""TMOP mesh optimisation (the ALE mesh-optimisation phase) on the B200.

Drop-in for `ale_minihydro.meshopt` (meshopt.py:1-588): the same names, constructor
arguments and return layouts.  The objective's two integrals, the gradient, the Hessian
action and the matrix-free Hessian diagonal run in libb200hydro.so (`hx_tmop_*`, one CTA
per element on the Lagrange phase's sum-factorised contractions, csrc/hx_tmop.cuh): the
target Jacobians T = A W^{-1}, the metric and its first and second derivatives are
evaluated at the quadrature points on the fly and assembled by the deterministic node pass.
Setup (targets, limiting radii, gamma) and the Newton orchestration stay on the host, as in
the reference; the inner Jacobi-PCG is `operators.cg_solve` on device vectors.

Restrictions of the device path: the quadrature must be the context's rule
(gauss_legendre(p + 2)); metrics are the reference's shape metrics of `metric_for(d)` and
their composite with `SizeMetric` (`metric_for(d, with_size=True)`, any weights).
"""

from __future__ import annotations

import ctypes as C
import weakref
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._device import context_for, empty, like, to_dev
from .fespace import FiniteElementSpace, HighOrderMesh, compute_geometric_factors
from .kernel_exec import SEQ, ExecPlace
from .operators import CGError, cg_solve

__all__ = [
    "ShapeMetric2D",
    "ShapeMetric3D",
    "SizeMetric",
    "CompositeMetric",
    "TargetTransform",
    "TMOPObjective",
    "build_targets",
    "metric_for",
    "newton_solve",
    "NewtonResult",
]


# ---------------------------------------------------------------------------
# quality metrics (host evaluators over a flat (N, d, d) stack; the device kernels use the
# same closed forms).  d2mu is returned as the 4-tensor (N, m, n, k, l) built from the
# directional derivative of dmu along the unit matrices e_k e_l^T.

def _cof(T):
    """Cofactor matrix d det / dT and det, (N, d, d)."""
    d = T.shape[-1]
    if d == 2:
        C_ = np.stack([np.stack([T[:, 1, 1], -T[:, 1, 0]], -1), np.stack([-T[:, 0, 1], T[:, 0, 0]], -1)], 1)
        return C_, T[:, 0, 0] * T[:, 1, 1] - T[:, 0, 1] * T[:, 1, 0]
    C_ = np.empty_like(T)
    for m in range(3):
        m1, m2 = (m + 1) % 3, (m + 2) % 3
        for n in range(3):
            n1, n2 = (n + 1) % 3, (n + 2) % 3
            C_[:, m, n] = T[:, m1, n1] * T[:, m2, n2] - T[:, m1, n2] * T[:, m2, n1]
    return C_, np.einsum("nj,nj->n", T[:, 0], C_[:, 0])


def _dcof(T, dT):
    d = T.shape[-1]
    if d == 2:
        return _cof(dT)[0]
    out = np.empty_like(T)
    for m in range(3):
        m1, m2 = (m + 1) % 3, (m + 2) % 3
        for n in range(3):
            n1, n2 = (n + 1) % 3, (n + 2) % 3
            out[:, m, n] = (dT[:, m1, n1] * T[:, m2, n2] + T[:, m1, n1] * dT[:, m2, n2]) - (
                dT[:, m1, n2] * T[:, m2, n1] + T[:, m1, n2] * dT[:, m2, n1])
    return out


def _ddot(a, b):
    return np.einsum("nij,nij->n", a, b)


class _Metric:
    dim = None

    def dd(self, T, dT):  # directional derivative of dmu at T along dT
        raise NotImplementedError

    def d2mu(self, T):
        d = T.shape[-1]
        out = np.empty((T.shape[0], d, d, d, d))
        for k in range(d):
            for l in range(d):
                E = np.zeros_like(T)
                E[:, k, l] = 1.0
                out[..., k, l] = self.dd(T, E)
        return out


class ShapeMetric2D(_Metric):
    """mu = |T|^2 / (2 det T) - 1 (meshopt.py:46-83)."""

    dim = 2

    def mu(self, T):
        _, tau = _cof(T)
        return _ddot(T, T) / (2.0 * tau) - 1.0

    def dmu(self, T):
        C_, tau = _cof(T)
        f = _ddot(T, T)
        return T / tau[:, None, None] - (f / (2.0 * tau * tau))[:, None, None] * C_

    def dd(self, T, dT):
        C_, tau = _cof(T)
        f = _ddot(T, T)
        cd, td = _ddot(C_, dT)[:, None, None], _ddot(T, dT)[:, None, None]
        it = (1.0 / tau)[:, None, None]
        return dT * it - (T * cd + C_ * td) * it**2 + f[:, None, None] * it**3 * cd * C_ - (
            f / (2.0 * tau * tau))[:, None, None] * _dcof(T, dT)


class ShapeMetric3D(_Metric):
    """mu = |T|^2 |T^-1|^2 / 9 - 1 (meshopt.py:86-122)."""

    dim = 3

    @staticmethod
    def _parts(T):
        C_, tau = _cof(T)
        S = np.swapaxes(C_, 1, 2) / tau[:, None, None]
        f, g = _ddot(T, T), _ddot(S, S)
        N = np.einsum("nam,nab,nzb->nmz", S, S, S)
        return S, f, g, N

    def mu(self, T):
        _, f, g, _ = self._parts(T)
        return f * g / 9.0 - 1.0

    def dmu(self, T):
        _, f, g, N = self._parts(T)
        return (2.0 * g[:, None, None] * T - 2.0 * f[:, None, None] * N) / 9.0

    def dd(self, T, dT):
        S, f, g, N = self._parts(T)
        StS, SSt = np.einsum("nkm,nkz->nmz", S, S), np.einsum("nmk,nzk->nmz", S, S)
        dN = -(np.einsum("nkm,nlk,nlz->nmz", S, dT, N) + np.einsum("nmk,nkl,nlz->nmz", StS, dT, SSt)
               + np.einsum("nml,nkl,nzk->nmz", N, dT, S))
        nd, td = _ddot(N, dT)[:, None, None], _ddot(T, dT)[:, None, None]
        return (2.0 * g[:, None, None] * dT - 4.0 * (nd * T + td * N) - 2.0 * f[:, None, None] * dN) / 9.0


class SizeMetric(_Metric):
    """mu = (det T + 1/det T)/2 - 1 (meshopt.py:125-166)."""

    def __init__(self, dim: int):
        self.dim = dim

    def mu(self, T):
        _, tau = _cof(T)
        return 0.5 * (tau + 1.0 / tau) - 1.0

    def dmu(self, T):
        C_, tau = _cof(T)
        return (0.5 * (1.0 - 1.0 / (tau * tau)))[:, None, None] * C_

    def dd(self, T, dT):
        C_, tau = _cof(T)
        return (_ddot(C_, dT) / tau**3)[:, None, None] * C_ + (0.5 * (1.0 - 1.0 / (tau * tau)))[:, None, None] * _dcof(
            T, dT)


class CompositeMetric(_Metric):
    """Weighted sum of metrics (meshopt.py:169-182)."""

    def __init__(self, parts):
        self.parts = list(parts)

    def mu(self, T):
        return sum(w * m.mu(T) for w, m in self.parts)

    def dmu(self, T):
        return sum(w * m.dmu(T) for w, m in self.parts)

    def dd(self, T, dT):
        return sum(w * m.dd(T, dT) for w, m in self.parts)


def metric_for(dim: int, with_size: bool = False):
    """Shape metric of the dimension, optionally plus the size metric (meshopt.py:185-190)."""
    shape = ShapeMetric2D() if dim == 2 else ShapeMetric3D()
    return CompositeMetric([(1.0, shape), (1.0, SizeMetric(dim))]) if with_size else shape


def _device_metric(metric, dim):
    """(composite, w_shape, w_size) of the device kernels; accepts this module's metrics
    and the reference's (by class name)."""
    name = type(metric).__name__
    if name in ("ShapeMetric2D", "ShapeMetric3D") and metric.dim == dim:
        return 0, 1.0, 0.0
    if name == "CompositeMetric":
        parts = list(metric.parts)
        if (len(parts) == 2 and type(parts[0][1]).__name__ == ("ShapeMetric2D" if dim == 2 else "ShapeMetric3D")
                and type(parts[1][1]).__name__ == "SizeMetric"):
            return 1, float(parts[0][0]), float(parts[1][0])
    raise NotImplementedError(f"metric {name} has no device kernel (shape, or shape + size composite)")


# ---------------------------------------------------------------------------
# targets (host setup, meshopt.py:196-245)

@dataclass
class TargetTransform:
    """Per-point target Jacobians W (d,d,nq,NE), the reference's inverse and det W (nq,NE)."""

    w: np.ndarray
    winv: np.ndarray
    detw: np.ndarray


def _ref_det_inv(w):
    """det and the reference's _det_inv second output (fespace.py:280-302): the adjugate in
    2D, the cofactor matrix in 3D (so winv = J^{-T} there, a reference quirk kept for parity)."""
    d = w.shape[0]
    flat = np.moveaxis(w.reshape(d, d, -1), -1, 0)
    C_, det = _cof(flat)
    inv = np.swapaxes(C_, 1, 2) if d == 2 else C_
    return det.reshape(w.shape[2:]), np.moveaxis(inv, 0, -1).reshape(w.shape)


def _interp_nodal(mesh: HighOrderMesh, quad, field) -> np.ndarray:
    """Nodal H1 scalar -> all quadrature points (nq, NE) by 1D basis contractions."""
    from .tensor_basis import eval_basis

    d, n1, ne = mesh.dim, mesh.order + 1, mesh.num_elements
    B = eval_basis(mesh.lobatto_nodes, quad).B  # (Q, D1)
    t = np.asarray(field, dtype=float)[mesh.node_dofmap].reshape((n1,) * d + (ne,), order="F")
    for ax in range(d):  # x = axis 0 here (node index x fastest)
        t = np.moveaxis(np.tensordot(B, t, axes=(1, ax)), 0, ax)
    return t.reshape(-1, ne, order="F")


def build_targets(mesh0: HighOrderMesh, quad, mode: str = "ideal-uniform", xi=None) -> TargetTransform:
    """ideal-uniform: the mean Jacobian of the initial mesh at every point; size-adapted: that
    target scaled pointwise by xi^(1/d) (meshopt.py:204-229)."""
    d = mesh0.dim
    jac0 = np.asarray(like(to_dev(compute_geometric_factors(mesh0, quad).jac), np.empty(0)))
    nq, ne = jac0.shape[2:]
    w = np.broadcast_to(jac0.mean(axis=(2, 3))[:, :, None, None], (d, d, nq, ne)).copy()
    if mode == "size-adapted":
        if xi is None:
            raise ValueError("size-adapted targets need a xi field")
        xq = _interp_nodal(mesh0, quad, xi)
        if np.any(xq <= 0.0):
            raise ValueError("xi must be positive wherever it scales the target")
        w = w * (xq ** (1.0 / d))[None, None]
    elif mode != "ideal-uniform":
        raise ValueError(f"unknown target mode {mode!r}")
    detw, inv = _ref_det_inv(w)
    if np.any(detw <= 0.0):
        raise ValueError("target Jacobians must have positive determinant")
    return TargetTransform(w=w, winv=inv / detw, detw=detw)


# ---------------------------------------------------------------------------
# objective

class TMOPObjective:
    """F(x) = sum_q w_q detW mu(T(x)) + gamma * limiting term (meshopt.py:248-486), with the
    quadrature loops on the device."""

    def __init__(self, mesh: HighOrderMesh, quad, targets: TargetTransform, metric=None,
                 gamma: float | str = 0.0, x0=None, place: ExecPlace = SEQ):
        self.mesh, self.quad, self.targets, self.place = mesh, quad, targets, place
        self.d = d = mesh.dim
        self.metric = metric_for(d) if metric is None else metric
        self.scalar = FiniteElementSpace(mesh, "H1")
        self.basis = self.scalar.basis(quad)
        self.x0 = np.array(mesh.coords if x0 is None else x0, dtype=float)
        wq = quad.weights
        for _ in range(d - 1):
            wq = np.multiply.outer(wq, quad.weights)
        self.wdetw = wq.reshape(-1)[:, None] * np.asarray(targets.detw)
        self.dlim = self._node_sizes()
        comp, ws, wz = _device_metric(self.metric, d)
        self._ctx = ctx = context_for(mesh, quad)
        h = C.c_void_p()
        W, WD, X0, DL = (to_dev(np.asarray(a)) for a in (targets.winv, self.wdetw, self.x0, self.dlim))
        ctx.sync_stream()
        ctx.check(ctx.lib.hx_tmop_create(ctx.h, _lib.ptr(W), _lib.ptr(WD), _lib.ptr(X0), _lib.ptr(DL), comp, ws, wz,
                                         0.0, C.byref(h)), "TMOPObjective")
        self._h = h
        self._fin = weakref.finalize(self, ctx.lib.hx_tmop_destroy, h)
        if gamma == "auto":
            self.gamma = 0.0
            self.gamma = self._auto_gamma()
        else:
            self.gamma = float(gamma)

    @property
    def gamma(self) -> float:
        return self._gamma

    @gamma.setter
    def gamma(self, g):
        self._gamma = float(g)
        if getattr(self, "_h", None) is not None:
            self._ctx.check(self._ctx.lib.hx_tmop_set_gamma(self._h, self._gamma), "gamma")

    def _node_sizes(self) -> np.ndarray:
        """Per-node limiting radius: the mean local element size of the initial mesh."""
        geom = compute_geometric_factors(self.mesh, self.quad, x=self.x0)
        size = np.asarray(like(to_dev(geom.wdetj), np.empty(0))).sum(axis=0) ** (1.0 / self.d)
        tot = self.scalar.scatter_add(np.ascontiguousarray(np.broadcast_to(size, (self.scalar.nloc, self.mesh.num_elements))))
        return np.asarray(like(to_dev(tot), np.empty(0))) / np.asarray(like(to_dev(self.scalar.multiplicity()),
                                                                              np.empty(0)))

    def free_interior_mask(self) -> np.ndarray:
        mask = np.ones((self.mesh.num_nodes, self.d), dtype=bool)
        mask[self.mesh.boundary_nodes()] = False
        return mask

    def _terms(self, x, want_limit):
        X = to_dev(x)
        mu, lim, ok = C.c_double(), C.c_double(), C.c_int()
        self._ctx.sync_stream()
        self._ctx.check(self._ctx.lib.hx_tmop_terms(self._h, _lib.ptr(X), 1 if want_limit else 0, C.byref(mu),
                                                    C.byref(lim), C.byref(ok)), "TMOP objective")
        return (mu.value if ok.value else np.inf), lim.value

    def _mu_term(self, x) -> float:
        return float(self._terms(x, False)[0])

    def _limit_term(self, x, gamma=None) -> float:
        g = self.gamma if gamma is None else gamma
        if g == 0.0:
            return 0.0
        return g * float(self._terms(x, True)[1])

    def _auto_gamma(self) -> float:
        """Balance the two integrals under the reference's deterministic 0.1 h perturbation."""
        rng = np.random.default_rng(20201717)
        free = self.free_interior_mask()
        dx = np.zeros_like(self.x0)
        dx[free] = rng.uniform(-1.0, 1.0, size=int(free.sum()))
        x_ref = self.x0 + dx * (0.1 * self.dlim[:, None])
        f_mu, lim = self._terms(x_ref, True)
        return 0.0 if lim <= 0.0 else f_mu / lim

    def objective(self, x) -> float:
        """F(x); +inf when det A <= 0 at any point (the line search's sentinel)."""
        f_mu, lim = self._terms(x, self.gamma != 0.0)
        if not np.isfinite(f_mu):
            return np.inf
        return f_mu + (self.gamma * lim if self.gamma != 0.0 else 0.0)

    def _derivative(self, fn, what, x, *more):
        X = to_dev(x)
        args = [to_dev(m) for m in more]
        out = empty(tuple(X.shape))
        self._ctx.sync_stream()
        rc = fn(self._h, _lib.ptr(X), *[_lib.ptr(a) for a in args], _lib.ptr(out))
        if rc == _lib.HX_EINVERTED:
            raise ValueError(f"{what} undefined: mesh has non-positive Jacobians")
        self._ctx.check(rc, what)
        return like(out, x)

    def gradient(self, x):
        return self._derivative(self._ctx.lib.hx_tmop_gradient, "gradient", x)

    def hessian_action(self, x, dx):
        return self._derivative(self._ctx.lib.hx_tmop_hessian_action, "Hessian", x, dx)

    def hessian_diagonal(self, x):
        return self._derivative(self._ctx.lib.hx_tmop_hessian_diagonal, "diagonal", x)


# ---------------------------------------------------------------------------
# Newton solver (meshopt.py:488-566): host orchestration of the device derivatives

@dataclass
class NewtonResult:
    x: np.ndarray
    iterations: int
    converged: bool
    objective_history: list
    grad_norm: float


def _backtrack(obj, x, step, f):
    """Largest alpha in 1, 1/2, ..., 2^-19 with F(x + alpha step) < f, or None."""
    alpha = 1.0
    for _ in range(20):
        ft = obj.objective(x + alpha * step)
        if ft < f:
            return alpha, ft
        alpha *= 0.5
    return None, None


def newton_solve(obj: TMOPObjective, x_init, rel_tol: float = 1e-10, abs_tol: float = 1e-12, max_newton: int = 30,
                 cg_tol: float = 1e-8, cg_max_iter: int = 100, free_mask=None) -> NewtonResult:
    """Newton with a Jacobi-PCG inner solve on the free nodes and a backtracking line search
    that never accepts det A <= 0; falls back to gradient descent when the Hessian is
    indefinite or the Newton step does not decrease F."""
    free = obj.free_interior_mask() if free_mask is None else np.asarray(free_mask, dtype=bool)
    x = np.array(x_init, dtype=float)
    f = obj.objective(x)
    if not np.isfinite(f):
        raise ValueError("initial mesh is invalid (det A <= 0 somewhere)")
    hist = [f]
    grad = lambda y: np.where(free, np.asarray(obj.gradient(y)), 0.0)  # noqa: E731
    g = grad(x)
    g0 = gn = float(np.linalg.norm(g))
    it = 0
    while it < max_newton and gn > max(rel_tol * g0, abs_tol):
        dg = np.where(free, np.asarray(obj.hessian_diagonal(x)), 1.0)
        dg = np.where(dg > 1e-14, dg, 1.0)

        def hop(v):
            v = np.where(free, np.asarray(v).reshape(x.shape), 0.0)
            return np.where(free, np.asarray(obj.hessian_action(x, v)), v).ravel()

        try:
            s, _ = cg_solve(hop, -g.ravel(), precond_diag=dg.ravel(), rel_tol=cg_tol, max_iter=cg_max_iter)
            step = np.where(free, np.asarray(s).reshape(x.shape), 0.0)
        except CGError:
            step = np.where(free, -g, 0.0)
        alpha, ft = _backtrack(obj, x, step, f)
        if alpha is None:
            step = np.where(free, -g, 0.0)
            alpha, ft = _backtrack(obj, x, step, f)
            if alpha is None:
                return NewtonResult(x, it, False, hist, gn)
        x = x + alpha * step
        f = ft
        hist.append(f)
        g = grad(x)
        gn = float(np.linalg.norm(g))
        it += 1
    return NewtonResult(x, it, gn <= max(rel_tol * g0, abs_tol), hist, gn)
