"""1D quadrature rules and nodal Lagrange bases (host-side setup tables).

Drop-in for `ale_minihydro.tensor_basis` (tensor_basis.py:24-172).  These
tables are computed once on the host and uploaded to the device context
(`hx_create`); every contraction that uses them runs in the sm_100a kernels
(csrc/hx_core.cuh).  The Newton iterations reproduce the reference's nodes and
weights bit for bit (checked against tests/golden/basis.npz), so both sides
start from identical B/G tables.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = [
    "QuadratureRule1D",
    "Basis1D",
    "gauss_legendre",
    "gauss_lobatto_nodes",
    "eval_basis",
    "lagrange_eval",
]


@dataclass(frozen=True)
class QuadratureRule1D:
    """Gauss rule on [-1, 1] (tensor_basis.py:41-50)."""

    points: np.ndarray
    weights: np.ndarray

    @property
    def n(self) -> int:
        return len(self.points)


@dataclass(frozen=True)
class Basis1D:
    """B[q, i] = phi_i(x_q), G[q, i] = phi_i'(x_q), shaped (Q1D, D1D) (tensor_basis.py:53-72)."""

    order: int
    nodes: np.ndarray
    B: np.ndarray
    G: np.ndarray

    @property
    def d1d(self) -> int:
        return self.order + 1

    @property
    def q1d(self) -> int:
        return self.B.shape[0]


def _legendre_pair(n: int, x: np.ndarray):
    # three-term recurrence for P_n and P_n' (tensor_basis.py:75-84)
    lo = np.ones_like(x)
    if n == 0:
        return lo, np.zeros_like(x)
    hi = x.copy()
    for k in range(1, n):
        lo, hi = hi, ((2 * k + 1) * x * hi - k * lo) / (k + 1)
    return hi, n * (x * hi - lo) / (x * x - 1.0)


def gauss_legendre(n: int) -> QuadratureRule1D:
    """n-point Gauss-Legendre rule; Newton from Chebyshev guesses (tensor_basis.py:87-109)."""
    if n < 1:
        raise ValueError("need at least one quadrature point")
    if n == 1:
        return QuadratureRule1D(np.zeros(1), np.full(1, 2.0))
    x = np.cos(np.pi * (np.arange(n) + 0.75) / (n + 0.5))
    for _ in range(100):
        pn, dpn = _legendre_pair(n, x)
        dx = pn / dpn
        x -= dx
        if np.max(np.abs(dx)) < 1e-15:
            break
    x = np.sort(0.5 * (x - x[::-1]))
    _, dpn = _legendre_pair(n, x)
    return QuadratureRule1D(x, 2.0 / ((1.0 - x * x) * dpn * dpn))


def gauss_lobatto_nodes(p: int) -> np.ndarray:
    """p+1 Gauss-Lobatto nodes (tensor_basis.py:112-131)."""
    if p < 1:
        raise ValueError("Lobatto nodes need order >= 1")
    if p == 1:
        return np.array([-1.0, 1.0])
    x = np.cos(np.pi * np.arange(1, p) / p)
    for _ in range(100):
        pv, dp = _legendre_pair(p, x)
        dx = dp / ((2.0 * x * dp - p * (p + 1) * pv) / (1.0 - x * x))
        x -= dx
        if np.max(np.abs(dx)) < 1e-15:
            break
    x = 0.5 * (x - x[::-1])
    out = np.empty(p + 1)
    out[0], out[-1] = -1.0, 1.0
    out[1:-1] = np.sort(x)
    return out


def lagrange_eval(nodes, x):
    """Lagrange basis values and derivatives by product formulas (tensor_basis.py:134-155)."""
    nodes = np.asarray(nodes, dtype=float)
    x = np.atleast_1d(np.asarray(x, dtype=float))
    n = len(nodes)
    vals = np.ones((len(x), n))
    ders = np.zeros((len(x), n))
    for i in range(n):
        rest = [j for j in range(n) if j != i]
        for j in rest:
            vals[:, i] *= (x - nodes[j]) / (nodes[i] - nodes[j])
        for m in rest:
            term = np.full(len(x), 1.0 / (nodes[i] - nodes[m]))
            for j in rest:
                if j != m:
                    term *= (x - nodes[j]) / (nodes[i] - nodes[j])
            ders[:, i] += term
    return vals, ders


def eval_basis(nodes, quad) -> Basis1D:
    """B/G at the rule's points, rows renormalised (sum B = 1, sum G = 0) (tensor_basis.py:158-172)."""
    nodes = np.asarray(nodes, dtype=float)
    if len(np.unique(nodes)) != len(nodes):
        raise ValueError("basis nodes must be distinct")
    pts = quad.points if hasattr(quad, "points") else np.asarray(quad, dtype=float)
    B, G = lagrange_eval(nodes, pts)
    B /= B.sum(axis=1, keepdims=True)
    G -= G.mean(axis=1, keepdims=True)
    return Basis1D(order=len(nodes) - 1, nodes=nodes, B=B, G=G)
