"""High-order meshes, H1/L2 spaces, E<->L restriction and geometric factors.

Drop-in for `ale_minihydro.fespace` on the hot path: `gather` / `scatter_add`
(fespace.py:221-234) and `compute_geometric_factors` (fespace.py:326-346) run in
libb200hydro.so (`hx_gather`, `hx_scatter_add`, `hx_geometry`).  The scatter
sums each node's element contributions in ascending element order starting from
0.0, which is bit-identical to the reference's `np.add.at`.

Mesh topology helpers that only TMOP/remap use (face orientation maps, mesh
text I/O) are out of scope; `boundary_nodes` is kept because the sealed-box
setup and the reference's test meshes use it.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._device import context_for, is_torch, like, to_dev, empty
from .tensor_basis import Basis1D, eval_basis, gauss_lobatto_nodes

__all__ = [
    "HighOrderMesh",
    "FiniteElementSpace",
    "GeometricFactors",
    "InvertedElementError",
    "cartesian_mesh",
    "compute_geometric_factors",
]


class InvertedElementError(RuntimeError):
    """det J <= 0 at (element, point); the first offender in q-major order (fespace.py:37-41)."""

    def __init__(self, element: int, point: int, detj: float):
        super().__init__(f"det J = {detj:.3e} <= 0 in element {element} at point {point}")
        self.element = element
        self.point = point


class HighOrderMesh:
    """Conforming quad/hex mesh with an order-p nodal coordinate field (fespace.py:63-102)."""

    def __init__(self, dim: int, order: int, node_dofmap: np.ndarray, coords: np.ndarray):
        if dim not in (2, 3):
            raise ValueError("mesh dimension must be 2 or 3")
        self.dim = dim
        self.order = order
        self.node_dofmap = np.ascontiguousarray(node_dofmap, dtype=np.int64)
        self.coords = np.ascontiguousarray(coords, dtype=float)
        self.num_nodes = self.coords.shape[0]
        self.lobatto_nodes = gauss_lobatto_nodes(order)
        if self.node_dofmap.shape[0] != (order + 1) ** dim:
            raise ValueError("node map does not match (p+1)^d local nodes")

    @property
    def num_elements(self) -> int:
        return self.node_dofmap.shape[1]

    def corner_ids(self) -> np.ndarray:
        """Corner node ids per element, (2^d, NE), x-fastest corners (fespace.py:82-90)."""
        p, d = self.order, self.dim
        loc = [sum(((c >> a) & 1) * p * (p + 1) ** a for a in range(d)) for c in range(2**d)]
        return self.node_dofmap[loc, :]

    def boundary_nodes(self) -> np.ndarray:
        """Ids of nodes on faces owned by a single element (fespace.py:110-121)."""
        p, d = self.order, self.dim
        ne = self.num_elements
        corners = self.corner_ids()
        local = np.arange((p + 1) ** d).reshape((p + 1,) * d)
        keys, faces = [], []
        for a in range(d):
            for s in (0, 1):
                cs = [c for c in range(2**d) if ((c >> a) & 1) == s]
                keys.append(np.sort(corners[cs, :], axis=0).T)  # (NE, 2^{d-1})
                sl = [slice(None)] * d
                sl[d - 1 - a] = -1 if s else 0
                faces.append(local[tuple(sl)].ravel())
        allk = np.concatenate(keys, axis=0)
        _, inv, counts = np.unique(allk, axis=0, return_inverse=True, return_counts=True)
        single = (counts[inv.ravel()] == 1).reshape(2 * d, ne)
        ids = [self.node_dofmap[faces[f]][:, single[f]].ravel() for f in range(2 * d)]
        ids = np.concatenate(ids) if ids else np.array([], dtype=np.int64)
        return np.unique(ids)


class FiniteElementSpace:
    """H1 (continuous) or L2 (discontinuous) space (fespace.py:177-255)."""

    def __init__(self, mesh: HighOrderMesh, continuity: str, order: int | None = None, vdim: int = 1):
        if continuity not in ("H1", "L2"):
            raise ValueError("continuity must be 'H1' or 'L2'")
        self.mesh = mesh
        self.continuity = continuity
        self.order = mesh.order if order is None else order
        self.vdim = vdim
        d = mesh.dim
        nloc = (self.order + 1) ** d
        if continuity == "H1":
            if self.order != mesh.order:
                raise ValueError("H1 spaces are supported at the mesh order only")
            self.dofmap = mesh.node_dofmap
            self.ndof = mesh.num_nodes
        else:
            ne = mesh.num_elements
            self.dofmap = np.arange(nloc * ne, dtype=np.int64).reshape(ne, nloc).T.copy()
            self.ndof = nloc * ne
        self.nloc = nloc
        self.nodes1d = np.zeros(1) if self.order == 0 else gauss_lobatto_nodes(self.order)
        self._basis_cache: dict = {}
        self._mult = None

    def basis(self, quad) -> Basis1D:
        key = (quad.n, quad.points.tobytes())
        b = self._basis_cache.get(key)
        if b is None:
            b = eval_basis(self.nodes1d, quad)
            self._basis_cache[key] = b
        return b

    def tshape(self, q1d: int) -> tuple:
        return (q1d,) * self.mesh.dim

    def _ctx(self):
        from .tensor_basis import gauss_legendre

        return context_for(self.mesh, gauss_legendre(self.mesh.order + 2))

    def gather(self, gvec):
        """G: (ndof, ...) -> E-vector (nloc, NE, ...) on the device (hx_gather)."""
        if gvec.shape[0] != self.ndof:
            raise ValueError(f"global vector has leading size {gvec.shape[0]}, expected {self.ndof}")
        extra = tuple(gvec.shape[1:])
        nc = int(np.prod(extra)) if extra else 1
        ne = self.mesh.num_elements
        L = to_dev(gvec)
        if self.continuity == "L2":
            E = L.reshape(ne, self.nloc, nc).transpose(0, 1).contiguous()
            return like(E.reshape((self.nloc, ne) + extra), gvec)
        ctx = self._ctx()
        E = empty((self.nloc, ne) + extra)
        ctx.sync_stream()
        ctx.check(ctx.lib.hx_gather(ctx.h, _lib.HX_SPACE_H1, _lib.ptr(L), nc, _lib.ptr(E)), "gather")
        return like(E, gvec)

    def scatter_add(self, evec):
        """G^T: ascending-element accumulation from 0.0 (hx_scatter_add), bit-identical to np.add.at."""
        expect = (self.nloc, self.mesh.num_elements)
        if tuple(evec.shape[:2]) != expect:
            raise ValueError(f"E-vector has shape {tuple(evec.shape)}, expected {expect} (+ components)")
        extra = tuple(evec.shape[2:])
        nc = int(np.prod(extra)) if extra else 1
        E = to_dev(evec)
        if self.continuity == "L2":
            ne = self.mesh.num_elements
            L = E.reshape(self.nloc, ne, nc).transpose(0, 1).contiguous() + 0.0  # 0.0 + x like add.at
            return like(L.reshape((self.ndof,) + extra), evec)
        ctx = self._ctx()
        L = empty((self.ndof,) + extra)
        ctx.sync_stream()
        ctx.check(ctx.lib.hx_scatter_add(ctx.h, _lib.HX_SPACE_H1, _lib.ptr(E), nc, _lib.ptr(L)), "scatter_add")
        return like(L, evec)

    def multiplicity(self):
        if self._mult is None:
            self._mult = self.scatter_add(np.ones((self.nloc, self.mesh.num_elements)))
        return self._mult

    def e_tensor(self, evec, extra: tuple = ()):
        """(nloc, NE, *extra) -> (n1,)*d + extra + (NE,) (layout only, fespace.py:243-250)."""
        d, n1, ne = self.mesh.dim, self.order + 1, self.mesh.num_elements
        if is_torch(evec):
            t = torch.movedim(evec.reshape((self.nloc, ne) + extra), 1, -1)
            return t.reshape((n1,) * d + extra + (ne,)).contiguous()
        t = np.moveaxis(evec.reshape((self.nloc, ne) + extra), 1, -1)
        return np.ascontiguousarray(t.reshape((n1,) * d + extra + (ne,)))

    def e_flat(self, t, extra: tuple = ()):
        ne = self.mesh.num_elements
        if is_torch(t):
            return torch.movedim(t.reshape((self.nloc,) + extra + (ne,)), -1, 1).contiguous()
        return np.ascontiguousarray(np.moveaxis(t.reshape((self.nloc,) + extra + (ne,)), -1, 1))


@dataclass
class GeometricFactors:
    """jac[a, b, q, e] = d x_a / d xi_b; detj, wdetj (nq, NE) (fespace.py:261-277).

    `jinv` follows the reference convention (fespace.py:280-302): J^{-1} in 2D,
    cof(J)/det = J^{-T} in 3D.  `x` records the positions the factors came from.
    """

    jac: object
    detj: object
    jinv: object
    wdetj: object
    quad: object
    basis: Basis1D
    x: object = None

    @property
    def volume(self) -> float:
        return float(self.wdetj.sum())


def compute_geometric_factors(mesh: HighOrderMesh, quad, x=None) -> GeometricFactors:
    """Jacobian, determinant, inverse, weighted determinant on the device (hx_geometry).

    Raises InvertedElementError naming the first (q-major) point with det J <= 0.
    """
    d = mesh.dim
    coords = mesh.coords if x is None else x
    ctx = context_for(mesh, quad)
    X = to_dev(coords)
    nq, ne = quad.n**d, mesh.num_elements
    jac, jinv = empty((d, d, nq, ne)), empty((d, d, nq, ne))
    detj, wdetj = empty((nq, ne)), empty((nq, ne))
    inv = _lib.Inverted()
    ctx.sync_stream()
    rc = ctx.lib.hx_geometry(ctx.h, _lib.ptr(X), _lib.ptr(jac), _lib.ptr(detj), _lib.ptr(jinv),
                             _lib.ptr(wdetj), inv)
    if rc == _lib.HX_EINVERTED:
        raise InvertedElementError(int(inv.element), int(inv.point), float(inv.detj))
    ctx.check(rc, "compute_geometric_factors")
    basis = eval_basis(mesh.lobatto_nodes, quad)
    return GeometricFactors(jac=like(jac, coords), detj=like(detj, coords), jinv=like(jinv, coords),
                            wdetj=like(wdetj, coords), quad=quad, basis=basis, x=coords)


def cartesian_mesh(dim: int, extents, counts, order: int) -> HighOrderMesh:
    """Axis-aligned box at tensor Lobatto nodes (fespace.py:352-385), vectorised.

    Global node id = sum_a (c_a*p + l_a) * stride_a with x fastest, identical to
    the reference numbering (restriction indices are bit-exact, tests/golden/mesh.npz).
    """
    extents = np.atleast_1d(np.asarray(extents, dtype=float))
    counts = np.atleast_1d(np.asarray(counts, dtype=int))
    if len(extents) != dim or len(counts) != dim:
        raise ValueError("extents and counts must match the dimension")
    if np.any(counts < 1):
        raise ValueError("element counts must be >= 1")
    p = order
    lob = (gauss_lobatto_nodes(p) + 1.0) / 2.0
    axes = []
    for a in range(dim):
        h = extents[a] / counts[a]
        pts = np.empty(counts[a] * p + 1)
        for c in range(counts[a]):
            pts[c * p : (c + 1) * p + 1] = c * h + lob * h
        axes.append(pts)
    nper = [len(ax) for ax in axes]
    grids = np.meshgrid(*axes, indexing="ij")
    coords = np.stack([g.reshape(-1, order="F") for g in grids], axis=1)
    ne = int(np.prod(counts))
    nl = (p + 1) ** dim
    strides = np.cumprod([1] + nper[:-1])
    ec = np.unravel_index(np.arange(ne), counts, order="F")
    lc = np.unravel_index(np.arange(nl), [p + 1] * dim, order="F")
    dofmap = np.zeros((nl, ne), dtype=np.int64)
    for a in range(dim):
        dofmap += (np.asarray(ec[a])[None, :] * p + np.asarray(lc[a])[:, None]) * strides[a]
    return HighOrderMesh(dim=dim, order=p, node_dofmap=dofmap, coords=coords)
