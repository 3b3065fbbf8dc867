"""Initial conditions of the BASELINE.json configs, as (rho0_fn, v0_fn, e0_fn)
triples for `LagrangeHydro.initial_state` (hydro.py:189-218 calling convention:
rho0_fn(xq (d, nq, NE)), v0_fn(x (NN, d)), e0_fn(pts (d, nt, NE))).

The reference ships no presets (SPEC.md:791 lists no Sedov); these follow the
Laghos conventions named in SURVEY.md section 8d.
"""

from __future__ import annotations

import numpy as np

__all__ = ["sedov", "taylor_green", "triple_point", "triple_point_multi"]


def sedov(dim, extents, counts, energy=0.25):
    """rho0 = 1, v0 = 0, e = energy / V_elem in the element at the origin corner."""
    cell = np.asarray(extents, float) / np.asarray(counts, float)
    vol = float(np.prod(cell))

    def rho0(xq):
        return np.ones(xq.shape[1:])

    def v0(x):
        return np.zeros_like(x)

    def e0(pts):
        centroid = pts.mean(axis=1)
        at_origin = np.all(centroid < cell[:, None], axis=0)
        return np.where(at_origin[None, :], energy / vol, 0.0) * np.ones(pts.shape[1:])

    return rho0, v0, e0


def taylor_green(dim, gamma=5.0 / 3.0):
    """Unit box, rho = 1, v = (sin x cos y cos z, -cos x sin y cos z, 0) (pi-scaled),
    p = 100 + ((cos 2x + cos 2y)(cos 2z + 2) - 2)/16."""

    def rho0(xq):
        return np.ones(xq.shape[1:])

    def v0(x):
        s = np.pi * x
        if dim == 3:
            cz = np.cos(s[:, 2])
            return np.stack([np.sin(s[:, 0]) * np.cos(s[:, 1]) * cz,
                             -np.cos(s[:, 0]) * np.sin(s[:, 1]) * cz, np.zeros(len(x))], axis=1)
        return np.stack([np.sin(s[:, 0]) * np.cos(s[:, 1]), -np.cos(s[:, 0]) * np.sin(s[:, 1])], axis=1)

    def e0(pts):
        s = 2 * np.pi * pts
        if dim == 3:
            pr = 100.0 + ((np.cos(s[0]) + np.cos(s[1])) * (np.cos(s[2]) + 2.0) - 2.0) / 16.0
        else:
            pr = 100.0 + (np.cos(s[0]) + np.cos(s[1])) / 4.0
        return pr / (gamma - 1.0)

    return rho0, v0, e0


def triple_point(dim, gamma=1.5):
    """[0,7]x[0,3](x[0,1.5]): x<1 (rho,p)=(1,1); x>=1,y<1.5 (1,0.1); x>=1,y>=1.5 (0.125,0.1).
    Single gamma (the reference has one MaterialModel)."""

    def fields(pts):
        left, low = pts[0] < 1.0, pts[1] < 1.5
        rho = np.where(left, 1.0, np.where(low, 1.0, 0.125))
        return rho, np.where(left, 1.0, 0.1)

    def rho0(xq):
        return fields(xq)[0]

    def v0(x):
        return np.zeros_like(x)

    def e0(pts):
        rho, pr = fields(pts)
        return pr / ((gamma - 1.0) * rho)

    return rho0, v0, e0


TRIPLE_GAMMA = (1.5, 1.4, 1.5)  # Laghos triple point: left, lower-right, upper-right


def _triple_region(x, y):
    """0: x < 1; 1: x >= 1, y < 1.5; 2: x >= 1, y >= 1.5."""
    return np.where(x < 1.0, 0, np.where(y < 1.5, 1, 2))


def triple_point_multi(dim, counts, extents=(7.0, 3.0, 1.5)):
    """Multi-material triple point (Laghos convention): the three regions of `triple_point`
    with their own adiabatic index (1.5, 1.4, 1.5).  Returns (rho0_fn, v0_fn, e0_fn,
    gamma_e) with one gamma per element (element regions from the centroids; the region
    boundaries x = 1, y = 1.5 must be element faces).  A multi-material extension: the
    reference's MaterialModel has one gamma (hydro.py:40-48), so parity is against the
    oracle with the same per-element gamma."""
    ext = np.asarray(extents[:dim], float)
    cnt = np.asarray(counts[:dim], int)
    h = ext / cnt
    for a, b in ((0, 1.0), (1, 1.5)):
        if abs(b / h[a] - round(b / h[a])) > 1e-9:
            raise ValueError("triple-point region boundaries must be element faces")
    ne = int(np.prod(cnt))
    ec = np.array(np.unravel_index(np.arange(ne), cnt, order="F"), dtype=float)
    cen = (ec + 0.5) * h[:, None]
    reg = _triple_region(cen[0], cen[1])
    gamma_e = np.asarray(TRIPLE_GAMMA)[reg]

    def fields(pts):
        r = _triple_region(pts[0], pts[1])
        rho = np.where(r == 2, 0.125, 1.0)
        return rho, np.where(r == 0, 1.0, 0.1), np.asarray(TRIPLE_GAMMA)[r]

    def rho0(xq):
        return fields(xq)[0]

    def v0(x):
        return np.zeros_like(x)

    def e0(pts):
        rho, pr, g = fields(pts)
        return pr / ((g - 1.0) * rho)

    return rho0, v0, e0, gamma_e
