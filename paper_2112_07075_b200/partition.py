"""Brick domain decomposition of a cartesian hex/quad mesh (the paper's P operator).

The reference runs single-process (P = identity; PAPER.md:217-225,295
describes the MPI decomposition).  Here the element grid of `cartesian_mesh` is split
into px*py*pz bricks, one per rank.  Each rank gets

  * a local cartesian mesh over its brick (local lexicographic numbering, x fastest),
    with coordinates copied from the global mesh;
  * `l2g`: local node id -> global node id, with the invariant
        global.node_dofmap[:, g_elems[e]] == l2g[local.node_dofmap[:, e]]   (bit-exact);
  * the shared-node halo plan: for every node on an inter-rank interface, the ranks
    that hold it (ascending), and per neighbour the shared local nodes sorted by global id;
  * `owned`: 1 where this rank is the lowest rank holding the node (dot products count
    every node once);
  * the wall mask restricted from the GLOBAL box (subdomain faces are not walls).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .fespace import HighOrderMesh, cartesian_mesh

__all__ = ["Subdomain", "rank_grid", "brick_partition"]


def rank_grid(nranks: int, dim: int, counts) -> tuple:
    """px*py(*pz) = nranks, splitting the longest element axis first."""
    dims = [1] * dim
    n = nranks
    f = 2
    factors = []
    while n > 1:
        while n % f == 0:
            factors.append(f)
            n //= f
        f += 1
    for fac in sorted(factors, reverse=True):
        per = [counts[a] / dims[a] for a in range(dim)]
        a = int(np.argmax(per))
        dims[a] *= fac
    for a in range(dim):
        if dims[a] > counts[a]:
            raise ValueError(f"cannot split {counts[a]} elements over {dims[a]} ranks on axis {a}")
    return tuple(dims)


def _split(n: int, parts: int):
    base, extra = divmod(n, parts)
    sizes = [base + (1 if i < extra else 0) for i in range(parts)]
    starts = np.concatenate(([0], np.cumsum(sizes)))
    return [(int(starts[i]), int(starts[i + 1])) for i in range(parts)]


@dataclass
class Subdomain:
    rank: int
    nranks: int
    grid: tuple
    coord: tuple
    mesh: HighOrderMesh            # local mesh (global coordinates)
    l2g: np.ndarray                # (NN_local,) global node ids
    g_elems: np.ndarray            # (NE_local,) global element ids
    owned: np.ndarray              # (NN_local,) bool
    neighbors: list                # ranks sharing at least one node, ascending
    shared: dict                   # neighbor rank -> local node ids sorted by global id
    sharers: dict = field(default_factory=dict)  # local node id -> tuple of ranks (ascending), interface nodes only
    bc_mask: np.ndarray | None = None


def brick_partition(dim: int, extents, counts, order: int, nranks: int, bc_mask_global=None):
    """Split cartesian_mesh(dim, extents, counts, order) into nranks bricks.

    Returns (global_mesh, [Subdomain for each rank])."""
    counts = tuple(int(c) for c in counts)
    gmesh = cartesian_mesh(dim, extents, counts, order)
    grid = rank_grid(nranks, dim, counts)
    p = order
    nper = [c * p + 1 for c in counts]
    strides = np.cumprod([1] + nper[:-1])
    ranges = [_split(counts[a], grid[a]) for a in range(dim)]
    # node index ranges per rank per axis (inclusive of the shared interface layer)
    subs = []
    coords_of = {}
    for r in range(nranks):
        c = np.unravel_index(r, grid, order="F")
        coords_of[r] = tuple(int(x) for x in c)
    node_ranges = {r: [(ranges[a][coords_of[r][a]][0] * p, ranges[a][coords_of[r][a]][1] * p)
                       for a in range(dim)] for r in range(nranks)}
    for r in range(nranks):
        cr = coords_of[r]
        ecount = [ranges[a][cr[a]][1] - ranges[a][cr[a]][0] for a in range(dim)]
        estart = [ranges[a][cr[a]][0] for a in range(dim)]
        lmesh = cartesian_mesh(dim, np.ones(dim), ecount, p)
        # local node (i0, i1, i2) -> global node id
        lper = [ecount[a] * p + 1 for a in range(dim)]
        lidx = np.unravel_index(np.arange(lmesh.num_nodes), lper, order="F")
        l2g = np.zeros(lmesh.num_nodes, dtype=np.int64)
        for a in range(dim):
            l2g += (lidx[a] + estart[a] * p) * strides[a]
        lmesh.coords = gmesh.coords[l2g].copy()
        lmesh._hx_ctx = {}
        eidx = np.unravel_index(np.arange(lmesh.num_elements), ecount, order="F")
        g_elems = np.zeros(lmesh.num_elements, dtype=np.int64)
        gstr = np.cumprod([1] + list(counts[:-1]))
        for a in range(dim):
            g_elems += (eidx[a] + estart[a]) * gstr[a]
        # sharers of every local node: ranks whose node box contains it
        gcoord = [lidx[a] + estart[a] * p for a in range(dim)]
        holders = [[] for _ in range(lmesh.num_nodes)]
        sharers = {}
        for q in range(nranks):
            inside = np.ones(lmesh.num_nodes, dtype=bool)
            for a in range(dim):
                lo, hi = node_ranges[q][a]
                inside &= (gcoord[a] >= lo) & (gcoord[a] <= hi)
            for i in np.flatnonzero(inside):
                holders[i].append(q)
        owned = np.array([min(h) == r for h in holders])
        neighbors = sorted({q for h in holders for q in h if q != r})
        shared = {}
        for q in neighbors:
            ids = np.array([i for i, h in enumerate(holders) if q in h], dtype=np.int64)
            shared[q] = ids[np.argsort(l2g[ids], kind="stable")]
        for i, h in enumerate(holders):
            if len(h) > 1:
                sharers[i] = tuple(sorted(h))
        sub = Subdomain(rank=r, nranks=nranks, grid=grid, coord=cr, mesh=lmesh, l2g=l2g, g_elems=g_elems,
                        owned=owned, neighbors=neighbors, shared=shared, sharers=sharers)
        if bc_mask_global is not None:
            sub.bc_mask = np.asarray(bc_mask_global)[l2g]
        subs.append(sub)
    return gmesh, subs
