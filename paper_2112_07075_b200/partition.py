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

__all__ = ["Subdomain", "rank_grid", "brick_partition", "max_shared_nodes"]


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


def _axes(dim, extents, counts, p):
    """The 1D node coordinates of cartesian_mesh along every axis (same arithmetic, so the
    local coordinates below are bit-identical to the global mesh's)."""
    from .tensor_basis import gauss_lobatto_nodes

    lob = (gauss_lobatto_nodes(p) + 1.0) / 2.0
    ext = np.atleast_1d(np.asarray(extents, dtype=float))
    axes = []
    for a in range(dim):
        h = ext[a] / counts[a]
        pts = np.empty(counts[a] * p + 1)
        for c in range(counts[a]):
            pts[c * p:(c + 1) * p + 1] = c * h + lob * h
        axes.append(pts)
    return axes


def _layout(dim, counts, order, nranks):
    grid = rank_grid(nranks, dim, counts)
    ranges = [_split(counts[a], grid[a]) for a in range(dim)]
    coords_of = [tuple(int(x) for x in np.unravel_index(r, grid, order="F")) for r in range(nranks)]
    # node index ranges per rank per axis (inclusive of the shared interface layer)
    node_ranges = [[(ranges[a][coords_of[r][a]][0] * order, ranges[a][coords_of[r][a]][1] * order)
                    for a in range(dim)] for r in range(nranks)]
    return grid, ranges, coords_of, node_ranges


def max_shared_nodes(dim: int, counts, order: int, nranks: int) -> int:
    """Largest number of nodes two ranks share (the mailbox receive block size), from the
    brick layout alone -- no mesh is built (every rank computes the same value)."""
    counts = tuple(int(c) for c in counts)
    _, _, _, nr = _layout(dim, counts, order, nranks)
    best = 1
    for r in range(nranks):
        for q in range(nranks):
            if q == r:
                continue
            n = 1
            for a in range(dim):
                lo, hi = max(nr[r][a][0], nr[q][a][0]), min(nr[r][a][1], nr[q][a][1])
                n *= max(hi - lo + 1, 0)
            best = max(best, n)
    return best


def brick_partition(dim: int, extents, counts, order: int, nranks: int, bc_mask_global=None, ranks=None,
                    build_global: bool = True):
    """Split cartesian_mesh(dim, extents, counts, order) into nranks bricks.

    Returns (global_mesh, [Subdomain for each rank]).  `ranks` restricts the work to the
    listed ranks (the other entries are None) and `build_global=False` skips the global
    mesh (returned as None): one process per GPU then builds only its own brick, with the
    global box's wall mask computed from the global node coordinates (identical to
    box_velocity_bc(global_mesh)[l2g])."""
    counts = tuple(int(c) for c in counts)
    p = order
    gmesh = cartesian_mesh(dim, extents, counts, order) if build_global else None
    grid, ranges, coords_of, node_ranges = _layout(dim, counts, p, nranks)
    axes = _axes(dim, extents, counts, p)
    nper = [c * p + 1 for c in counts]
    strides = np.cumprod([1] + nper[:-1])
    gstr = np.cumprod([1] + list(counts[:-1]))
    want = range(nranks) if ranks is None else sorted(set(int(r) for r in ranks))
    subs = [None] * nranks
    for r in want:
        cr = coords_of[r]
        ecount = [ranges[a][cr[a]][1] - ranges[a][cr[a]][0] for a in range(dim)]
        estart = [ranges[a][cr[a]][0] for a in range(dim)]
        lmesh = cartesian_mesh(dim, np.ones(dim), ecount, p)
        # local node (i0, i1, i2) -> global node id
        lper = [ecount[a] * p + 1 for a in range(dim)]
        lidx = np.unravel_index(np.arange(lmesh.num_nodes), lper, order="F")
        gcoord = [np.asarray(lidx[a]) + estart[a] * p for a in range(dim)]
        l2g = np.zeros(lmesh.num_nodes, dtype=np.int64)
        for a in range(dim):
            l2g += gcoord[a] * strides[a]
        lmesh.coords = np.stack([axes[a][gcoord[a]] for a in range(dim)], axis=1)
        lmesh._hx_ctx = {}
        eidx = np.unravel_index(np.arange(lmesh.num_elements), ecount, order="F")
        g_elems = np.zeros(lmesh.num_elements, dtype=np.int64)
        for a in range(dim):
            g_elems += (np.asarray(eidx[a]) + estart[a]) * gstr[a]
        # H[q, i]: rank q's node box holds local node i (vectorised over nodes)
        H = np.ones((nranks, lmesh.num_nodes), dtype=bool)
        for q in range(nranks):
            for a in range(dim):
                lo, hi = node_ranges[q][a]
                H[q] &= (gcoord[a] >= lo) & (gcoord[a] <= hi)
        owned = np.argmax(H, axis=0) == r  # lowest holding rank
        neighbors = [q for q in range(nranks) if q != r and H[q].any()]
        shared = {}
        for q in neighbors:
            ids = np.flatnonzero(H[q]).astype(np.int64)
            shared[q] = ids[np.argsort(l2g[ids], kind="stable")]
        multi = np.flatnonzero(H.sum(axis=0) > 1)
        Hm = H[:, multi]
        sharers = {int(i): tuple(int(q) for q in np.flatnonzero(Hm[:, j])) for j, i in enumerate(multi)}
        sub = Subdomain(rank=r, nranks=nranks, grid=grid, coord=cr, mesh=lmesh, l2g=l2g, g_elems=g_elems,
                        owned=owned, neighbors=neighbors, shared=shared, sharers=sharers)
        if bc_mask_global is not None:
            sub.bc_mask = np.asarray(bc_mask_global)[l2g]
        elif not build_global:
            sub.bc_mask = _box_mask_local(lmesh.coords, axes)
        subs[r] = sub
    return gmesh, subs


def _box_mask_local(coords, axes, tol=1e-10):
    """box_velocity_bc of the GLOBAL box (hydro.py:118-131) restricted to local nodes: the
    global min / max coordinates are the first / last global 1D nodes."""
    d = coords.shape[1]
    mask = np.zeros(coords.shape, dtype=bool)
    for a in range(d):
        lo, hi = axes[a][0], axes[a].max()
        scale = max(hi - lo, 1.0)
        mask[:, a] = (np.abs(coords[:, a] - lo) < tol * scale) | (np.abs(coords[:, a] - hi) < tol * scale)
    return mask
