"""CPU oracle for the PA Lagrange hot path -- TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference algorithm
(`/root/reference/pkg/src/ale_minihydro`, the `ale_minihydro` package).  It is
the checker: only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s
cpu_baseline / `--impl reference` leg may import it.  The product package
(`paper_2112_07075_b200`) never imports or calls anything here.

Parity pinning: the oracle is checked against golden vectors produced by the
real reference in this container (`tests/golden/make_golden.py` imports
`/root/reference/pkg/src` and writes `tests/golden/*.npz`;
`tests/test_oracle_golden.py` compares).  See DESIGN.md section "Oracle".

Layouts follow the reference API (tensor_basis.py:7-13, fespace.py:243-255):
  element tensors (n_{d-1}, ..., n_0, NE), x fastest, NE last;
  E-vectors (nloc, NE[, comps]); H1 vector fields (NN, d); L2 fields (NE*nt,)
  element-major; point data (nq, NE); jacobians (d, d, nq, NE).

Every function cites the reference file:line it restates.
"""

from __future__ import annotations

import numpy as np

# ---------------------------------------------------------------------------
# 1D rules and bases (tensor_basis.py:75-172)


def _legendre(n, x):
    """P_n and P_n' by the three-term recurrence (tensor_basis.py:75-84)."""
    prev = np.ones_like(x)
    if n == 0:
        return prev, np.zeros_like(x)
    cur = x.copy()
    for k in range(1, n):
        prev, cur = cur, ((2 * k + 1) * x * cur - k * prev) / (k + 1)
    return cur, n * (x * cur - prev) / (x * x - 1.0)


def gauss_legendre(n):
    """(points, weights) of the n-point Gauss rule (tensor_basis.py:87-109)."""
    if n < 1:
        raise ValueError("need at least one quadrature point")
    if n == 1:
        return np.zeros(1), np.full(1, 2.0)
    x = np.cos(np.pi * (np.arange(n) + 0.75) / (n + 0.5))
    for _ in range(100):
        pn, dpn = _legendre(n, x)
        step = pn / dpn
        x -= step
        if np.max(np.abs(step)) < 1e-15:
            break
    x = np.sort(0.5 * (x - x[::-1]))
    _, dpn = _legendre(n, x)
    return x, 2.0 / ((1.0 - x * x) * dpn * dpn)


def gauss_lobatto(p):
    """p+1 Gauss-Lobatto nodes (tensor_basis.py:112-131)."""
    if p < 1:
        raise ValueError("Lobatto nodes need order >= 1")
    if p == 1:
        return np.array([-1.0, 1.0])
    x = np.cos(np.pi * np.arange(1, p) / p)
    for _ in range(100):
        pv, dp = _legendre(p, x)
        step = dp / ((2.0 * x * dp - p * (p + 1) * pv) / (1.0 - x * x))
        x -= step
        if np.max(np.abs(step)) < 1e-15:
            break
    x = 0.5 * (x - x[::-1])
    return np.concatenate(([-1.0], np.sort(x), [1.0]))


def basis_tables(nodes, pts):
    """B[q,i]=phi_i(x_q), G[q,i]=phi_i'(x_q), row-renormalised
    (lagrange_eval tensor_basis.py:134-155, eval_basis :158-172)."""
    nodes = np.asarray(nodes, float)
    pts = np.atleast_1d(np.asarray(pts, float))
    n = len(nodes)
    B = np.ones((len(pts), n))
    G = np.zeros((len(pts), n))
    for i in range(n):
        rest = [j for j in range(n) if j != i]
        for j in rest:
            B[:, i] *= (pts - nodes[j]) / (nodes[i] - nodes[j])
        for m in rest:
            t = np.full(len(pts), 1.0 / (nodes[i] - nodes[m]))
            for j in rest:
                if j != m:
                    t *= (pts - nodes[j]) / (nodes[i] - nodes[j])
            G[:, i] += t
    B /= B.sum(axis=1, keepdims=True)
    G -= G.mean(axis=1, keepdims=True)
    return B, G


def l2_nodes(order):
    """L2 nodes: Lobatto for order>=1, the origin for order 0 (fespace.py:199-202)."""
    return np.zeros(1) if order == 0 else gauss_lobatto(order)


# ---------------------------------------------------------------------------
# sum-factorised contractions (tensor_basis.py:207-273)


def along(mat, t, axis):
    """Apply mat (m_out, m_in) along tensor axis `axis` (contract_dim, :207-226)."""
    out = np.tensordot(mat, t, axes=(1, axis))
    return np.ascontiguousarray(np.moveaxis(out, 0, axis))


def interp(B, t, d):
    """B on every reference axis a; axis a is tensor axis a as written by the
    reference loop (tensor_interp :234-238)."""
    for a in range(d):
        t = along(B, t, a)
    return t


def interp_t(B, t, d):
    for a in range(d):
        t = along(B.T, t, a)
    return t


def grad(B, G, t, d):
    """[d t/d xi_a for a in 0..d-1]; ref axis b is tensor axis d-1-b (:248-261)."""
    out = []
    for a in range(d):
        g = t
        for b in range(d):
            g = along(G if b == a else B, g, d - 1 - b)
        out.append(g)
    return out


def grad_t(B, G, comps, d):
    acc = None
    for a in range(d):
        g = comps[a]
        for b in range(d):
            g = along(G.T if b == a else B.T, g, d - 1 - b)
        acc = g if acc is None else acc + g
    return acc


# ---------------------------------------------------------------------------
# mesh, restriction (fespace.py:184-255, 352-385)


def box_mesh(dim, extents, counts, p):
    """(dofmap (nl, NE) int64, coords (NN, dim)) of cartesian_mesh (fespace.py:352-385)."""
    extents = np.atleast_1d(np.asarray(extents, float))
    counts = np.atleast_1d(np.asarray(counts, int))
    lob = (gauss_lobatto(p) + 1.0) / 2.0
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
    # global node id = sum_a (ec_a * p + lc_a) * stride_a, x fastest for both
    strides = np.cumprod([1] + nper[:-1])
    ne = int(np.prod(counts))
    ecoord = np.array(np.unravel_index(np.arange(ne), counts, order="F"))  # (dim, NE)
    nl = (p + 1) ** dim
    lcoord = np.array(np.unravel_index(np.arange(nl), [p + 1] * dim, order="F"))  # (dim, nl)
    dofmap = np.zeros((nl, ne), dtype=np.int64)
    for a in range(dim):
        dofmap += (ecoord[a][None, :] * p + lcoord[a][:, None]) * strides[a]
    return dofmap, coords


def l2_dofmap(nl, ne):
    """L2 numbering: element-major (fespace.py:194-197)."""
    return np.arange(nl * ne, dtype=np.int64).reshape(ne, nl).T.copy()


def gather(dofmap, gvec):
    """G (fespace.py:221-225)."""
    return gvec[dofmap]


def scatter_add(dofmap, evec, ndof):
    """G^T, ascending-element accumulation from 0.0 (fespace.py:227-234)."""
    out = np.zeros((ndof,) + evec.shape[2:])
    np.add.at(out, dofmap.T, np.swapaxes(evec, 0, 1))
    return out


def e_tensor(evec, n1, d, extra=()):
    """E-vector (nl, NE, *extra) -> (n1,)*d + extra + (NE,) (fespace.py:243-250)."""
    nl, ne = evec.shape[0], evec.shape[1]
    t = np.moveaxis(evec.reshape((nl, ne) + extra), 1, -1)
    return np.ascontiguousarray(t.reshape((n1,) * d + extra + (ne,)))


def e_flat(t, nl, extra=()):
    """Inverse of e_tensor (fespace.py:252-255)."""
    ne = t.shape[-1]
    return np.ascontiguousarray(np.moveaxis(t.reshape((nl,) + extra + (ne,)), -1, 1))


# ---------------------------------------------------------------------------
# geometry (fespace.py:280-346)


class Inverted(Exception):
    """det J <= 0; carries the first (q-major) offender (fespace.py:37-41, 335-337)."""

    def __init__(self, element, point, detj):
        super().__init__(f"det J = {detj:.3e} <= 0 in element {element} at point {point}")
        self.element, self.point, self.detj = element, point, detj


def det_and_inv(jac):
    """det and the reference's 'inverse' (fespace.py:280-302).

    2D: adj(J)/det = J^{-1}.  3D: the reference fills inv[j, i] with the
    cofactor C_{ji}, i.e. cof(J)/det = J^{-T}.  Parity follows the code.
    """
    d = jac.shape[0]
    if d == 2:
        det = jac[0, 0] * jac[1, 1] - jac[0, 1] * jac[1, 0]
        inv = np.empty_like(jac)
        inv[0, 0], inv[0, 1] = jac[1, 1], -jac[0, 1]
        inv[1, 0], inv[1, 1] = -jac[1, 0], jac[0, 0]
        return det, inv
    det = (
        jac[0, 0] * (jac[1, 1] * jac[2, 2] - jac[1, 2] * jac[2, 1])
        - jac[0, 1] * (jac[1, 0] * jac[2, 2] - jac[1, 2] * jac[2, 0])
        + jac[0, 2] * (jac[1, 0] * jac[2, 1] - jac[1, 1] * jac[2, 0])
    )
    inv = np.empty_like(jac)
    for r in range(3):
        for c in range(3):
            rr = [k for k in range(3) if k != r]
            cc = [k for k in range(3) if k != c]
            minor = jac[rr[0], cc[0]] * jac[rr[1], cc[1]] - jac[rr[0], cc[1]] * jac[rr[1], cc[0]]
            inv[r, c] = minor if (r + c) % 2 == 0 else -minor
    return det, inv


def weights_nd(w, d):
    """Tensor weights laid out like the point index, x fastest (fespace.py:339-344)."""
    wq = w
    for _ in range(d - 1):
        wq = np.multiply.outer(wq, w)
    return wq.reshape(-1)


def geometry(dofmap, x, p, qpts, qw, d):
    """jac, detj, jinv, wdetj (element_jacobians :305-323, compute_geometric_factors :326-346)."""
    B, G = basis_tables(gauss_lobatto(p), qpts)
    ne = dofmap.shape[1]
    nq = len(qpts) ** d
    xe = x[dofmap]  # (nl, NE, d)
    jac = np.empty((d, d, nq, ne))
    for a in range(d):
        t = e_tensor(xe[:, :, a], p + 1, d)
        g = grad(B, G, t, d)
        for b in range(d):
            jac[a, b] = g[b].reshape(nq, ne)
    det, inv = det_and_inv(jac)
    bad = det <= 0.0
    if np.any(bad):
        q, e = np.argwhere(bad)[0]
        raise Inverted(int(e), int(q), float(det[q, e]))
    return jac, det, inv / det, weights_nd(qw, d)[:, None] * det


# ---------------------------------------------------------------------------
# PA operators (operators.py:84-324)


def mass_apply(dofmap, D, B, x, d):
    """y = G^T B^T D B G x per component (MassPA._apply_scalar/apply, operators.py:97-115)."""
    ndof = x.shape[0]
    n1 = B.shape[1]
    nq1 = B.shape[0]
    nl = dofmap.shape[0]

    def one(xs):
        t = e_tensor(gather(dofmap, xs), n1, d)
        q = interp(B, t, d)
        q = q * D.reshape((nq1,) * d + (-1,))
        return scatter_add(dofmap, e_flat(interp_t(B, q, d), nl), ndof)

    if x.ndim == 1:
        return one(x)
    return np.stack([one(x[:, c]) for c in range(x.shape[1])], axis=1)


def mass_diag(dofmap, D, B, ndof, d):
    """diag(M) via squared-basis contractions (MassPA.diagonal, operators.py:117-124)."""
    nq1 = B.shape[0]
    t = D.reshape((nq1,) * d + (-1,))
    B2 = B * B
    for a in range(d):
        t = along(B2.T, t, a)
    return scatter_add(dofmap, e_flat(t, dofmap.shape[0]), ndof)


def force_D(sigma, jinv, wdetj):
    """D_F[a,l] = sum_b sigma[a,b] jinv[l,b] wdetj (ForcePA.__init__, operators.py:258)."""
    return np.einsum("abqe,lbqe,qe->alqe", sigma, jinv, wdetj)


def force_apply(kin_dofmap, nn, DF, Bk, Gk, Bt, e_field, d):
    """(F e)_{a,i}, an (NN, d) array (ForcePA.apply, operators.py:264-280)."""
    ne = kin_dofmap.shape[1]
    nt1 = Bt.shape[1]
    nq1 = Bt.shape[0]
    nt = nt1**d
    te = e_tensor(gather(l2_dofmap(nt, ne), e_field), nt1, d)
    q = interp(Bt, te, d)
    Dq = DF.reshape((d, d) + (nq1,) * d + (ne,))
    nl = kin_dofmap.shape[0]
    cols = []
    for a in range(d):
        ta = grad_t(Bk, Gk, [Dq[a, l] * q for l in range(d)], d)
        cols.append(scatter_add(kin_dofmap, e_flat(ta, nl), nn))
    return np.stack(cols, axis=1)


def force_apply_t(kin_dofmap, DF, Bk, Gk, Bt, v, d):
    """(F^T v)_j (ForcePA.apply_transpose, operators.py:282-300)."""
    ne = kin_dofmap.shape[1]
    nq1 = Bt.shape[0]
    nt1 = Bt.shape[1]
    n1 = Bk.shape[1]
    tv = e_tensor(gather(kin_dofmap, v), n1, d, extra=(d,))
    Dq = DF.reshape((d, d) + (nq1,) * d + (ne,))
    s = None
    for a in range(d):
        g = grad(Bk, Gk, tv[(Ellipsis, a, slice(None))], d)
        for l in range(d):
            term = Dq[a, l] * g[l]
            s = term if s is None else s + term
    out = interp_t(Bt, s, d)
    return scatter_add(l2_dofmap(nt1**d, ne), e_flat(out, nt1**d), nt1**d * ne)


def diffusion_D(jinv, wdetj, nu=None):
    """D[a,c] = sum_b jinv[a,b] jinv[c,b] wdetj (nu) (DiffusionPA.__init__, operators.py:145-149)."""
    scal = wdetj if nu is None else wdetj * nu
    return np.einsum("abqe,cbqe,qe->acqe", jinv, jinv, scal)


def diffusion_apply(dofmap, D, B, G, x, d):
    """y = sum_a G_a^T (sum_b D[a,b] G_b x) (DiffusionPA.apply, operators.py:151-168)."""
    n1, nq1, nl = B.shape[1], B.shape[0], dofmap.shape[0]
    ne = dofmap.shape[1]
    t = e_tensor(gather(dofmap, x), n1, d)
    Dq = D.reshape((d, d) + (nq1,) * d + (ne,))
    g = grad(B, G, t, d)
    comps = []
    for a in range(d):
        s = Dq[a, 0] * g[0]
        for b in range(1, d):
            s = s + Dq[a, b] * g[b]
        comps.append(s)
    return scatter_add(dofmap, e_flat(grad_t(B, G, comps, d), nl), x.shape[0])


def convection_D(jinv, u_points, wdetj):
    """D[l] = sum_b jinv[l,b] u[b] wdetj (ConvectionPA.__init__, operators.py:194-198)."""
    return np.einsum("lbqe,bqe,qe->lqe", jinv, u_points, wdetj)


def convection_apply(dofmap, D, B, G, x, d):
    """y = B^T (sum_l D[l] G_l x) (ConvectionPA.apply, operators.py:200-214)."""
    n1, nq1, nl = B.shape[1], B.shape[0], dofmap.shape[0]
    ne = dofmap.shape[1]
    t = e_tensor(gather(dofmap, x), n1, d)
    Dq = D.reshape((d,) + (nq1,) * d + (ne,))
    g = grad(B, G, t, d)
    s = Dq[0] * g[0]
    for l in range(1, d):
        s = s + Dq[l] * g[l]
    return scatter_add(dofmap, e_flat(interp_t(B, s, d), nl), x.shape[0])


class CGFailure(Exception):
    def __init__(self, msg, residuals):
        super().__init__(msg)
        self.residuals = residuals


def cg(apply_op, b, precond_diag=None, rel_tol=1e-8, max_iter=1000):
    """Jacobi PCG, x0 = 0 (cg_solve, operators.py:333-366)."""
    b = np.asarray(b, float)
    x = np.zeros_like(b)
    if not np.any(b):
        return x, 0
    inv_diag = None if precond_diag is None else 1.0 / precond_diag
    r = b.copy()
    z = r if inv_diag is None else inv_diag * r
    p = z.copy()
    rz = float(np.vdot(r, z))
    norm0 = np.sqrt(rz)
    hist = [norm0]
    for it in range(1, max_iter + 1):
        Ap = apply_op(p)
        pAp = float(np.vdot(p, Ap))
        if pAp <= 0.0:
            raise CGFailure(f"CG breakdown: p^T A p = {pAp:.3e} <= 0", hist)
        alpha = rz / pAp
        x += alpha * p
        r -= alpha * Ap
        z = r if inv_diag is None else inv_diag * r
        rz_new = float(np.vdot(r, z))
        hist.append(np.sqrt(max(rz_new, 0.0)))
        if hist[-1] <= rel_tol * norm0:
            return x, it
        p = z + (rz_new / rz) * p
        rz = rz_new
    raise CGFailure(f"CG did not converge in {max_iter} iterations", hist)


# ---------------------------------------------------------------------------
# Lagrange phase (hydro.py:118-423)


class Underflow(Exception):
    pass


def box_mask(coords, extents=None, tol=1e-10):
    """Sealed-box wall mask (box_velocity_bc, hydro.py:118-131)."""
    d = coords.shape[1]
    lo = coords.min(axis=0)
    hi = coords.max(axis=0) if extents is None else np.asarray(extents, float)
    mask = np.zeros(coords.shape, dtype=bool)
    for a in range(d):
        s = max(hi[a] - lo[a], 1.0)
        mask[:, a] = (np.abs(coords[:, a] - lo[a]) < tol * s) | (np.abs(coords[:, a] - hi[a]) < tol * s)
    return mask


class Hydro:
    """Restatement of LagrangeHydro (hydro.py:134-423) for one phase.

    State is a dict {x, v, e, qdata0, t} with the reference layouts.
    """

    def __init__(self, dim, p, dofmap, coords, gamma, q1=0.5, q2=2.0, bc_mask=None,
                 momentum_rel_tol=1e-8, q1d=None, thermo_order=None):
        self.d, self.p = dim, p
        self.dofmap = dofmap
        self.coords0 = coords
        self.nn, self.ne = coords.shape[0], dofmap.shape[1]
        # gamma: one value (the reference) or one per element (multi-material extension)
        self.gamma = np.asarray(gamma, dtype=float)[None, :] if np.ndim(gamma) > 0 else gamma
        self.q1, self.q2 = q1, q2
        if np.any(np.asarray(gamma) <= 1.0):
            raise ValueError("adiabatic index must exceed 1")
        self.tol = momentum_rel_tol
        self.qpts, self.qw = gauss_legendre(p + 2 if q1d is None else q1d)
        self.nq1 = len(self.qpts)
        self.nq = self.nq1**dim
        self.to = max(p - 1, 0) if thermo_order is None else thermo_order
        self.tnodes = l2_nodes(self.to)
        self.nt1 = len(self.tnodes)
        self.nt = self.nt1**dim
        self.Bk, self.Gk = basis_tables(gauss_lobatto(p), self.qpts)
        self.Bt, _ = basis_tables(self.tnodes, self.qpts)
        self.mask = np.zeros((self.nn, dim), bool) if bc_mask is None else bc_mask
        self.tmap = l2_dofmap(self.nt, self.ne)
        self.ones_t = np.ones(self.nt * self.ne)
        self.clamps = 0

    # -- setup (hydro.py:176-232)
    def geom(self, x):
        return geometry(self.dofmap, x, self.p, self.qpts, self.qw, self.d)

    def points_physical(self, x):
        d = self.d
        xe = e_tensor(x[self.dofmap], self.p + 1, d, extra=(d,))
        return np.stack([interp(self.Bk, np.ascontiguousarray(xe[..., a, :]), d).reshape(self.nq, self.ne)
                         for a in range(d)])

    def initial_state(self, rho0_fn, v0_fn, e0_fn):
        d = self.d
        x = self.coords0.copy()
        _, det0, _, _ = self.geom(x)
        qdata0 = rho0_fn(self.points_physical(x)) * det0
        v = np.where(self.mask, 0.0, v0_fn(x))
        Bn, _ = basis_tables(gauss_lobatto(self.p), self.tnodes)
        xe = e_tensor(x[self.dofmap], self.p + 1, d, extra=(d,))
        pts = np.stack([interp(Bn, np.ascontiguousarray(xe[..., a, :]), d).reshape(self.nt, self.ne)
                        for a in range(d)])
        e = scatter_add(self.tmap, e0_fn(pts), self.nt * self.ne)
        st = dict(x=x, v=v, e=e, qdata0=qdata0, t=0.0)
        self.begin_phase(st)
        return st

    def begin_phase(self, st):
        _, det0, _, wdetj0 = self.geom(st["x"])
        Dm = (wdetj0 / det0) * st["qdata0"]
        self.Dm = Dm
        self.mdiag = mass_diag(self.dofmap, Dm, self.Bk, self.nn, self.d)
        Bfull = np.ones((1, 1))
        for _ in range(self.d):
            Bfull = np.kron(Bfull, self.Bt)
        self.Minv = np.linalg.inv(np.einsum("qi,qe,qj->eij", Bfull, Dm, Bfull))

    # -- point data (hydro.py:254-315)
    def stress(self, st, geo):
        d, ne, nq, g = self.d, self.ne, self.nq, self.gamma
        _, det, jinv, _ = geo
        rho = st["qdata0"] / det
        ep = interp(self.Bt, e_tensor(gather(self.tmap, st["e"]), self.nt1, d), d).reshape(nq, ne)
        neg = ep < 0.0
        if np.any(neg):
            self.clamps += int(neg.sum())
            ep = np.where(neg, 0.0, ep)
        pres = (g - 1.0) * rho * ep
        cs = np.sqrt(g * (g - 1.0) * ep)
        vt = e_tensor(gather(self.dofmap, st["v"]), self.p + 1, d, extra=(d,))
        gv = np.empty((d, d, nq, ne))
        vq = np.empty((d, nq, ne))
        for a in range(d):
            comp = np.ascontiguousarray(vt[..., a, :])
            refs = np.stack([r.reshape(nq, ne) for r in grad(self.Bk, self.Gk, comp, d)])
            gv[a] = np.einsum("lqe,lbqe->bqe", refs, jinv)
            vq[a] = interp(self.Bk, comp, d).reshape(nq, ne)
        sig = np.zeros((d, d, nq, ne))
        for a in range(d):
            sig[a, a] = -pres
        div = np.trace(gv, axis1=0, axis2=1)
        if self.q1 > 0.0 or self.q2 > 0.0:
            h = det ** (1.0 / d)
            mu = rho * h * (self.q1 * cs + self.q2 * h * np.abs(div))
            mu = np.where(div < 0.0, mu, 0.0)
            sig += mu * (0.5 * (gv + np.swapaxes(gv, 0, 1)))
        speed = cs + np.sqrt(np.sum(vq**2, axis=0))
        hh = det ** (1.0 / d)
        with np.errstate(divide="ignore"):
            ratio = np.where(speed > 0.0, hh / np.maximum(speed, 1e-300), np.inf)
        return sig, float(ratio.min())

    # -- semi-discrete rhs (hydro.py:319-360)
    def mass_op(self, x):
        return mass_apply(self.dofmap, self.Dm, self.Bk, x, self.d)

    def solve_momentum(self, rhs_v, rel_tol=None):
        m = self.mask
        rhs = np.where(m, 0.0, rhs_v)

        def op(w):
            w2 = w.reshape(rhs.shape)
            out = self.mass_op(np.where(m, 0.0, w2))
            return np.where(m, w2, out).ravel()

        diag = np.where(m, 1.0, self.mdiag[:, None] * np.ones_like(rhs))
        x, it = cg(op, rhs.ravel(), diag.ravel(), self.tol if rel_tol is None else rel_tol, 2000)
        self.last_cg_iters = it
        return x.reshape(rhs.shape)

    def solve_energy(self, rhs_e):
        return np.einsum("eij,ej->ei", self.Minv, rhs_e.reshape(self.ne, self.nt)).reshape(-1)

    def rates(self, st, rel_tol=None):
        geo = self.geom(st["x"])
        c0 = self.clamps
        sig, ratio = self.stress(st, geo)
        DF = force_D(sig, geo[2], geo[3])
        rhs_v = -force_apply(self.dofmap, self.nn, DF, self.Bk, self.Gk, self.Bt, self.ones_t, self.d)
        dv = self.solve_momentum(rhs_v, rel_tol)
        de = self.solve_energy(force_apply_t(self.dofmap, DF, self.Bk, self.Gk, self.Bt, st["v"], self.d))
        return dict(dx=st["v"].copy(), dv=dv, de=de, ratio=ratio, clamped=self.clamps - c0)

    # -- stepping (hydro.py:364-405)
    def timestep_estimate(self, st, cfl, dt_min=1e-12, dt_max=1.0, t_final=1.0):
        _, ratio = self.stress(st, self.geom(st["x"]))
        dt = min(cfl * ratio, dt_max, t_final - st["t"])
        if dt < dt_min:
            raise Underflow(f"dt = {dt:.3e} fell below dt_min = {dt_min:.3e} at t = {st['t']:.6e}")
        return dt

    def rk2_step(self, st, dt, max_retries=5):
        attempt = dt
        for _ in range(max_retries + 1):
            try:
                r0 = self.rates(st)
                half = attempt / 2.0
                mid = dict(x=st["x"] + half * r0["dx"], v=st["v"] + half * r0["dv"],
                           e=st["e"] + half * r0["de"], qdata0=st["qdata0"], t=st["t"] + half)
                r1 = self.rates(mid)
                new = dict(x=st["x"] + attempt * r1["dx"], v=st["v"] + attempt * r1["dv"],
                           e=st["e"] + attempt * r1["de"], qdata0=st["qdata0"], t=st["t"] + attempt)
                self.geom(new["x"])
                return new, {"dt": attempt, "min_h_over_speed": r1["ratio"]}
            except Inverted:
                attempt /= 2.0
        raise Underflow(f"step rejected {max_retries + 1} times from dt = {dt:.3e}")

    # -- diagnostics (hydro.py:242-252, 409-423)
    def kinetic_energy(self, st):
        return 0.5 * float(np.vdot(st["v"], self.mass_op(st["v"])))

    def internal_energy(self, st):
        d = self.d
        ep = interp(self.Bt, e_tensor(gather(self.tmap, st["e"]), self.nt1, d), d).reshape(self.nq, self.ne)
        return float(np.sum(weights_nd(self.qw, d)[:, None] * st["qdata0"] * ep))

    def total_energy(self, st):
        return self.kinetic_energy(st) + self.internal_energy(st)

    def total_mass(self, st):
        return float(np.sum(weights_nd(self.qw, self.d)[:, None] * st["qdata0"]))


# ---------------------------------------------------------------------------
# problem generators (BASELINE.json configs)


def sedov_fns(dim, extents, counts, energy=0.25):
    """Sedov: rho0=1, v0=0, e = energy/V_elem in the origin-corner element.

    e0_fn receives the thermo node coordinates (d, nt, NE) (hydro.py:204-218);
    the corner element is the one whose node centroid lies in the first cell.
    """
    h = np.asarray(extents, float) / np.asarray(counts, float)
    vol = float(np.prod(h))

    def rho0(xq):
        return np.ones(xq.shape[1:])

    def v0(x):
        return np.zeros_like(x)

    def e0(pts):
        cen = pts.mean(axis=1)  # (d, NE)
        corner = np.all(cen < h[:, None], axis=0)
        return np.where(corner[None, :], energy / vol, 0.0) * np.ones(pts.shape[1:])

    return rho0, v0, e0


def taylor_green_fns(dim, gamma=5.0 / 3.0):
    """Taylor-Green (Laghos convention), unit box, rho=1."""

    def rho0(xq):
        return np.ones(xq.shape[1:])

    def v0(x):
        X, Y = np.pi * x[:, 0], np.pi * x[:, 1]
        if dim == 3:
            Z = np.pi * x[:, 2]
            return np.stack([np.sin(X) * np.cos(Y) * np.cos(Z), -np.cos(X) * np.sin(Y) * np.cos(Z),
                             np.zeros_like(X)], axis=1)
        return np.stack([np.sin(X) * np.cos(Y), -np.cos(X) * np.sin(Y)], axis=1)

    def e0(pts):
        X, Y = 2 * np.pi * pts[0], 2 * np.pi * pts[1]
        if dim == 3:
            Z = 2 * np.pi * pts[2]
            pr = 100.0 + ((np.cos(X) + np.cos(Y)) * (np.cos(Z) + 2.0) - 2.0) / 16.0
        else:
            pr = 100.0 + (np.cos(X) + np.cos(Y)) / 4.0
        return pr / (gamma - 1.0)

    return rho0, v0, e0


def triple_point_fns(dim, gamma=1.5):
    """Triple point (Laghos convention, single gamma): [0,7]x[0,3](x[0,1.5]).
    Left x<1: rho=1,p=1; right-bottom y<1.5: rho=1,p=0.1; right-top: rho=0.125,p=0.1."""

    def region(pts):
        left = pts[0] < 1.0
        bottom = pts[1] < 1.5
        rho = np.where(left, 1.0, np.where(bottom, 1.0, 0.125))
        pr = np.where(left, 1.0, 0.1)
        return rho, pr

    def rho0(xq):
        return region(xq)[0]

    def v0(x):
        return np.zeros_like(x)

    def e0(pts):
        rho, pr = region(pts)
        return pr / ((gamma - 1.0) * rho)

    return rho0, v0, e0
