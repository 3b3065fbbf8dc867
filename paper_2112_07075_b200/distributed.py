"""Distributed Lagrange step over a brick decomposition (torch.distributed: NCCL or gloo).

Per rank, the element work (geometry, stress, force, PA mass action, energy solve)
runs on the local subdomain through a `LocalOps` backend -- `DeviceOps` calls
libb200hydro.so; the CPU tests plug in the oracle.  This module adds the exchange
steps the single-process reference does not need (P = identity):

  * halo_sum: shared-node partial sums of an H1 field, combined in ascending rank
    order, so every rank ends with bit-identical values at shared nodes;
  * dot: sum over owned nodes (each node once), allreduce-sum;
  * allreduce-min of the CFL ratio, allreduce-max of "inverted" and clamp counts.

The step follows the reference control flow exactly (timestep_estimate hydro.py:364-373,
rk2_step :375-405, rates :346-360, _solve_momentum :319-337, cg_solve operators.py:333-366).
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

__all__ = ["Halo", "DistributedLagrange", "DeviceOps"]


class Halo:
    """Shared-node exchange plan of one subdomain."""

    def __init__(self, sub, device):
        self.sub = sub
        self.device = device
        self.rank = sub.rank
        self.nbrs = list(sub.neighbors)
        self.send_idx = {q: torch.as_tensor(sub.shared[q], device=device) for q in self.nbrs}
        ids = sorted(sub.sharers)
        self.nodes = torch.as_tensor(np.array(ids, dtype=np.int64), device=device)
        # for every shared node and every sharer (ascending), where its partial lives:
        # column j of `src` indexes the concatenation [own values; recv from nbr0; recv from nbr1; ...]
        pos = {q: {int(n): i for i, n in enumerate(sub.shared[q])} for q in self.nbrs}
        offs, o = {}, len(ids)
        for q in self.nbrs:
            offs[q] = o
            o += len(sub.shared[q])
        maxs = max((len(sub.sharers[i]) for i in ids), default=1)
        src = np.full((len(ids), maxs), -1, dtype=np.int64)
        for row, i in enumerate(ids):
            for j, q in enumerate(sub.sharers[i]):
                src[row, j] = row if q == self.rank else offs[q] + pos[q][i]
        self.src = torch.as_tensor(src, device=device)
        self.owned = torch.as_tensor(sub.owned, device=device)
        # gloo moves host tensors; NCCL moves device tensors directly over NVLink
        self.comm = "cpu" if dist.get_backend() == "gloo" else device

    def sum(self, vec: torch.Tensor) -> torch.Tensor:
        """Complete the shared-node sums of a locally scattered H1 field (NN_local[, d])."""
        if not self.nbrs:
            return vec
        sends = {q: vec[self.send_idx[q]].contiguous().to(self.comm) for q in self.nbrs}
        recvs = {q: torch.empty_like(sends[q]) for q in self.nbrs}
        ops = []
        for q in self.nbrs:
            ops.append(dist.P2POp(dist.isend, sends[q], q))
            ops.append(dist.P2POp(dist.irecv, recvs[q], q))
        for req in dist.batch_isend_irecv(ops):
            req.wait()
        own = vec[self.nodes]
        cat = torch.cat([own] + [recvs[q].to(vec.device) for q in self.nbrs], dim=0)
        total = torch.zeros_like(own)
        for j in range(self.src.shape[1]):  # ascending rank order, from 0.0
            col = self.src[:, j]
            have = col >= 0
            add = cat[col.clamp(min=0)]
            if vec.dim() > 1:
                have = have[:, None]
            total = torch.where(have, total + add, total)
        out = vec.clone()
        out[self.nodes] = total
        return out

    def dot(self, a: torch.Tensor, b: torch.Tensor) -> float:
        w = self.owned if a.dim() == 1 else self.owned[:, None]
        s = torch.sum(torch.where(w, a * b, torch.zeros((), dtype=a.dtype, device=a.device)), dtype=torch.float64)
        s = s.reshape(1).to(torch.float64).to(self.comm)
        dist.all_reduce(s, op=dist.ReduceOp.SUM)
        return float(s.item())

    def any_nonzero(self, a: torch.Tensor) -> bool:
        t = torch.tensor([1.0 if bool(torch.any(a != 0)) else 0.0], dtype=torch.float64, device=self.comm)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return bool(t.item() > 0)

    def amin(self, x: float) -> float:
        t = torch.tensor([x], dtype=torch.float64, device=self.comm)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        return float(t.item())

    def amax(self, x: float) -> float:
        t = torch.tensor([x], dtype=torch.float64, device=self.comm)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def asum(self, x: float) -> float:
        t = torch.tensor([x], dtype=torch.float64, device=self.comm)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())


class DistributedLagrange:
    """The reference Lagrange step on a brick partition (one rank per subdomain)."""

    def __init__(self, sub, ops, gamma, q1=0.5, q2=2.0, momentum_rel_tol=1e-8, device="cpu"):
        self.sub, self.ops = sub, ops
        self.halo = Halo(sub, device)
        self.device = device
        self.gamma, self.q1, self.q2 = gamma, q1, q2
        self.tol = momentum_rel_tol
        self.mask = torch.as_tensor(np.asarray(sub.bc_mask, dtype=bool), device=device)
        self.clamps = 0

    def T(self, a):
        return torch.as_tensor(np.asarray(a) if not isinstance(a, torch.Tensor) else a, device=self.device,
                               dtype=torch.float64)

    def begin_phase(self, x, qdata0):
        self.ops.begin_phase(x, qdata0)
        d = self.halo.sum(self.T(self.ops.mass_diagonal()))
        md = d[:, None].expand(-1, self.sub.mesh.dim)
        self.precond = torch.where(self.mask, torch.ones((), dtype=torch.float64, device=self.device), md)
        self.inv_diag = 1.0 / self.precond

    # -- CG (cg_solve operators.py:333-366 with the wall rows of hydro.py:319-337) --
    def solve_momentum(self, rhs_v):
        m = self.mask
        zero = torch.zeros((), dtype=torch.float64, device=self.device)
        b = torch.where(m, zero, rhs_v)
        x = torch.zeros_like(b)
        if not self.halo.any_nonzero(b):
            return x, 0
        r = b.clone()
        z = self.inv_diag * r
        p = z.clone()
        rz = self.halo.dot(r, z)
        norm0 = np.sqrt(rz)
        for it in range(1, 2001):
            Ap = self.halo.sum(self.T(self.ops.mass_apply(torch.where(m, zero, p))))
            Ap = torch.where(m, p, Ap)
            pAp = self.halo.dot(p, Ap)
            if pAp <= 0.0:
                raise RuntimeError(f"CG breakdown: p^T A p = {pAp:.3e} <= 0")
            alpha = rz / pAp
            x = x + alpha * p
            r = r - alpha * Ap
            z = self.inv_diag * r
            rz_new = self.halo.dot(r, z)
            if np.sqrt(max(rz_new, 0.0)) <= self.tol * norm0:
                return x, it
            p = z + (rz_new / rz) * p
            rz = rz_new
        raise RuntimeError("CG did not converge in 2000 iterations")

    def rates(self, x, v, e, qdata0):
        """(dx, dv, de, ratio, clamped) or raises Inverted if any rank's geometry is inverted."""
        res = self.ops.stress_force(x, v, e, qdata0, self.gamma, self.q1, self.q2)
        bad = self.halo.amax(1.0 if res["inverted"] else 0.0)
        if bad > 0:
            raise Inverted()
        rhs_v = -self.halo.sum(self.T(res["F1"]))
        dv, it = self.solve_momentum(rhs_v)
        de = self.T(self.ops.energy_solve(res["Ftv"]))
        clamped = int(self.halo.asum(float(res["clamped"])))
        return v.clone(), dv, de, self.halo.amin(res["ratio"]), clamped, it

    def timestep_estimate(self, x, v, e, qdata0, t, cfl, dt_min=1e-12, dt_max=1.0, t_final=1.0):
        res = self.ops.stress_force(x, v, e, qdata0, self.gamma, self.q1, self.q2, ratio_only=True)
        if self.halo.amax(1.0 if res["inverted"] else 0.0) > 0:
            raise Inverted()
        self.clamps += int(self.halo.asum(float(res["clamped"])))
        dt = min(cfl * self.halo.amin(res["ratio"]), dt_max, t_final - t)
        if dt < dt_min:
            raise RuntimeError(f"dt = {dt:.3e} fell below dt_min")
        return dt

    def rk2_step(self, x, v, e, qdata0, t, dt, max_retries=5):
        attempt = dt
        for _ in range(max_retries + 1):
            try:
                dx0, dv0, de0, _, c0, _ = self.rates(x, v, e, qdata0)
                self.clamps += c0
                half = attempt / 2.0
                xm, vm, em = x + half * dx0, v + half * dv0, e + half * de0
                dx1, dv1, de1, ratio1, c1, _ = self.rates(xm, vm, em, qdata0)
                self.clamps += c1
                xn, vn, en = x + attempt * dx1, v + attempt * dv1, e + attempt * de1
                ok = self.ops.geometry_ok(xn)
                if self.halo.amax(0.0 if ok else 1.0) > 0:
                    raise Inverted()
                return (xn, vn, en, t + attempt), {"dt": attempt, "min_h_over_speed": ratio1}
            except Inverted:
                attempt /= 2.0
        raise RuntimeError(f"step rejected {max_retries + 1} times")


class Inverted(Exception):
    pass


class DeviceOps:
    """LocalOps on the B200 library for one subdomain."""

    def __init__(self, sub, gamma, q1, q2):
        from .hydro import LagrangeHydro, MaterialModel, ViscosityModel
        from .tensor_basis import gauss_legendre

        self.sub = sub
        p = sub.mesh.order
        self.quad = gauss_legendre(p + 2)
        self.hy = LagrangeHydro(sub.mesh, self.quad, MaterialModel(gamma), ViscosityModel(q1, q2),
                                bc_mask=np.zeros_like(sub.bc_mask))

    def begin_phase(self, x, qdata0):
        from .hydro import HydroState

        st = HydroState(x, x, x, qdata0)
        self.hy.begin_phase(st)

    def mass_diagonal(self):
        return self.hy.mass_pa.diagonal()

    def mass_apply(self, x):
        return self.hy.mass_pa.apply(x)

    def stress_force(self, x, v, e, qdata0, gamma, q1, q2, ratio_only=False):
        from .fespace import InvertedElementError, compute_geometric_factors
        from .hydro import HydroState
        from .operators import ForcePA

        try:
            geom = compute_geometric_factors(self.sub.mesh, self.quad, x=x)
        except InvertedElementError:
            return {"inverted": True, "clamped": 0, "ratio": float("inf")}
        st = HydroState(x, v, e, qdata0)
        c0 = self.hy.clamp_warnings
        sigma, ratio = self.hy.stress_qdata(st, geom)
        out = {"inverted": False, "clamped": self.hy.clamp_warnings - c0, "ratio": ratio}
        if not ratio_only:
            f = ForcePA(self.hy.kin, self.hy.thermo, geom, sigma)
            out["F1"] = f.apply(torch.ones(self.hy.thermo.ndof, dtype=torch.float64, device=x.device)
                                if isinstance(x, torch.Tensor) else np.ones(self.hy.thermo.ndof))
            out["Ftv"] = f.apply_transpose(v)
        return out

    def energy_solve(self, rhs):
        return self.hy.solve_energy(rhs)

    def geometry_ok(self, x):
        from .fespace import InvertedElementError, compute_geometric_factors

        try:
            compute_geometric_factors(self.sub.mesh, self.quad, x=x)
            return True
        except InvertedElementError:
            return False
