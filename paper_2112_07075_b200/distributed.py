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

__all__ = ["Halo", "DistributedLagrange", "DeviceOps", "PeerExchange", "peer_plan", "max_shared"]


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
        if getattr(self.ops, "peer", None) is not None:  # device-resident CG (hx_peer_*)
            return self.ops.solve_momentum(rhs_v, self.precond, self.mask, self.tol)
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

    peer = None  # PeerExchange once connected

    def solve_momentum(self, rhs, precond, mask, tol):
        """Jacobi PCG of the whole distributed mass system on the device: interface sums
        and world dot products move through the peer mailboxes inside the loop."""
        x, it = self.hy.mass_pa.solve(rhs, precond_diag=precond, bc_mask=mask, rel_tol=tol, max_iter=2000)
        return x, it

    def geometry_ok(self, x):
        from .fespace import InvertedElementError, compute_geometric_factors

        try:
            compute_geometric_factors(self.sub.mesh, self.quad, x=x)
            return True
        except InvertedElementError:
            return False


# ---------------------------------------------------------------------------
# device-resident CG exchange (libb200hydro.so hx_peer_*, csrc/hx_peer.cuh)

def max_shared(subs) -> int:
    """Longest shared-node list over all rank pairs (the mailbox receive block size)."""
    return max([len(ids) for s in subs for ids in s.shared.values()] + [1])


def peer_plan(sub):
    """Flat exchange plan of one subdomain (include/b200hydro.h, hx_peer_setup)."""
    snode, sdst, sidx = [], [], []
    for q in sub.neighbors:
        ids = sub.shared[q]
        snode.extend(int(n) for n in ids)
        sdst.extend([q] * len(ids))
        sidx.extend(range(len(ids)))
    pos = {q: {int(n): i for i, n in enumerate(sub.shared[q])} for q in sub.neighbors}
    hnode = sorted(sub.sharers)
    hoff, hsrc = [0], []
    for n in hnode:
        for q in sub.sharers[n]:  # ascending rank
            hsrc.append(-1 if q == sub.rank else (q << 24) | pos[q][n])
        hoff.append(len(hsrc))
    i32 = lambda a: np.ascontiguousarray(np.asarray(a, dtype=np.int32).reshape(-1))
    return dict(snode=i32(snode), sdst=i32(sdst), sidx=i32(sidx), hnode=i32(hnode), hoff=i32(hoff),
                hsrc=i32(hsrc), nbr=i32(sub.neighbors), owned=np.ascontiguousarray(sub.owned, dtype=np.uint8))


class PeerExchange:
    """Mailbox of one rank's device context; connect() maps every rank's mailbox.

    Ranks in one process (tests on one GPU): connect_local([...]).  One process per GPU:
    connect_ipc() exchanges CUDA IPC handles through torch.distributed."""

    def __init__(self, target, sub, maxh):
        """target: a DeviceOps (its MassPA's CG exchanges; the rest of the step stays in
        DistributedLagrange) or a LagrangeHydro on the subdomain (its whole step graph --
        rates, F.1 halo, CG, status, validity -- exchanges on the device).  Connect before
        LagrangeHydro.begin_phase: the mass diagonal's interface sums are exchanged there."""
        import ctypes as C

        from . import _lib
        from ._device import context_for

        self.ops, self.sub, self.maxh = target, sub, int(maxh)
        if hasattr(target, "hy"):
            self._ctx = context_for(sub.mesh, target.quad)  # the context MassPA runs its CG in
        else:
            self._ctx = target._ctx  # LagrangeHydro's private context: hx_phase_begin / hx_step
        lib, h = self._ctx.lib, self._ctx.h
        self.plan = pl = peer_plan(sub)
        ptr = lambda a: a.ctypes.data_as(C.c_void_p) if a.size else None
        mb = C.c_void_p()
        rc = lib.hx_peer_setup(h, sub.rank, sub.nranks, self.maxh, int(pl["snode"].size), ptr(pl["snode"]),
                               ptr(pl["sdst"]), ptr(pl["sidx"]), int(pl["hnode"].size), ptr(pl["hnode"]),
                               ptr(pl["hoff"]), ptr(pl["hsrc"]), int(pl["nbr"].size), ptr(pl["nbr"]),
                               ptr(pl["owned"]), C.byref(mb))
        self._ctx.check(rc, "hx_peer_setup")
        self.mailbox = int(mb.value)
        self._opened = []
        self._C, self._lib = C, _lib

    def _connect(self, ptrs):
        C = self._C
        arr = (C.c_void_p * len(ptrs))(*[C.c_void_p(p) for p in ptrs])
        self._ctx.check(self._ctx.lib.hx_peer_connect(self._ctx.h, arr), "hx_peer_connect")
        self.ops.peer = self

    def _warm(self):
        """Run one solo CG (zero right-hand side) so that every CG kernel is loaded before
        ranks sharing a process start spinning on each other (lazy module loading)."""
        import torch

        nn, d = self.sub.mesh.num_nodes, self.sub.mesh.dim
        z = torch.zeros((nn, d), dtype=torch.float64, device="cuda")
        self.ops.hy.mass_pa.solve(z, precond_diag=torch.ones_like(z), bc_mask=None, rel_tol=1e-8, max_iter=8)
        torch.cuda.synchronize()

    @staticmethod
    def connect_local(exchanges):
        """Ranks sharing one process (and one GPU): mailboxes are plain device pointers."""
        ptrs = [x.mailbox for x in sorted(exchanges, key=lambda x: x.sub.rank)]
        for x in exchanges:
            if hasattr(x.ops, "hy"):
                x._warm()
            x._connect(ptrs)

    def connect_ipc(self):
        C, lib = self._C, self._ctx.lib
        hbuf = (C.c_char * 64)()
        self._ctx.check(lib.hx_peer_ipc_handle(C.c_void_p(self.mailbox), hbuf), "hx_peer_ipc_handle")
        handles = [None] * self.sub.nranks
        dist.all_gather_object(handles, bytes(hbuf))
        ptrs = []
        for q, hq in enumerate(handles):
            if q == self.sub.rank:
                ptrs.append(self.mailbox)
                continue
            p = C.c_void_p()
            self._ctx.check(lib.hx_peer_ipc_open(C.create_string_buffer(hq, 64), C.byref(p)), "hx_peer_ipc_open")
            self._opened.append(p.value)
            ptrs.append(p.value)
        self._connect(ptrs)

    def close(self):
        """Leave the exchange after the last step: wait for this rank's queued work, detach
        the context (hx_peer_disconnect: peer pointers and exchange graphs dropped), wait
        for every rank to get here, then unmap the other ranks' IPC mailboxes.  Steps on
        this context afterwards run solo (call begin_phase again first)."""
        C = self._C
        self._ctx.check(self._ctx.lib.hx_peer_disconnect(self._ctx.h), "hx_peer_disconnect")
        if self.ops is not None and getattr(self.ops, "peer", None) is self:
            self.ops.peer = None
        if self._opened and dist.is_available() and dist.is_initialized():
            dist.barrier()  # no rank unmaps (or frees) a mailbox another rank may still write
        for p in self._opened:
            self._ctx.lib.hx_peer_ipc_close(C.c_void_p(p))
        self._opened = []
