"""Multi-rank path on CPU: brick partition maps and the distributed Lagrange step
(world size 2, gloo, 127.0.0.1) against the single-domain oracle.

The per-rank element work uses the oracle (test infrastructure); the exchange logic
under test (partition.py, distributed.Halo / DistributedLagrange) is the same code
the GPU ranks run with DeviceOps over NCCL.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import rel
from oracle import pa_oracle as O


@pytest.mark.parametrize("dim,counts,p,nranks", [(2, (6, 4), 2, 2), (2, (5, 5), 3, 4), (3, (4, 3, 2), 2, 2),
                                                  (3, (4, 4, 4), 1, 8), (3, (3, 2, 2), 3, 2)])
def test_partition_index_maps_bitwise(dim, counts, p, nranks):
    from paper_2112_07075_b200.partition import brick_partition

    gmesh, subs = brick_partition(dim, (1.0,) * dim, counts, p, nranks)
    covered = np.zeros(gmesh.num_nodes, dtype=int)
    owners = np.zeros(gmesh.num_nodes, dtype=int)
    elems = []
    for s in subs:
        # restriction indices: global dofmap == l2g[local dofmap], bit-exact
        assert np.array_equal(gmesh.node_dofmap[:, s.g_elems], s.l2g[s.mesh.node_dofmap])
        assert np.array_equal(s.mesh.coords, gmesh.coords[s.l2g])
        covered[s.l2g] += 1
        owners[s.l2g[s.owned]] += 1
        elems.append(s.g_elems)
        for q in s.neighbors:
            mine = s.l2g[s.shared[q]]
            theirs = subs[q].l2g[subs[q].shared[s.rank]]
            assert np.array_equal(mine, theirs)
            assert np.all(np.diff(mine) > 0)
    assert np.all(covered >= 1) and np.all(owners == 1)
    assert np.array_equal(np.sort(np.concatenate(elems)), np.arange(gmesh.num_elements))


class OracleOps:
    """LocalOps backed by the CPU oracle (tests only)."""

    def __init__(self, sub, p):
        self.sub, self.p, self.d = sub, p, sub.mesh.dim
        self.qpts, self.qw = O.gauss_legendre(p + 2)
        self.dofmap = sub.mesh.node_dofmap
        self.nn = sub.mesh.num_nodes
        self.B, self.G = O.basis_tables(O.gauss_lobatto(p), self.qpts)
        self.Bt, _ = O.basis_tables(O.l2_nodes(p - 1), self.qpts)
        self.nt = max(p, 1) ** self.d

    def _np(self, a):
        return a.detach().cpu().numpy() if isinstance(a, torch.Tensor) else np.asarray(a)

    def begin_phase(self, x, qdata0):
        _, det, _, wdetj = O.geometry(self.dofmap, self._np(x), self.p, self.qpts, self.qw, self.d)
        self.Dm = (wdetj / det) * self._np(qdata0)
        Bf = np.ones((1, 1))
        for _ in range(self.d):
            Bf = np.kron(Bf, self.Bt)
        self.Minv = np.linalg.inv(np.einsum("qi,qe,qj->eij", Bf, self.Dm, Bf))

    def mass_diagonal(self):
        return O.mass_diag(self.dofmap, self.Dm, self.B, self.nn, self.d)

    def mass_apply(self, x):
        return O.mass_apply(self.dofmap, self.Dm, self.B, self._np(x), self.d)

    def stress_force(self, x, v, e, qdata0, gamma, q1, q2, ratio_only=False):
        try:
            geo = O.geometry(self.dofmap, self._np(x), self.p, self.qpts, self.qw, self.d)
        except O.Inverted:
            return {"inverted": True, "clamped": 0, "ratio": float("inf")}
        hy = O.Hydro(self.d, self.p, self.dofmap, self._np(x), gamma, q1, q2)
        st = dict(x=self._np(x), v=self._np(v), e=self._np(e), qdata0=self._np(qdata0))
        sig, ratio = hy.stress(st, geo)
        out = {"inverted": False, "clamped": hy.clamps, "ratio": ratio}
        if not ratio_only:
            DF = O.force_D(sig, geo[2], geo[3])
            out["F1"] = O.force_apply(self.dofmap, self.nn, DF, self.B, self.G, self.Bt,
                                      np.ones(self.nt * self.sub.mesh.num_elements), self.d)
            out["Ftv"] = O.force_apply_t(self.dofmap, DF, self.B, self.G, self.Bt, st["v"], self.d)
        return out

    def energy_solve(self, rhs):
        r = self._np(rhs)
        ne = self.sub.mesh.num_elements
        return np.einsum("eij,ej->ei", self.Minv, r.reshape(ne, self.nt)).reshape(-1)

    def geometry_ok(self, x):
        try:
            O.geometry(self.dofmap, self._np(x), self.p, self.qpts, self.qw, self.d)
            return True
        except O.Inverted:
            return False


CASES = {
    "2d_q2_r2": (dict(dim=2, p=2, counts=(8, 6), extents=(1.0, 1.0), gamma=1.4, cfl=0.05, steps=6), 2),
    "3d_q2_r4": (dict(dim=3, p=2, counts=(4, 4, 2), extents=(1.0, 1.0, 1.0), gamma=1.4, cfl=0.02, steps=3), 4),
}


def _global_initial(case):
    d, p, counts = case["dim"], case["p"], case["counts"]
    dofmap, coords = O.box_mesh(d, case["extents"], counts, p)
    mask = O.box_mask(coords)
    hy = O.Hydro(d, p, dofmap, coords, case["gamma"], 0.5, 2.0, bc_mask=mask)
    st = hy.initial_state(*O.sedov_fns(d, case["extents"], counts))
    return hy, st, mask


def _worker(rank, world, port, case, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2112_07075_b200.distributed import DistributedLagrange
    from paper_2112_07075_b200.partition import brick_partition

    hy, st, mask = _global_initial(case)
    d, p = case["dim"], case["p"]
    _, subs = brick_partition(d, case["extents"], case["counts"], p, world, bc_mask_global=mask)
    sub = subs[rank]
    nt = max(p, 1) ** d
    T = lambda a: torch.as_tensor(a, dtype=torch.float64)
    x, v = T(st["x"][sub.l2g]), T(st["v"][sub.l2g])
    e = T(st["e"].reshape(-1, nt)[sub.g_elems].reshape(-1))
    q0 = T(st["qdata0"][:, sub.g_elems])
    dl = DistributedLagrange(sub, OracleOps(sub, p), case["gamma"])
    dl.begin_phase(x, q0)
    t = 0.0
    dts = []
    for _ in range(case["steps"]):
        dt = dl.timestep_estimate(x, v, e, q0, t, case["cfl"], dt_max=1.0, t_final=10.0)
        (x, v, e, t), info = dl.rk2_step(x, v, e, q0, t, dt)
        dts.append(info["dt"])
    np.savez(out_path + f".{rank}.npz", x=x.numpy(), v=v.numpy(), e=e.numpy(), l2g=sub.l2g, g_elems=sub.g_elems,
             dts=np.array(dts), clamps=dl.clamps)
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("name", sorted(CASES))
def test_distributed_sedov_matches_single_domain(tmp_path, name):
    case, world = CASES[name]
    out = str(tmp_path / "res")
    mp.spawn(_worker, args=(world, _free_port(), case, out), nprocs=world, join=True)
    hy, st, mask = _global_initial(case)
    dts = []
    for _ in range(case["steps"]):
        dt = hy.timestep_estimate(st, case["cfl"], dt_max=1.0, t_final=10.0)
        st, info = hy.rk2_step(st, dt)
        dts.append(info["dt"])
    nt = max(case["p"], 1) ** case["dim"]
    X = np.full_like(st["x"], np.nan)
    V = np.full_like(st["v"], np.nan)
    E = np.full(st["e"].reshape(-1, nt).shape, np.nan)
    clamps = 0
    for r in range(world):
        z = np.load(out + f".{r}.npz")
        X[z["l2g"]] = z["x"]
        V[z["l2g"]] = z["v"]
        E[z["g_elems"]] = z["e"].reshape(-1, nt)
        assert np.allclose(z["dts"], dts, rtol=1e-12, atol=0)
        clamps = int(z["clamps"])
    assert not np.isnan(X).any() and not np.isnan(E).any()
    assert rel(X, st["x"]) < 1e-10
    assert rel(V, st["v"]) < 1e-10
    assert rel(E.reshape(-1), st["e"]) < 1e-10
    assert clamps == hy.clamps


@pytest.mark.parametrize("d,counts,world", [(3, (4, 4, 2), 4), (3, (4, 4, 4), 8), (2, (6, 4), 2)])
def test_peer_plan_consistent(d, counts, world):
    """Exchange plan of the device-resident CG (distributed.peer_plan / hx_peer_setup):
    every (node, neighbour) entry lands at an index both sides agree on, every
    interface node lists all its sharers in ascending rank order, and exactly one rank
    owns each global node."""
    from paper_2112_07075_b200.distributed import max_shared, peer_plan
    from paper_2112_07075_b200.partition import brick_partition

    gm, subs = brick_partition(d, (1.0,) * d, counts, 2, world)
    mx = max_shared(subs)
    plans = [peer_plan(s) for s in subs]
    owners = np.zeros(gm.num_nodes, dtype=int)
    for s, pl in zip(subs, plans):
        owners[s.l2g[pl["owned"].astype(bool)]] += 1
        # sender side: entry j goes to rank sdst[j] at index sidx[j]
        for n, q, i in zip(pl["snode"], pl["sdst"], pl["sidx"]):
            assert 0 <= i < mx
            assert subs[q].l2g[subs[q].shared[s.rank][i]] == s.l2g[n]
        # receiver side: sharers ascending, -1 = self, else (q << 24) | index into q's block
        for h, n in enumerate(pl["hnode"]):
            srcs = pl["hsrc"][pl["hoff"][h]:pl["hoff"][h + 1]]
            ranks = [s.rank if v < 0 else int(v) >> 24 for v in srcs]
            assert ranks == sorted(ranks) and s.rank in ranks and len(ranks) >= 2
            for v in srcs:
                if v >= 0:
                    q, i = int(v) >> 24, int(v) & 0xFFFFFF
                    assert s.l2g[s.shared[q][i]] == s.l2g[n]
    assert np.all(owners == 1)
