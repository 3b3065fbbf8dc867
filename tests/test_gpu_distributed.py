"""Device backend through the distributed driver: two ranks share one B200 (gloo
transport, since gpurun exposes a single GPU), each runs its subdomain's element
work in libb200hydro.so; the gathered state is checked against the CPU oracle's
single-domain run at 1e-10."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import rel
from oracle import pa_oracle as O

pytestmark = pytest.mark.gpu

CASE = dict(dim=3, p=2, counts=(4, 2, 2), extents=(1.0, 1.0, 1.0), gamma=1.4, cfl=0.02, steps=3)


def _initial(case):
    d, p, counts = case["dim"], case["p"], case["counts"]
    dofmap, coords = O.box_mesh(d, case["extents"], counts, p)
    mask = O.box_mask(coords)
    hy = O.Hydro(d, p, dofmap, coords, case["gamma"], 0.5, 2.0, bc_mask=mask)
    return hy, hy.initial_state(*O.sedov_fns(d, case["extents"], counts)), mask


def _worker(rank, world, port, case, out, peer=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2112_07075_b200.distributed import DeviceOps, DistributedLagrange
    from paper_2112_07075_b200.partition import brick_partition

    _, st, mask = _initial(case)
    d, p = case["dim"], case["p"]
    _, subs = brick_partition(d, case["extents"], case["counts"], p, world, bc_mask_global=mask)
    sub = subs[rank]
    nt = max(p, 1) ** d
    T = lambda a: torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")
    x, v = T(st["x"][sub.l2g]), T(st["v"][sub.l2g])
    e = T(st["e"].reshape(-1, nt)[sub.g_elems].reshape(-1))
    q0 = T(st["qdata0"][:, sub.g_elems])
    dl = DistributedLagrange(sub, DeviceOps(sub, case["gamma"], 0.5, 2.0), case["gamma"], device="cuda")
    dl.begin_phase(x, q0)
    if peer:  # device-resident CG; mailboxes mapped across the two processes with CUDA IPC
        from paper_2112_07075_b200.distributed import PeerExchange, max_shared

        PeerExchange(dl.ops, sub, max_shared(subs)).connect_ipc()
    t, dts = 0.0, []
    for _ in range(case["steps"]):
        dt = dl.timestep_estimate(x, v, e, q0, t, case["cfl"], dt_max=1.0, t_final=10.0)
        (x, v, e, t), info = dl.rk2_step(x, v, e, q0, t, dt)
        dts.append(info["dt"])
    np.savez(out + f".{rank}.npz", x=x.cpu().numpy(), v=v.cpu().numpy(), e=e.cpu().numpy(), l2g=sub.l2g,
             g_elems=sub.g_elems, dts=np.array(dts), clamps=dl.clamps)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("peer", [False, True], ids=["host_cg", "peer_cg"])
def test_device_ranks_match_single_domain_oracle(tmp_path, peer):
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    out = str(tmp_path / "res")
    world = 2
    mp.spawn(_worker, args=(world, port, CASE, out, peer), nprocs=world, join=True)
    hy, st, _ = _initial(CASE)
    dts = []
    for _ in range(CASE["steps"]):
        dt = hy.timestep_estimate(st, CASE["cfl"], dt_max=1.0, t_final=10.0)
        st, info = hy.rk2_step(st, dt)
        dts.append(info["dt"])
    nt = max(CASE["p"], 1) ** CASE["dim"]
    X, V = np.full_like(st["x"], np.nan), np.full_like(st["v"], np.nan)
    E = np.full(st["e"].reshape(-1, nt).shape, np.nan)
    for r in range(world):
        z = np.load(out + f".{r}.npz")
        X[z["l2g"]], V[z["l2g"]] = z["x"], z["v"]
        E[z["g_elems"]] = z["e"].reshape(-1, nt)
        assert np.allclose(z["dts"], dts, rtol=1e-12, atol=0)
        assert int(z["clamps"]) == hy.clamps
    assert rel(X, st["x"]) < 1e-10 and rel(V, st["v"]) < 1e-10 and rel(E.reshape(-1), st["e"]) < 1e-10


def _graph_worker(rank, world, port, case, out):
    """One rank of the device-resident distributed step: LagrangeHydro on the brick, the
    whole step one CUDA graph with the exchanges inside (hx_peer over CUDA IPC)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2112_07075_b200.distributed import PeerExchange, max_shared
    from paper_2112_07075_b200.hydro import HydroState, LagrangeHydro, MaterialModel, StepControls, ViscosityModel
    from paper_2112_07075_b200.partition import brick_partition
    from paper_2112_07075_b200.tensor_basis import gauss_legendre

    _, st, mask = _initial(case)
    d, p = case["dim"], case["p"]
    _, subs = brick_partition(d, case["extents"], case["counts"], p, world, bc_mask_global=mask)
    sub = subs[rank]
    nt = max(p, 1) ** d
    hy = LagrangeHydro(sub.mesh, gauss_legendre(p + 2), MaterialModel(case["gamma"]), ViscosityModel(0.5, 2.0),
                       bc_mask=sub.bc_mask)
    PeerExchange(hy, sub, max_shared(subs)).connect_ipc()
    s0 = HydroState(st["x"][sub.l2g].copy(), st["v"][sub.l2g].copy(),
                    st["e"].reshape(-1, nt)[sub.g_elems].reshape(-1).copy(), st["qdata0"][:, sub.g_elems].copy(), 0.0)
    hy.begin_phase(s0)
    cur = hy.to_device(s0)
    ctl = StepControls(cfl=case["cfl"], dt_max=1.0, t_final=10.0)
    dts = []
    for _ in range(case["steps"]):
        cur, info = hy.step(cur, ctl)
        dts.append(info["dt"])
    h = hy.to_host(cur)
    np.savez(out + f".{rank}.npz", x=h.x, v=h.v, e=h.e, l2g=sub.l2g, g_elems=sub.g_elems, dts=np.array(dts),
             clamps=hy.clamp_warnings)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_graph_step_ranks_match_single_domain_oracle(tmp_path, world):
    """Device-resident distributed step (two or four processes sharing one B200, 2x1x1 /
    2x2x1 bricks: four ranks put interior edge nodes on four sharers): every exchange --
    mass-diagonal and F.1 interface sums, CG halo and world scalars, CFL / clamp /
    inversion status -- runs inside each rank's step graph."""
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    out = str(tmp_path / "res")
    case = CASE if world == 2 else dict(CASE, counts=(4, 4, 2))
    mp.spawn(_graph_worker, args=(world, port, case, out), nprocs=world, join=True)
    hy, st, _ = _initial(case)
    dts = []
    for _ in range(case["steps"]):
        dt = hy.timestep_estimate(st, case["cfl"], dt_max=1.0, t_final=10.0)
        st, info = hy.rk2_step(st, dt)
        dts.append(info["dt"])
    nt = max(case["p"], 1) ** case["dim"]
    X, V = np.full_like(st["x"], np.nan), np.full_like(st["v"], np.nan)
    E = np.full(st["e"].reshape(-1, nt).shape, np.nan)
    for r in range(world):
        z = np.load(out + f".{r}.npz")
        X[z["l2g"]], V[z["l2g"]] = z["x"], z["v"]
        E[z["g_elems"]] = z["e"].reshape(-1, nt)
        assert np.allclose(z["dts"], dts, rtol=1e-12, atol=0)
        assert int(z["clamps"]) == hy.clamps
    assert rel(X, st["x"]) < 1e-10 and rel(V, st["v"]) < 1e-10 and rel(E.reshape(-1), st["e"]) < 1e-10
