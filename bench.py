#!/usr/bin/env python
"""Benchmark of the PA Lagrange step on B200: megadofs x timesteps / s (fp64).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = timestep_estimate + rk2_step (hydro.py:364-405) of the 3D Sedov blast,
Q3-Q2, 23^3 elements per GPU (1,029,000 velocity dofs), the BASELINE.json
weak-scaling configuration.  dofs = velocity dofs V = d * NN.

value  : device time of K steps (CUDA events on the launching stream, max over
         ranks), state resident in HBM, L2 flushed (256 MiB write) before every step.
e2e    : the same steps through the C-ABI entry a host caller binds
         (hx_step_host) with pinned HOST state buffers: H2D of x, v, e, the step,
         D2H of the new x, v, e -- all inside the timed region.
roofline: dominant kernel's algorithmic bytes / its average launch time (CUDA
         events recorded by the library around each launch during the timed steps)
         against MEASURED_PEAKS.json hbm_gbs.
cpu_baseline / --impl reference: the unmodified reference package (baseline/_ref,
         tools/install_reference.sh) through its public API, ExecPlace.sequential()
         with the fastest BLAS thread count on the host cores, on a bounded sample of
         the same workload (12^3 elements); the oracle port only if it is not installed.
window : every arm advances steps 0..HORIZON-1 of the run and restarts from the
         initial state outside the timed region (the workload underflows at step 42
         in the reference algorithm itself).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "megadofs x timesteps/sec (Lagrange step, fp64)"
UNIT = "Mdof*steps/s"
K_NAMES = ["rates", "mass_cg", "cg_node", "cg_init", "axpy", "validity", "other"]


def algorithmic_bytes(d, p, ne, nn, layout="brick"):
    """Per-launch algorithmic bytes of each kernel class: SURVEY.md section 8(d)'s per-unit
    figures (the HBM traffic the operation must move at minimum, index maps included,
    layout-specific intermediates such as the element-major E-vector excluded):
      mass     B_mass = 8 NE nq + 16 V + 4 NE nl
      cg_node  the rest of a CG iteration's vector traffic: B_CG,vec/iter - 16 V = 80 V
      rates    fused qpoint + F.1 + F^T v + energy solve, D_F kept on chip:
               x, v (16 V) + e + qdata0 + index map in, F.1 (8 V) out,
               M_e^-1 (8 NE nt^2) in, de (8 NE nt) out
      cg_init  F.1 in, r, (z, p), x out: 48 V;  axpy: x, v, e and rates in, new state out
      validity x in + index map"""
    nl, nq, nt = (p + 1) ** d, (p + 2) ** d, max(p, 1) ** d
    V = d * nn
    return {
        "mass_cg": 8 * ne * nq + 16 * V + 4 * ne * nl,
        "cg_node": 80 * V,
        "rates": 24 * V + 16 * ne * nt + 8 * ne * nq + 4 * ne * nl + 8 * ne * nt * nt,
        "cg_init": 48 * V,
        "axpy": 3 * 2 * 8 * V + 3 * 8 * ne * nt,
        "validity": 8 * V + 4 * ne * nl,
    }


def algorithmic_flops(d, p, ne):
    """Per-launch algorithmic fp64 flops (2 per multiply-add) of the contraction kernels.

    Sum-factorised contractions as the kernels perform them; the
    point physics of the rates kernel (EOS, viscosity, D_F, det J^-1) is not counted, so
    the rates figure is a lower bound."""
    if d != 3:
        return {}
    D1, Q, Dt = p + 1, p + 2, max(p, 1)
    nq, nt = Q ** 3, Dt ** 3
    sf = Q * D1 ** 3 + Q ** 2 * D1 ** 2 + Q ** 3 * D1  # one 3D interpolation (MACs)
    rates = (6 * D1 * D1 * Q * D1 * 2 + Dt * Dt * Q * Dt          # x stage (B, G) + thermo
             + 6 * D1 * Q * Q * D1 * 3 + Dt * Q * Q * Dt          # y stage (BB, GB, BG) + thermo
             + nq * (6 * D1 * 3 + 3 * D1 + Dt)                    # z stage: grads, v, e at points
             + 3 * Q * Q * Q * D1 * 3 + Q * Q * Q * Dt            # transposed z
             + 3 * D1 * Q * Q * D1 * 3 + Dt * Q * Q * Dt          # transposed y
             + 3 * D1 * D1 * D1 * Q * 2 + Dt * Dt * Dt * Q        # transposed x
             + nt * nt)                                           # M_e^-1 matvec
    valid = 3 * D1 * D1 * Q * D1 * 2 + 3 * D1 * Q * Q * D1 * 3 + nq * 3 * D1 * 3
    return {"mass_cg": 2 * d * (2 * sf + nq) * ne, "rates": 2 * rates * ne, "validity": 2 * valid * ne}


def fp64_peak(lib):
    """Live fp64 FMA peak of this device (hx_fp64_peak), TFLOP/s."""
    import ctypes

    v = ctypes.c_double(0.0)
    if lib.hx_fp64_peak(ctypes.byref(v)) != 0:
        return None
    return v.value


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap,utilization.gpu")

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        loaded = [r for r in self.rows if (num(r[6]) or 0) > 0] or self.rows
        sm = [num(r[0]) for r in loaded if num(r[0]) is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": num(self.rows[0][1]),
                "reasons": reasons, "samples": len(self.rows)}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic():
    """dram bytes per launch from the committed ncu --set full summary, if present."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            return json.load(f)
    except (OSError, ValueError):
        return {}


# ---------------------------------------------------------------------------
# The timed window.  The 23^3 Q3 Sedov run (CFL 0.05) is valid for a bounded number of
# steps in the reference algorithm itself: the oracle and the GPU both collapse dt after
# step ~26 and underflow (TimestepUnderflow) at step 42, t = 6.579338e-04.  Every arm
# therefore advances the SAME window of the run: steps 0 .. HORIZON-1 from the initial
# state, restarting from the initial state (a copy outside the timed region) whenever
# the window is exhausted.  Any --steps/--warmup is valid; `config.window` records the
# cycle indices of the timed steps.

HORIZON = 20


class Window:
    """Step counter of the cyclic window: restart() is due when pos hits HORIZON."""

    def __init__(self, horizon=HORIZON):
        self.horizon = horizon
        self.pos = 0

    def due(self):
        return self.pos % self.horizon == 0

    def advance(self):
        self.pos += 1

    def index(self):
        return self.pos % self.horizon


# ---------------------------------------------------------------------------
# CPU arms: the unmodified reference package (baseline/_ref, installed by
# tools/install_reference.sh from /root/reference) through its own public API;
# the oracle port only where the reference is not installed.

REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def sedov_ic(d, n, energy=0.25):
    """Sedov initial condition as the reference's initial_state callables (hydro.py:189-218):
    rho0 = 1, v0 = 0, e = energy / V_elem in the element at the origin corner (unit cube)."""
    cell = 1.0 / n
    vol = cell ** d

    def rho0(xq):
        return np.ones(xq.shape[1:])

    def v0(x):
        return np.zeros_like(x)

    def e0(pts):
        at_origin = np.all(pts.mean(axis=1) < cell, axis=0)
        return np.where(at_origin[None, :], energy / vol, 0.0) * np.ones(pts.shape[1:])

    return rho0, v0, e0


def reference_available():
    return os.path.isdir(os.path.join(REF_DIR, "ale_minihydro"))


def cpu_reference_run(p, n, steps, warmup, cfl, threads, window=None):
    """Time the reference's timestep_estimate + rk2_step (hydro.py:364-405) on an n^3 Q{p}
    Sedov sample with ExecPlace.sequential() and `threads` BLAS threads.  Returns
    (V, per-step seconds, kind)."""
    from threadpoolctl import threadpool_limits

    d = 3
    window = window or Window()
    with threadpool_limits(limits=threads):
        if reference_available():
            if REF_DIR not in sys.path:
                sys.path.insert(0, REF_DIR)
            from ale_minihydro.fespace import cartesian_mesh
            from ale_minihydro.hydro import LagrangeHydro, MaterialModel, StepControls, ViscosityModel, box_velocity_bc
            from ale_minihydro.kernel_exec import ExecPlace
            from ale_minihydro.tensor_basis import gauss_legendre

            mesh = cartesian_mesh(d, (1.0,) * d, (n,) * d, p)
            hy = LagrangeHydro(mesh, gauss_legendre(p + 2), MaterialModel(1.4), ViscosityModel(0.5, 2.0),
                               bc_mask=box_velocity_bc(mesh), place=ExecPlace.sequential())
            st0 = hy.initial_state(*sedov_ic(d, n))
            ctl = StepControls(cfl=cfl, dt_max=1.0, t_final=1e9)

            def one(st):
                dt = hy.timestep_estimate(st, ctl)
                return hy.rk2_step(st, dt)[0]
            V, kind = d * mesh.num_nodes, "reference"
        else:
            from oracle import pa_oracle as O

            dofmap, coords = O.box_mesh(d, (1.0,) * d, (n,) * d, p)
            ohy = O.Hydro(d, p, dofmap, coords, 1.4, 0.5, 2.0, bc_mask=O.box_mask(coords))
            st0 = ohy.initial_state(*O.sedov_fns(d, (1.0,) * d, (n,) * d))

            def one(st):
                dt = ohy.timestep_estimate(st, cfl, dt_max=1.0, t_final=1e9)
                return ohy.rk2_step(st, dt)[0]
            V, kind = d * coords.shape[0], "port"
        times = []
        st = st0
        for i in range(warmup + steps):
            if window.due():
                st = st0
            t0 = time.perf_counter()
            st = one(st)
            dtm = time.perf_counter() - t0
            window.advance()
            if i >= warmup:
                times.append(dtm)
    return V, times, kind


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def best_threads(p, n, cfl):
    """BLAS thread count the reference runs fastest with on this host (1 vs all cores vs
    half): its dgemms are small, so more threads can be slower (the reference's own
    ExecPlace.threaded is GIL-bound and slower still)."""
    cores = os.cpu_count() or 1
    cands = sorted({1, max(1, cores // 2), cores})
    best, best_t = cores, None
    for th in cands:
        _, t, _ = cpu_reference_run(p, n, 1, 1, cfl, th)
        if best_t is None or t[0] < best_t:
            best, best_t = th, t[0]
    return best, cands


def run_reference(args, rank):
    """--impl reference: the reference's own CPU path on this host's cores, rank 0 only."""
    if rank != 0:
        return
    n = args.cpu_n
    threads, cands = best_threads(args.p, n, args.cfl)
    V, times, kind = cpu_reference_run(args.p, n, args.steps, args.warmup, args.cfl, threads)
    tot = sum(times)
    val = V * len(times) / tot / 1e6
    # the 1-core figure (OMP/OpenBLAS threads = 1) on a short sample of the same window
    V1, t1, _ = cpu_reference_run(args.p, n, 2, 1, args.cfl, 1)
    one_core = V1 * len(t1) / sum(t1) / 1e6
    src = "baseline/_ref ale_minihydro, ExecPlace.sequential()" if kind == "reference" else "oracle/pa_oracle.py"
    sample = (f"3D Sedov blast Q{args.p}-Q{args.p - 1} {n}^3 elements ({V} velocity dofs), CFL {args.cfl}, "
              f"{len(times)} timed steps after {args.warmup} warm-up, window of {HORIZON} steps; {src}, "
              f"{threads} BLAS threads (fastest of {cands}) on {os.cpu_count()} x {cpu_model()}")
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / len(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        # the GPU arm's workload name; the CPU times a stated sample of it per step
        "config": {"workload": f"{problem_setup(args)[3]}, {3 * (args.p * args.n + 1) ** 3} velocity dofs per GPU, "
                               f"CFL {args.cfl}",
                   "sample": f"{n}^3 elements per CPU step ({V} velocity dofs), same window", "global_batch": V,
                   "seq_len": None, "parallelism": "cpu", "window_steps": HORIZON},
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": threads, "kind": kind, "sample": sample,
                         "one_core": {"value": one_core, "unit": UNIT, "cores": 1,
                                      "sample": f"{len(t1)} steps after 1 warm-up, BLAS threads = 1"}},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# B200 arm


def problem_setup(args):
    """(extents, counts, gamma, name) of the benchmark problem (BASELINE.json configs)."""
    n = args.n
    if args.problem == "sedov":
        return (1.0, 1.0, 1.0), (n, n, n), 1.4, f"3D Sedov blast Q{args.p}-Q{args.p - 1}, {n}^3 hex elements per GPU"
    if args.problem == "tgv":
        return (1.0, 1.0, 1.0), (n, n, n), 5.0 / 3.0, (f"3D Taylor-Green vortex Q{args.p}-Q{args.p - 1} (inviscid), "
                                                        f"{n}^3 elements")
    # multi-material triple point [0,7]x[0,3]x[0,1.5], gamma (1.5, 1.4, 1.5) by region;
    # n = elements per unit length (even, so that x = 1 and y = 1.5 are element faces)
    k = max(2, n - n % 2)
    c = (7 * k, 3 * k, 3 * k // 2)
    return (7.0, 3.0, 1.5), c, None, (f"3D triple point Q{args.p}-Q{args.p - 1}, multi-material "
                                       f"(per-element gamma 1.5/1.4/1.5), {c[0]}x{c[1]}x{c[2]} elements")


def run_distributed(args, world, rank, local):
    """N>1: one brick of n^3 elements per rank (weak scaling) of a global Sedov mesh;
    element work on the device, shared-node halo sums and CG/CFL scalars over NCCL
    (paper_2112_07075_b200.distributed)."""
    import torch
    import torch.distributed as dist

    from paper_2112_07075_b200 import problems
    from paper_2112_07075_b200.distributed import DeviceOps, DistributedLagrange, PeerExchange
    from paper_2112_07075_b200.hydro import HydroState, LagrangeHydro, MaterialModel, StepControls, ViscosityModel
    from paper_2112_07075_b200.partition import brick_partition, max_shared_nodes
    from paper_2112_07075_b200.tensor_basis import gauss_legendre

    d, p, n = 3, args.p, args.n
    # choose global counts so that every brick is n^3
    gg = [1, 1, 1]
    f = world
    ax = 0
    while f > 1:
        gg[ax % 3] *= 2
        f //= 2
        ax += 1
    counts = [n * gg[a] for a in range(3)]
    # each rank builds only its own brick (no global mesh): local coordinates, numbering
    # maps and the global box's wall mask come from the brick layout; the initial state is
    # sampled on the brick, which equals the global sampling restricted to it (the Sedov
    # source element is found by position)
    t_setup = time.perf_counter()
    _, subs = brick_partition(d, (1.0,) * d, counts, p, world, ranks=[rank], build_global=False)
    sub = subs[rank]
    maxh = max_shared_nodes(d, counts, p, world)
    lhy = LagrangeHydro(sub.mesh, gauss_legendre(p + 2), MaterialModel(1.4), ViscosityModel(0.5, 2.0),
                        bc_mask=sub.bc_mask)
    st0 = lhy.initial_state(*problems.sedov(d, (1.0,) * d, counts))
    T = lambda a: torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")
    x, v, e, q0 = T(st0.x), T(st0.v), T(st0.e), T(st0.qdata0)
    setup_s = time.perf_counter() - t_setup
    ctl = StepControls(cfl=args.cfl, dt_max=1.0, t_final=1e9)
    V_global = d * int(np.prod([c * p + 1 for c in counts]))
    win = Window()
    # device-resident exchanges need every pair of ranks to map each other's mailbox (CUDA
    # IPC + peer access); if any rank cannot, every rank falls back to the host-driven step
    use_peer = not args.host_cg
    if use_peer:
        ok, pex = 1, None
        try:
            pex = PeerExchange(lhy, sub, maxh)
            pex.connect_ipc()
        except Exception as exc:  # noqa: BLE001
            ok = 0
            print(f"[rank {rank}] peer-memory exchange unavailable ({exc}); host-driven fallback", file=sys.stderr)
        flag = torch.tensor([ok], dtype=torch.int32, device="cpu" if dist.get_backend() == "gloo" else "cuda")
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        if int(flag.item()) == 0:
            if ok and pex is not None:
                pex.close()
            use_peer = False
    if not use_peer:
        ops = DeviceOps(sub, 1.4, 0.5, 2.0)
        dl = DistributedLagrange(sub, ops, 1.4, device="cuda")
        dl.begin_phase(x, q0)
        cg_mode = "host-driven step (DistributedLagrange: torch.distributed collectives per CG iteration)"
        x0, v0, e0 = x.clone(), v.clone(), e.clone()
        t = 0.0

        def restart_if_due():
            nonlocal x, v, e, t
            if win.due():
                x, v, e, t = x0.clone(), v0.clone(), e0.clone(), 0.0

        def step():
            nonlocal x, v, e, t
            dt = dl.timestep_estimate(x, v, e, q0, t, args.cfl, dt_max=1.0, t_final=1e9)
            (x, v, e, t), _ = dl.rk2_step(x, v, e, q0, t, dt)
            win.advance()
    else:
        # device-resident step: each rank runs the single-GPU step graph on its brick with
        # every exchange inside (F.1 / diagonal interface sums, CG halo + world scalars,
        # CFL / clamp / inversion status) over CUDA-IPC-mapped peer mailboxes
        hy = lhy
        hy.begin_phase(HydroState(x, v, e, q0, 0.0))  # again: the mass diagonal's interface sums
        bufs = [(torch.empty_like(x), torch.empty_like(v), torch.empty_like(e)) for _ in range(2)]
        cg_mode = "device-resident step graph per rank (peer-memory exchanges, one host sync per step)"
        cur = [None, 0]

        def restart_if_due():
            if win.due():
                for dst, src in zip(bufs[0], (x, v, e)):
                    dst.copy_(src)
                cur[0], cur[1] = HydroState(bufs[0][0], bufs[0][1], bufs[0][2], q0, 0.0), 0

        def step():
            st, _ = hy.step(cur[0], ctl, out=bufs[1 - cur[1]])
            cur[0], cur[1] = st, 1 - cur[1]
            win.advance()

    for _ in range(args.warmup):
        restart_if_due()
        step()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    stream = torch.cuda.current_stream()
    dist.barrier()
    torch.cuda.synchronize()
    launches0 = hy._ctx.launches() if use_peer else 0
    tot = 0.0
    timed_idx = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            restart_if_due()
            timed_idx.append(win.index())
            flush.zero_()
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record(stream)
            step()
            ev1.record(stream)
            ev1.synchronize()
            tot += ev0.elapsed_time(ev1)
    tt = torch.tensor([tot], dtype=torch.float64, device="cpu" if dist.get_backend() == "gloo" else "cuda")
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    tot = float(tt.item())
    launches = None
    if use_peer:
        ll = torch.tensor([float(hy._ctx.launches() - launches0)], dtype=torch.float64,
                          device="cpu" if dist.get_backend() == "gloo" else "cuda")
        dist.all_reduce(ll)
        launches = int(ll.item())

    # ---- e2e: every rank steps its brick through the C-ABI host entry (hx_step_host:
    # pinned host x, v, e -> H2D, the step graph with its peer exchanges, D2H), the same
    # window; time = max over ranks of the host wall clock around the call
    e2e = None
    if not args.no_e2e and use_peer:
        from paper_2112_07075_b200 import _lib

        nx, nvv, ne_ = x.numel(), v.numel(), e.numel()
        arena = torch.empty(nx + nvv + ne_, dtype=torch.float64).pin_memory()
        hx_, hv_, he_ = arena[:nx], arena[nx:nx + nvv], arena[nx + nvv:]
        init = torch.cat([a.reshape(-1).cpu() for a in (x, v, e)])
        prm = hy._params(ctl)
        t_state = [0.0]
        info_c = _lib.StepInfo()
        hwin = Window()
        lib, h = hy._ctx.lib, hy._ctx.h

        def host_step():
            if hwin.due():
                arena.copy_(init)
                t_state[0] = 0.0
            hy._ctx.sync_stream()
            rc = lib.hx_step_host(h, _lib.C.byref(prm), float(t_state[0]), hx_.data_ptr(), hv_.data_ptr(),
                                  he_.data_ptr(), _lib.C.byref(info_c))
            if rc != 0:
                raise RuntimeError(f"hx_step_host failed: rc {rc}, info.code {info_c.code}")
            t_state[0] = info_c.t_new
            hwin.advance()

        for _ in range(args.warmup):
            host_step()
        e2e_s = 0.0
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            dist.barrier()
            t0 = time.perf_counter()
            host_step()
            e2e_s += time.perf_counter() - t0
        te = torch.tensor([e2e_s], dtype=torch.float64, device="cpu" if dist.get_backend() == "gloo" else "cuda")
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e_s = float(te.item())
        nb = 8 * (nx + nvv + ne_) * world
        e2e = {"value": V_global * args.steps / e2e_s / 1e6, "unit": UNIT, "h2d_bytes_per_step": nb,
               "d2h_bytes_per_step": nb, "ms_per_step": 1e3 * e2e_s / args.steps,
               "path": "hx_step_host (C-ABI) from pinned host x, v, e on every rank; max over ranks"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": V_global * args.steps / (tot / 1e3) / 1e6, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"3D Sedov blast Q{p}-Q{p - 1}, {n}^3 hex elements per GPU, global {counts}, "
                                   f"CFL {args.cfl}", "global_batch": V_global, "seq_len": None,
                       "parallelism": f"domain decomposition {list(sub.grid)}: {cg_mode}",
                       "l2": "flushed before every timed step",
                       "window": {"horizon_steps": HORIZON, "timed_cycle_indices": timed_idx},
                       "setup_s_rank0": setup_s},
            "e2e": e2e, "gpu_launches": launches, "roofline": None, "cpu_baseline": None, "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", "--elems", dest="n", type=int, default=23, help="elements per direction per GPU")
    ap.add_argument("--p", type=int, default=3, help="kinematic order (Q_p - Q_{p-1})")
    ap.add_argument("--cfl", type=float, default=0.05)
    ap.add_argument("--problem", default="sedov", choices=["sedov", "tgv", "triple"])
    ap.add_argument("--cpu-n", type=int, default=12, help="CPU sample: elements per direction")
    ap.add_argument("--cpu-steps", type=int, default=3)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--peer-self", action="store_true",
                    help="N=1 with the multi-GPU exchange launches active on a one-rank partition")
    ap.add_argument("--ktime", default="events", choices=["events", "dup", "both"],
                    help="per-kernel timing: CUDA events around every launch of a plain-launch replay of "
                         "the timed steps (events), in-graph duplication (dup), or both")
    ap.add_argument("--host-cg", action="store_true",
                    help="N>1: the host-driven distributed step instead of the device-resident step graph")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        run_reference(args, rank)
        return

    import torch

    # HX_BENCH_ONE_GPU=1: every rank on cuda:0 with gloo host collectives -- a functional
    # check of the N>1 path where only one GPU exists (ranks time-share it: no scaling number)
    one_gpu = os.environ.get("HX_BENCH_ONE_GPU") == "1"
    if one_gpu:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    if world > 1:
        run_distributed(args, world, rank, local)
        return

    from paper_2112_07075_b200 import _lib, problems
    from paper_2112_07075_b200.fespace import cartesian_mesh
    from paper_2112_07075_b200.hydro import (HydroState, LagrangeHydro, MaterialModel, StepControls,
                                             ViscosityModel, box_velocity_bc)
    from paper_2112_07075_b200.tensor_basis import gauss_legendre

    d, p, n = 3, args.p, args.n
    extents, counts, gamma, pname = problem_setup(args)
    mesh = cartesian_mesh(d, extents, counts, p)
    # Taylor-Green runs inviscid (as the reference's own TG test, test_hydro.py:279-297): the
    # flow is divergence-free, so the viscosity switch would act on rounding noise and the
    # reference itself collapses dt (checked with the oracle)
    visc = ViscosityModel(0.0, 0.0) if args.problem == "tgv" else ViscosityModel(0.5, 2.0)
    if args.problem == "sedov":
        fns = problems.sedov(d, extents, counts)
    elif args.problem == "tgv":
        fns = problems.taylor_green(d, gamma)
    else:
        *fns, gamma = problems.triple_point_multi(d, counts, extents)
    hy = LagrangeHydro(mesh, gauss_legendre(p + 2), MaterialModel(gamma), visc, bc_mask=box_velocity_bc(mesh))
    st0 = hy.initial_state(*fns)
    if args.peer_self:
        # the multi-GPU exchange launches on a one-rank partition (no neighbours, flags to
        # itself): measures what the exchanges add to a step besides the NVLink flag round trip
        from paper_2112_07075_b200.distributed import PeerExchange
        from paper_2112_07075_b200.partition import brick_partition

        _, subs1 = brick_partition(d, extents, counts, p, 1)
        PeerExchange.connect_local([PeerExchange(hy, subs1[0], 1)])
        hy.begin_phase(st0)
    ctl = StepControls(cfl=args.cfl, dt_max=1.0, t_final=1e9)
    V = d * mesh.num_nodes
    lib, h = hy._ctx.lib, hy._ctx.h
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    stream = torch.cuda.current_stream()

    # ---- device-resident steps over the cyclic window (see Window): the state lives in
    # two ping-pong buffer sets; a window restart copies the resident initial state into
    # the current set outside the timed region, so the step graphs keep their buffers
    st0d = hy.to_device(st0)
    bufs = [tuple(torch.empty_like(a) for a in (st0d.x, st0d.v, st0d.e)) for _ in range(2)]
    win = Window()
    cur = [None, 0]  # state, buffer index

    def restart_if_due():
        if win.due():
            b = bufs[0]
            for dst, src in zip(b, (st0d.x, st0d.v, st0d.e)):
                dst.copy_(src)
            cur[0], cur[1] = HydroState(b[0], b[1], b[2], st0d.qdata0, st0d.t), 0

    def dev_step():
        st, info = hy.step(cur[0], ctl, out=bufs[1 - cur[1]])
        cur[0], cur[1] = st, 1 - cur[1]
        win.advance()
        return info

    for i in range(args.warmup):
        restart_if_due()
        dev_step()
    torch.cuda.synchronize()
    # snapshot of the post-warm-up position: the kernel pass below replays the timed steps
    snap = (win.pos, cur[1], tuple(a.clone() for a in bufs[cur[1]]), cur[0].t)
    launches0 = hy._ctx.launches()
    step_ms, cg_iters, dts, timed_idx = [], [], [], []
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            restart_if_due()
            timed_idx.append(win.index())
            flush.zero_()  # L2 flush (outside the per-step events)
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record(stream)
            info = dev_step()
            ev1.record(stream)
            ev1.synchronize()
            step_ms.append(ev0.elapsed_time(ev1))
            cg_iters.append(info["cg_iterations"])
            dts.append(info["dt"])
    torch.cuda.synchronize()
    launches = hy._ctx.launches() - launches0

    # ---- kernel breakdown by duplication: the SAME timed steps replayed from the
    # post-warm-up snapshot through step graphs in which every launch of one kernel class
    # runs twice (hx_prof_dup; the CG node pass's twin is a dry copy writing to scratch).
    # A class's in-step cost per launch = (T_dup - T_plain) / (duplicates that did work),
    # both timed with CUDA events around whole steps on the launching stream, L2 flushed
    # before every step as in the timed region.  Unlike events around single launches in
    # a graph (which stall the pipeline between kernels) this leaves the step unperturbed.
    def restore():
        win.pos, cur[1] = snap[0], snap[1]
        for dst, src in zip(bufs[cur[1]], snap[2]):
            dst.copy_(src)
        b = bufs[cur[1]]
        cur[0] = HydroState(b[0], b[1], b[2], st0d.qdata0, snap[3])

    def replay(dup):
        lib.hx_prof_dup(h, dup)
        restore()
        for _ in range(2):  # capture this variant's graphs (both buffer sets) untimed
            restart_if_due()
            dev_step()
        restore()
        torch.cuda.synchronize()
        lib.hx_prof_reset(h)
        tot = 0.0
        for _ in range(args.steps):
            restart_if_due()
            flush.zero_()
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record(stream)
            dev_step()
            ev1.record(stream)
            ev1.synchronize()
            tot += ev0.elapsed_time(ev1)
        cnt = 0
        if dup >= 0:
            t_, c_ = _lib.C.c_double(), _lib.C.c_int64()
            lib.hx_prof_read(h, dup, _lib.C.byref(t_), _lib.C.byref(c_))
            cnt = int(c_.value)
        lib.hx_prof_dup(h, -1)
        return tot, cnt

    # ---- kernel breakdown by CUDA events around every launch: the same timed steps
    # replayed from the snapshot as plain stream launches (HX graph off while profiling),
    # the library recording an event pair on the launching stream around each launch
    def replay_events():
        restore()
        torch.cuda.synchronize()
        lib.hx_prof_enable(h, 1)
        lib.hx_prof_reset(h)
        tot = 0.0
        for _ in range(args.steps):
            restart_if_due()
            flush.zero_()
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record(stream)
            dev_step()
            ev1.record(stream)
            ev1.synchronize()
            tot += ev0.elapsed_time(ev1)
        out = {}
        for k, name in enumerate(K_NAMES):
            t_, c_ = _lib.C.c_double(), _lib.C.c_int64()
            lib.hx_prof_read(h, k, _lib.C.byref(t_), _lib.C.byref(c_))
            if c_.value:
                out[name] = (float(t_.value), int(c_.value))
        lib.hx_prof_enable(h, 0)
        return tot, out

    # two replays, per kernel class the lower average (a replay occasionally runs all the
    # memory-bound launches ~1.5x slower; the timed region above is not affected)
    ev_ms, ev_times = replay_events()
    ev_ms2, ev_times2 = replay_events()
    for name, (t2, c2) in ev_times2.items():
        if name not in ev_times or (c2 and t2 / c2 < ev_times[name][0] / max(ev_times[name][1], 1)):
            ev_times[name] = (t2, c2)
    ev_ms = min(ev_ms, ev_ms2)
    ktimes_dup = {}
    prof_base = None
    if args.ktime in ("dup", "both"):
        prof_base, _ = replay(-1)
        for k, name in enumerate(K_NAMES[:6]):
            tot, cnt = replay(k)
            if cnt:
                ktimes_dup[name] = (max(tot - prof_base, 0.0), cnt)  # ms over the K steps, working launches
    if args.ktime == "dup":
        ktimes, prof_ms = ktimes_dup, prof_base
    else:
        ktimes, prof_ms = ev_times, ev_ms
    total_ms = sum(step_ms)
    ms_per_step = total_ms / args.steps
    value = V * args.steps / (total_ms / 1e3) / 1e6

    # ---- e2e through the C-ABI with pinned host buffers
    e2e = None
    if not args.no_e2e:
        # the same window: from the initial state, W warm-up steps, then K timed steps,
        # restarting from the initial host state (outside the timed region) as above
        hst = st0
        # the host state lives in one pinned arena (x | v | e): separately pinned small
        # blocks measured ~40% slower for H2D on this host (tools/pcie_probe.py)
        nx, nvv, ne_ = hst.x.size, hst.v.size, hst.e.size
        arena = torch.empty(nx + nvv + ne_, dtype=torch.float64).pin_memory()
        hx_ = arena[:nx].view(hst.x.shape)
        hv_ = arena[nx:nx + nvv].view(hst.v.shape)
        he_ = arena[nx + nvv:].view(hst.e.shape)
        init = torch.cat([torch.from_numpy(np.ascontiguousarray(a)).reshape(-1) for a in (hst.x, hst.v, hst.e)])
        prm = hy._params(ctl)
        t_state = [hst.t]
        info_c = _lib.StepInfo()
        hwin = Window()

        def host_restart_if_due():
            if hwin.due():
                arena.copy_(init)
                t_state[0] = hst.t

        def host_step():
            hy._ctx.sync_stream()
            rc = lib.hx_step_host(h, _lib.C.byref(prm), float(t_state[0]), hx_.data_ptr(), hv_.data_ptr(),
                                  he_.data_ptr(), _lib.C.byref(info_c))
            if rc != 0:
                raise RuntimeError(f"hx_step_host failed: rc {rc}, info.code {info_c.code}")
            t_state[0] = info_c.t_new
            hwin.advance()

        for _ in range(args.warmup):
            host_restart_if_due()
            host_step()
        e2e_s = 0.0
        for _ in range(args.steps):
            host_restart_if_due()
            flush.zero_()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            host_step()
            e2e_s += time.perf_counter() - t0
        nb = 8 * (hst.x.size + hst.v.size + hst.e.size)
        e2e = {"value": V * args.steps / e2e_s / 1e6, "unit": UNIT, "h2d_bytes_per_step": nb,
               "d2h_bytes_per_step": nb, "ms_per_step": 1e3 * e2e_s / args.steps,
               "path": "hx_step_host (C-ABI) from pinned host x, v, e"}

    # ---- the reference-API call sequence a drop-in script makes per step
    # (timestep_estimate + rk2_step, hydro.py:364-405) on the same resident window: one
    # fused ratio launch, then the rk2 step graph; host syncs as the API implies
    api = None
    if not args.no_e2e:
        awin = Window()
        ast = [None]

        def api_restart_if_due():
            if awin.due():
                ast[0] = HydroState(st0d.x.clone(), st0d.v.clone(), st0d.e.clone(), st0d.qdata0, st0d.t)

        def api_step():
            dt = hy.timestep_estimate(ast[0], ctl)
            ast[0], _ = hy.rk2_step(ast[0], dt)
            awin.advance()

        for _ in range(args.warmup):
            api_restart_if_due()
            api_step()
        api_ms = 0.0
        for _ in range(args.steps):
            api_restart_if_due()
            flush.zero_()
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record(stream)
            api_step()
            ev1.record(stream)
            ev1.synchronize()
            api_ms += ev0.elapsed_time(ev1)
        api = {"value": V * args.steps / (api_ms / 1e3) / 1e6, "unit": UNIT, "ms_per_step": api_ms / args.steps,
               "path": "LagrangeHydro.timestep_estimate + rk2_step (hx_timestep_ratio + hx_rk2_step), state resident"}

    # ---- roofline of the dominant kernel
    pk, pk_src = peaks()
    layout = hy._ctx.layout()
    ab = algorithmic_bytes(d, p, mesh.num_elements, mesh.num_nodes, layout)
    traffic = ncu_traffic()
    af = algorithmic_flops(d, p, mesh.num_elements)
    f64pk = fp64_peak(lib) if rank == 0 else None
    kern = {}
    for name, (tot, cnt) in ktimes.items():
        avg_s = tot / cnt / 1e3
        kb = ab.get(name)
        kern[name] = {"launches": cnt, "avg_us": avg_s * 1e6, "share": tot / max(prof_ms, 1e-30),
                      "alg_bytes": kb, "gbs": (kb / avg_s / 1e9) if kb else None,
                      "hbm_frac": (kb / avg_s / 1e9 / pk) if kb else None}
        if name in af:
            tf = af[name] / avg_s / 1e12
            kern[name].update({"alg_flops": af[name], "fp64_tflops": tf,
                               "fp64_frac": (tf / f64pk) if f64pk else None})
    dom = max(kern, key=lambda k: ktimes[k][0]) if kern else None
    roof = None
    if dom:
        ach = kern[dom]["gbs"]
        roof = {"kernel": dom, "bound": "hbm", "achieved": ach, "peak": pk, "unit": "GB/s",
                "frac": ach / pk if ach else None, "traffic": traffic.get(dom), "peak_source": pk_src,
                "alg_bytes_per_launch": kern[dom]["alg_bytes"],
                "fp64": {"achieved": kern[dom].get("fp64_tflops"), "peak": f64pk, "unit": "TFLOP/s",
                         "frac": kern[dom].get("fp64_frac"), "alg_flops_per_launch": kern[dom].get("alg_flops"),
                         "peak_source": "measured live (hx_fp64_peak: DFMA chains, full occupancy)"}}

    # ---- CPU baseline (rank 0, N=1 only): the reference itself on a bounded sample
    cpu = None
    if rank == 0 and not args.no_cpu:
        cores, _ = best_threads(p, args.cpu_n, args.cfl)
        Vc, times, kind = cpu_reference_run(p, args.cpu_n, args.cpu_steps, 1, args.cfl, cores)
        src = ("baseline/_ref ale_minihydro (the unmodified reference), ExecPlace.sequential()"
               if kind == "reference" else "oracle/pa_oracle.py (reference not installed)")
        cpu = {"value": Vc * len(times) / sum(times) / 1e6, "unit": UNIT, "cores": cores, "kind": kind,
               "sample": f"3D Sedov Q{p}-Q{p - 1} {args.cpu_n}^3 elements ({Vc} velocity dofs), CFL {args.cfl}, "
                         f"{len(times)} steps after 1 warm-up; {src}; {cores} BLAS threads (the fastest count) on "
                         f"{os.cpu_count()} x {cpu_model()}"}

    if args.ktime == "dup":
        kpass = {"method": "dup",
                 "note": "per-launch kernel cost in the step graph by duplication: the same timed steps replayed "
                         "from the post-warm-up snapshot with every launch of one class doubled (CG node pass: "
                         "dry twin writing to scratch); avg_us = (T_dup - T_plain) / working duplicates, CUDA "
                         "events around whole steps",
                 "ms_per_step_plain_replay": prof_ms / args.steps}
    else:
        kpass = {"method": "events",
                 "note": "the same timed steps replayed (twice) from the post-warm-up snapshot as plain stream "
                         "launches; the library records a CUDA event pair on the launching stream around every "
                         "launch; per class the replay with the lower average; share = class time / replay step time",
                 "ms_per_step_replay": prof_ms / args.steps}
        if ktimes_dup:
            kpass["graph_dup_avg_us"] = {k: 1e3 * t / c for k, (t, c) in ktimes_dup.items()}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{pname}, {V} velocity dofs per GPU, CFL {args.cfl}",
                       "global_batch": V, "seq_len": None, "parallelism": "single",
                       "l2": "flushed (256 MiB write) before every timed step",
                       "layout": layout,
                       "window": {"horizon_steps": HORIZON, "timed_cycle_indices": timed_idx,
                                  "note": "steps 0..horizon-1 of the run from the initial state, restarted "
                                          "from it outside the timed region (the workload underflows at "
                                          "step 42 in the reference algorithm)"},
                       "cg_iterations": cg_iters, "dt": dts},
            "e2e": e2e, "api": api, "gpu_launches": launches, "roofline": roof, "kernels": kern,
            "kernel_pass": kpass,
            "cpu_baseline": cpu,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)

if __name__ == "__main__":
    main()
