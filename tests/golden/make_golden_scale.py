"""At-scale fixture from the REAL reference: the bench workload itself (run in the build
container; the GPU box only reads the committed .npz).

    python tests/golden/make_golden_scale.py [--ref /root/reference/pkg/src] [--n 23]

3D Sedov blast Q3-Q2 on n^3 elements (the BASELINE.json per-GPU configuration, 12,167
elements, 1,029,000 velocity dofs), CFL 0.05, via the reference's timestep_estimate +
rk2_step (hydro.py:364-405).  Records
  * the bench window (steps 0..19): dt, clamp count, total energy per step, and the
    final x, v, e as norms plus a strided subsample (the full state is 19 MB);
  * the same window from e0 * (1 + 1e-15): the reference's own noise floor;
  * the horizon: the unperturbed run continued until TimestepUnderflow (hydro.py:370-372),
    its step index, t and dt sequence.
"""

from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
STRIDE = 97  # subsample stride of the final state


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/root/reference/pkg/src")
    ap.add_argument("--n", type=int, default=23)
    ap.add_argument("--window", type=int, default=20)
    ap.add_argument("--pert", type=float, default=0.0)
    ap.add_argument("--horizon", action="store_true")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    sys.path.insert(0, args.ref)
    from ale_minihydro import fespace, hydro, tensor_basis

    n, p, d = args.n, 3, 3
    cell = 1.0 / n
    vol = cell ** d

    def rho0(xq):
        return np.ones(xq.shape[1:])

    def v0(x):
        return np.zeros_like(x)

    def e0(pts):
        at = np.all(pts.mean(axis=1) < cell, axis=0)
        return np.where(at[None, :], 0.25 / vol, 0.0) * np.ones(pts.shape[1:]) * (1.0 + args.pert)

    t0 = time.time()
    mesh = fespace.cartesian_mesh(d, (1.0,) * d, (n,) * d, p)
    hy = hydro.LagrangeHydro(mesh, tensor_basis.gauss_legendre(p + 2), hydro.MaterialModel(1.4),
                             hydro.ViscosityModel(0.5, 2.0), bc_mask=hydro.box_velocity_bc(mesh))
    st = hy.initial_state(rho0, v0, e0)
    ctl = hydro.StepControls(cfl=0.05, dt_max=1.0, t_final=1e9)
    out = {"n": n, "p": p, "cfl": 0.05, "window": args.window, "stride": STRIDE, "pert": args.pert}
    dts, clamps, energies, ratios = [], [], [hy.total_energy(st)], []
    step = 0
    under = None
    while True:
        c0 = hy.clamp_warnings
        try:
            dt = hy.timestep_estimate(st, ctl)
        except hydro.TimestepUnderflow as exc:
            under = str(exc)
            break
        st, info = hy.rk2_step(st, dt)
        step += 1
        dts.append(info["dt"])
        ratios.append(info["min_h_over_speed"])
        clamps.append(hy.clamp_warnings - c0)
        if step <= args.window:
            energies.append(hy.total_energy(st))
        print(f"step {step} dt={info['dt']:.6e} t={st.t:.9e} clamps={clamps[-1]} ({time.time() - t0:.0f}s)",
              flush=True)
        if step == args.window:
            out.update(x_sub=st.x.reshape(-1)[::STRIDE], v_sub=st.v.reshape(-1)[::STRIDE],
                       e_sub=st.e.reshape(-1)[::STRIDE], x_norm=np.linalg.norm(st.x),
                       v_norm=np.linalg.norm(st.v), e_norm=np.linalg.norm(st.e), t_window=st.t,
                       x_sum=st.x.sum(), v_sum=st.v.sum(), e_sum=st.e.sum(),
                       v_absmax=np.abs(st.v).max(), e_absmax=np.abs(st.e).max())
            if not args.horizon:
                break
    out.update(dts=np.array(dts), ratios=np.array(ratios), clamps=np.array(clamps),
               energies=np.array(energies), steps=step)
    if under is not None:
        out.update(underflow_step=step + 1, underflow_t=st.t, underflow_msg=under)
    name = args.out or f"scale_sedov{n}_q3{'_pert' if args.pert else ''}.npz"
    np.savez_compressed(os.path.join(HERE, name), **out)
    print(f"wrote {name}: {step} steps, {time.time() - t0:.0f}s, underflow={under}", flush=True)


if __name__ == "__main__":
    main()
