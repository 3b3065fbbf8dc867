"""Generate golden vectors from the REAL reference package (run in the build container).

    python tests/golden/make_golden.py [--ref /root/reference/pkg/src]

Imports `ale_minihydro` from the read-only reference tree and writes small
`.npz` fixtures next to this script.  The GPU box never runs this (the
reference does not exist there); it only reads the committed fixtures.

Fixtures
  basis.npz          Gauss/Lobatto rules and B/G tables, p = 1..4
  mesh.npz           cartesian dofmaps/coords (restriction indices, bit-exact)
  ops_{d}d_p{p}.npz  operator-level results on randomly perturbed meshes
                     (geometry, mass apply/diag, force apply/apply_t, gather,
                     scatter_add, stress_qdata, momentum CG, energy solve, rates)
  remap_{d}d_p{p}.npz DiffusionPA / ConvectionPA D tables and applies (remap phase)
  run_*.npz          N-step Lagrange runs of the BASELINE configs at parity size,
                     with the noise floor (1e-15 relative perturbation of e0)
"""

from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))


def perturbed_mesh(cartesian_mesh, dim, counts, order, seed, amount=0.15):
    """Same recipe as the reference tests' random_mesh (test_operators.py:12-18)."""
    mesh = cartesian_mesh(dim, (1.0,) * dim, counts, order)
    rng = np.random.default_rng(seed)
    interior = np.setdiff1d(np.arange(mesh.num_nodes), mesh.boundary_nodes())
    h = 1.0 / (max(counts) * order)
    mesh.coords[interior] += amount * h * rng.uniform(-1, 1, size=(len(interior), dim))
    return mesh


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/root/reference/pkg/src")
    ap.add_argument("--only", default=None)
    args = ap.parse_args()
    sys.path.insert(0, args.ref)
    from ale_minihydro import fespace, hydro, operators, tensor_basis

    # ---- basis
    if args.only in (None, "basis"):
        out = {}
        for p in range(1, 5):
            q = tensor_basis.gauss_legendre(p + 2)
            lob = tensor_basis.gauss_lobatto_nodes(p)
            kb = tensor_basis.eval_basis(lob, q)
            tnodes = np.zeros(1) if p == 1 else tensor_basis.gauss_lobatto_nodes(p - 1)
            tb = tensor_basis.eval_basis(tnodes, q)
            out[f"qpts_{p}"], out[f"qw_{p}"] = q.points, q.weights
            out[f"lob_{p}"] = lob
            out[f"B_{p}"], out[f"G_{p}"] = kb.B, kb.G
            out[f"Bt_{p}"], out[f"Gt_{p}"] = tb.B, tb.G
        for n in range(1, 9):
            q = tensor_basis.gauss_legendre(n)
            out[f"gl_pts_{n}"], out[f"gl_w_{n}"] = q.points, q.weights
        np.savez_compressed(os.path.join(HERE, "basis.npz"), **out)

    # ---- meshes (restriction indices)
    if args.only in (None, "mesh"):
        out = {}
        cases = [(2, (3, 2), 2), (2, (16, 16), 2), (3, (2, 3, 2), 1), (3, (2, 3, 2), 2),
                 (3, (2, 3, 2), 3), (3, (2, 2, 3), 4), (3, (4, 4, 4), 3)]
        for i, (d, counts, p) in enumerate(cases):
            m = fespace.cartesian_mesh(d, (1.0,) * d, counts, p)
            out[f"dofmap_{i}"] = m.node_dofmap
            out[f"coords_{i}"] = m.coords
            out[f"case_{i}"] = np.array([d, p] + list(counts) + [0] * (3 - len(counts)))
        np.savez_compressed(os.path.join(HERE, "mesh.npz"), **out)

    # ---- remap-phase PA operators (DiffusionPA, ConvectionPA; operators.py:143-236)
    if args.only in (None, "remap"):
        for d in (2, 3):
            for p in (1, 2, 3, 4):
                counts = (3, 2) if d == 2 else (2, 2, 2)
                seed = 500 + 10 * d + p
                mesh = perturbed_mesh(fespace.cartesian_mesh, d, counts, p, seed)
                quad = tensor_basis.gauss_legendre(p + 2)
                geom = fespace.compute_geometric_factors(mesh, quad)
                h1 = fespace.FiniteElementSpace(mesh, "H1")
                rng = np.random.default_rng(900 + seed)
                nq, ne = quad.n**d, mesh.num_elements
                nu = 1.0 + 0.5 * rng.uniform(size=(nq, ne))
                dif = operators.DiffusionPA(h1, geom, nu=nu)
                dif1 = operators.DiffusionPA(h1, geom)
                u = rng.normal(size=(d, nq, ne))
                con = operators.ConvectionPA(h1, geom, u)
                x = rng.normal(size=h1.ndof)
                np.savez_compressed(os.path.join(HERE, f"remap_{d}d_p{p}.npz"), coords=mesh.coords,
                                    dofmap=mesh.node_dofmap, jinv=geom.jinv, wdetj=geom.wdetj, nu=nu,
                                    diff_D=dif.D, diff_x=x, diff_y=dif.apply(x), diff1_D=dif1.D,
                                    diff1_y=dif1.apply(x), conv_u=u, conv_D=con.D, conv_y=con.apply(x))

    # ---- operator-level fixtures
    if args.only in (None, "ops"):
        for d in (2, 3):
            for p in (1, 2, 3, 4):
                counts = (3, 2) if d == 2 else (2, 2, 2)
                seed = 10 * d + p
                mesh = perturbed_mesh(fespace.cartesian_mesh, d, counts, p, seed)
                quad = tensor_basis.gauss_legendre(p + 2)
                geom = fespace.compute_geometric_factors(mesh, quad)
                h1 = fespace.FiniteElementSpace(mesh, "H1")
                kin = fespace.FiniteElementSpace(mesh, "H1", vdim=d)
                thermo = fespace.FiniteElementSpace(mesh, "L2", order=max(p - 1, 0))
                rng = np.random.default_rng(100 + seed)
                nq = quad.n**d
                ne = mesh.num_elements
                o = dict(coords=mesh.coords, dofmap=mesh.node_dofmap, jac=geom.jac, detj=geom.detj,
                         jinv=geom.jinv, wdetj=geom.wdetj)
                # restriction
                L = rng.normal(size=(h1.ndof, d))
                E = rng.normal(size=(h1.nloc, ne, d))
                o["gather_in"], o["gather_out"] = L, h1.gather(L)
                o["scatter_in"], o["scatter_out"] = E, h1.scatter_add(E)
                Es = rng.normal(size=(h1.nloc, ne))
                o["scatter1_in"], o["scatter1_out"] = Es, h1.scatter_add(Es)
                # mass
                coeff = 1.0 + 0.5 * rng.uniform(size=(nq, ne))
                m = operators.MassPA(h1, geom, coeff=coeff)
                u1 = rng.normal(size=h1.ndof)
                u3 = rng.normal(size=(h1.ndof, d))
                o.update(mass_coeff=coeff, mass_D=m.D, mass_u1=u1, mass_y1=m.apply(u1),
                         mass_u3=u3, mass_y3=m.apply(u3), mass_diag=m.diagonal())
                # force
                sig = rng.normal(size=(d, d, nq, ne))
                f = operators.ForcePA(kin, thermo, geom, sig)
                ef = rng.normal(size=thermo.ndof)
                vf = rng.normal(size=(kin.ndof, d))
                o.update(force_sigma=sig, force_D=f.D, force_e=ef, force_Fe=f.apply(ef),
                         force_v=vf, force_Ftv=f.apply_transpose(vf),
                         force_F1=f.apply(np.ones(thermo.ndof)))
                # CG on the mass operator with Jacobi
                b = rng.normal(size=h1.ndof)
                xs, it = operators.cg_solve(m.apply, b, precond_diag=m.diagonal(), rel_tol=1e-8,
                                            max_iter=500)
                o.update(cg_b=b, cg_x=xs, cg_iters=np.array(it))
                # hydro-level: stress, momentum solve, energy solve, rates
                hy = hydro.LagrangeHydro(mesh, quad, hydro.MaterialModel(1.4),
                                         hydro.ViscosityModel(0.5, 2.0),
                                         bc_mask=hydro.box_velocity_bc(mesh))
                vfield = lambda x: 0.3 * np.stack(
                    [np.sin(np.pi * x[:, a] + a) * np.cos(np.pi * x[:, (a + 1) % d]) for a in range(d)],
                    axis=1) - 0.2 * (x - 0.5)
                st = hy.initial_state(lambda xq: 1.0 + 0.3 * xq[0] + 0.1 * xq[1],
                                      vfield,
                                      lambda pts: 1.0 + 0.5 * pts[0] - 1.2 * pts[d - 1] ** 2)
                sig2, ratio = hy.stress_qdata(st, geom)
                clamps_stress = hy.clamp_warnings
                r = hy.rates(st)
                rhs_e = rng.normal(size=thermo.ndof)
                o.update(st_x=st.x, st_v=st.v, st_e=st.e, st_qdata0=st.qdata0,
                         bc_mask=hy.bc_mask, stress_sigma=sig2, stress_ratio=np.array(ratio),
                         stress_clamps=np.array(clamps_stress),
                         rates_dv=r.dv, rates_de=r.de, rates_ratio=np.array(r.min_h_over_speed),
                         rates_clamped=np.array(r.clamped),
                         minv=hy._m_e_inv, mdiag=hy._mass_diag, mass_D_phase=hy.mass_pa.D,
                         esolve_rhs=rhs_e, esolve_out=hy.solve_energy(rhs_e),
                         ke=np.array(hy.kinetic_energy(st)), ie=np.array(hy.internal_energy(st)),
                         mass_total=np.array(hy.total_mass(st)))
                # one rk2 step
                new, info = hy.rk2_step(st, 1e-3)
                o.update(step_x=new.x, step_v=new.v, step_e=new.e, step_dt=np.array(info["dt"]))
                np.savez_compressed(os.path.join(HERE, f"ops_{d}d_p{p}.npz"), **o)
                print(f"ops {d}d p{p}: NE={ne} NN={mesh.num_nodes} cg_it={it}", flush=True)

    # ---- N-step runs
    if args.only in (None, "runs"):
        sys.path.insert(0, os.path.join(HERE, "..", ".."))
        from oracle.pa_oracle import sedov_fns, taylor_green_fns, triple_point_fns

        runs = [
            # name, dim, p, extents, counts, gamma, problem, cfl, steps
            # Taylor-Green is divergence-free: the viscosity compression switch
            # (hydro.py:301) would be decided by rounding noise in div v, so it runs
            # inviscid like the reference's own TG test (test_hydro.py:279-297).
            ("sedov2d_q2", 2, 2, (1.0, 1.0), (16, 16), 1.4, "sedov", 0.05, 50),
            ("sedov3d_q3", 3, 3, (1.0, 1.0, 1.0), (4, 4, 4), 1.4, "sedov", 0.02, 30),
            ("sedov3d_q2", 3, 2, (1.0, 1.0, 1.0), (4, 4, 4), 1.4, "sedov", 0.02, 30),
            ("triple3d_q3", 3, 3, (7.0, 3.0, 1.5), (7, 3, 2), 1.5, "triple", 0.05, 8),
            ("tgv3d_q4", 3, 4, (1.0, 1.0, 1.0), (2, 2, 2), 5.0 / 3.0, "tgv", 0.05, 10),
        ]
        for name, d, p, ext, counts, gamma, prob, cfl, nsteps in runs:
            q1, q2 = (0.0, 0.0) if prob == "tgv" else (0.5, 2.0)
            if prob == "sedov":
                fns = sedov_fns(d, ext, counts)
            elif prob == "tgv":
                fns = taylor_green_fns(d, gamma)
            else:
                fns = triple_point_fns(d, gamma)

            def run(pert):
                mesh = fespace.cartesian_mesh(d, ext, counts, p)
                quad = tensor_basis.gauss_legendre(p + 2)
                hy = hydro.LagrangeHydro(mesh, quad, hydro.MaterialModel(gamma),
                                         hydro.ViscosityModel(q1, q2),
                                         bc_mask=hydro.box_velocity_bc(mesh))
                e0 = fns[2]
                st = hy.initial_state(fns[0], fns[1], (lambda pts: e0(pts) * (1.0 + pert)))
                ctl = hydro.StepControls(cfl=cfl, dt_max=1.0, t_final=10.0)
                E0 = hy.total_energy(st)
                dts, energies = [], [E0]
                for _ in range(nsteps):
                    dt = hy.timestep_estimate(st, ctl)
                    st, info = hy.rk2_step(st, dt)
                    dts.append(info["dt"])
                    energies.append(hy.total_energy(st))
                return mesh, hy, st, np.array(dts), np.array(energies)

            t0 = time.time()
            mesh, hy, st, dts, energies = run(0.0)
            _, _, st_p, _, en_p = run(1e-15)
            floor = max(
                np.linalg.norm(st_p.x - st.x) / np.linalg.norm(st.x),
                np.linalg.norm(st_p.v - st.v) / max(np.linalg.norm(st.v), 1e-300),
                np.linalg.norm(st_p.e - st.e) / np.linalg.norm(st.e),
                abs(en_p[-1] - energies[-1]) / abs(energies[-1]),
            )
            np.savez_compressed(
                os.path.join(HERE, f"run_{name}.npz"),
                dim=d, p=p, extents=np.array(ext), counts=np.array(counts), gamma=gamma,
                problem=prob, cfl=cfl, nsteps=nsteps, q1=q1, q2=q2,
                x=st.x, v=st.v, e=st.e, t=st.t, dts=dts, energies=energies,
                clamps=hy.clamp_warnings, noise_floor=floor,
            )
            print(f"run {name}: {time.time() - t0:.1f}s floor={floor:.2e} "
                  f"E0={energies[0]:.6e} E={energies[-1]:.6e} clamps={hy.clamp_warnings}", flush=True)


if __name__ == "__main__":
    main()
