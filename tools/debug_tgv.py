"""Stage-by-stage comparison of the device path and the oracle on the TGV Q4 config."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import pa_oracle as O
from paper_2112_07075_b200 import problems
from paper_2112_07075_b200.fespace import cartesian_mesh, compute_geometric_factors
from paper_2112_07075_b200.hydro import LagrangeHydro, MaterialModel, StepControls, ViscosityModel, box_velocity_bc, HydroState
from paper_2112_07075_b200.tensor_basis import gauss_legendre

def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)

d, p, counts, g = 3, int(sys.argv[1]) if len(sys.argv) > 1 else 4, (2, 2, 2), 5/3
mesh = cartesian_mesh(d, (1.,)*3, counts, p)
hy = LagrangeHydro(mesh, gauss_legendre(p+2), MaterialModel(g), ViscosityModel(0.5, 2.0), bc_mask=box_velocity_bc(mesh))
st = hy.initial_state(*problems.taylor_green(d, g))
oh = O.Hydro(d, p, mesh.node_dofmap, mesh.coords, g, 0.5, 2.0, bc_mask=O.box_mask(mesh.coords))
ost = oh.initial_state(*O.taylor_green_fns(d, g))
print("init x v e q0", rel(st.x, ost["x"]), rel(st.v, ost["v"]), rel(st.e, ost["e"]), rel(st.qdata0, ost["qdata0"]))
geo = compute_geometric_factors(mesh, hy.quad, x=st.x)
sig, ratio = hy.stress_qdata(st, geo)
ogeo = oh.geom(ost["x"])
osig, oratio = oh.stress(ost, ogeo)
print("stress", rel(sig, osig), ratio, oratio)
r = hy.rates(st)
orr = oh.rates(ost)
print("rates dv de", rel(r.dv, orr["dv"]), rel(r.de, orr["de"]), r.min_h_over_speed, orr["ratio"], "it", oh.last_cg_iters)
print("mass diag", rel(hy._mass_diag, oh.mdiag), "minv", rel(hy._m_e_inv, oh.Minv))
# rhs
DF = O.force_D(osig, ogeo[2], ogeo[3])
F1 = O.force_apply(oh.dofmap, oh.nn, DF, oh.Bk, oh.Gk, oh.Bt, oh.ones_t, d)
from paper_2112_07075_b200.operators import ForcePA
f = ForcePA(hy.kin, hy.thermo, geo, sig)
print("F1", rel(f.apply(np.ones(hy.thermo.ndof)), F1), "Ftv", rel(f.apply_transpose(st.v), O.force_apply_t(oh.dofmap, DF, oh.Bk, oh.Gk, oh.Bt, ost["v"], d)))
dvs = hy._solve_momentum(-F1)
print("solve", rel(dvs, oh.solve_momentum(-F1)), oh.last_cg_iters)
