/*
 * b200hydro.h -- C-ABI of libb200hydro.so, the B200 (sm_100a) matrix-free
 * partial-assembly Lagrange hot path.
 *
 * Every entry point replaces one call of the reference Python package
 * `ale_minihydro` (/root/reference/pkg/src/ale_minihydro); the cited
 * file:line is the reference interface it stands in for.  The reference has no
 * FFI of its own: its backend plug-in point is `place: ExecPlace`
 * (kernel_exec.py:39-66, hydro.py:150, operators.py:67).  INTEGRATION.md shows
 * the ctypes binding a maintainer adds behind that parameter.
 *
 * Conventions
 *   - Plain C types only.  Array arguments are DEVICE pointers (cudaMalloc'd or
 *     torch CUDA storage) unless the name ends in `_host`.
 *   - Layouts are the reference API layouts (C-contiguous float64, element index
 *     fastest in point data): H1 vector fields (NN, d) node-major; L2 fields
 *     (NE*nt) element-major; point data (nq, NE); jacobians (d, d, nq, NE);
 *     E-vectors (nl, NE[, ncomp]); boundary mask (NN, d) uint8.
 *   - All calls are ordered on the context's stream (hx_set_stream).  Calls that
 *     report a status or a scalar synchronise that stream before returning.
 *   - Return value: HX_OK or one of the HX_E* codes below.  Inverted-element,
 *     CG and time-step failures carry details in the out-structs, so the Python
 *     layer can raise the reference's exception types with the same fields.
 *   - Results are deterministic: no floating-point atomics on any result path.
 */
#ifndef B200HYDRO_H
#define B200HYDRO_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes (map to the reference exceptions) */
enum {
  HX_OK = 0,
  HX_EINVAL = 1,        /* ValueError (fespace.py:223-231, tensor_basis.py:216-222) */
  HX_EINVERTED = 2,     /* InvertedElementError(element, point, detj) (fespace.py:37-41) */
  HX_ECG_BREAKDOWN = 3, /* CGError "p^T A p <= 0" (operators.py:354-355) */
  HX_ECG_MAXITER = 4,   /* CGError "did not converge" (operators.py:366) */
  HX_ECUDA = 5,         /* CUDA runtime error */
  HX_ENCCL = 6,         /* multi-GPU exchange error (a peer stopped answering) */
  HX_EUNDERFLOW = 7     /* TimestepUnderflow (hydro.py:82-83, 369-372, 405) */
};

enum { HX_SPACE_H1 = 0, HX_SPACE_L2 = 1 };

typedef struct hx_ctx hx_ctx;
typedef struct hx_mass hx_mass;
typedef struct hx_force hx_force;
typedef struct hx_op hx_op;
typedef struct hx_tmop hx_tmop;

/* Mesh + discretisation description (HighOrderMesh fespace.py:63-80,
 * FiniteElementSpace fespace.py:177-208, QuadratureRule1D tensor_basis.py:41-50,
 * eval_basis tensor_basis.py:158-172).  Host pointers; copied by hx_create. */
typedef struct {
  int32_t dim;             /* 2 or 3 */
  int32_t order;           /* kinematic order p (1..4) */
  int32_t q1d;             /* quadrature points per direction (must be p+2) */
  int32_t thermo_order;    /* L2 order (must be max(p-1, 0)) */
  int64_t num_elements;    /* NE */
  int64_t num_nodes;       /* NN */
  const int64_t* dofmap_host;  /* (nl, NE) node ids, reference layout */
  const double* B_host;    /* (Q, p+1) kinematic basis at quadrature points */
  const double* G_host;    /* (Q, p+1) its derivative */
  const double* Bt_host;   /* (Q, Dt) thermodynamic basis at quadrature points */
  const double* qweights_host; /* (Q) 1D Gauss weights */
  int32_t device;          /* CUDA ordinal */
} hx_mesh_desc;

/* Physics + solver controls (MaterialModel hydro.py:40-48, ViscosityModel :51-65,
 * StepControls :68-79, LagrangeHydro(momentum_rel_tol) :152, _solve_momentum
 * max_iter :335, rk2_step(max_retries) :375). */
typedef struct {
  double gamma, q1, q2;
  double rel_tol;
  int32_t max_iter;
  int32_t max_retries;
  double cfl, dt_min, dt_max, t_final;
} hx_params;

/* Inverted element: the first (q-major) point with det J <= 0 (fespace.py:335-337). */
typedef struct {
  int32_t inverted;
  int64_t element;
  int64_t point;
  double detj;
} hx_inverted;

/* CG outcome (cg_solve operators.py:333-366). */
typedef struct {
  int32_t code;            /* HX_OK, HX_ECG_BREAKDOWN, HX_ECG_MAXITER */
  int32_t iterations;
  int32_t n_residuals;     /* entries written to the residual history */
} hx_cg_info;

/* Outcome of one rates() / step() call. */
typedef struct {
  int32_t code;            /* HX_OK or the failure code */
  int32_t cg_iterations[2];/* momentum CG iterations of stage 1 and 2 */
  int32_t retries;         /* halvings performed by rk2_step */
  int64_t clamped;         /* clamp_warnings increment (hydro.py:275-278) */
  double dt;               /* accepted time step */
  double min_h_over_speed; /* stage-2 ratio (rk2_step info, hydro.py:402) */
  double t_new;
  hx_inverted inv;         /* for HX_EINVERTED */
  int32_t failed_stage;    /* 0: S (timestep_estimate), 1: midpoint, 2: new state */
} hx_step_info;

/* ---- context --------------------------------------------------------- */

/* Replaces the construction of LagrangeHydro / FiniteElementSpace (hydro.py:142-172,
 * fespace.py:184-208): uploads dofmap, builds the transpose (node -> element entries,
 * ascending element) used by the deterministic scatter, basis tables. */
int hx_create(const hx_mesh_desc* desc, hx_ctx** out);
int hx_destroy(hx_ctx* ctx);
/* stream: a cudaStream_t (0 = legacy default stream). */
int hx_set_stream(hx_ctx* ctx, void* stream);
/* Human-readable message of the last error on this context. */
const char* hx_last_error(hx_ctx* ctx);
/* Number of kernels this context launched so far (evidence counter). */
int64_t hx_kernel_launches(hx_ctx* ctx);
/* Restriction layout chosen by hx_create: 1 = structured brick (the dofmap is the
 * lexicographic numbering of cartesian_mesh, fespace.py:352-385: index-free CG kernels,
 * element-major E-vectors), 0 = generic CSR transpose map.  Results are identical. */
int hx_layout(hx_ctx* ctx);
/* Multi-material extension (not in the reference, whose MaterialModel has one gamma,
 * hydro.py:40-48): per-element adiabatic index gamma_e (NE, device) used by the stress /
 * rates kernels instead of hx_params.gamma; NULL restores the single gamma. */
int hx_set_material(hx_ctx* ctx, const double* gamma_e);

/* ---- restriction (fespace.py:221-234) -------------------------------- */

/* FiniteElementSpace.gather: E[l, e, c] = L[dofmap[l, e], c]  (fespace.py:221-225) */
int hx_gather(hx_ctx* ctx, int space, const double* L, int ncomp, double* E);
/* FiniteElementSpace.scatter_add: ascending-element accumulation from 0.0,
 * bit-identical to np.add.at (fespace.py:227-234) */
int hx_scatter_add(hx_ctx* ctx, int space, const double* E, int ncomp, double* L);

/* ---- geometry (fespace.py:305-346) ----------------------------------- */

/* compute_geometric_factors(mesh, quad, x): jac (d,d,nq,NE), detj, jinv
 * (reference convention: 2D J^{-1}, 3D cof(J)/det = J^{-T}, fespace.py:280-302),
 * wdetj (nq,NE).  Any output pointer may be NULL.  On det<=0 returns
 * HX_EINVERTED with *inv filled. */
int hx_geometry(hx_ctx* ctx, const double* x, double* jac, double* detj, double* jinv,
                double* wdetj, hx_inverted* inv);

/* ---- PA mass (operators.py:84-124) ----------------------------------- */

/* MassPA(space, geom, qdata=D): D (nq, NE) */
int hx_mass_create(hx_ctx* ctx, const double* D, hx_mass** out);
int hx_mass_destroy(hx_mass* m);
/* MassPA.apply: x (NN, ncomp) -> y (NN, ncomp), ncomp in 1..3 (operators.py:97-115) */
int hx_mass_apply(hx_mass* m, const double* x, int ncomp, double* y);
/* MassPA.diagonal (operators.py:117-124) */
int hx_mass_diagonal(hx_mass* m, double* diag);
/* Jacobi PCG on the mass operator (cg_solve operators.py:333-366) with identity rows
 * on masked components (_solve_momentum hydro.py:319-337).  rhs, x: (NN, ncomp);
 * bcmask (NN, ncomp) uint8 or NULL; precond_diag (NN, ncomp) or NULL (no
 * preconditioner); residuals (max_iter+1 doubles, device) may be NULL. */
int hx_mass_cg(hx_mass* m, const double* rhs, int ncomp, const uint8_t* bcmask,
               const double* precond_diag, double rel_tol, int max_iter, double* x,
               double* residuals, hx_cg_info* info);

/* ---- PA force (operators.py:239-300) --------------------------------- */

/* ForcePA(kin, thermo, geom, sigma): D_F = sum_b sigma[a,b] jinv[l,b] wdetj  (operators.py:258)
 * sigma, jinv: (d,d,nq,NE); wdetj (nq,NE).  D_out (d,d,nq,NE) may be NULL. */
int hx_force_create(hx_ctx* ctx, const double* sigma, const double* jinv, const double* wdetj,
                    double* D_out, hx_force** out);
int hx_force_destroy(hx_force* f);
/* ForcePA.apply: e (NE*nt) -> y (NN, d)  (operators.py:264-280) */
int hx_force_apply(hx_force* f, const double* e, double* y);
/* ForcePA.apply_transpose: v (NN, d) -> y (NE*nt)  (operators.py:282-300) */
int hx_force_apply_t(hx_force* f, const double* v, double* y);

/* ---- remap-phase PA operators (operators.py:143-236) --------------------
 * Scalar H1 operators on the same sum-factorised machinery (not on the Lagrange path).
 * hx_diffusion_create: D[a][c] = sum_b jinv[a][b] jinv[c][b] wdetj (nu)   (DiffusionPA.__init__ :145-149)
 * hx_convection_create: D[l] = sum_b jinv[l][b] u[b] wdetj               (ConvectionPA.__init__ :194-198)
 * jinv (d,d,nq,NE), wdetj/nu (nq,NE), u_points (d,nq,NE); D_out (reference layout) may be NULL.
 * hx_op_apply: y = sum_a G_a^T (sum_b D G_b x) (DiffusionPA.apply :151-168) or
 *              y = B^T (sum_l D[l] G_l x)       (ConvectionPA.apply :200-214); x, y (NN). */
int hx_diffusion_create(hx_ctx* ctx, const double* jinv, const double* wdetj, const double* nu, double* D_out,
                        hx_op** out);
int hx_convection_create(hx_ctx* ctx, const double* jinv, const double* u_points, const double* wdetj,
                         double* D_out, hx_op** out);
int hx_op_apply(hx_op* op, const double* x, double* y);
int hx_op_destroy(hx_op* op);

/* ---- TMOP mesh optimisation (meshopt.py:248-486) ------------------------- */

/* TMOPObjective.__init__ (meshopt.py:257-287): the per-point target inverses winv
 * (d,d,nq,NE), wdetW = w_q det W (nq,NE), the anchor positions x0 (NN,d) and the limiting
 * radii d(x0) (NN), device pointers in the reference layouts (copied).  composite = 0: the
 * shape metric of metric_for(d) (2D |T|^2/(2 det T) - 1, 3D |T|^2|T^-1|^2/9 - 1); 1:
 * w_shape * shape + w_size * SizeMetric (metric_for(d, with_size=True): 1, 1). */
int hx_tmop_create(hx_ctx* ctx, const double* winv, const double* wdetw, const double* x0,
                   const double* dlim, int composite, double w_shape, double w_size, double gamma,
                   hx_tmop** out);
/* gamma (the "auto" value is computed by the caller from hx_tmop_terms, meshopt.py:300-312). */
int hx_tmop_set_gamma(hx_tmop* op, double gamma);
/* _mu_term / _limit_term (meshopt.py:335-356): mu_sum = sum w detW mu(T(x)); lim_sum (if
 * want_limit) = sum_a sum_q w detW ((x - x0)/d)_a^2 without gamma; valid = 0 when det A <= 0
 * at some point (the objective's +inf sentinel, meshopt.py:357-362). */
int hx_tmop_terms(hx_tmop* op, const double* x, int want_limit, double* mu_sum, double* lim_sum,
                  int* valid);
/* gradient (meshopt.py:376-389, 391-405): dF/dx (NN,d), HX_EINVERTED on an invalid mesh. */
int hx_tmop_gradient(hx_tmop* op, const double* x, double* grad);
/* hessian_action (meshopt.py:407-440): H(x) dx (NN,d). */
int hx_tmop_hessian_action(hx_tmop* op, const double* x, const double* dx, double* out);
/* hessian_diagonal (meshopt.py:442-486): diag H(x) (NN,d), matrix-free. */
int hx_tmop_hessian_diagonal(hx_tmop* op, const double* x, double* diag);
int hx_tmop_destroy(hx_tmop* op);

/* ---- Lagrange phase (hydro.py:220-405) ------------------------------- */

/* begin_phase (hydro.py:220-232): mass qdata = (wdetj/detj)*qdata0 at x, its
 * diagonal, and the per-element inverse thermodynamic mass.  bcmask (NN,d) or NULL.
 * mass_D_out (nq,NE), mass_diag_out (NN), minv_out (NE,nt,nt) may be NULL. */
int hx_phase_begin(hx_ctx* ctx, const double* x, const double* qdata0, const uint8_t* bcmask,
                   double* mass_D_out, double* mass_diag_out, double* minv_out);
/* stress_qdata (hydro.py:254-315): sigma (d,d,nq,NE) (may be NULL), min ratio, clamp count. */
int hx_stress(hx_ctx* ctx, const hx_params* prm, const double* x, const double* v,
              const double* e, const double* qdata0, double* sigma, double* min_ratio,
              int64_t* clamped, hx_inverted* inv);
/* timestep_estimate's ratio (hydro.py:364-367 -> compute_geometric_factors fespace.py:305-346
 * + stress_qdata hydro.py:254-315): min h/(c_s+|v|), clamp count and the first inverted
 * point, fused (no geometry or sigma written); after hx_phase_begin; 3D, p >= 2. */
int hx_timestep_ratio(hx_ctx* ctx, const hx_params* prm, const double* x, const double* v,
                      const double* e, double* min_ratio, int64_t* clamped, hx_inverted* inv);
/* solve_energy (hydro.py:339-344): out = M_e^{-1} rhs per element (after hx_phase_begin). */
int hx_energy_solve(hx_ctx* ctx, const double* rhs, double* out);
/* rates (hydro.py:346-360): fused quadrature-point setup + F.1 + F^T v + M_e^{-1},
 * then the masked momentum CG.  dv (NN,d), de (NE*nt). */
int hx_rates(hx_ctx* ctx, const hx_params* prm, const double* x, const double* v,
             const double* e, double* dv, double* de, hx_step_info* info);
/* One Lagrange step = timestep_estimate (hydro.py:364-373) + rk2_step (hydro.py:375-405)
 * on device-resident state, one host synchronisation.  Output buffers must not
 * alias inputs.  t is the state time; info->t_new = t + dt. */
int hx_step(hx_ctx* ctx, const hx_params* prm, double t, const double* x, const double* v,
            const double* e, double* x_out, double* v_out, double* e_out, hx_step_info* info);
/* rk2_step(state, dt) alone (hydro.py:375-405): the caller supplies dt. */
int hx_rk2_step(hx_ctx* ctx, const hx_params* prm, double t, double dt, const double* x, const double* v,
                const double* e, double* x_out, double* v_out, double* e_out, hx_step_info* info);
/* Same step with HOST state buffers (pinned or pageable): H2D, step, D2H in one call
 * -- the end-to-end entry a host-side caller binds. In/out may alias.  On a 3D brick the
 * H2D is streamed in z-slabs behind the step's launch (HX_STREAM_IN slabs, default 3; 0 =
 * one up-front copy) and overlaps the stage-1 rates kernel; x' and e' are read back while
 * stage 2 runs.  Results are bit-identical to hx_step on the same state. */
int hx_step_host(hx_ctx* ctx, const hx_params* prm, double t, double* x_host, double* v_host,
                 double* e_host, hx_step_info* info);
/* kinetic_energy / internal_energy (hydro.py:409-420) with the phase mass. */
int hx_energies(hx_ctx* ctx, const double* v, const double* e, const double* qdata0,
                double* kinetic, double* internal);

/* ---- live kernel timing (CUDA events around instrumented launches) ------------
 * classes: 0 fused rates, 1 PA mass (CG), 2 CG node update, 3 CG init,
 * 4 state axpy, 5 geometry validity, 6 other. */
int hx_prof_enable(hx_ctx* ctx, int on);
int hx_prof_read(hx_ctx* ctx, int kclass, double* total_ms, int64_t* count);
int hx_prof_reset(hx_ctx* ctx);
/* Step graphs captured after this call duplicate every launch of kernel class `kclass`
 * (0 rates, 1 mass, 2 CG node pass, 3 CG init, 4 state update, 5 validity; -1 restores
 * plain graphs).  The CG node pass's duplicate is a dry copy writing to scratch.  A
 * class's in-step cost is (step time with duplicates - plain step time) / the number of
 * duplicates that did work, which hx_prof_read(kclass) counts (bench.py).  Measurement
 * hook; replaces no reference call. */
int hx_prof_dup(hx_ctx* ctx, int kclass);
/* Diagnostic (no reference counterpart): fp64 FMA peak of the current device, measured
 * with independent DFMA chains at full occupancy (best of 5 CUDA-event-timed launches);
 * the denominator of the fp64 roofline fractions bench.py reports. */
int hx_fp64_peak(double* tflops);

/* ---- multi-GPU (domain decomposition; the reference's P = identity) -- */

/* Device-resident exchange of the momentum CG (hx_mass_cg) over peer memory, one
 * brick subdomain per rank (paper_2112_07075_b200/partition.py).  Each rank owns a
 * MAILBOX (flags, scalar slots, halo receive blocks) that every rank maps; inside the
 * CG the interface-node sums and the p.Ap / r.z world sums move by P2P stores plus
 * release/acquire sequence flags (no host round trip, no NCCL call in the loop), summed
 * in ascending rank order so all sharers hold identical values.  Replaces the P operator
 * the reference leaves as identity inside cg_solve (operators.py:333-366).
 *   snode/sdst/sidx (nsh): for every (shared node, neighbour) pair, the local node, the
 *     neighbour rank and the node's index in the list of nodes the two ranks share
 *     (sorted by global id: the same index on both sides), < maxh;
 *   hnode (nh), hoff (nh+1), hsrc: interface nodes and their sharers in ascending rank,
 *     -1 = this rank, else (rank << 24) | index;
 *   nbr (nnbr): neighbour ranks; owned (NN host bytes): 1 where this rank owns the node;
 *   maxh: the same on every rank (max shared-list length over all rank pairs).
 * hx_peer_setup allocates the mailbox and returns its device pointer; hx_peer_connect
 * takes every rank's mailbox pointer in this address space (hx_peer_ipc_open for other
 * processes, the pointer itself for ranks sharing a process).  All ranks must then run
 * the same sequence of hx_mass_cg calls concurrently. */
int hx_peer_setup(hx_ctx* ctx, int rank, int nranks, int maxh, int nsh, const int32_t* snode,
                  const int32_t* sdst, const int32_t* sidx, int nh, const int32_t* hnode,
                  const int32_t* hoff, const int32_t* hsrc, int nnbr, const int32_t* nbr,
                  const uint8_t* owned, void** mailbox);
int hx_peer_connect(hx_ctx* ctx, void* const* mailboxes);
/* CUDA IPC export / import of a mailbox (64-byte handle) for ranks in other processes. */
/* Detach from the exchange (after the last exchanging step, before the peers' mailboxes are
 * unmapped or freed): synchronises the context's streams, clears the peer pointers and drops
 * the step graphs that contain exchange launches.  Replaces no reference call (the
 * reference's P operator is the identity). */
int hx_peer_disconnect(hx_ctx* ctx);
int hx_peer_ipc_handle(const void* mailbox, void* handle_out);
int hx_peer_ipc_open(const void* handle, void** ptr_out);
int hx_peer_ipc_close(void* ptr);
/* Diagnostic: out[0] = exchange counter, out[1] = timeout flag, out[2 + q] = last
 * sequence number rank q posted to this rank (2 + 64 values). */
int hx_peer_state(hx_ctx* ctx, uint64_t* out);
/* 1 once hx_peer_connect succeeded. */
int hx_comm_active(hx_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* B200HYDRO_H */
