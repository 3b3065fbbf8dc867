// hx_kernels.cuh -- sm_100a kernels of the PA Lagrange hot path (fp64).
//
// Device layouts (internal, chosen for coalescing; the C-ABI converts at the edge):
//   emap   (NE, nl) int32       element-major node ids (dofmap transposed)
//   csr    node -> E-vector entries e*nl+l in ascending element order (deterministic G^T)
//   own    (NE, nl) uint8       1 on the first (lowest-element) occurrence of each node
//   Dm     (NE, nq)             mass point data  w*rho0*detJ0  (operators.py:85-95)
//   qd0    (NE, nq)             rho0*detJ0  (hydro.py:195)
//   DF     (NE, d*d, nq)        force point data (operators.py:258)
//   minv   (NE, nt, nt)         inverse thermodynamic mass blocks (hydro.py:229-232)
//   evec   (NE, nl, ncomp)      element results before the scatter
#pragma once

#include "hx_core.cuh"

namespace hx {

// ---------------------------------------------------------------------------
// shared argument blocks

struct Tables {
  const double* B;    // (Q, D1)
  const double* G;    // (Q, D1)
  const double* Bt;   // (Q, DT)
  const double* wnd;  // (nq) tensor weights, x fastest (fespace.py:339-344)
  const double* psi1; // (nq) thermodynamic interpolant of the constant 1
};

template <int Q, int D1, int DT>
__device__ __forceinline__ void load_tables(const Tables& t, double* sB, double* sG, double* sBt) {
  for (int i = threadIdx.x; i < Q * D1; i += blockDim.x) {
    sB[i] = t.B[i];
    sG[i] = t.G[i];
  }
  for (int i = threadIdx.x; i < Q * DT; i += blockDim.x) sBt[i] = t.Bt[i];
}

// Packed symmetric storage of the inverse thermodynamic mass (3D, p <= 3, i.e. whenever
// k_minv_warp builds it): the lower triangle row by row, entry (i, j <= i) at
// i (i + 1) / 2 + j, nt (nt + 1) / 2 doubles per element (hydro.py:229-232: M_e is SPD, so
// its inverse is symmetric; 378 instead of 729 doubles at nt = 27).
template <int DIM, int P>
__host__ __device__ constexpr bool minv_packed() { return DIM == 3 && P <= 3; }
__host__ __device__ constexpr int tri(int i) { return i * (i + 1) / 2; }

struct StatusDev {
  unsigned long long inv_key;  // min over det<=0 points of q*NE+e (~0ull if none)
  unsigned long long clamps;   // e<0 clamps (hydro.py:275-278)
  double min_ratio;            // min h/(c_s+|v|)  (hydro.py:311-315)
  int pad;
};

// ---------------------------------------------------------------------------
// per-point physics (hydro.py:271-315, fespace.py:280-302, operators.py:258)

template <int DIM>
struct PointOut {
  double det;
  double jinv[DIM][DIM];
  double sigma[DIM][DIM];
  double ratio;
  int clamped;
};

// dx[a][b] = d x_a / d xi_b ; reference "inverse": 2D adj/det, 3D cof/det
template <int DIM>
__device__ __forceinline__ double det_inv(const double (&J)[DIM][DIM], double (&inv)[DIM][DIM]) {
  if constexpr (DIM == 2) {
    const double det = J[0][0] * J[1][1] - J[0][1] * J[1][0];
    inv[0][0] = J[1][1] / det;
    inv[0][1] = -J[0][1] / det;
    inv[1][0] = -J[1][0] / det;
    inv[1][1] = J[0][0] / det;
    return det;
  } else {
    const double det = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) -
                       J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
                       J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const int r0 = r == 0 ? 1 : 0, r1 = r == 2 ? 1 : 2;
        const int c0 = c == 0 ? 1 : 0, c1 = c == 2 ? 1 : 2;
        const double m = J[r0][c0] * J[r1][c1] - J[r0][c1] * J[r1][c0];
        inv[r][c] = (((r + c) & 1) ? -m : m) / det;
      }
    return det;
  }
}

template <int DIM>
__device__ __forceinline__ void point_physics(const double (&J)[DIM][DIM], const double (&dv)[DIM][DIM],
                                              const double (&vq)[DIM], double eq, double qd0,
                                              double gamma, double q1, double q2, PointOut<DIM>& o) {
  o.det = det_inv<DIM>(J, o.jinv);
  const double det = o.det;
  const double rho = qd0 / det;
  o.clamped = 0;
  if (eq < 0.0) {
    o.clamped = 1;
    eq = 0.0;
  }
  const double p = (gamma - 1.0) * rho * eq;
  const double cs = sqrt(gamma * (gamma - 1.0) * eq);
  double gv[DIM][DIM];
#pragma unroll
  for (int a = 0; a < DIM; ++a)
#pragma unroll
    for (int b = 0; b < DIM; ++b) {
      double s = 0.0;
#pragma unroll
      for (int l = 0; l < DIM; ++l) s = fma(dv[a][l], o.jinv[l][b], s);
      gv[a][b] = s;
    }
#pragma unroll
  for (int a = 0; a < DIM; ++a)
#pragma unroll
    for (int b = 0; b < DIM; ++b) o.sigma[a][b] = (a == b) ? -p : 0.0;
  double div = 0.0;
#pragma unroll
  for (int a = 0; a < DIM; ++a) div += gv[a][a];
  const double h = (DIM == 3) ? pow(det, 1.0 / 3.0) : pow(det, 0.5);
  if (q1 > 0.0 || q2 > 0.0) {
    double mu = rho * h * (q1 * cs + q2 * h * fabs(div));
    mu = div < 0.0 ? mu : 0.0;
#pragma unroll
    for (int a = 0; a < DIM; ++a)
#pragma unroll
      for (int b = 0; b < DIM; ++b) o.sigma[a][b] += mu * (0.5 * (gv[a][b] + gv[b][a]));
  }
  double v2 = 0.0;
#pragma unroll
  for (int a = 0; a < DIM; ++a) v2 += vq[a] * vq[a];
  const double speed = cs + sqrt(v2);
  o.ratio = speed > 0.0 ? h / fmax(speed, 1e-300) : __longlong_as_double(0x7ff0000000000000ll);
}

// D_F[a][l] = sum_b sigma[a][b] jinv[l][b] wdetj  (operators.py:258)
template <int DIM>
__device__ __forceinline__ void force_point(const double (&sig)[DIM][DIM], const double (&jinv)[DIM][DIM],
                                            double wdetj, double (&DF)[DIM][DIM]) {
#pragma unroll
  for (int a = 0; a < DIM; ++a)
#pragma unroll
    for (int l = 0; l < DIM; ++l) {
      double s = 0.0;
#pragma unroll
      for (int b = 0; b < DIM; ++b) s = fma(sig[a][b], jinv[l][b], s);
      DF[a][l] = s * wdetj;
    }
}

// block-level status publication: ratio min, clamp sum, inversion key
template <int NT>
__device__ __forceinline__ void publish_status(StatusDev* st, double rmin, long long clamps,
                                               unsigned long long key, double* sbuf) {
  rmin = warp_min(rmin);
  clamps = warp_sum_ll(clamps);
  if ((threadIdx.x & 31) == 0) {
    if (clamps) atomicAdd(&st->clamps, (unsigned long long)clamps);
    atomic_min_nonneg(&st->min_ratio, rmin);
  }
  if (key != ~0ull) atomicMin(&st->inv_key, key);
  (void)sbuf;
}

// ---------------------------------------------------------------------------
// K_rates: fused quadrature-point setup + F.1 + F^T v + M_e^{-1}
// (LagrangeHydro.rates hydro.py:346-360 minus the momentum solve: geometry
//  fespace.py:305-346, stress_qdata hydro.py:254-315, ForcePA operators.py:247-300,
//  solve_energy hydro.py:339-344).  One CTA per element; D_F never leaves smem.

struct RatesArgs {
  const double* x;     // (NN, d)
  const double* v;     // (NN, d)
  const double* e;     // (NE*nt)
  const double* qd0;   // (NE, nq)
  const int* emap;     // (NE, nl)
  const int* slot;     // (NE, nl) position of (e, l) in the node-sorted E-vector
  const double* minv;  // (NE, nt, nt)
  Tables tab;
  double gamma, q1, q2;
  const double* gam;   // per-element adiabatic index (multi-material extension) or null
  long long ne;
  double* evec;        // (NE, nl, d)  element F.1
  double* de;          // (NE*nt)      M_e^{-1} F^T v
  StatusDev* st;
  int mode;            // 0: full rates; 1: geometry validity only
};

template <int DIM, int P>
struct RatesSmem {
  using D = Disc<DIM, P>;
  static constexpr int NCG = 2 * DIM;
  static constexpr int A = cmax(NCG * D::NL, DIM == 3 ? 3 * NCG * D::Q * D::Q * D::D1 : 0);
  static constexpr int S = 2 * NCG * D::Q * ipow(D::D1, DIM - 1);
  static constexpr int OUT = NCG * (DIM + 1) * D::NQ;
  static constexpr int TH = 2 * D::NQ;
  static constexpr int TABS = 2 * D::Q * D::D1 + D::Q * D::DT;
  static constexpr int RED = 32;
  static constexpr int TOTAL = TABS + A + S + OUT + TH + D::NT + RED;
  static constexpr size_t bytes = sizeof(double) * TOTAL;
};

template <int DIM, int P, int NT>
__global__ void __launch_bounds__(NT) k_rates(RatesArgs a) {
  using D = Disc<DIM, P>;
  using SM = RatesSmem<DIM, P>;
  constexpr int D1 = D::D1, Q = D::Q, DT = D::DT, NL = D::NL, NQ = D::NQ, NTH = D::NT;
  constexpr int NCG = SM::NCG;
  extern __shared__ double smem[];
  double* sB = smem;
  double* sG = sB + Q * D1;
  double* sBt = sG + Q * D1;
  double* rA = sBt + Q * DT;
  double* rS = rA + SM::A;
  double* rOut = rS + SM::S;
  double* rTH = rOut + SM::OUT;
  double* rMV = rTH + SM::TH;
  double* red = rMV + NTH;
  const int tid = threadIdx.x;
  const long long e = blockIdx.x;
  load_tables<Q, D1, DT>(a.tab, sB, sG, sBt);

  // gather x and v (components 0..DIM-1 = x, DIM..2DIM-1 = v), and e
  const int* em = a.emap + e * NL;
  for (int i = tid; i < NL * DIM; i += NT) {
    const int l = i / DIM, c = i - l * DIM;
    const long long n = em[l];
    rA[c * NL + l] = a.x[n * DIM + c];
    if (a.mode == 0) rA[(DIM + c) * NL + l] = a.v[n * DIM + c];
  }
  if (a.mode == 0)
    for (int i = tid; i < NTH; i += NT) rTH[i] = a.e[e * NTH + i];
  __syncthreads();
  if (a.mode == 1) {
    grad<DIM, D1, Q, DIM, DIM + 1, NT>(sB, sG, rA, rS, rA, rOut, tid);
    __syncthreads();
    unsigned long long key = ~0ull;
    for (int q = tid; q < NQ; q += NT) {
      double J[DIM][DIM], inv[DIM][DIM];
#pragma unroll
      for (int c = 0; c < DIM; ++c)
#pragma unroll
        for (int b = 0; b < DIM; ++b) J[c][b] = rOut[(c * (DIM + 1) + b) * NQ + q];
      const double det = det_inv<DIM>(J, inv);
      if (det <= 0.0) {
        const unsigned long long k = (unsigned long long)q * a.ne + e;
        key = k < key ? k : key;
      }
    }
    if (key != ~0ull) atomicMin(&a.st->inv_key, key);
    return;
  }
  grad<DIM, D1, Q, NCG, DIM + 1, NT>(sB, sG, rA, rS, rA, rOut, tid);
  double* eq = interp<DIM, DT, Q, 1, NT>(sBt, rTH, rTH + NQ, tid);
  double* sq = (eq == rTH) ? rTH + NQ : rTH;
  __syncthreads();

  // per-point physics; the point owner rewrites its slots in place:
  //   rOut[c][l][q] (c < DIM) <- D_F[c][l] * psi1_q  (F.1 components)
  //   sq[q]                   <- sum_{a,l} D_F[a][l] dv_a/dxi_l  (F^T v integrand)
  double rmin = __longlong_as_double(0x7ff0000000000000ll);
  long long clamps = 0;
  unsigned long long key = ~0ull;
  for (int q = tid; q < NQ; q += NT) {
    double J[DIM][DIM], dv[DIM][DIM], vq[DIM];
#pragma unroll
    for (int c = 0; c < DIM; ++c) {
#pragma unroll
      for (int b = 0; b < DIM; ++b) {
        J[c][b] = rOut[(c * (DIM + 1) + b) * NQ + q];
        dv[c][b] = rOut[((DIM + c) * (DIM + 1) + b) * NQ + q];
      }
      vq[c] = rOut[((DIM + c) * (DIM + 1) + DIM) * NQ + q];
    }
    PointOut<DIM> po;
    point_physics<DIM>(J, dv, vq, eq[q], a.qd0[e * NQ + q], a.gam ? __ldg(a.gam + e) : a.gamma, a.q1, a.q2, po);
    if (po.det <= 0.0) {
      const unsigned long long k = (unsigned long long)q * a.ne + e;
      key = k < key ? k : key;
    }
    clamps += po.clamped;
    rmin = fmin(rmin, po.ratio);
    double DF[DIM][DIM];
    force_point<DIM>(po.sigma, po.jinv, a.tab.wnd[q] * po.det, DF);
    const double p1 = a.tab.psi1[q];
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < DIM; ++c)
#pragma unroll
      for (int l = 0; l < DIM; ++l) {
        s += DF[c][l] * dv[c][l];
        rOut[(c * (DIM + 1) + l) * NQ + q] = DF[c][l] * p1;
      }
    sq[q] = s;
  }
  publish_status<NT>(a.st, rmin, clamps, key, red);
  __syncthreads();
  // F.1 element vector: grad_t over the x-slots; result into the dead v-slots
  double* fout = rOut + DIM * (DIM + 1) * NQ;
  grad_t<DIM, D1, Q, DIM, (DIM + 1) * NQ, NT>(sB, sG, rOut, rA, rS, fout, tid);
  // F^T v: thermodynamic transpose interpolation (operators.py:297)
  double* fv = interp_t<DIM, DT, Q, 1, NT>(sBt, sq, eq, tid);
  __syncthreads();
  for (int i = tid; i < NL * DIM; i += NT) {
    const int l = i / DIM, c = i - l * DIM;
    // node-sorted position (generic CSR path) or element-major (structured brick, coalesced)
    const long long pos = a.slot ? (long long)a.slot[e * NL + l] * DIM + c : e * (NL * DIM) + i;
    a.evec[pos] = fout[c * NL + l];
  }
  // de = M_e^{-1} (F^T v)_e   (einsum "eij,ej->ei", hydro.py:343)
  constexpr bool PK = minv_packed<DIM, P>();
  const double* mi = a.minv + e * (PK ? tri(NTH) : NTH * NTH);
  for (int i = tid; i < NTH; i += NT) {
    double s = 0.0;
    for (int j = 0; j < NTH; ++j) s = fma(mi[PK ? (j <= i ? tri(i) + j : tri(j) + i) : i * NTH + j], fv[j], s);
    a.de[e * NTH + i] = s;
  }
  (void)rMV;
}

// ---------------------------------------------------------------------------
// K_mass: PA mass action, one warp per element (MassPA._apply_scalar operators.py:97-115).
// CG mode fuses the direction update p = z + beta p_old, the wall mask of
// _solve_momentum (hydro.py:323-327) and the element-wise p.Ap partial:
//   p.Ap = sum_e sum_q D (B w_e)^2 + sum_{masked} p^2.

// ---------------------------------------------------------------------------
// multi-GPU peer-memory primitives (mailbox layout and protocol: hx_peer.cuh)

#define HX_MAXR 64
constexpr int SLOTW = 8;                               // doubles per (parity, source) slot
constexpr int MB_FLAG = 0;                             // u64 flag[src]
constexpr int MB_SLOT = HX_MAXR;                       // double slot[2][HX_MAXR][SLOTW]
constexpr int MB_BCF = HX_MAXR + 2 * SLOTW * HX_MAXR;  // u64: CTA-0 broadcast flag (local, gpu scope)
constexpr int MB_BC = MB_BCF + 8;                      // double bc[2][SLOTW]: world values for the other CTAs
constexpr int MB_RECV = MB_BC + 2 * SLOTW;             // double recv[src][maxh][nc]
constexpr unsigned long long PEER_SPIN_LIMIT = 1ull << 25;  // ~seconds: a stuck peer ends the CG with code 6

struct PeerDev {
  int rank, nranks, maxh;
  int nsh;                      // shared (node, neighbour) entries
  int nh;                       // interface nodes
  int nnbr;
  unsigned long long* seq;      // this rank's exchange counter
  int* err;                     // set to 1 on a peer timeout
  double* mb[HX_MAXR];          // every rank's mailbox in this address space
  int nbr[HX_MAXR];             // neighbour ranks
  const int* snode;             // per shared entry: local node
  const int* sdst;              //   destination rank
  const int* sidx;              //   index in the destination's recv block from this rank
  const int* hnode;             // interface nodes
  const int* hoff;              // (nh + 1) offsets into hsrc
  const int* hsrc;              // sharers in ascending rank: -1 = this rank, else (q << 24) | index
  const uint8_t* owned;         // (NN) lowest-rank sharer owns a node (dot products count it once)
  const int* ifx;               // (NN) interface index h of a node, -1 inside the subdomain
};

// what a CG launch's prologue needs for a world sum, passed by value in the kernel
// arguments (no dependent loads on the latency path)
struct PeerLite {
  double* me;               // this rank's mailbox
  double* const* mbs;       // every rank's mailbox (device array)
  unsigned long long* seq;  // exchange counter
  int rank, nranks;
  int post;                 // PEER_POST_*: the CG's world scalars posted by their producer launch
};
// producer-side posting of the CG's per-iteration world scalars (r.z_k by the node launch,
// p.Ap_k by the halo pack launch, or by the mass launch on a rank without neighbours): the
// last CTA of the producer to finish reduces the per-CTA partials and posts this rank's value
// to every rank, so the consumer launch's CTAs only poll flags that are usually already set
// (the post overlaps the launch gap instead of the consumer's prologue)
constexpr int PEER_POST_ON = 1, PEER_POST_MASS = 2;

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
#ifndef PEER_WORLD_PURE
#define PEER_WORLD_PURE 0
#endif
#ifndef PEER_SPIN_PURE
#define PEER_SPIN_PURE 0
#endif
#ifndef PEER_SLEEP_NS
#define PEER_SLEEP_NS 64
#endif
#ifndef PEER_ALL_CTAS
#define PEER_ALL_CTAS 1
#endif
#ifndef PEER_BC_SLEEP
#define PEER_BC_SLEEP 32
#endif
#ifndef PEER_FENCE_GPU
#define PEER_FENCE_GPU 0
#endif
__device__ __forceinline__ void fence_acq_rel_sys() {
#if PEER_FENCE_GPU
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
#else
  asm volatile("fence.acq_rel.sys;" ::: "memory");
#endif
}
// spin until *flag >= seq: relaxed polls (pure spin first, then backing off), one
// acquire fence after success; false after PEER_SPIN_LIMIT polls
__device__ __forceinline__ bool spin_flag(const unsigned long long* flag, unsigned long long seq) {
  unsigned long long spins = 0;
  while (ld_relaxed_sys(flag) < seq) {
    if (++spins > PEER_SPIN_PURE) __nanosleep(PEER_SLEEP_NS);
    if (spins > PEER_SPIN_LIMIT) return false;
  }
  fence_acq_rel_sys();
  return true;
}
__device__ __forceinline__ unsigned long long* mb_flag(double* mb, int src) {
  return reinterpret_cast<unsigned long long*>(mb) + MB_FLAG + src;
}
// wait until every listed rank published seq; false on timeout
__device__ __forceinline__ bool peer_wait(const PeerDev& pd, const int* ranks, int n, unsigned long long seq) {
  double* me = pd.mb[pd.rank];
  for (int j = 0; j < n; ++j) {
    const int q = ranks ? ranks[j] : j;
    if (q == pd.rank) continue;
    if (!spin_flag(mb_flag(me, q), seq)) return false;
  }
  return true;
}

// world sum of NV values inside a CG launch's prologue (multi-GPU): block 0 posts this
// rank's values to every rank's slot and publishes seq; every CTA waits for all ranks
// (itself included) and sums the slots in ascending rank order, so all CTAs of all ranks
// hold the same values.  False on a peer timeout.
__device__ __forceinline__ void st_release_gpu(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_gpu(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Block 0 alone talks to the other ranks (system scope: one release per rank, one acquire
// fence); it then broadcasts the world values to the launch's other CTAs through its own
// mailbox with a gpu-scope release, which they poll at gpu scope.
template <int NV>
__device__ __forceinline__ bool peer_world(const PeerLite& pl, unsigned long long seq, double (&v)[NV]) {
  __shared__ double wv[NV];
  __shared__ int wok;
  if (threadIdx.x == 0) {
    const int par = (int)(seq & 1);
    unsigned long long* bcf = reinterpret_cast<unsigned long long*>(pl.me) + MB_BCF;
    double* bc = pl.me + MB_BC + par * SLOTW;
    int ok = 1;
#if PEER_ALL_CTAS
    // every CTA reads the ranks' flags itself: relaxed polls, then one system-scope
    // acquire load per flag (no fence, no broadcast step)
    if (blockIdx.x == 0) {
      for (int q = 0; q < pl.nranks; ++q) {
        double* s = pl.mbs[q] + MB_SLOT + (par * HX_MAXR + pl.rank) * SLOTW;
#pragma unroll
        for (int t = 0; t < NV; ++t) s[t] = v[t];
      }
      for (int q = 0; q < pl.nranks; ++q) st_release_sys(mb_flag(pl.mbs[q], pl.rank), seq);
      *pl.seq = seq;
    }
    for (int q = 0; q < pl.nranks && ok; ++q) {
      unsigned long long spins = 0;
      const unsigned long long* f = mb_flag(pl.me, q);
      while (ld_relaxed_sys(f) < seq) {
        if (spins >= PEER_WORLD_PURE) __nanosleep(32);  // pure polls first, then back off
        if (++spins > PEER_SPIN_LIMIT) {
          ok = 0;
          break;
        }
      }
      if (ok) (void)ld_acquire_sys(f);
    }
    if (ok) {
      const double* s = pl.me + MB_SLOT + par * HX_MAXR * SLOTW;
#pragma unroll
      for (int t = 0; t < NV; ++t) {
        double tot = 0.0;
        for (int q = 0; q < pl.nranks; ++q) tot += __ldcg(s + q * SLOTW + t);
        wv[t] = tot;
      }
    }
    (void)bcf;
    (void)bc;
#else
    if (blockIdx.x == 0) {
      for (int q = 0; q < pl.nranks; ++q) {
        double* s = pl.mbs[q] + MB_SLOT + (par * HX_MAXR + pl.rank) * SLOTW;
#pragma unroll
        for (int t = 0; t < NV; ++t) s[t] = v[t];
      }
      // the release stores order this thread's slot writes; the halo data were fenced at
      // system scope by k_halo_pack, which completed before this launch
      for (int q = 0; q < pl.nranks; ++q) st_release_sys(mb_flag(pl.mbs[q], pl.rank), seq);
      *pl.seq = seq;
      for (int q = 0; q < pl.nranks && ok; ++q) ok = spin_flag(mb_flag(pl.me, q), seq) ? 1 : 0;
      const double* s = pl.me + MB_SLOT + par * HX_MAXR * SLOTW;
#pragma unroll
      for (int t = 0; t < NV; ++t) {
        double tot = 0.0;
        for (int q = 0; q < pl.nranks; ++q) tot += __ldcg(s + q * SLOTW + t);
        wv[t] = tot;
        bc[t] = tot;
      }
      bc[NV] = ok ? 1.0 : 0.0;
      st_release_gpu(bcf, seq);
    } else {
      unsigned long long spins = 0;
      while (ld_acquire_gpu(bcf) < seq) {
        if (PEER_BC_SLEEP) __nanosleep(PEER_BC_SLEEP);
        if (++spins > PEER_SPIN_LIMIT) {
          ok = 0;
          break;
        }
      }
      if (ok) {
#pragma unroll
        for (int t = 0; t < NV; ++t) wv[t] = __ldcg(bc + t);
        ok = __ldcg(bc + NV) != 0.0;
      }
    }
#endif
    wok = ok;
  }
  __syncthreads();
#pragma unroll
  for (int t = 0; t < NV; ++t) v[t] = wv[t];
  return wok != 0;
}
__device__ __forceinline__ PeerLite peer_lite(const PeerDev* pd) {
  return PeerLite{pd->mb[pd->rank], pd->mb, pd->seq, pd->rank, pd->nranks, 0};
}

// fixed-order sum of n grid partials, broadcast to every thread of the CTA
template <int NT>
__device__ __forceinline__ double reduce_bcast(const double* parts, int n, double* red) {
  __shared__ double bc;
  const double v = reduce_partials<NT>(parts, n, red);
  if (threadIdx.x == 0) bc = v;
  __syncthreads();
  return bc;
}

// world sum of NV values posted by the ranks' producer launches (cg_post_last): every CTA
// polls the ranks' flags (relaxed, then one acquire per flag) and sums the slots in ascending
// rank order, this rank's own included.  False on a peer timeout.
template <int NV>
__device__ __forceinline__ bool peer_recv(const PeerLite& pl, unsigned long long seq, double (&v)[NV]) {
  __shared__ double wv[NV];
  __shared__ int wok;
  if (threadIdx.x == 0) {
    const int par = (int)(seq & 1);
    int ok = 1;
    for (int q = 0; q < pl.nranks && ok; ++q) {
      unsigned long long spins = 0;
      const unsigned long long* f = mb_flag(pl.me, q);
      while (ld_relaxed_sys(f) < seq) {
        if (spins >= PEER_WORLD_PURE) __nanosleep(32);
        if (++spins > PEER_SPIN_LIMIT) {
          ok = 0;
          break;
        }
      }
      if (ok) (void)ld_acquire_sys(f);
    }
    if (ok) {
      const double* s = pl.me + MB_SLOT + par * HX_MAXR * SLOTW;
#pragma unroll
      for (int t = 0; t < NV; ++t) {
        double tot = 0.0;
        for (int q = 0; q < pl.nranks; ++q) tot += __ldcg(s + q * SLOTW + t);
        wv[t] = tot;
      }
    }
    wok = ok;
  }
  __syncthreads();
#pragma unroll
  for (int t = 0; t < NV; ++t) v[t] = wv[t];
  return wok != 0;
}

// end of a producer launch: every CTA has written its partial (and, for the halo pack, its
// system-fenced halo entries); the last CTA to arrive reduces the partials in the same fixed
// order the consumers used to (reduce_bcast) and posts the rank's value with seq to every
// rank's slot, then resets the arrival counter for the next launch.
template <int NT>
__device__ __forceinline__ void cg_post_last(const PeerLite& pl, const double* parts, int nparts, unsigned* counter,
                                             unsigned long long seq, double* red) {
  __shared__ int is_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    is_last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  const double v = reduce_bcast<NT>(parts, nparts, red);
  if (threadIdx.x == 0) {
    *counter = 0u;
    const int par = (int)(seq & 1);
    for (int q = 0; q < pl.nranks; ++q) pl.mbs[q][MB_SLOT + (par * HX_MAXR + pl.rank) * SLOTW] = v;
    for (int q = 0; q < pl.nranks; ++q) st_release_sys(mb_flag(pl.mbs[q], pl.rank), seq);
    *pl.seq = seq;
  }
}

// interface node sum (multi-GPU): the sharers' partials in ascending rank order from 0.0,
// this rank's own from the local E-vector, the others from the receive blocks
template <int NC>
__device__ __forceinline__ double peer_node_sum(const PeerDev* pd, double own, int h, int c) {
  const double* recv = pd->mb[pd->rank] + MB_RECV;
  double tot = 0.0;
  for (int s = __ldg(pd->hoff + h); s < __ldg(pd->hoff + h + 1); ++s) {
    const int src = __ldg(pd->hsrc + s);
    tot += src < 0 ? own : __ldcg(recv + ((long long)(src >> 24) * pd->maxh + (src & 0xffffff)) * NC + c);
  }
  return tot;
}

// Device CG state.  Each iteration k is a mass launch M(k) and a node launch N(k).
// Grid reductions are finished by the CONSUMER launch: every CTA of N(k) sums M(k)'s
// per-CTA p.Ap partials in the same fixed order (-> alpha_k), every CTA of M(k+1)
// sums N(k)'s r.z partials (-> stop test, beta_{k+1}); block 0 publishes the scalars.
// No fences, atomics or last-block tails on the iteration path.  Scalars that a
// launch reads while its block 0 writes the next value are ping-ponged by parity.
struct CGDev {
  double rz, norm0, alpha, beta, tol;
  double rz2[2];      // rz_k at [k & 1]
  double alpha2[2];   // alpha_k at [k & 1]
  int pend;           // x lags one iteration: k (odd) whose x += a_k p_k is still to apply, else 0
  int it_m, it_n;     // iteration index of the next mass / node launch
  int nparts_m, nparts_n;
  const double* parts_m;  // per-CTA p.Ap partials of the last mass launch
  const double* parts_n;  // per-CTA r.z partials of the last node launch
  double* hist;
  int it, active, code, iters, max_iter, nres;
  unsigned int cnt[4];
  unsigned long long cond;  // cudaGraphConditionalHandle of the WHILE node (graph mode)
  int use_cond;
  const PeerDev* peer;      // multi-GPU exchange (null on one GPU)
  unsigned long long seq0;  // exchange counter at the start of this solve
};

// Packed element map used by the CG kernels: node id | owner<<27 | wall-mask(c)<<(28+c)
// (one load per local node instead of node id + owner byte + mask byte).
__device__ __forceinline__ long long emf_node(int w) { return (long long)(w & 0x07ffffff); }
__device__ __forceinline__ bool emf_own(int w) { return (w >> 27) & 1; }
__device__ __forceinline__ bool emf_mask(int w, int c) { return (w >> (28 + c)) & 1; }

// CG direction p_k = z_{k-1} + beta p_{k-1} from the interleaved (z, p) pair
__device__ __forceinline__ double cg_dir(const double* zp, long long j, double beta) {
  const double2 q = __ldcg(reinterpret_cast<const double2*>(zp) + j);
  return __dadd_rn(q.x, __dmul_rn(beta, q.y));
}

// publish the CG "continue" flag to the enclosing WHILE graph node
__device__ __forceinline__ void cg_publish(const CGDev* g) {
  if (g->use_cond) cudaGraphSetConditional((cudaGraphConditionalHandle)g->cond, g->active ? 1u : 0u);
}


// mass-launch prologue of iteration k = it_m: for k >= 2 finish N(k-1)'s r.z
// reduction, stop test (operators.py:361-362) and beta_k = rz_{k-1}/rz_{k-2}.
// Returns false when this launch has nothing to do.
template <int NT, bool PEER = true>
__device__ __forceinline__ bool cg_mass_begin(CGDev* g, double* red, double& beta, int& k,
                                              const PeerLite* pl = nullptr) {
  if (!g->active) return false;
  k = g->it_m;
  if (k == 1) {  // finish k_cg_init's reduction: rz_0, any(b != 0)
    __shared__ double b2[2];
    double t = 0.0, nz = 0.0;
    for (int i = threadIdx.x; i < g->nparts_n; i += NT) {
      t += __ldcg(g->parts_n + 2 * i);
      nz += __ldcg(g->parts_n + 2 * i + 1);
    }
    t = block_sum<NT>(t, red);
    nz = block_sum<NT>(nz, red);
    if (threadIdx.x == 0) {
      b2[0] = t;
      b2[1] = nz;
    }
    __syncthreads();
    t = b2[0];
    nz = b2[1];
    if (PEER && g->peer) {  // world r.z_0 and nnz(b)
      double w[2] = {t, nz};
      if (!peer_world<2>(pl ? *pl : peer_lite(g->peer), g->seq0 + 1, w)) {
        if (threadIdx.x == 0) {  // any block that timed out stops the CG
          g->code = 6;
          g->active = 0;
          cg_publish(g);
        }
        return false;
      }
      t = w[0];
      nz = w[1];
    }
    const bool none = nz == 0.0, maxed = !none && g->max_iter <= 0;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      if (!none) {
        g->norm0 = sqrt(t);
        if (g->hist) g->hist[0] = g->norm0;
      }
      g->nres = none ? 0 : 1;
      if (none || maxed) {
        if (maxed) g->code = 4;
        g->active = 0;
        cg_publish(g);
      } else {
        g->rz = t;
        g->rz2[0] = t;
      }
    }
    beta = 0.0;
    return !(none || maxed);
  }
  double rzk = 0.0;
  const bool posted = PEER && g->peer && pl && (pl->post & PEER_POST_ON);
  if (!posted) rzk = reduce_bcast<NT>(g->parts_n, g->nparts_n, red);
  if (PEER && g->peer) {  // world r.z_{k-1}
    double w[1] = {rzk};
    const bool okw = posted ? peer_recv<1>(*pl, g->seq0 + 2ull * k - 1, w)
                            : peer_world<1>(pl ? *pl : peer_lite(g->peer), g->seq0 + 2ull * k - 1, w);
    if (!okw) {
      if (threadIdx.x == 0) {  // any block that timed out stops the CG (same values from every block)
        g->code = 6;
        g->active = 0;
        cg_publish(g);
      }
      return false;
    }
    rzk = w[0];
  }
  const double res = sqrt(fmax(rzk, 0.0));
  const bool conv = res <= g->tol * g->norm0;
  const bool maxed = !conv && (k - 1 >= g->max_iter);
  const double rzp = g->rz2[(k - 2) & 1];
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (g->hist) g->hist[k - 1] = res;
    g->nres = k;
    if (conv || maxed) {
      g->iters = k - 1;
      if (maxed) g->code = 4;
      g->active = 0;
      cg_publish(g);
    } else {
      g->rz2[(k - 1) & 1] = rzk;
      g->rz = rzk;
      g->beta = rzk / rzp;
      g->it_n = k;
    }
  }
  if (conv || maxed) return false;
  beta = rzk / rzp;
  return true;
}

// node-launch prologue of iteration k = it_n: finish M(k)'s p.Ap reduction,
// breakdown test (operators.py:354-355), alpha_k = rz_{k-1}/pAp.
template <int NT, bool PEER = true>
__device__ __forceinline__ bool cg_node_begin(CGDev* g, double* red, double& alpha, double& alpha_prev, int& k,
                                              const PeerLite* pl = nullptr) {
  if (!g->active) return false;
  k = g->it_n;
  double pAp = 0.0;
  const bool posted = PEER && g->peer && pl && (pl->post & PEER_POST_ON);
  if (!posted) pAp = reduce_bcast<NT>(g->parts_m, g->nparts_m, red);
  if (PEER && g->peer) {  // world p.Ap_k; the flag also publishes this rank's halo (k_halo_pack)
    double w[1] = {pAp};
    const bool okw = posted ? peer_recv<1>(*pl, g->seq0 + 2ull * k, w)
                            : peer_world<1>(pl ? *pl : peer_lite(g->peer), g->seq0 + 2ull * k, w);
    if (!okw) {
      if (threadIdx.x == 0) {  // any block that timed out stops the CG (same values from every block)
        g->code = 6;
        g->active = 0;
        cg_publish(g);
      }
      return false;
    }
    pAp = w[0];
  }
  if (pAp <= 0.0) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      g->code = 3;
      g->active = 0;
      cg_publish(g);
    }
    return false;
  }
  alpha = g->rz2[(k - 1) & 1] / pAp;
  alpha_prev = g->alpha2[(k - 1) & 1];
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    g->alpha2[k & 1] = alpha;
    g->alpha = alpha;
    g->it = k;
    g->it_m = k + 1;
    g->pend = (k & 1) ? k : 0;
  }
  return true;
}

// per-CTA partial of a CG launch (block 0 also records the grid size for the consumer)
__device__ __forceinline__ void cg_partial(double* parts, int* nparts, double v) {
  if (threadIdx.x == 0) {
    parts[blockIdx.x] = v;
    if (blockIdx.x == 0) *nparts = (int)gridDim.x;
  }
}

struct MassArgs {
  const double* x;      // apply: input (NN, NC)
  const double* pold;   // unused
  double* pbuf0;        // cg: interleaved (z, p) pairs, ping-pong: iteration k reads pbuf[(k-1)&1]
  double* pbuf1;
  const uint8_t* mask;  // (NN, NC) or null
  const uint8_t* own;   // (NE, nl)
  const int* emapf;     // cg: packed element map (node | owner | wall mask)
  const double* D;      // (NE, nq)
  const int* emap;
  const int* slot;      // (NE, nl) node-sorted E-vector position
  const double* B;      // (Q, D1)
  long long ne;
  double* evec;         // (NE, nl, NC)
  CGDev* cg;
  double* partials;
};

template <int DIM, int P>
struct MassCfg {
  using D = Disc<DIM, P>;
  static constexpr int WARPS = 4;
  static constexpr int NT = 32 * WARPS;
};

template <int DIM, int P, int NC, bool CG>
__global__ void __launch_bounds__(128) k_mass(MassArgs a) {
  using D = Disc<DIM, P>;
  constexpr int D1 = D::D1, Q = D::Q, NL = D::NL, NQ = D::NQ;
  constexpr int WARPS = 4;
  constexpr int BUF = NC * NQ;
  extern __shared__ double smem[];
  __shared__ double red[32];
  double* sB = smem;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* A = smem + Q * D1 + warp * 2 * BUF;
  double* Bf = A + BUF;
  double cg_beta = 0.0;
  int cg_k = 0;
  if constexpr (CG)
    if (!cg_mass_begin<128>(a.cg, red, cg_beta, cg_k)) return;
  for (int i = threadIdx.x; i < Q * D1; i += blockDim.x) sB[i] = a.B[i];
  __syncthreads();
  const long long e = (long long)blockIdx.x * WARPS + warp;
  double acc = 0.0;
  double beta = 0.0;
  const double* pz = a.x;
  const double* po = nullptr;
  if constexpr (CG) {
    beta = cg_beta;
    po = (cg_k & 1) ? a.pbuf0 : a.pbuf1;  // (z, p)_{k-1} lives in pbuf[(k-1)&1]
  }
  if (e < a.ne) {
    const int* em = a.emap + e * NL;
    for (int i = lane; i < NL * NC; i += 32) {
      const int l = i / NC, c = i - l * NC;
      double val;
      if constexpr (CG) {
        const int w = a.emapf[e * NL + l];
        const long long n = emf_node(w);
        const double p = cg_dir(po, n * NC + c, beta);
        const bool m = emf_mask(w, c);
        if (m && emf_own(w)) acc = fma(p, p, acc);
        val = m ? 0.0 : p;
      } else {
        const long long n = em[l];
        val = pz[n * NC + c];
      }
      A[c * NL + l] = val;
    }
    __syncwarp();
    double* qv = interp<DIM, D1, Q, NC, 32>(sB, A, Bf, lane);
    __syncwarp();
    const double* De = a.D + e * NQ;
    for (int i = lane; i < NQ * NC; i += 32) {
      const int q = i % NQ;
      const double u = qv[i];
      const double du = u * De[q];
      if constexpr (CG) acc = fma(du, u, acc);
      qv[i] = du;
    }
    __syncwarp();
    double* other = (qv == A) ? Bf : A;
    double* r = interp_t<DIM, D1, Q, NC, 32>(sB, qv, other, lane);
    __syncwarp();
    for (int i = lane; i < NL * NC; i += 32) {
      const int l = i / NC, c = i - l * NC;
      a.evec[(long long)a.slot[e * NL + l] * NC + c] = r[c * NL + l];
    }
  }
  if constexpr (CG) {
    cg_partial(a.partials, &a.cg->nparts_m, block_sum<128>(acc, red));
  }
}

// Fixed 1D tables per order p, in the constant bank: the z-direction stages read
// them with warp-uniform addresses, so DFMA takes them as c[][] operands (no
// register or shared-memory traffic).  hx_create uploads them and refuses a
// context whose tables differ (they depend only on p: Lobatto nodes, p+2 Gauss points).
__constant__ double c_B[4][30];

// ---------------------------------------------------------------------------
// Warp-per-element 3D PA mass ("line" mapping).  Each lane owns whole tensor
// lines of a 1D contraction (MI inputs -> MO outputs), so all lanes read the same
// basis entry at the same time: the basis is a constant-bank operand of DFMA
// (c_B, warp-uniform) and every shared-memory load feeds MO FMAs.  Tensors use an
// odd x-pitch so line-strided accesses are bank-conflict free.  Only __syncwarp
// between stages.  CG fusion as in k_mass (direction update, wall mask, p.Ap).

__constant__ double c_G[4][30];
__constant__ double c_Bt[4][30];  // thermodynamic basis (Q x DT) per order, like c_B

template <int P, int TAB>
__device__ __forceinline__ double cmat(int i) {
  if constexpr (TAB == 0) return c_B[P - 1][i];
  else return c_G[P - 1][i];
}

__host__ __device__ constexpr int oddp(int n) { return n | 1; }

// out = M.in along axis AX; M is the (Q x D1) table TAB, applied D1->Q (TR=false)
// or transposed Q->D1 (TR=true).  in: (N0,N1,N2) with x-pitch P0; out x-pitch oddp(O0).
template <int P, int TAB, bool TR, int N0, int N1, int N2, int AX, int NC>
__device__ __forceinline__ void wline(const double* in, double* out, int lane) {
  constexpr int D1 = P + 1;
  constexpr int MI = AX == 0 ? N0 : (AX == 1 ? N1 : N2);
  constexpr int MO = TR ? D1 : P + 2;
  constexpr int O0 = AX == 0 ? MO : N0, O1 = AX == 1 ? MO : N1, O2 = AX == 2 ? MO : N2;
  constexpr int P0 = oddp(N0), Q0 = oddp(O0);
  constexpr int CSI = N2 * N1 * P0, CSO = O2 * O1 * Q0;
  constexpr int NLN = N0 * N1 * N2 / MI;
  constexpr int ROUNDS = (NLN * NC + 31) / 32;
  constexpr int IST = AX == 0 ? 1 : (AX == 1 ? P0 : N1 * P0);
  constexpr int OST = AX == 0 ? 1 : (AX == 1 ? Q0 : O1 * Q0);
#pragma unroll
  for (int r = 0; r < ROUNDS; ++r) {
    const int w = lane + 32 * r;
    if (w < NLN * NC) {
      const int c = w / NLN, l = w - c * NLN;
      int ib, ob;
      if constexpr (AX == 0) {
        ib = l * P0;  // l = i2*N1 + i1
        ob = l * Q0;
      } else if constexpr (AX == 1) {
        const int i0 = l % N0, i2 = l / N0;
        ib = i2 * N1 * P0 + i0;
        ob = i2 * O1 * Q0 + i0;
      } else {
        const int i0 = l % N0, i1 = l / N0;
        ib = i1 * P0 + i0;
        ob = i1 * Q0 + i0;
      }
      const double* src = in + c * CSI + ib;
      double* dst = out + c * CSO + ob;
      double x[MI];
#pragma unroll
      for (int j = 0; j < MI; ++j) x[j] = src[j * IST];
#pragma unroll
      for (int k = 0; k < MO; ++k) {
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < MI; ++j) s = fma(cmat<P, TAB>(TR ? j * D1 + k : k * D1 + j), x[j], s);
        dst[k * OST] = s;
      }
    }
  }
}

template <int P, int NC>
struct Mass3W {
  static constexpr int D1 = P + 1, Q = P + 2;
  static constexpr int BUF = NC * Q * Q * oddp(Q);  // largest stage tensor
  static constexpr int WPB = 4;
  static constexpr size_t bytes = sizeof(double) * WPB * 2 * BUF;
};

template <int P, int NC, bool CG, int MINB>
__global__ void __launch_bounds__(128, MINB) k_mass3w(MassArgs a) {
  constexpr int D1 = P + 1, Q = P + 2, NL = D1 * D1 * D1, NQ = Q * Q * Q, Q2 = Q * Q;
  constexpr int WPB = Mass3W<P, NC>::WPB, BUF = Mass3W<P, NC>::BUF;
  constexpr int PD = oddp(D1), PQ = oddp(Q);
  constexpr int GR = (NL + 31) / 32;          // gather rounds (nodes per lane)
  constexpr int ZR = (Q2 * NC + 31) / 32;     // z-stage rounds (columns per lane)
  extern __shared__ double smem[];
  __shared__ double red[32];
  double cg_beta = 0.0;
  int cg_k = 0;
  if constexpr (CG)
    if (!cg_mass_begin<32 * WPB>(a.cg, red, cg_beta, cg_k)) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* A = smem + warp * 2 * BUF;
  double* Bb = A + BUF;
  double acc = 0.0;
  // persistent: the grid covers the resident capacity, warps stride over elements
  for (long long e = (long long)blockIdx.x * WPB + warp; e < a.ne; e += (long long)gridDim.x * WPB) {
    // gather: lane owns nodes lane, lane+32, ... (all loads issued before use)
    double beta = 0.0;
    const double* po = nullptr;
    if constexpr (CG) {
      beta = cg_beta;
      po = (cg_k & 1) ? a.pbuf0 : a.pbuf1;
    }
    const int* em = (CG ? a.emapf : a.emap) + e * NL;
    int wd[GR];
#pragma unroll
    for (int k = 0; k < GR; ++k) {
      const int l = lane + 32 * k;
      wd[k] = l < NL ? __ldg(em + l) : -1;
    }
    double vv[GR][NC];
#pragma unroll
    for (int k = 0; k < GR; ++k) {
      if (wd[k] >= 0) {
        const long long n = CG ? emf_node(wd[k]) : (long long)wd[k];
#pragma unroll
        for (int c = 0; c < NC; ++c) vv[k][c] = CG ? cg_dir(po, n * NC + c, beta) : __ldcg(a.x + n * NC + c);
      }
    }
#pragma unroll
    for (int k = 0; k < GR; ++k) {
      const int l = lane + 32 * k;
      if (wd[k] >= 0) {
        const int dx = l % D1, dy = (l / D1) % D1, dz = l / (D1 * D1);
        const int si = (dz * D1 + dy) * PD + dx;
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          double val = vv[k][c];
          if constexpr (CG) {
            const bool m = emf_mask(wd[k], c);
            if (m && emf_own(wd[k])) acc = fma(val, val, acc);
            val = m ? 0.0 : val;
          }
          A[c * D1 * D1 * PD + si] = val;
        }
      }
    }
    __syncwarp();
    wline<P, 0, false, D1, D1, D1, 0, NC>(A, Bb, lane);  // (Q, D1, D1)
    __syncwarp();
    // point data of this lane's z columns, in flight during the y stage
    double Dq[ZR][Q];
#pragma unroll
    for (int r = 0; r < ZR; ++r) {
      const int w = lane + 32 * r;
      const int l = (w < Q2 * NC) ? w % Q2 : 0;
#pragma unroll
      for (int qz = 0; qz < Q; ++qz) Dq[r][qz] = __ldg(a.D + e * NQ + qz * Q2 + l);
    }
    wline<P, 0, false, Q, D1, D1, 1, NC>(Bb, A, lane);   // (Q, Q, D1)
    __syncwarp();
    // z stage: B, D, B^T on each (qx, qy) column in registers; in place in A
#pragma unroll
    for (int r = 0; r < ZR; ++r) {
      const int w = lane + 32 * r;
      if (w < Q2 * NC) {
        const int c = w / Q2, l = w - c * Q2;
        const int qx = l % Q, qy = l / Q;
        double* col = A + c * D1 * Q * PQ + qy * PQ + qx;  // (Q,Q,D1) tensor, z stride Q*PQ
        double xin[D1];
#pragma unroll
        for (int dz = 0; dz < D1; ++dz) xin[dz] = col[dz * Q * PQ];
        double u[Q];
#pragma unroll
        for (int qz = 0; qz < Q; ++qz) {
          double s = 0.0;
#pragma unroll
          for (int dz = 0; dz < D1; ++dz) s = fma(cmat<P, 0>(qz * D1 + dz), xin[dz], s);
          const double du = s * Dq[r][qz];
          if constexpr (CG) acc = fma(du, s, acc);
          u[qz] = du;
        }
#pragma unroll
        for (int dz = 0; dz < D1; ++dz) {
          double s = 0.0;
#pragma unroll
          for (int qz = 0; qz < Q; ++qz) s = fma(cmat<P, 0>(qz * D1 + dz), u[qz], s);
          col[dz * Q * PQ] = s;
        }
      }
    }
    __syncwarp();
    wline<P, 0, true, Q, Q, D1, 1, NC>(A, Bb, lane);     // (Q, D1, D1)
    __syncwarp();
    wline<P, 0, true, Q, D1, D1, 0, NC>(Bb, A, lane);    // (D1, D1, D1)
    __syncwarp();
    // node-sorted E-vector: lanes over (node, component), 24 contiguous bytes per node
    const int* sl = a.slot + e * NL;
#pragma unroll
    for (int k = 0; k < GR; ++k) {
      const int l = lane + 32 * k;
      if (l < NL) {
        const int dx = l % D1, dy = (l / D1) % D1, dz = l / (D1 * D1);
        const int si = (dz * D1 + dy) * PD + dx;
        const long long o = (long long)__ldg(sl + l) * NC;
#pragma unroll
        for (int c = 0; c < NC; ++c) a.evec[o + c] = A[c * D1 * D1 * PD + si];
      }
    }
    __syncwarp();
  }
  if constexpr (CG) {
    cg_partial(a.partials, &a.cg->nparts_m, block_sum<32 * WPB>(acc, red));
  }
}

// ---------------------------------------------------------------------------
// 3D PA mass, "plane + column" decomposition.  A thread owns one (component,
// z-plane) of an element and runs the x and y contractions of that plane in
// registers (basis entries are warp-uniform constant-bank operands); threads
// owning (qx, qy) columns then run z, the point scaling D and z^T on all
// components at once (one D column load serves NC components).  Shared memory only
// carries the (Q x Q) plane images between the two phases: 4 * NC * D1 * Q^2
// doubles per element, odd plane stride -> conflict-free.  Persistent CTAs.
template <int P, int NC>
struct MassPC {
  static constexpr int D1 = P + 1, Q = P + 2, QQ = Q * Q;
  static constexpr int PLN = NC * D1;       // planes per element
  static constexpr int EPC = 128 / PLN;     // elements per CTA pass
  static constexpr int TS = NC * D1 * QQ;   // smem doubles per element (plane stride QQ is odd for odd Q...)
  static constexpr size_t bytes = sizeof(double) * EPC * TS;
};

template <int P, int NC, bool CG>
__global__ void __launch_bounds__(128, 4) k_mass_pc(MassArgs a) {
  using M = MassPC<P, NC>;
  constexpr int D1 = P + 1, Q = P + 2, NL = D1 * D1 * D1, NQ = Q * Q * Q, QQ = Q * Q, DD = D1 * D1;
  constexpr int PLN = M::PLN, EPC = M::EPC, TS = M::TS;
  const double* cB = c_B[P - 1];
  extern __shared__ double smem[];
  __shared__ double red[32];
  double cg_beta = 0.0;
  int cg_k = 0;
  if constexpr (CG)
    if (!cg_mass_begin<128>(a.cg, red, cg_beta, cg_k)) return;
  const int t = threadIdx.x;
  double acc = 0.0;
  double beta = 0.0;
  const double* po = nullptr;
  if constexpr (CG) {
    beta = cg_beta;
    po = (cg_k & 1) ? a.pbuf0 : a.pbuf1;
  }
  const int pe = t / PLN, pr = t - pe * PLN;
  const int pc = pr / D1, pz = pr - pc * D1;  // plane: component pc, z index pz
  for (long long e0 = (long long)blockIdx.x * EPC; e0 < a.ne; e0 += (long long)gridDim.x * EPC) {
    const long long e = e0 + pe;
    const bool pact = pe < EPC && e < a.ne;
    double* T = smem + pe * TS + pr * QQ;
    // ---- phase 1 (planes): gather, x and y contractions in registers
    if (pact) {
      double u[DD];
      if constexpr (CG) {
        const int* em = a.emapf + e * NL + pz * DD;
        int wd[DD];
#pragma unroll
        for (int k = 0; k < DD; ++k) wd[k] = __ldg(em + k);
#pragma unroll
        for (int k = 0; k < DD; ++k) u[k] = cg_dir(po, emf_node(wd[k]) * NC + pc, beta);
#pragma unroll
        for (int k = 0; k < DD; ++k) {
          const bool m = emf_mask(wd[k], pc);
          if (m && emf_own(wd[k])) acc = fma(u[k], u[k], acc);
          u[k] = m ? 0.0 : u[k];
        }
      } else {
        const int* em = a.emap + e * NL + pz * DD;
#pragma unroll
        for (int k = 0; k < DD; ++k) u[k] = a.x[(long long)__ldg(em + k) * NC + pc];
      }
      double v[D1][Q];  // after x: v[dy][qx]
#pragma unroll
      for (int dy = 0; dy < D1; ++dy)
#pragma unroll
        for (int qx = 0; qx < Q; ++qx) {
          double s = 0.0;
#pragma unroll
          for (int dx = 0; dx < D1; ++dx) s = fma(cB[qx * D1 + dx], u[dy * D1 + dx], s);
          v[dy][qx] = s;
        }
#pragma unroll
      for (int qy = 0; qy < Q; ++qy)
#pragma unroll
        for (int qx = 0; qx < Q; ++qx) {
          double s = 0.0;
#pragma unroll
          for (int dy = 0; dy < D1; ++dy) s = fma(cB[qy * D1 + dy], v[dy][qx], s);
          T[qy * Q + qx] = s;
        }
    }
    __syncthreads();
    // ---- phase 2 (columns): z, D, z^T for all components of a (qx, qy) column
    for (int it = t; it < EPC * QQ; it += 128) {
      const int ce = it / QQ, l = it - ce * QQ;
      const long long ee = e0 + ce;
      if (ee >= a.ne) continue;
      double Dq[Q];
#pragma unroll
      for (int qz = 0; qz < Q; ++qz) Dq[qz] = __ldg(a.D + ee * NQ + qz * QQ + l);
      double* base = smem + ce * TS + l;
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        double col[D1];
#pragma unroll
        for (int dz = 0; dz < D1; ++dz) col[dz] = base[(c * D1 + dz) * QQ];
        double w[Q];
#pragma unroll
        for (int qz = 0; qz < Q; ++qz) {
          double s = 0.0;
#pragma unroll
          for (int dz = 0; dz < D1; ++dz) s = fma(cB[qz * D1 + dz], col[dz], s);
          const double du = s * Dq[qz];
          if constexpr (CG) acc = fma(du, s, acc);
          w[qz] = du;
        }
#pragma unroll
        for (int dz = 0; dz < D1; ++dz) {
          double s = 0.0;
#pragma unroll
          for (int qz = 0; qz < Q; ++qz) s = fma(cB[qz * D1 + dz], w[qz], s);
          base[(c * D1 + dz) * QQ] = s;
        }
      }
    }
    __syncthreads();
    // ---- phase 3 (planes): y^T, x^T in registers, node-sorted E-vector out
    if (pact) {
      double Tq[QQ];
#pragma unroll
      for (int k = 0; k < QQ; ++k) Tq[k] = T[k];
      double v[D1][Q];  // after y^T: v[dy][qx]
#pragma unroll
      for (int dy = 0; dy < D1; ++dy)
#pragma unroll
        for (int qx = 0; qx < Q; ++qx) {
          double s = 0.0;
#pragma unroll
          for (int qy = 0; qy < Q; ++qy) s = fma(cB[qy * D1 + dy], Tq[qy * Q + qx], s);
          v[dy][qx] = s;
        }
      const int* sl = a.slot + e * NL + pz * DD;
#pragma unroll
      for (int dy = 0; dy < D1; ++dy)
#pragma unroll
        for (int dx = 0; dx < D1; ++dx) {
          double s = 0.0;
#pragma unroll
          for (int qx = 0; qx < Q; ++qx) s = fma(cB[qx * D1 + dx], v[dy][qx], s);
          a.evec[(long long)__ldg(sl + dy * D1 + dx) * NC + pc] = s;
        }
    }
    __syncthreads();
  }
  if constexpr (CG) {
    cg_partial(a.partials, &a.cg->nparts_m, block_sum<128>(acc, red));
  }
}

// ---------------------------------------------------------------------------
// node-side kernels: deterministic G^T through the transpose map

// E is node-sorted: the entries of node n are E[off[n]..off[n+1]) in ascending element
// order.  Up to MAXDEG entries are requested at once (absent ones read as +0.0,
// which never changes a sum that starts from 0.0), then added in order: the result
// is bit-identical to the sequential ascending-element accumulation (fespace.py:227-234).
template <int NC>
__device__ __forceinline__ double node_sum1(const int* off, const double* E, long long n, int c) {
  constexpr int MAXDEG = 8;
  const int b = __ldg(off + n), f = __ldg(off + n + 1);
  double s = 0.0;
  if (f - b <= MAXDEG) {
    double v[MAXDEG];
#pragma unroll
    for (int j = 0; j < MAXDEG; ++j) v[j] = (b + j < f) ? __ldcg(E + (long long)(b + j) * NC + c) : 0.0;
#pragma unroll
    for (int j = 0; j < MAXDEG; ++j) s += v[j];
  } else {
    for (long long k = b; k < f; ++k) s += __ldcg(E + k * NC + c);
  }
  return s;
}

template <int NC>
__device__ __forceinline__ void node_sum(const int* off, const int* idx, const double* E, long long n,
                                         double (&s)[NC]) {
#pragma unroll
  for (int c = 0; c < NC; ++c) s[c] = node_sum1<NC>(off, E, n, c);
  (void)idx;
}

#ifndef NODE_U
#define NODE_U 2
#endif
#ifndef NODE_MINB
#define NODE_MINB 4
#endif
#ifndef NODE_PEER_MINB
#define NODE_PEER_MINB NODE_MINB
#endif
struct NodeArgs {
  const int* off;
  const int* idx;
  const double* evec;   // (NE, nl, NC)
  const uint8_t* mask;
  const double* invd;   // (NN, NC) 1/diag (masked rows -> 1)
  const double* invdn;  // or null; else (NN) 1/diag per node, masked components -> 1 (the
                        // same value for every unmasked component, a third of the bytes)
  double* x;
  double* r;
  double* z;            // unused by the CG (z lives in the (z, p) pairs)
  double* pbuf0;        // interleaved (z, p) pairs, ping-pong
  double* pbuf1;
  const double* rhs;    // cg_init from an explicit rhs (NN, NC) or null
  double* out;          // scatter output
  long long nn;
  CGDev* cg;
  double* partials;     // this launch's per-CTA partials (node launches: r.z)
  double* pm;           // cg_init: where the mass launches put their p.Ap partials
  double* hist;
  int negate;           // cg_init from evec: rhs = -sum
  double tol;           // cg_init: stop tolerance and iteration cap
  int max_iter;
  unsigned long long cond;
  int use_cond;
  const uint8_t* owned;  // multi-GPU: r.z counts a node on its owning rank only (null: every node)
  const PeerDev* peer;   // multi-GPU exchange (device copy) or null
  PeerLite pl;           // its prologue essentials, by value
};

// plain scatter: out = G^T evec (internal layout)
template <int NC>
__global__ void __launch_bounds__(256) k_scatter(NodeArgs a) {
  const long long n = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= a.nn) return;
  double s[NC];
  node_sum<NC>(a.off, a.idx, a.evec, n, s);
#pragma unroll
  for (int c = 0; c < NC; ++c) a.out[n * NC + c] = s[c];
}

// CG start (cg_solve operators.py:340-350): r = b, z = D^{-1} r, x = 0, p_0 = 0, and the
// per-CTA partials of r.z and of the nonzero count of b; M(1) finishes the reduction
// (norm0, the b == 0 and max_iter tests).  b is rhs, or -(G^T evec) masked
// (rhs_v = -F.1, hydro.py:351, 320).  Persistent grid-stride over (node, component),
// two items in flight per thread.
template <int NC, class SUM>
__global__ void __launch_bounds__(256, 4) k_cg_init(NodeArgs a, SUM sum) {
  __shared__ double red[32];
  double rz = 0.0, nz = 0.0;
  const long long N = a.nn * NC;
  const long long stride = (long long)gridDim.x * blockDim.x;
  constexpr int U = 2;
  for (long long j0 = (long long)blockIdx.x * blockDim.x + threadIdx.x; j0 < N; j0 += U * stride) {
    double s[U], d[U];
    bool m[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long j = j0 + u * stride;
      if (j < N) {
        const long long n = j / NC;
        const int c = (int)(j - n * NC);
        s[u] = a.rhs ? a.rhs[j] : sum(n, c);
        m[u] = a.mask && a.mask[j];
        d[u] = a.invdn ? (m[u] ? 1.0 : __ldg(a.invdn + n)) : a.invd[j];
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long j = j0 + u * stride;
      if (j < N) {
        double b = a.negate ? -s[u] : s[u];
        if (m[u]) b = 0.0;
        const double z = d[u] * b;
        a.r[j] = b;
        reinterpret_cast<double2*>(a.pbuf0)[j] = make_double2(z, 0.0);  // (z_0, p_0 = 0)
        a.x[j] = 0.0;
        if (!a.owned || a.owned[j / NC]) rz = fma(b, z, rz);
        if (b != 0.0 || b != b) nz += 1.0;
      }
    }
  }
  const double brz = block_sum<256>(rz, red);
  const double bnz = block_sum<256>(nz, red);
  if (threadIdx.x == 0) {
    a.partials[2 * blockIdx.x] = brz;
    a.partials[2 * blockIdx.x + 1] = bnz;
    if (blockIdx.x == 0) {
      CGDev* g = a.cg;
      g->code = 0;
      g->beta = 0.0;
      g->alpha = 0.0;
      g->alpha2[0] = g->alpha2[1] = 0.0;
      g->pend = 0;
      g->it_m = 1;
      g->it_n = 1;
      g->nparts_n = (int)gridDim.x;  // M(1) reads the (r.z, nonzero) pairs from here
      g->parts_m = a.pm;
      g->parts_n = a.partials;
      g->hist = a.hist;
      g->it = 1;
      g->iters = 0;
      g->nres = 0;
      g->tol = a.tol;
      g->max_iter = a.max_iter;
      g->cond = a.cond;
      g->use_cond = a.use_cond;
      g->peer = a.peer;
      g->seq0 = a.peer ? *a.peer->seq : 0ull;
      g->cnt[2] = g->cnt[3] = 0u;  // producer-post arrival counters
      g->active = 1;
    }
  }
}

// CG iteration tail (operators.py:352-365): p_k = z + beta p_{k-1} (written),
// Ap = G^T evec (identity on masked rows), x += alpha p, r -= alpha Ap, z = D^{-1} r,
// rz_new = r.z; stop test sqrt(max(rz_new,0)) <= tol*norm0; beta = rz_new/rz.
template <int NC, class SUM>
__global__ void __launch_bounds__(256, NODE_MINB) k_cg_node(NodeArgs a, SUM sum) {
  __shared__ double red[32];
  CGDev* g = a.cg;
  double alpha, alpha_prev;
  int k;
  if (!cg_node_begin<256, false>(g, red, alpha, alpha_prev, k)) return;
  const double beta = g->beta;
  const double* po = (k & 1) ? a.pbuf0 : a.pbuf1;
  double* pn = (k & 1) ? a.pbuf1 : a.pbuf0;
  // x is stored every second iteration: at even k, x_k = (x_{k-2} + a_{k-1} p_{k-1}) +
  // a_k p_k evaluated in registers -- the reference's two roundings, one store
  // (p_{k-1} is the old pair's second half).  k_cg_finish applies a pending odd step.
  const bool xk = (k & 1) == 0;
  double rz = 0.0;
  // grid-stride over (node, component), U items per thread per trip so that all
  // their loads are in flight together
  constexpr int U = NODE_U;
  const long long N = a.nn * NC;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long j0 = (long long)blockIdx.x * blockDim.x + threadIdx.x; j0 < N; j0 += U * stride) {
    double2 zp[U];
    double xj[U], rj[U], dj[U], s[U];
    bool m[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long j = j0 + u * stride;
      if (j < N) {
        const long long n = j / NC;
        const int c = (int)(j - n * NC);
        zp[u] = __ldcg(reinterpret_cast<const double2*>(po) + j);
        if (xk) xj[u] = __ldcg(a.x + j);
        rj[u] = __ldcg(a.r + j);
        m[u] = a.mask && a.mask[j];
        dj[u] = a.invdn ? (m[u] ? 1.0 : __ldg(a.invdn + n)) : __ldg(a.invd + j);
        s[u] = sum(n, c);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long j = j0 + u * stride;
      if (j < N) {
        const double p = __dadd_rn(zp[u].x, __dmul_rn(beta, zp[u].y));
        const double ap = m[u] ? p : s[u];
        if (xk) a.x[j] = __dadd_rn(__dadd_rn(xj[u], __dmul_rn(alpha_prev, zp[u].y)), __dmul_rn(alpha, p));
        const double r = __dsub_rn(rj[u], __dmul_rn(alpha, ap));
        a.r[j] = r;
        const double z = __dmul_rn(dj[u], r);
        reinterpret_cast<double2*>(pn)[j] = make_double2(z, p);
        rz = fma(r, z, rz);
      }
    }
  }
  cg_partial(a.partials, &g->nparts_n, block_sum<256>(rz, red));
}

// multi-GPU variant: the first trip's own-data loads are issued before the prologue's
// world p.Ap handshake; interface nodes add the neighbours' partials afterwards
// (PEER = false: the same prologue overlap on one GPU, NODE_PF)
template <int NC, class SUM, bool PEER = true>
__global__ void __launch_bounds__(256, PEER ? NODE_PEER_MINB : NODE_MINB) k_cg_node_peer(NodeArgs a, SUM sum) {
  __shared__ double red[32];
  CGDev* g = a.cg;
  if (!g->active) return;
  const int k = g->it_n;  // the iteration cg_node_begin finishes
  const double* po = (k & 1) ? a.pbuf0 : a.pbuf1;
  double* pn = (k & 1) ? a.pbuf1 : a.pbuf0;
  // x is stored every second iteration: at even k, x_k = (x_{k-2} + a_{k-1} p_{k-1}) +
  // a_k p_k evaluated in registers -- the reference's two roundings, one store
  // (p_{k-1} is the old pair's second half).  k_cg_finish applies a pending odd step.
  const bool xk = (k & 1) == 0;
  const PeerDev* pd = PEER ? g->peer : nullptr;
  const int* ifx = PEER ? pd->ifx : nullptr;
  // grid-stride over (node, component), U items per thread per trip so that all
  // their loads are in flight together
  constexpr int U = NODE_U;
  const long long N = a.nn * NC;
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long jfirst = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  double2 zp[U];
  double xj[U], rj[U], dj[U], s[U];
  bool m[U];
  int hh[U];
  auto load = [&](long long j0) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long j = j0 + u * stride;
      if (j < N) {
        const long long n = j / NC;
        const int c = (int)(j - n * NC);
        zp[u] = __ldcg(reinterpret_cast<const double2*>(po) + j);
        if (xk) xj[u] = __ldcg(a.x + j);
        rj[u] = __ldcg(a.r + j);
        m[u] = a.mask && a.mask[j];
        dj[u] = a.invdn ? (m[u] ? 1.0 : __ldg(a.invdn + n)) : __ldg(a.invd + j);
        s[u] = sum(n, c);  // own (local elements) part
        hh[u] = PEER ? __ldg(ifx + n) : -1;
      }
    }
  };
  // the first trip's loads are in flight while the prologue finishes the p.Ap reduction
  // (and, multi-GPU, waits for the world value and the neighbours' halo)
  load(jfirst);
  double alpha, alpha_prev;
  int kk;
  if (!cg_node_begin<256, PEER>(g, red, alpha, alpha_prev, kk, &a.pl)) return;
  const double beta = g->beta;
  double rz = 0.0;
  for (long long j0 = jfirst; j0 < N; j0 += U * stride) {
    if (j0 != jfirst) load(j0);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long j = j0 + u * stride;
      if (j < N) {
        if constexpr (PEER) {
          if (hh[u] >= 0) s[u] = peer_node_sum<NC>(pd, s[u], hh[u], (int)(j % NC));
        }
        const double p = __dadd_rn(zp[u].x, __dmul_rn(beta, zp[u].y));
        const double ap = m[u] ? p : s[u];
        if (xk) a.x[j] = __dadd_rn(__dadd_rn(xj[u], __dmul_rn(alpha_prev, zp[u].y)), __dmul_rn(alpha, p));
        const double r = __dsub_rn(rj[u], __dmul_rn(alpha, ap));
        a.r[j] = r;
        const double z = __dmul_rn(dj[u], r);
        reinterpret_cast<double2*>(pn)[j] = make_double2(z, p);
        // r.z counts a node on its owning rank only (multi-GPU: only interface nodes can
        // be owned elsewhere)
        if (!PEER || hh[u] < 0 || a.owned[j / NC]) rz = fma(r, z, rz);
      }
    }
  }
  cg_partial(a.partials, &g->nparts_n, block_sum<256>(rz, red));
  if constexpr (PEER) {  // post this rank's r.z_k (consumed by M(k+1)'s prologue)
    if (a.pl.post & PEER_POST_ON) cg_post_last<256>(a.pl, a.partials, gridDim.x, &g->cnt[2], g->seq0 + 2ull * kk + 1, red);
  }
}

// CG epilogue: apply the x update of a final odd iteration (x_k = x_{k-1} + a_k p_k;
// p_k is the second half of the last pairs written, alpha still a_k)
__global__ void __launch_bounds__(256) k_cg_finish(const CGDev* g, const double* pbuf0, const double* pbuf1,
                                                   double* x, long long n) {
  const int k = g->pend;
  if (!k) return;
  const double* pk = (k & 1) ? pbuf1 : pbuf0;  // pairs written by iteration k
  const double alpha = g->alpha2[k & 1];
  for (long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (long long)gridDim.x * blockDim.x)
    x[j] = __dadd_rn(x[j], __dmul_rn(alpha, __ldcg(pk + 2 * j + 1)));
}

// ---------------------------------------------------------------------------
// state updates (rk2_step hydro.py:385-399)

struct AxpyArgs {
  const double* x;
  const double* v;
  const double* e;
  const double* dxs;   // velocity used as dx (state.v for stage 1, mid.v for stage 2)
  const double* dv;
  const double* de;
  double* xo;
  double* vo;
  double* eo;
  const double* dtp;   // device attempt dt
  double scale;        // 0.5 (midpoint) or 1.0
  long long nv;        // NN*d
  long long nte;       // NE*nt
  double* xf;          // midpoint launch only, or null: the step's final x = x + dt v_half (the
                       // reference's S + dt r1 position, hydro.py:392-396), computed as soon as
                       // v_half exists so the rest of the step can overlap its use
};

// y = a + h*b on pairs of entries (16-byte accesses when every array is 16-byte aligned)
__device__ __forceinline__ void axpy2(const double* a, const double* b, double* y, double h, long long i, long long n,
                                      bool vec) {
  if (vec && i + 1 < n) {
    const double2 p = *reinterpret_cast<const double2*>(a + i);
    const double2 q = *reinterpret_cast<const double2*>(b + i);
    *reinterpret_cast<double2*>(y + i) = make_double2(__dadd_rn(p.x, __dmul_rn(h, q.x)),
                                                      __dadd_rn(p.y, __dmul_rn(h, q.y)));
  } else {
    for (long long j = i; j < n && j < i + 2; ++j) y[j] = __dadd_rn(a[j], __dmul_rn(h, b[j]));
  }
}

__global__ void __launch_bounds__(256) k_axpy_state(AxpyArgs a) {
  const double h = a.scale == 1.0 ? *a.dtp : (*a.dtp / 2.0);
  const long long i = 2 * ((long long)blockIdx.x * blockDim.x + threadIdx.x);
  const bool vec = ((reinterpret_cast<unsigned long long>(a.x) | reinterpret_cast<unsigned long long>(a.v) |
                     reinterpret_cast<unsigned long long>(a.e) | reinterpret_cast<unsigned long long>(a.dxs) |
                     reinterpret_cast<unsigned long long>(a.dv) | reinterpret_cast<unsigned long long>(a.de) |
                     reinterpret_cast<unsigned long long>(a.xo) | reinterpret_cast<unsigned long long>(a.vo) |
                     reinterpret_cast<unsigned long long>(a.eo)) & 15ull) == 0;
  if (i < a.nv) {
    if (a.xo) axpy2(a.x, a.dxs, a.xo, h, i, a.nv, vec);
    if (a.vo) axpy2(a.v, a.dv, a.vo, h, i, a.nv, vec);
    if (a.xf) {  // x + dt * v_half from the just-rounded v_half
      const double dt = *a.dtp;
      for (long long j = i; j < a.nv && j < i + 2; ++j) a.xf[j] = __dadd_rn(a.x[j], __dmul_rn(dt, a.vo[j]));
    }
  }
  if (i < a.nte && a.eo) axpy2(a.e, a.de, a.eo, h, i, a.nte, vec);
}

// dt = min(cfl*ratio, dt_max, t_final - t) / 2^retry  (timestep_estimate hydro.py:364-373)
struct DtArgs {
  const StatusDev* st;
  double* dt;        // [0] = estimate, [1] = attempt
  double cfl, dt_max, t_final, t;
  double dt_fixed;   // >= 0: rk2_step(state, dt) with a caller-given dt
  int retry;
  const double* tptr;  // graph mode: {state time, caller-given dt} on the device, or null (use t, dt_fixed)
};
__global__ void k_dt(DtArgs a) {
  double dt;
  if (a.dt_fixed >= 0.0) {
    dt = a.tptr ? a.tptr[1] : a.dt_fixed;
  } else {
    const double t = a.tptr ? *a.tptr : a.t;
    dt = a.cfl * a.st->min_ratio;
    dt = fmin(dt, a.dt_max);
    dt = fmin(dt, a.t_final - t);
  }
  a.dt[0] = dt;
  double att = dt;
  for (int i = 0; i < a.retry; ++i) att /= 2.0;
  a.dt[1] = att;
}

// pack node id | owner << 27 | wall mask(c) << (28 + c) for the CG kernels
__global__ void k_build_emapf(const int* emap, const uint8_t* own, const uint8_t* mask, int nc, long long n_entries,
                              int* out) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_entries) return;
  const int node = emap[t];
  int w = node | (own[t] ? (1 << 27) : 0);
  if (mask)
    for (int c = 0; c < nc; ++c)
      if (mask[(long long)node * nc + c]) w |= 1 << (28 + c);
  out[t] = w;
}

__global__ void k_status_reset(StatusDev* st, int n) {
  const int i = threadIdx.x;
  if (i < n) {
    st[i].inv_key = ~0ull;
    st[i].clamps = 0;
    st[i].min_ratio = __longlong_as_double(0x7ff0000000000000ll);
    st[i].pad = 0;
  }
}

// ---------------------------------------------------------------------------
// API-level kernels (reference layouts in, reference layouts out)

// gather to the reference E-vector layout (nl, NE, ncomp)
__global__ void k_gather_ref(const double* L, const int* emap, int nl, long long ne, int nc, double* E) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long tot = (long long)nl * ne * nc;
  if (t >= tot) return;
  const int c = (int)(t % nc);
  const long long le = t / nc;  // l*NE + e
  const long long e = le % ne, l = le / ne;
  E[t] = L[(long long)emap[e * nl + l] * nc + c];
}

// scatter from the reference E-vector layout, ascending element per node (bit-exact np.add.at)
__global__ void k_scatter_ref(const double* E, const int* off, const int* idx, int nl, long long ne,
                              long long nn, int nc, double* L) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nn * nc) return;
  const long long n = t / nc;
  const int c = (int)(t % nc);
  double s = 0.0;
  for (int k = off[n]; k < off[n + 1]; ++k) {
    const long long j = idx[k];
    const long long e = j / nl, l = j % nl;
    s += E[(l * ne + e) * nc + c];
  }
  L[t] = s;
}

// L2 space: E (nt, NE, nc) <-> L (NE*nt, nc) is a transpose
__global__ void k_l2_gather(const double* L, int nt, long long ne, int nc, double* E, int transpose_back) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)nt * ne * nc) return;
  const int c = (int)(t % nc);
  const long long le = t / nc;
  const long long e = le % ne, l = le / ne;
  if (!transpose_back) E[t] = L[(e * nt + l) * nc + c];
  else E[(e * nt + l) * nc + c] = L[t];
}

// (nq, NE) <-> (NE, nq) transposes and general point-data transposes
__global__ void k_transpose(const double* in, long long rows, long long cols, double* out) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= rows * cols) return;
  const long long r = t / cols, c = t % cols;
  out[c * rows + r] = in[t];
}

// geometry in reference layouts (compute_geometric_factors, fespace.py:326-346)
struct GeomArgs {
  const double* x;
  const int* emap;
  Tables tab;
  long long ne;
  double* jac;
  double* detj;
  double* jinv;
  double* wdetj;
  double* Dm_int;       // optional (NE, nq): (wdetj/detj)*qdata0 (hydro.py:223-224)
  double* Dm_ref;       // optional (nq, NE)
  const double* qdata0; // (nq, NE) ref layout
  StatusDev* st;
};

template <int DIM, int P>
struct GeomSmem {
  using D = Disc<DIM, P>;
  static constexpr int A = cmax(DIM * D::NL, DIM == 3 ? 3 * DIM * D::Q * D::Q * D::D1 : 0);
  static constexpr int S = 2 * DIM * D::Q * ipow(D::D1, DIM - 1);
  static constexpr int OUT = DIM * (DIM + 1) * D::NQ;
  static constexpr int TOTAL = 2 * D::Q * D::D1 + D::Q * D::DT + A + S + OUT;
  static constexpr size_t bytes = sizeof(double) * TOTAL;
};

template <int DIM, int P, int NT>
__global__ void __launch_bounds__(NT) k_geom(GeomArgs a) {
  using D = Disc<DIM, P>;
  using SM = GeomSmem<DIM, P>;
  constexpr int D1 = D::D1, Q = D::Q, DT = D::DT, NL = D::NL, NQ = D::NQ;
  extern __shared__ double smem[];
  double* sB = smem;
  double* sG = sB + Q * D1;
  double* sBt = sG + Q * D1;
  double* rA = sBt + Q * DT;
  double* rS = rA + SM::A;
  double* rOut = rS + SM::S;
  const int tid = threadIdx.x;
  const long long e = blockIdx.x;
  const long long ne = a.ne;
  load_tables<Q, D1, DT>(a.tab, sB, sG, sBt);
  const int* em = a.emap + e * NL;
  for (int i = tid; i < NL * DIM; i += NT) {
    const int l = i / DIM, c = i - l * DIM;
    rA[c * NL + l] = a.x[(long long)em[l] * DIM + c];
  }
  __syncthreads();
  grad<DIM, D1, Q, DIM, DIM + 1, NT>(sB, sG, rA, rS, rA, rOut, tid);
  __syncthreads();
  unsigned long long key = ~0ull;
  for (int q = tid; q < NQ; q += NT) {
    double J[DIM][DIM], inv[DIM][DIM];
#pragma unroll
    for (int c = 0; c < DIM; ++c)
#pragma unroll
      for (int b = 0; b < DIM; ++b) J[c][b] = rOut[(c * (DIM + 1) + b) * NQ + q];
    const double det = det_inv<DIM>(J, inv);
    if (det <= 0.0) {
      const unsigned long long k = (unsigned long long)q * ne + e;
      key = k < key ? k : key;
    }
    const long long pe = (long long)q * ne + e;
    const double wd = a.tab.wnd[q] * det;
#pragma unroll
    for (int r = 0; r < DIM; ++r)
#pragma unroll
      for (int c = 0; c < DIM; ++c) {
        if (a.jac) a.jac[(long long)(r * DIM + c) * NQ * ne + pe] = J[r][c];
        if (a.jinv) a.jinv[(long long)(r * DIM + c) * NQ * ne + pe] = inv[r][c];
      }
    if (a.detj) a.detj[pe] = det;
    if (a.wdetj) a.wdetj[pe] = wd;
    if (a.Dm_int || a.Dm_ref) {
      const double dm = (wd / det) * a.qdata0[pe];
      if (a.Dm_int) a.Dm_int[e * NQ + q] = dm;
      if (a.Dm_ref) a.Dm_ref[pe] = dm;
    }
  }
  if (key != ~0ull && a.st) atomicMin(&a.st->inv_key, key);
}

// stress_qdata in reference layout (hydro.py:254-315), geometry recomputed from x
struct StressArgs {
  const double* x;
  const double* v;
  const double* e;
  const double* qdata0;  // (nq, NE)
  const int* emap;
  Tables tab;
  double gamma, q1, q2;
  const double* gam;   // per-element adiabatic index (multi-material extension) or null
  long long ne;
  double* sigma;         // (d,d,nq,NE) or null
  StatusDev* st;
};

template <int DIM, int P, int NT>
__global__ void __launch_bounds__(NT) k_stress(StressArgs a) {
  using D = Disc<DIM, P>;
  using SM = RatesSmem<DIM, P>;
  constexpr int D1 = D::D1, Q = D::Q, DT = D::DT, NL = D::NL, NQ = D::NQ, NTH = D::NT;
  constexpr int NCG = SM::NCG;
  extern __shared__ double smem[];
  double* sB = smem;
  double* sG = sB + Q * D1;
  double* sBt = sG + Q * D1;
  double* rA = sBt + Q * DT;
  double* rS = rA + SM::A;
  double* rOut = rS + SM::S;
  double* rTH = rOut + SM::OUT;
  double* red = rTH + SM::TH + NTH;
  const int tid = threadIdx.x;
  const long long e = blockIdx.x, ne = a.ne;
  load_tables<Q, D1, DT>(a.tab, sB, sG, sBt);
  const int* em = a.emap + e * NL;
  for (int i = tid; i < NL * DIM; i += NT) {
    const int l = i / DIM, c = i - l * DIM;
    const long long n = em[l];
    rA[c * NL + l] = a.x[n * DIM + c];
    rA[(DIM + c) * NL + l] = a.v[n * DIM + c];
  }
  for (int i = tid; i < NTH; i += NT) rTH[i] = a.e[e * NTH + i];
  __syncthreads();
  grad<DIM, D1, Q, NCG, DIM + 1, NT>(sB, sG, rA, rS, rA, rOut, tid);
  double* eq = interp<DIM, DT, Q, 1, NT>(sBt, rTH, rTH + NQ, tid);
  __syncthreads();
  double rmin = __longlong_as_double(0x7ff0000000000000ll);
  long long clamps = 0;
  unsigned long long key = ~0ull;
  for (int q = tid; q < NQ; q += NT) {
    double J[DIM][DIM], dv[DIM][DIM], vq[DIM];
#pragma unroll
    for (int c = 0; c < DIM; ++c) {
#pragma unroll
      for (int b = 0; b < DIM; ++b) {
        J[c][b] = rOut[(c * (DIM + 1) + b) * NQ + q];
        dv[c][b] = rOut[((DIM + c) * (DIM + 1) + b) * NQ + q];
      }
      vq[c] = rOut[((DIM + c) * (DIM + 1) + DIM) * NQ + q];
    }
    const long long pe = (long long)q * ne + e;
    PointOut<DIM> po;
    point_physics<DIM>(J, dv, vq, eq[q], a.qdata0[pe], a.gam ? __ldg(a.gam + e) : a.gamma, a.q1, a.q2, po);
    if (po.det <= 0.0) {
      const unsigned long long k = (unsigned long long)q * ne + e;
      key = k < key ? k : key;
    }
    clamps += po.clamped;
    rmin = fmin(rmin, po.ratio);
    if (a.sigma)
#pragma unroll
      for (int r = 0; r < DIM; ++r)
#pragma unroll
        for (int c = 0; c < DIM; ++c) a.sigma[(long long)(r * DIM + c) * NQ * ne + pe] = po.sigma[r][c];
  }
  publish_status<NT>(a.st, rmin, clamps, key, red);
}

// D_F from reference-layout sigma, jinv, wdetj -> internal (NE, d*d, nq)
template <int DIM>
__global__ void k_force_D(const double* sigma, const double* jinv, const double* wdetj, long long ne,
                          int nq, double* DFint, double* DFref) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= ne * nq) return;
  const long long q = t / ne, e = t % ne;  // t = q*NE + e
  const long long P = (long long)nq * ne;
  double sg[DIM][DIM], ji[DIM][DIM], DF[DIM][DIM];
#pragma unroll
  for (int r = 0; r < DIM; ++r)
#pragma unroll
    for (int c = 0; c < DIM; ++c) {
      sg[r][c] = sigma[(r * DIM + c) * P + t];
      ji[r][c] = jinv[(r * DIM + c) * P + t];
    }
  force_point<DIM>(sg, ji, wdetj[t], DF);
#pragma unroll
  for (int r = 0; r < DIM; ++r)
#pragma unroll
    for (int c = 0; c < DIM; ++c) {
      DFint[(e * DIM * DIM + r * DIM + c) * nq + q] = DF[r][c];
      if (DFref) DFref[(r * DIM + c) * P + t] = DF[r][c];
    }
}

// ForcePA.apply (operators.py:264-280) / apply_transpose (:282-300), one CTA per element
struct ForceArgs {
  const double* in;     // apply: e (NE*nt); apply_t: v (NN, d)
  const double* DF;     // (NE, d*d, nq)
  const int* emap;
  const int* slot;
  Tables tab;
  long long ne;
  double* evec;         // apply: (NE, nl, d)
  double* out;          // apply_t: (NE*nt)
};

template <int DIM, int P>
struct ForceSmem {
  using D = Disc<DIM, P>;
  static constexpr int A = cmax(DIM * D::NL, DIM == 3 ? 3 * DIM * D::Q * D::Q * D::D1 : 0);
  static constexpr int S = 2 * DIM * D::Q * ipow(D::D1, DIM - 1);
  static constexpr int OUT = DIM * (DIM + 1) * D::NQ;
  static constexpr int TH = 2 * D::NQ;
  static constexpr int TOTAL = 2 * D::Q * D::D1 + D::Q * D::DT + A + S + OUT + TH + DIM * D::NL;
  static constexpr size_t bytes = sizeof(double) * TOTAL;
};

template <int DIM, int P, int NT, bool TRANS>
__global__ void __launch_bounds__(NT) k_force(ForceArgs a) {
  using D = Disc<DIM, P>;
  using SM = ForceSmem<DIM, P>;
  constexpr int D1 = D::D1, Q = D::Q, DT = D::DT, NL = D::NL, NQ = D::NQ, NTH = D::NT;
  extern __shared__ double smem[];
  double* sB = smem;
  double* sG = sB + Q * D1;
  double* sBt = sG + Q * D1;
  double* rA = sBt + Q * DT;
  double* rS = rA + SM::A;
  double* rOut = rS + SM::S;
  double* rTH = rOut + SM::OUT;
  double* rF = rTH + SM::TH;
  const int tid = threadIdx.x;
  const long long e = blockIdx.x;
  load_tables<Q, D1, DT>(a.tab, sB, sG, sBt);
  const double* DFe = a.DF + e * DIM * DIM * NQ;
  if constexpr (!TRANS) {
    for (int i = tid; i < NTH; i += NT) rTH[i] = a.in[e * NTH + i];
    __syncthreads();
    double* eq = interp<DIM, DT, Q, 1, NT>(sBt, rTH, rTH + NQ, tid);
    __syncthreads();
    for (int i = tid; i < DIM * DIM * NQ; i += NT) {
      const int q = i % NQ, al = i / NQ, c = al / DIM, l = al % DIM;
      rOut[(c * (DIM + 1) + l) * NQ + q] = DFe[i] * eq[q];
    }
    __syncthreads();
    grad_t<DIM, D1, Q, DIM, (DIM + 1) * NQ, NT>(sB, sG, rOut, rA, rS, rF, tid);
    __syncthreads();
    for (int i = tid; i < NL * DIM; i += NT) {
      const int l = i / DIM, c = i - l * DIM;
      a.evec[(long long)a.slot[e * NL + l] * DIM + c] = rF[c * NL + l];
    }
  } else {
    const int* em = a.emap + e * NL;
    for (int i = tid; i < NL * DIM; i += NT) {
      const int l = i / DIM, c = i - l * DIM;
      rA[c * NL + l] = a.in[(long long)em[l] * DIM + c];
    }
    __syncthreads();
    grad<DIM, D1, Q, DIM, DIM + 1, NT>(sB, sG, rA, rS, rA, rOut, tid);
    __syncthreads();
    for (int q = tid; q < NQ; q += NT) {
      double s = 0.0;
#pragma unroll
      for (int c = 0; c < DIM; ++c)
#pragma unroll
        for (int l = 0; l < DIM; ++l) s += DFe[(c * DIM + l) * NQ + q] * rOut[(c * (DIM + 1) + l) * NQ + q];
      rTH[q] = s;
    }
    __syncthreads();
    double* fv = interp_t<DIM, DT, Q, 1, NT>(sBt, rTH, rTH + NQ, tid);
    __syncthreads();
    for (int i = tid; i < NTH; i += NT) a.out[e * NTH + i] = fv[i];
  }
}

// MassPA.diagonal (operators.py:117-124): contract D with (B*B)^T on every axis
template <int DIM, int P>
__global__ void __launch_bounds__(128) k_mass_diag(const double* D, const double* B, const int* slot, long long ne,
                                                   double* evec) {
  using Dd = Disc<DIM, P>;
  constexpr int D1 = Dd::D1, Q = Dd::Q, NL = Dd::NL, NQ = Dd::NQ;
  __shared__ double sB2[Q * D1];
  __shared__ double buf[4][2][NQ];
  for (int i = threadIdx.x; i < Q * D1; i += blockDim.x) sB2[i] = B[i] * B[i];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long e = (long long)blockIdx.x * 4 + warp;
  if (e >= ne) return;
  double* A = buf[warp][0];
  double* Bf = buf[warp][1];
  for (int i = lane; i < NQ; i += 32) A[i] = D[e * NQ + i];
  __syncwarp();
  double* r = interp_t<DIM, D1, Q, 1, 32>(sB2, A, Bf, lane);
  __syncwarp();
  for (int i = lane; i < NL; i += 32) evec[slot[e * NL + i]] = r[i];
}

// per-element thermodynamic mass blocks M_e = Bth^T diag(D) Bth and their inverse
// (hydro.py:229-232): Gauss-Jordan with partial pivoting, one CTA per element.
// Thermodynamic mass inverses, one warp per element (3D, nt <= 32): M_e = B_t^T diag(D) B_t
// (hydro.py:229-231) assembled by sum factorisation (x, y, z pairs of basis rows), then
// inverted in place by Gauss-Jordan with lane j holding column j in registers (M_e is SPD:
// no pivoting; the reference's LAPACK getri differs at rounding level only).
template <int P>
__global__ void __launch_bounds__(256) k_minv_warp(const double* Dm /*(NE,nq)*/, long long ne, double* minv,
                                                   double* minv_ref) {
  constexpr int Q = P + 2, DT = P, N = DT * DT * DT, NQ = Q * Q * Q, D2 = DT * DT;
  static_assert(N <= 32, "one column per lane");
  constexpr int WPB = 8;
  constexpr int AX = D2 * Q * Q;        // A_x[(ix,jx)][qy][qz]
  constexpr int AXY = D2 * D2 * Q;      // A_xy[(ix,jx)][(iy,jy)][qz]
  constexpr int PER = NQ + AX + AXY;
  extern __shared__ double smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* sD = smem + warp * PER;
  double* sAx = sD + NQ;
  double* sAxy = sAx + AX;
  const double* bt = c_Bt[P - 1];  // (Q, DT)
  for (long long e = (long long)blockIdx.x * WPB + warp; e < ne; e += (long long)gridDim.x * WPB) {
    for (int q = lane; q < NQ; q += 32) sD[q] = __ldg(Dm + e * NQ + q);
    __syncwarp();
    // x: A_x[ix,jx][qy,qz] = sum_qx Bt[qx][ix] Bt[qx][jx] D[qz][qy][qx]
    for (int o = lane; o < AX; o += 32) {
      const int ij = o / (Q * Q), r = o - ij * (Q * Q);  // r = qz*Q + qy
      const int ix = ij / DT, jx = ij - ix * DT;
      double s = 0.0;
#pragma unroll
      for (int qx = 0; qx < Q; ++qx) s = fma(bt[qx * DT + ix] * bt[qx * DT + jx], sD[r * Q + qx], s);
      sAx[o] = s;
    }
    __syncwarp();
    // y: A_xy[ij_x][iy,jy][qz] = sum_qy Bt[qy][iy] Bt[qy][jy] A_x[ij_x][qz][qy]
    for (int o = lane; o < AXY; o += 32) {
      const int ijx = o / (D2 * Q), r = o - ijx * (D2 * Q);
      const int ijy = r / Q, qz = r - ijy * Q;
      const int iy = ijy / DT, jy = ijy - iy * DT;
      double s = 0.0;
#pragma unroll
      for (int qy = 0; qy < Q; ++qy)
        s = fma(bt[qy * DT + iy] * bt[qy * DT + jy], sAx[ijx * Q * Q + qz * Q + qy], s);
      sAxy[o] = s;
    }
    __syncwarp();
    // z: column j = (jx, jy, jz) of M_e in registers of lane j (row i = (ix, iy, iz), x fastest)
    double col[N];
    const int j = lane < N ? lane : 0;
    const int jx = j % DT, jy = (j / DT) % DT, jz = j / D2;
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const int ix = i % DT, iy = (i / DT) % DT, iz = i / D2;
      const double* a = sAxy + ((ix * DT + jx) * D2 + (iy * DT + jy)) * Q;
      double s = 0.0;
#pragma unroll
      for (int qz = 0; qz < Q; ++qz) s = fma(bt[qz * DT + iz] * bt[qz * DT + jz], a[qz], s);
      col[i] = s;
    }
    __syncwarp();
    // in-place Gauss-Jordan: after step k, column k holds -A[i][k]/p (i != k) and 1/p
#pragma unroll
    for (int kk = 0; kk < N; ++kk) {
      const double p = __shfl_sync(0xffffffffu, col[kk], kk);
      const double rp = 1.0 / p;
      const double akj = col[kk] * rp;
      const bool own = lane == kk;
#pragma unroll
      for (int i = 0; i < N; ++i) {
        const double aik = __shfl_sync(0xffffffffu, col[i], kk);
        if (i == kk) continue;
        col[i] = own ? -aik * rp : fma(-aik, akj, col[i]);
      }
      col[kk] = own ? rp : akj;
    }
    if (lane < N) {
#pragma unroll
      for (int i = 0; i < N; ++i) {
        if (lane <= i) minv[e * tri(N) + tri(i) + lane] = col[i];  // packed lower triangle
        if (minv_ref) minv_ref[(e * N + i) * N + lane] = col[i];
      }
    }
    __syncwarp();
  }
}

template <int DIM, int P>
__global__ void __launch_bounds__(128) k_minv(const double* Dm /*(NE,nq)*/, const double* Bt, long long ne,
                                             double* minv, double* minv_ref) {
  using Dd = Disc<DIM, P>;
  constexpr int Q = Dd::Q, DT = Dd::DT, NQ = Dd::NQ, N = Dd::NT;
  extern __shared__ double smem[];
  double* M = smem;              // N x 2N augmented
  double* Bf = M + N * 2 * N;    // full thermo basis (NQ x N)
  __shared__ int piv;
  const long long e = blockIdx.x;
  for (int i = threadIdx.x; i < NQ * N; i += blockDim.x) {
    const int q = i / N, j = i % N;
    // x-fastest point and node indices: q = (qz*Q + qy)*Q + qx
    double b = 1.0;
    int qq = q, jj = j;
    for (int d = 0; d < DIM; ++d) {
      b *= Bt[(qq % Q) * DT + (jj % DT)];
      qq /= Q;
      jj /= DT;
    }
    Bf[i] = b;
  }
  __syncthreads();
  const double* De = Dm + e * NQ;
  for (int i = threadIdx.x; i < N * N; i += blockDim.x) {
    const int r = i / N, c = i % N;
    double s = 0.0;
    for (int q = 0; q < NQ; ++q) s += Bf[q * N + r] * De[q] * Bf[q * N + c];
    M[r * 2 * N + c] = s;
    M[r * 2 * N + N + c] = (r == c) ? 1.0 : 0.0;
  }
  __syncthreads();
  for (int col = 0; col < N; ++col) {
    if (threadIdx.x == 0) {
      int best = col;
      double bv = fabs(M[col * 2 * N + col]);
      for (int r = col + 1; r < N; ++r) {
        const double v = fabs(M[r * 2 * N + col]);
        if (v > bv) {
          bv = v;
          best = r;
        }
      }
      piv = best;
    }
    __syncthreads();
    const int pr = piv;
    if (pr != col)
      for (int c = threadIdx.x; c < 2 * N; c += blockDim.x) {
        const double t = M[col * 2 * N + c];
        M[col * 2 * N + c] = M[pr * 2 * N + c];
        M[pr * 2 * N + c] = t;
      }
    __syncthreads();
    const double d = M[col * 2 * N + col];
    __syncthreads();
    for (int c = threadIdx.x; c < 2 * N; c += blockDim.x) M[col * 2 * N + c] /= d;
    __syncthreads();
    for (int i = threadIdx.x; i < N * 2 * N; i += blockDim.x) {
      const int r = i / (2 * N), c = i % (2 * N);
      if (r != col) {
        const double f = M[r * 2 * N + col];
        if (c != col) M[i] -= f * M[col * 2 * N + c];
      }
    }
    __syncthreads();
    for (int r = threadIdx.x; r < N; r += blockDim.x)
      if (r != col) M[r * 2 * N + col] = 0.0;
    __syncthreads();
  }
  for (int i = threadIdx.x; i < N * N; i += blockDim.x) {
    const int r = i / N, c = i % N;
    const double v = M[r * 2 * N + N + c];
    minv[e * N * N + i] = v;
    if (minv_ref) minv_ref[e * N * N + i] = v;
  }
}

// solve_energy: out[e,i] = sum_j minv[e,i,j] rhs[e,j]
// (packed: the symmetric lower-triangle storage of minv_packed)
__global__ void k_energy_solve(const double* minv, const double* rhs, int nt, long long ne, double* out, int packed) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= ne * nt) return;
  const long long e = t / nt;
  const int i = (int)(t % nt);
  const double* r = rhs + e * nt;
  double s = 0.0;
  if (packed) {
    const double* m = minv + e * tri(nt);
    for (int j = 0; j < nt; ++j) s = fma(m[j <= i ? tri(i) + j : tri(j) + i], r[j], s);
  } else {
    const double* m = minv + (e * nt + i) * nt;
    for (int j = 0; j < nt; ++j) s = fma(m[j], r[j], s);
  }
  out[t] = s;
}

// internal energy sum_q w_q qdata0 e_q (hydro.py:413-420) per element -> partials
template <int DIM, int P>
__global__ void __launch_bounds__(128) k_internal_energy(const double* e_field, const double* qd0 /*(NE,nq)*/,
                                                        const double* Bt, const double* wnd, long long ne,
                                                        double* per_elem) {
  using Dd = Disc<DIM, P>;
  constexpr int Q = Dd::Q, DT = Dd::DT, NQ = Dd::NQ, NT = Dd::NT;
  __shared__ double sBt[Q * DT];
  __shared__ double buf[4][2][NQ];
  for (int i = threadIdx.x; i < Q * DT; i += blockDim.x) sBt[i] = Bt[i];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long e = (long long)blockIdx.x * 4 + warp;
  if (e >= ne) return;
  double* A = buf[warp][0];
  for (int i = lane; i < NT; i += 32) A[i] = e_field[e * NT + i];
  __syncwarp();
  double* eq = interp<DIM, DT, Q, 1, 32>(sBt, A, buf[warp][1], lane);
  __syncwarp();
  double s = 0.0;
  for (int q = lane; q < NQ; q += 32) s += wnd[q] * qd0[e * NQ + q] * eq[q];
  s = warp_sum(s);
  if (lane == 0) per_elem[e] = s;
}

// fixed-order sum of n values into out[0] (one block)
__global__ void __launch_bounds__(256) k_sum(const double* v, long long n, double* out) {
  __shared__ double red[32];
  double acc = 0.0;
  for (long long i = threadIdx.x; i < n; i += 256) acc += v[i];
  const double s = block_sum<256>(acc, red);
  if (threadIdx.x == 0) *out = s;
}

// dot of two vectors, fixed order per thread then block tree
__global__ void __launch_bounds__(256) k_dot(const double* a, const double* b, long long n, double* out) {
  __shared__ double red[32];
  double acc = 0.0;
  for (long long i = threadIdx.x; i < n; i += 256) acc = fma(a[i], b[i], acc);
  const double s = block_sum<256>(acc, red);
  if (threadIdx.x == 0) *out = s;
}

}  // namespace hx
