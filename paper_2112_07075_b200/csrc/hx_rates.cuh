// hx_rates.cuh -- fused rates kernel (3D), the B200 mapping of LagrangeHydro.rates
// minus the momentum solve (hydro.py:346-360): geometry (fespace.py:305-346),
// stress_qdata (hydro.py:254-315), ForcePA F.1 and F^T v (operators.py:247-300) and
// M_e^{-1} (hydro.py:339-344).  D_F never leaves shared memory.
//
// A CTA of RATES_PC_NT (128) threads runs EPC elements per pass (one at p = 3, two at p = 2).  Every sum-factorisation stage is
// its own phase with one thread per 1D line, so no thread carries more than one
// line of one stage (short dependency chains, modest registers, all lanes busy):
//   A   prefetch one pass ahead: x, v node rows (6 fields) by cp.async -> G image;
//       e, qd0 and the packed M_e^{-1} (contiguous per pass) by bulk copies (TMA engine,
//       cp.async.bulk on an mbarrier)
//   B1  x stage, thread per (field, z, y) row: B_x u, G_x u          -> X image
//       (+ thermo rows B_x e -> the T image's thermo area)
//   B2  y stage, thread per (field, z, qx) line: B_y B_x, G_y B_x, B_y G_x -> T image
//   C1  z stage + point physics, thread per quadrature point: J, grad v, v, e at q
//       (e's y and z stages inline from the thermo rows),
//       EOS, tensor viscosity, CFL ratio, D_F; F.1 and F^T v integrands -> W image
//   C2  transposed z stage, thread per (comp, qx, qy) column           -> Z image
//   D1  transposed y stage, thread per (comp, z, qx) line              -> Y image
//   D2  transposed x stage, thread per (comp, z, y) row                -> staging
//   E   F.1 E-vector out (element-major or node-sorted) and de = M_e^{-1} F^T v
// MODE 1 (validity of the new geometry, hydro.py:400-401) runs A-C1 on x only.
// MODE 2 (timestep_estimate's CFL ratio, hydro.py:364-367) runs A-C1 with the point
// physics (ratio, clamp count, first inverted point) and writes nothing else.
// Shared images alias once dead: W over G+X, Z over T, Y over X, staging over G.
#pragma once

#include "hx_async.cuh"
#include "hx_brick.cuh"

namespace hx {

#ifndef RATES_PC_NT
#define RATES_PC_NT 128  // one element per CTA at p = 3 (measured: 123 vs 137 us with 2 per 256-thread CTA)
#endif
#ifndef RATES_PC_MINB
#define RATES_PC_MINB (512 / RATES_PC_NT)
#endif
template <int P>
struct RatesPC {
  static constexpr int D1 = P + 1, Q = P + 2, DT = P, DD = D1 * D1, QQ = Q * Q, NL = D1 * DD, NQ = Q * QQ;
  static constexpr int NT = DT * DT * DT, DTT = DT * DT;
  // p = 4 (216 points) keeps 256 threads: one point per thread in the z / physics stage
  // (128 threads measured 255 vs 189 us there)
  static constexpr int THREADS = P >= 4 ? 256 : RATES_PC_NT;
  static constexpr int EPC = THREADS / NQ > 0 ? THREADS / NQ : 1;
  static constexpr int XPL = 6 * D1;                   // field planes
  // G image: the node rows of x and of v as they lie in memory (D1 nodes x 3 comps per
  // row, 3 D1 contiguous doubles), rows padded to RP so that the x-stage threads (one per
  // (comp, z, y) row) read distinct bank pairs
  static constexpr int RP = 3 * D1 + 1, GRP = DD * RP;  // row pitch, field-group pitch
  static constexpr int GS = 2 * GRP;                    // G image (x rows, v rows)
  // X / Y images: row (plane, y) pitch XP, plane pitch XPP = Q (mod 16): the y-stage lines
  // (plane, qx) of consecutive planes fall on consecutive bank pairs
  static constexpr int XP = 2 * Q + 2;
  static constexpr int XPP = D1 * XP + ((Q - D1 * XP) % 16 + 16) % 16;
  static constexpr int XFS = XPL * XPP;                 // X image, field rows
  static constexpr int XS = XFS;                       // (thermo rows live in the T image)
  // plane pitch of the T and Z images: >= 3 QQ and = Q (mod 16) so that the lines of
  // consecutive planes (Q doubles each) fall on consecutive bank pairs
  static constexpr int PP = 3 * QQ + ((Q - 3 * QQ) % 16 + 16) % 16;
  static constexpr int TFS = XPL * PP;                 // T image, field planes
  static constexpr int TS = TFS + DTT * Q;             // + thermo x-stage rows (dz, dy, qx)
  static constexpr int WS = 10 * NQ;                   // W image (aliases G+X)
  static constexpr int ZS = 3 * D1 * PP + DT * QQ;     // Z image (aliases T)
  static constexpr int MN = minv_packed<3, P>() ? tri(NT) : NT * NT;  // M_e^{-1} doubles per element
  static constexpr int YFS = 3 * D1 * XPP;             // Y image (aliases X)
  static constexpr int YS = YFS + DTT * Q;
  // staging: per component DD rows of D1 nodes, row pitch OR (conflict-free x^T stage
  // stores), then the thermo F^T v block
  static constexpr int OR = D1 + 1, OPL = DD * OR;
  static constexpr int OS = 3 * OPL + NT;              // staging (aliases T)
  // prefetch buffer (double-buffered, filled one pass ahead):
  // [G images EPC x GS | e EPC x NT | qd0 EPC x NQ | M_e^{-1} EPC x MN], regions 16-byte aligned
  static constexpr int ev(int n) { return (n + 1) & ~1; }
  static constexpr int FE = ev(EPC * GS), FQ = FE + ev(EPC * NT), FM = FQ + ev(EPC * NQ), FS = FM + ev(EPC * MN);
  static constexpr int XR = (XS > WS ? (XS > YS ? XS : YS) : (WS > YS ? WS : YS));  // X / W / Y region
  static_assert(ZS <= TS && OS <= TS, "image aliasing");
  static constexpr int PER = XR + TS;                  // working images per element
  static constexpr size_t bytes = sizeof(double) * (2 * (size_t)FS + (size_t)EPC * PER + 2 * NQ) + 16;
};

struct RatesPCArgs {
  const double* x;     // (NN, 3)
  const double* v;     // (NN, 3)
  const double* e;     // (NE*nt)
  const double* qd0;   // (NE, nq)
  const int* emap;     // (NE, nl) (generic meshes)
  const int* slot;     // null: element-major E out; else node-sorted position
  const double* minv;  // (NE, nt, nt), or packed lower triangles (minv_packed)
  const double* wnd;   // (nq)
  const double* psi1;  // (nq)
  double gamma, q1, q2;
  const double* gam;   // per-element adiabatic index (multi-material extension) or null
  long long ne;
  double* evec;        // (NE, nl, 3) F.1 element vectors
  double* de;          // (NE*nt)
  StatusDev* st;
  Brick b;
  int brick;
  // hx_step_host streamed inputs (brick, MODE 0): inflag[0..in_ns) = epoch of each z-slab of
  // x, v, e that has landed, inflag[in_ns] = the epoch this launch needs (stream-ordered);
  // null when the inputs are resident
  const unsigned long long* inflag;
  unsigned long long* inerr;  // mapped host word: set on a wait that timed out (hx_step_host fails)
  int in_ns;  // slabs; inflag[in_ns + 1 + s] = end (exclusive) element layer of slab s
};

// streamed inputs: wait (thread 0, then the CTA) until the slab holding elements up to
// `last` has landed.  Every 128-byte line of x, v, e lies in one slab (host-side rounding),
// so no line read here can be cached from before its slab's copy.
__device__ __forceinline__ void rates_wait_inputs(const RatesPCArgs& a, long long last) {
  if (threadIdx.x == 0) {
    const int ez = (int)a.b.fnxy.div((unsigned)last);
    int s = 0;
    while (s < a.in_ns - 1 && (unsigned long long)ez >= __ldg(a.inflag + a.in_ns + 1 + s)) ++s;
    const unsigned long long need = *(volatile const unsigned long long*)(a.inflag + a.in_ns);
    unsigned long long spins = 0;
    while (ld_acquire_sys(a.inflag + s) < need)
      if (++spins > (1ull << 24)) {  // >= 1 s: the copy stream is stuck; report, do not hang
        st_release_sys(a.inerr, 1ull);
        break;
      } else {
        __nanosleep(64);
      }
  }
  __syncthreads();
}

// reference "inverse" (cof/det = J^{-T} in 3D, fespace.py:280-302,338) with one reciprocal
__device__ __forceinline__ double det_inv_fast(const double (&J)[3][3], double (&inv)[3][3]) {
  const double det = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) -
                     J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
                     J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
  const double rd = 1.0 / det;
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const int r0 = r == 0 ? 1 : 0, r1 = r == 2 ? 1 : 2;
      const int c0 = c == 0 ? 1 : 0, c1 = c == 2 ? 1 : 2;
      const double m = J[r0][c0] * J[r1][c1] - J[r0][c1] * J[r1][c0];
      inv[r][c] = (((r + c) & 1) ? -m : m) * rd;
    }
  return det;
}

// stress_qdata at one point (hydro.py:271-315) + D_F (operators.py:258): the
// arithmetic of point_physics with one reciprocal of det J and h = cbrt(det J)
// (the reference's detj ** (1/3) to within an ulp).
__device__ __forceinline__ void point_physics_fast(const double (&J)[3][3], const double (&dv)[3][3],
                                                   const double (&vq)[3], double eq, double qd0, double gamma,
                                                   double q1, double q2, PointOut<3>& o) {
  o.det = det_inv_fast(J, o.jinv);
  const double det = o.det;
  const double rho = qd0 / det;
  o.clamped = 0;
  if (eq < 0.0) {
    o.clamped = 1;
    eq = 0.0;
  }
  const double p = (gamma - 1.0) * rho * eq;
  const double cs = sqrt(gamma * (gamma - 1.0) * eq);
  double gv[3][3];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      double s = 0.0;
#pragma unroll
      for (int l = 0; l < 3; ++l) s = fma(dv[a][l], o.jinv[l][b], s);
      gv[a][b] = s;
    }
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) o.sigma[a][b] = (a == b) ? -p : 0.0;
  const double div = gv[0][0] + gv[1][1] + gv[2][2];
  const double h = cbrt(det);
  if (q1 > 0.0 || q2 > 0.0) {
    double mu = rho * h * (q1 * cs + q2 * h * fabs(div));
    mu = div < 0.0 ? mu : 0.0;
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) o.sigma[a][b] += mu * (0.5 * (gv[a][b] + gv[b][a]));
  }
  const double v2 = vq[0] * vq[0] + vq[1] * vq[1] + vq[2] * vq[2];
  const double speed = cs + sqrt(v2);
  o.ratio = speed > 0.0 ? h / fmax(speed, 1e-300) : __longlong_as_double(0x7ff0000000000000ll);
}

template <int P, int MODE>
__global__ void __launch_bounds__(RatesPC<P>::THREADS, P >= 4 ? 2 : RATES_PC_MINB) k_rates_pc(RatesPCArgs a) {
  using R = RatesPC<P>;
  constexpr int D1 = R::D1, Q = R::Q, DT = R::DT, DD = R::DD, QQ = R::QQ, NL = R::NL, NQ = R::NQ;
  constexpr int NTH = R::NT, DTT = R::DTT, EPC = R::EPC, RP = R::RP, GRP = R::GRP;
  constexpr int PER = R::PER, XP = R::XP, XPP = R::XPP, TFS = R::TFS, YFS = R::YFS, PP = R::PP;
  constexpr int OR = R::OR, OPL = R::OPL;
  constexpr int FS = R::FS, XR = R::XR;
  constexpr int NT = R::THREADS;
  constexpr int NF = MODE == 1 ? 3 : 6;  // fields gathered / contracted
  const double* cB = c_B[P - 1];
  const double* cG = c_G[P - 1];
  const double* cBt = c_Bt[P - 1];
  extern __shared__ __align__(16) double smem[];
  double* work = smem + 2 * FS;  // per element: X/W/Y region, T/Z/O region
  double* sw = work + EPC * PER;       // tensor weights
  double* sp = sw + NQ;                // psi1
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(sp + NQ);  // one per prefetch buffer
  constexpr int MN = R::MN;
  constexpr bool PK = minv_packed<3, P>();
  const int t = threadIdx.x;
  for (int i = t; i < NQ; i += NT) {
    sw[i] = a.wnd[i];
    sp[i] = a.psi1[i];
  }
  if constexpr (MODE != 1) {
    if (t == 0) {
      mbar_init(bar, 1);
      mbar_init(bar + 1, 1);
      mbar_fence_init();
    }
    __syncthreads();
  }
  unsigned ph0 = 0, ph1 = 0;  // mbarrier phase parity per buffer
  double rmin = __longlong_as_double(0x7ff0000000000000ll);
  long long clamps = 0;
  unsigned long long key = ~0ull;
  // A (prefetch): cp.async x, v node rows, bulk copies of e, qd0 and M_e^{-1} of the pass
  // at f0 into prefetch buffer b (G image: node rows as in memory, padded to RP)
  auto prefetch = [&](int b, long long f0) {
    if (f0 < a.ne) {
      const int fel = (int)((a.ne - f0) < EPC ? (a.ne - f0) : EPC);
      double* fb = smem + b * FS;
      if (MODE == 0 && a.inflag) rates_wait_inputs(a, f0 + fel - 1);
      constexpr int ROW = 3 * D1;  // doubles per node row (D1 nodes x 3 comps, contiguous)
      long long nb[EPC];  // brick: the pass's element base nodes, once per pass (not per item)
      if (a.brick) {
#pragma unroll
        for (int el = 0; el < EPC; ++el) {
          const unsigned ue = (unsigned)(f0 + el);
          const unsigned ez = a.b.fnxy.div(ue);
          const unsigned r2 = ue - ez * (unsigned)(a.b.nx * a.b.ny);
          const unsigned ey = a.b.fnx.div(r2), ex = r2 - ey * (unsigned)a.b.nx;
          nb[el] = (long long)(ex * P) + (long long)(ey * P) * a.b.Nx + (long long)(ez * P) * a.b.NxNy;
        }
      }
      for (int it = t; it < fel * DD * ROW; it += NT) {
        const int el = it / (DD * ROW), rem = it - el * (DD * ROW);
        const int row = rem / ROW, sidx = rem - row * ROW;  // row = dz*D1 + dy
        const int dz = row / D1, dy = row - dz * D1, dx = sidx / 3, c = sidx - dx * 3;
        const long long e = f0 + el;
        long long n;
        if (a.brick) {
          long long b0 = nb[0];
#pragma unroll
          for (int u = 1; u < EPC; ++u)
            if (el == u) b0 = nb[u];
          n = b0 + dx + (long long)dy * a.b.Nx + (long long)dz * a.b.NxNy;
        } else {
          n = __ldg(a.emap + e * NL + row * D1 + dx);
        }
        double* g = fb + el * R::GS + row * RP + sidx;
        cp_async8(g, a.x + n * 3 + c);
        if constexpr (MODE != 1) cp_async8(g + GRP, a.v + n * 3 + c);
      }
      if constexpr (MODE != 1) {
        // e, qd0, M_e^{-1} of the pass are contiguous: bulk copies on buffer b's mbarrier
        const double* se = a.e + f0 * NTH;
        const double* sq = a.qd0 + f0 * NQ;
        const double* sm = a.minv + f0 * MN;
        if (t == 0) {
          fence_proxy_async_smem();  // the generic reads of this buffer's last use are done
          mbar_expect_tx(bar + b, span_bulk_bytes(se, fel * NTH) + span_bulk_bytes(sq, fel * NQ) +
                                      (MODE == 0 ? span_bulk_bytes(sm, fel * MN) : 0u));
        }
        span_bulk<NT>(fb + R::FE, se, fel * NTH, t, bar + b);
        span_bulk<NT>(fb + R::FQ, sq, fel * NQ, t, bar + b);
        if constexpr (MODE == 0) span_bulk<NT>(fb + R::FM, sm, fel * MN, t, bar + b);
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  const long long stride = (long long)gridDim.x * EPC;
  prefetch(0, (long long)blockIdx.x * EPC);
  int buf = 0;

  for (long long e0 = (long long)blockIdx.x * EPC; e0 < a.ne; e0 += stride, buf ^= 1) {
    const int nel = (int)((a.ne - e0) < EPC ? (a.ne - e0) : EPC);
    const double* gcur = smem + buf * FS;
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    if constexpr (MODE != 1) {
      mbar_wait(bar + buf, buf ? ph1 : ph0);  // this pass's bulk copies landed
      if (buf) ph1 ^= 1; else ph0 ^= 1;
    }
    __syncthreads();  // this pass's prefetch landed; previous pass done with every image
    prefetch(buf ^ 1, e0 + stride);  // overlaps this pass's compute
    // ---- B1: x stage, thread per row
    {
      constexpr int FR = NF * D1 * D1;                 // field rows
      constexpr int TASKS = FR + (MODE != 1 ? DTT : 0);
#pragma unroll
      for (int rep = 0; rep < (EPC * TASKS + NT - 1) / NT; ++rep) {
        const int it = t + rep * NT;
        if (it >= nel * TASKS) break;
        const int el = it / TASKS, k = it - el * TASKS;
        const double* g = gcur + el * R::GS;
        double* X = work + el * PER;
        if (k < FR) {
          const int pl = k / D1, dy = k - pl * D1;  // pl = f*D1 + dz
          const int f = pl / D1, dz = pl - f * D1;
          const int grp = f >= 3, c = f - 3 * grp;
          double u[D1];
#pragma unroll
          for (int dx = 0; dx < D1; ++dx) u[dx] = g[grp * GRP + (dz * D1 + dy) * RP + dx * 3 + c];
          double* o = X + pl * XPP + dy * XP;
#pragma unroll
          for (int qx = 0; qx < Q; ++qx) {
            double sb = 0.0, sg = 0.0;
#pragma unroll
            for (int dx = 0; dx < D1; ++dx) {
              sb = fma(cB[qx * D1 + dx], u[dx], sb);
              sg = fma(cG[qx * D1 + dx], u[dx], sg);
            }
            o[qx] = sb;
            o[Q + qx] = sg;
          }
        } else {
          const int r = k - FR;  // dz_t * DT + dy_t
          double u[DT];
#pragma unroll
          for (int dx = 0; dx < DT; ++dx) u[dx] = gcur[R::FE + el * NTH + r * DT + dx];
          double* Th = work + el * PER + XR + TFS;  // thermo x-rows (the T image's thermo area)
#pragma unroll
          for (int qx = 0; qx < Q; ++qx) {
            double s = 0.0;
#pragma unroll
            for (int dx = 0; dx < DT; ++dx) s = fma(cBt[qx * DT + dx], u[dx], s);
            Th[r * Q + qx] = s;
          }
        }
      }
    }
    __syncthreads();
    // ---- B2: y stage, thread per (plane, qx) line
    {
      constexpr int FL = NF * D1 * Q;
      constexpr int TASKS = FL;  // (e's y stage runs inline in C1)
#pragma unroll
      for (int rep = 0; rep < (EPC * TASKS + NT - 1) / NT; ++rep) {
        const int it = t + rep * NT;
        if (it >= nel * TASKS) break;
        const int el = it / TASKS, k = it - el * TASKS;
        const double* X = work + el * PER;
        double* T = work + el * PER + XR;
        {
          const int pl = k / Q, qx = k - pl * Q;
          double vb[D1], vg[D1];
#pragma unroll
          for (int dy = 0; dy < D1; ++dy) {
            vb[dy] = X[pl * XPP + dy * XP + qx];
            vg[dy] = X[pl * XPP + dy * XP + Q + qx];
          }
          double* o = T + pl * PP + qx;
#pragma unroll
          for (int qy = 0; qy < Q; ++qy) {
            double bb = 0.0, gb = 0.0, bg = 0.0;
#pragma unroll
            for (int dy = 0; dy < D1; ++dy) {
              bb = fma(cB[qy * D1 + dy], vb[dy], bb);
              gb = fma(cG[qy * D1 + dy], vb[dy], gb);
              bg = fma(cB[qy * D1 + dy], vg[dy], bg);
            }
            o[qy * Q] = bb;
            o[QQ + qy * Q] = gb;
            o[2 * QQ + qy * Q] = bg;
          }
        }
      }
    }
    __syncthreads();
    // ---- C1: z stage + point physics, thread per point
#pragma unroll
    for (int rep = 0; rep < (EPC * NQ + NT - 1) / NT; ++rep) {
      const int it = t + rep * NT;
      if (it >= nel * NQ) break;
      // lanes run qz fastest: the Q points of a column share their T reads (broadcast)
      const int el = it / NQ, kq = it - el * NQ;
      const int col = kq / Q, qz = kq - col * Q;
      const int q = qz * QQ + col;
      const long long e = e0 + el;
      const double* T = work + el * PER + XR;
      double bz[D1], gz[D1];
#pragma unroll
      for (int dz = 0; dz < D1; ++dz) {
        bz[dz] = cB[qz * D1 + dz];
        gz[dz] = cG[qz * D1 + dz];
      }
      double J[3][3], dv[3][3], vq[3];
#pragma unroll
      for (int f = 0; f < NF; ++f) {
        double d0 = 0.0, d1 = 0.0, d2 = 0.0, iv = 0.0;
#pragma unroll
        for (int dz = 0; dz < D1; ++dz) {
          const double* tt = T + (f * D1 + dz) * PP + col;
          const double bb = tt[0], gb = tt[QQ], bg = tt[2 * QQ];
          d0 = fma(bz[dz], bg, d0);  // d/dxi_x: B_z B_y G_x
          d1 = fma(bz[dz], gb, d1);  // d/dxi_y: B_z G_y B_x
          d2 = fma(gz[dz], bb, d2);  // d/dxi_z: G_z B_y B_x
          if (f >= 3) iv = fma(bz[dz], bb, iv);
        }
        if (f < 3) {
          J[f][0] = d0;
          J[f][1] = d1;
          J[f][2] = d2;
        } else {
          dv[f - 3][0] = d0;
          dv[f - 3][1] = d1;
          dv[f - 3][2] = d2;
          vq[f - 3] = iv;
        }
      }
      if constexpr (MODE == 1) {
        double inv[3][3];
        const double det = det_inv_fast(J, inv);
        if (det <= 0.0) {
          const unsigned long long kk = (unsigned long long)q * a.ne + e;
          key = kk < key ? kk : key;
        }
      } else {
        // e at q: y stage (ascending dy from 0.0) then z stage, from the thermo x-rows
        const int qy = col / Q, qx = col - qy * Q;
        double eq = 0.0;
#pragma unroll
        for (int dz = 0; dz < DT; ++dz) {
          double sy = 0.0;
#pragma unroll
          for (int dy = 0; dy < DT; ++dy) sy = fma(cBt[qy * DT + dy], T[TFS + (dz * DT + dy) * Q + qx], sy);
          eq = fma(cBt[qz * DT + dz], sy, eq);
        }
        PointOut<3> po;
        point_physics_fast(J, dv, vq, eq, gcur[R::FQ + el * NQ + q], a.gam ? __ldg(a.gam + e) : a.gamma, a.q1,
                           a.q2, po);
        if (po.det <= 0.0) {
          const unsigned long long kk = (unsigned long long)q * a.ne + e;
          key = kk < key ? kk : key;
        }
        clamps += po.clamped;
        rmin = fmin(rmin, po.ratio);
        if constexpr (MODE == 0) {
        double DF[3][3];
        force_point<3>(po.sigma, po.jinv, sw[q] * po.det, DF);
        const double p1 = sp[q];
        double* W = work + el * PER;  // aliases X (dead)
        double s = 0.0;
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
          for (int l = 0; l < 3; ++l) {
            s += DF[c][l] * dv[c][l];
            W[(c * 3 + l) * NQ + kq] = DF[c][l] * p1;  // (col, qz) order: conflict-free stores
          }
        W[9 * NQ + kq] = s;
        }
      }
    }
    if constexpr (MODE != 0) continue;
    __syncthreads();
    // ---- C2: transposed z stage, thread per (comp, column) (+ F^T v per column)
    {
      constexpr int TASKS = 4 * QQ;
#pragma unroll
      for (int rep = 0; rep < (EPC * TASKS + NT - 1) / NT; ++rep) {
        const int it = t + rep * NT;
        if (it >= nel * TASKS) break;
        const int el = it / TASKS, k = it - el * TASKS;
        const int c = k / QQ, col = k - c * QQ;
        const double* W = work + el * PER;
        double* Z = work + el * PER + XR;  // aliases T (dead)
        if (c < 3) {
          double z0[D1], z1[D1], z2[D1];
#pragma unroll
          for (int dz = 0; dz < D1; ++dz) {
            z0[dz] = 0.0;
            z1[dz] = 0.0;
            z2[dz] = 0.0;
          }
#pragma unroll
          for (int qz = 0; qz < Q; ++qz) {
            const double s0 = W[(c * 3 + 0) * NQ + col * Q + qz];
            const double s1 = W[(c * 3 + 1) * NQ + col * Q + qz];
            const double s2 = W[(c * 3 + 2) * NQ + col * Q + qz];
#pragma unroll
            for (int dz = 0; dz < D1; ++dz) {
              z0[dz] = fma(cB[qz * D1 + dz], s0, z0[dz]);
              z1[dz] = fma(cB[qz * D1 + dz], s1, z1[dz]);
              z2[dz] = fma(cG[qz * D1 + dz], s2, z2[dz]);
            }
          }
#pragma unroll
          for (int dz = 0; dz < D1; ++dz) {
            Z[(c * D1 + dz) * PP + col] = z0[dz];
            Z[(c * D1 + dz) * PP + QQ + col] = z1[dz];
            Z[(c * D1 + dz) * PP + 2 * QQ + col] = z2[dz];
          }
        } else {
          double zt[DT];
#pragma unroll
          for (int dz = 0; dz < DT; ++dz) zt[dz] = 0.0;
#pragma unroll
          for (int qz = 0; qz < Q; ++qz) {
            const double s = W[9 * NQ + col * Q + qz];
#pragma unroll
            for (int dz = 0; dz < DT; ++dz) zt[dz] = fma(cBt[qz * DT + dz], s, zt[dz]);
          }
#pragma unroll
          for (int dz = 0; dz < DT; ++dz) Z[3 * D1 * PP + dz * QQ + col] = zt[dz];
        }
      }
    }
    __syncthreads();
    // ---- D1: transposed y stage, thread per (comp, z, qx) (+ thermo (z, qx))
    {
      constexpr int FL = 3 * D1 * Q;
      constexpr int TASKS = FL + DT * Q;
#pragma unroll
      for (int rep = 0; rep < (EPC * TASKS + NT - 1) / NT; ++rep) {
        const int it = t + rep * NT;
        if (it >= nel * TASKS) break;
        const int el = it / TASKS, k = it - el * TASKS;
        const double* Z = work + el * PER + XR;
        double* Y = work + el * PER;  // aliases W (dead)
        if (k < FL) {
          const int pl = k / Q, qx = k - pl * Q;  // pl = c*D1 + dz
          const double* z0 = Z + pl * PP + qx;
          const double* z1 = Z + pl * PP + QQ + qx;
          const double* z2 = Z + pl * PP + 2 * QQ + qx;
          double yg[D1], yb[D1];
#pragma unroll
          for (int dy = 0; dy < D1; ++dy) {
            yg[dy] = 0.0;
            yb[dy] = 0.0;
          }
#pragma unroll
          for (int qy = 0; qy < Q; ++qy) {
            const double r0 = z0[qy * Q], r1 = z1[qy * Q], r2 = z2[qy * Q];
#pragma unroll
            for (int dy = 0; dy < D1; ++dy) {
              yg[dy] = fma(cB[qy * D1 + dy], r0, yg[dy]);
              yb[dy] = fma(cG[qy * D1 + dy], r1, yb[dy]);
              yb[dy] = fma(cB[qy * D1 + dy], r2, yb[dy]);
            }
          }
#pragma unroll
          for (int dy = 0; dy < D1; ++dy) {
            Y[pl * XPP + dy * XP + qx] = yg[dy];
            Y[pl * XPP + dy * XP + Q + qx] = yb[dy];
          }
        } else {
          const int r = k - FL, dz = r / Q, qx = r - dz * Q;
          const double* z = Z + 3 * D1 * PP + dz * QQ + qx;
          double y[DT];
#pragma unroll
          for (int dy = 0; dy < DT; ++dy) y[dy] = 0.0;
#pragma unroll
          for (int qy = 0; qy < Q; ++qy) {
            const double zz = z[qy * Q];
#pragma unroll
            for (int dy = 0; dy < DT; ++dy) y[dy] = fma(cBt[qy * DT + dy], zz, y[dy]);
          }
#pragma unroll
          for (int dy = 0; dy < DT; ++dy) Y[YFS + (dz * DT + dy) * Q + qx] = y[dy];
        }
      }
    }
    __syncthreads();
    // ---- D2: transposed x stage, thread per (comp, z, y) row (+ thermo rows) -> staging
    {
      constexpr int FR = 3 * D1 * D1;
      constexpr int TASKS = FR + DTT;
#pragma unroll
      for (int rep = 0; rep < (EPC * TASKS + NT - 1) / NT; ++rep) {
        const int it = t + rep * NT;
        if (it >= nel * TASKS) break;
        const int el = it / TASKS, k = it - el * TASKS;
        const double* Y = work + el * PER;
        double* O = work + el * PER + XR;  // aliases Z (dead): [c][l] F.1, then fv
        if (k < FR) {
          const int c = k / DD, r = k - c * DD;  // r = dz*D1 + dy
          const int dz = r / D1, dy = r - dz * D1;
          double yg[Q], yb[Q];
#pragma unroll
          for (int qx = 0; qx < Q; ++qx) {
            yg[qx] = Y[(c * D1 + dz) * XPP + dy * XP + qx];
            yb[qx] = Y[(c * D1 + dz) * XPP + dy * XP + Q + qx];
          }
#pragma unroll
          for (int dx = 0; dx < D1; ++dx) {
            double s = 0.0;
#pragma unroll
            for (int qx = 0; qx < Q; ++qx) {
              s = fma(cG[qx * D1 + dx], yg[qx], s);
              s = fma(cB[qx * D1 + dx], yb[qx], s);
            }
            O[c * OPL + r * OR + dx] = s;
          }
        } else {
          const int r = k - FR;  // dz_t*DT + dy_t
          double y[Q];
#pragma unroll
          for (int qx = 0; qx < Q; ++qx) y[qx] = Y[YFS + r * Q + qx];
#pragma unroll
          for (int dx = 0; dx < DT; ++dx) {
            double s = 0.0;
#pragma unroll
            for (int qx = 0; qx < Q; ++qx) s = fma(cBt[qx * DT + dx], y[qx], s);
            O[3 * OPL + r * DT + dx] = s;
          }
        }
      }
    }
    __syncthreads();
    // ---- E: F.1 E-vector out, de = M_e^{-1} (F^T v)  (einsum "eij,ej->ei", hydro.py:343)
    for (int it = t; it < nel * NL * 3; it += NT) {
      const int el = it / (NL * 3), rem = it - el * (NL * 3);
      const int l = rem / 3, c = rem - l * 3;
      const double val = work[el * PER + XR + c * OPL + (l / D1) * OR + (l % D1)];
      const long long e = e0 + el;
      const long long pos = a.slot ? (long long)__ldg(a.slot + e * NL + l) * 3 + c : e * (NL * 3) + rem;
      a.evec[pos] = val;
    }
    for (int it = t; it < nel * NTH; it += NT) {
      const int el = it / NTH, i = it - el * NTH;
      const long long e = e0 + el;
      const double* fv = work + el * PER + XR + 3 * OPL;
      double s = 0.0;
      if constexpr (PK) {  // row i of the symmetric inverse: L[i][0..i], then L[j][i] for j > i
        const double* mi = gcur + R::FM + el * MN;
        const int ri = tri(i);
#pragma unroll
        for (int j = 0; j < NTH; ++j) s = fma(mi[j <= i ? ri + j : tri(j) + i], fv[j], s);
      } else {
        const double* mi = gcur + R::FM + (el * NTH + i) * NTH;
#pragma unroll
        for (int j = 0; j < NTH; ++j) s = fma(mi[j], fv[j], s);
      }
      a.de[e * NTH + i] = s;
    }
  }
  publish_status<NT>(a.st, rmin, clamps, key, nullptr);
}


// ---------------------------------------------------------------------------
// Geometry validity of a new state (rk2_step's check, hydro.py:400-401 ->
// compute_geometric_factors fespace.py:305-346): det J at every quadrature point,
// first inverted (q-major) point as the status key.  x only, so it gets its own lean
// kernel: 4 elements per pass, 4 CTAs per SM, no prefetch buffers.  J is formed with
// the same contraction order as k_rates_pc (x, y, z stages, ascending sums from 0.0)
// and det with det_inv_fast's expression, so both kernels agree on every det J.
#ifndef VALID_EPC
#define VALID_EPC 4
#endif
#ifndef VALID_MINB
#define VALID_MINB 4
#endif
template <int P>
struct ValidCfg {
  static constexpr int D1 = P + 1, Q = P + 2, DD = D1 * D1, QQ = Q * Q, NQ = Q * QQ;
  static constexpr int NT = 128, EPC = VALID_EPC;
  static constexpr int GP = DD + 1, GS = 3 * D1 * GP;         // gather image (c, dz) planes
  static constexpr int XP = 2 * Q + 1, XS = 3 * DD * XP;      // x-stage rows (c, dz, dy)
  static constexpr int PP = 3 * QQ + ((Q - 3 * QQ) % 16 + 16) % 16;
  static constexpr int TS = 3 * D1 * PP;                      // y-stage planes (c, dz), aliases G
  static constexpr int PER = XS + (TS > GS ? TS : GS);
  static constexpr size_t bytes = sizeof(double) * (size_t)EPC * PER;
};

template <int P>
__global__ void __launch_bounds__(128, VALID_MINB) k_valid(RatesPCArgs a) {
  using V = ValidCfg<P>;
  constexpr int D1 = V::D1, Q = V::Q, DD = V::DD, QQ = V::QQ, NQ = V::NQ, NL = D1 * DD;
  constexpr int NT = V::NT, EPC = V::EPC, GP = V::GP, XP = V::XP, PP = V::PP, PER = V::PER, XS = V::XS;
  const double* cB = c_B[P - 1];
  const double* cG = c_G[P - 1];
  extern __shared__ __align__(16) double smem[];
  const int t = threadIdx.x;
  unsigned long long key = ~0ull;
  for (long long e0 = (long long)blockIdx.x * EPC; e0 < a.ne; e0 += (long long)gridDim.x * EPC) {
    const int nel = (int)((a.ne - e0) < EPC ? (a.ne - e0) : EPC);
    // gather x node rows -> G image (aliases the T image of the previous pass); every
    // load of the thread is issued before the first shared store
    constexpr int ROW = 3 * D1, GI = EPC * DD * ROW, GU = (GI + NT - 1) / NT;
    long long nb[EPC];  // brick: the pass's element base nodes, once per pass
    if (a.brick) {
#pragma unroll
      for (int el = 0; el < EPC; ++el) {
        const unsigned ue = (unsigned)(e0 + el);
        const unsigned ez = a.b.fnxy.div(ue);
        const unsigned r2 = ue - ez * (unsigned)(a.b.nx * a.b.ny);
        const unsigned ey = a.b.fnx.div(r2), ex = r2 - ey * (unsigned)a.b.nx;
        nb[el] = (long long)(ex * P) + (long long)(ey * P) * a.b.Nx + (long long)(ez * P) * a.b.NxNy;
      }
    }
    {
      double xv[GU];
      int so[GU];
#pragma unroll
      for (int u = 0; u < GU; ++u) {
        const int it = t + u * NT;
        so[u] = -1;
        if (it < nel * DD * ROW) {
          const int el = it / (DD * ROW), rem = it - el * (DD * ROW);
          const int row = rem / ROW, sidx = rem - row * ROW;
          const int dz = row / D1, dy = row - dz * D1, dx = sidx / 3, c = sidx - dx * 3;
          const long long e = e0 + el;
          long long n;
          if (a.brick) {
            long long b0 = nb[0];
#pragma unroll
            for (int u = 1; u < EPC; ++u)
              if (el == u) b0 = nb[u];
            n = b0 + dx + (long long)dy * a.b.Nx + (long long)dz * a.b.NxNy;
          } else {
            n = __ldg(a.emap + e * NL + row * D1 + dx);
          }
          xv[u] = __ldg(a.x + n * 3 + c);
          so[u] = el * PER + XS + (c * D1 + dz) * GP + dy * D1 + dx;
        }
      }
#pragma unroll
      for (int u = 0; u < GU; ++u)
        if (so[u] >= 0) smem[so[u]] = xv[u];
    }
    __syncthreads();
    // x stage, thread per (c, dz, dy) row
    for (int it = t; it < nel * 3 * DD; it += NT) {
      const int el = it / (3 * DD), k = it - el * (3 * DD);
      const int pl = k / D1, dy = k - pl * D1;
      const double* g = smem + el * PER + XS + pl * GP + dy * D1;
      double u[D1];
#pragma unroll
      for (int dx = 0; dx < D1; ++dx) u[dx] = g[dx];
      double* o = smem + el * PER + k * XP;
#pragma unroll
      for (int qx = 0; qx < Q; ++qx) {
        double sb = 0.0, sg = 0.0;
#pragma unroll
        for (int dx = 0; dx < D1; ++dx) {
          sb = fma(cB[qx * D1 + dx], u[dx], sb);
          sg = fma(cG[qx * D1 + dx], u[dx], sg);
        }
        o[qx] = sb;
        o[Q + qx] = sg;
      }
    }
    __syncthreads();
    // y stage, thread per (c, dz, qx) line -> T (over the dead G image)
    for (int it = t; it < nel * 3 * D1 * Q; it += NT) {
      const int el = it / (3 * D1 * Q), k = it - el * (3 * D1 * Q);
      const int pl = k / Q, qx = k - pl * Q;
      const double* X = smem + el * PER;
      double vb[D1], vg[D1];
#pragma unroll
      for (int dy = 0; dy < D1; ++dy) {
        vb[dy] = X[(pl * D1 + dy) * XP + qx];
        vg[dy] = X[(pl * D1 + dy) * XP + Q + qx];
      }
      double* o = smem + el * PER + XS + pl * PP + qx;
#pragma unroll
      for (int qy = 0; qy < Q; ++qy) {
        double bb = 0.0, gb = 0.0, bg = 0.0;
#pragma unroll
        for (int dy = 0; dy < D1; ++dy) {
          bb = fma(cB[qy * D1 + dy], vb[dy], bb);
          gb = fma(cG[qy * D1 + dy], vb[dy], gb);
          bg = fma(cB[qy * D1 + dy], vg[dy], bg);
        }
        o[qy * Q] = bb;
        o[QQ + qy * Q] = gb;
        o[2 * QQ + qy * Q] = bg;
      }
    }
    __syncthreads();
    // z stage + det J, thread per point
    for (int it = t; it < nel * NQ; it += NT) {
      const int el = it / NQ, kq = it - el * NQ;
      const int col = kq / Q, qz = kq - col * Q;
      const int q = qz * QQ + col;
      const double* T = smem + el * PER + XS;
      double J[3][3];
#pragma unroll
      for (int f = 0; f < 3; ++f) {
        double d0 = 0.0, d1 = 0.0, d2 = 0.0;
#pragma unroll
        for (int dz = 0; dz < D1; ++dz) {
          const double* tt = T + (f * D1 + dz) * PP + col;
          d0 = fma(cB[qz * D1 + dz], tt[2 * QQ], d0);
          d1 = fma(cB[qz * D1 + dz], tt[QQ], d1);
          d2 = fma(cG[qz * D1 + dz], tt[0], d2);
        }
        J[f][0] = d0;
        J[f][1] = d1;
        J[f][2] = d2;
      }
      const double det = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) -
                         J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
                         J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
      if (det <= 0.0) {
        const unsigned long long kk = (unsigned long long)q * a.ne + (e0 + el);
        key = kk < key ? kk : key;
      }
    }
    __syncthreads();
  }
  publish_status<NT>(a.st, __longlong_as_double(0x7ff0000000000000ll), 0, key, nullptr);
}

}  // namespace hx
