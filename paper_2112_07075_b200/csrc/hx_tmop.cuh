// hx_tmop.cuh -- matrix-free TMOP mesh-optimisation kernels (the ALE mesh-optimisation
// phase, meshopt.py:248-486) on the Lagrange phase's contraction machinery.
//
// F(x) = sum_q w_q detW mu(T) + gamma sum_q w_q detW |(x - x0)/d(x0)|^2,  T = A W^{-1},
// A = dx/dxi at the point.  Per element (one CTA), everything at the points is computed
// on the fly from the gathered positions -- no point data is stored between calls
// ("there is no matrix D", SPEC tmop_mesh_opt / paper Sec. 3.4):
//   MODE 0  objective mu-term: per-element sum of w detW mu(T)          (meshopt.py:335-340)
//   MODE 1  gradient:    P = dmu(T) W^{-T} w detW, assembled by grad_t  (meshopt.py:364-389)
//   MODE 2  Hessian action on dx: dT = dA W^{-1}, dS = d2mu(T)[dT],
//           P = dS W^{-T} w detW, grad_t                                (meshopt.py:407-424)
//   MODE 3  Hessian diagonal: K_a[l1,l2] = W^{-1} h4[a,:,a,:] W^{-T} w detW contracted
//           with the per-axis basis products (B B, B G, G G)            (meshopt.py:442-486)
// and, with LIM (gamma != 0), the limiting term's pieces in the same element pass
// (meshopt.py:342-356, 391-405, 426-440, 480-484): r = (x - x0)/d (objective, gradient) or
// dx/d (Hessian action) formed at the gather with the reference's rounding, interpolated to
// the points: the per-element sum_a sum_q w detW r_a^2 (MODE 0) or the element vectors
// B^T (w detW r_a) (MODE 1, 2) into a second E-vector; MODE 3 adds (B o B)^T w detW.
// E-vectors are node-sorted and summed by the deterministic CSR node pass (scatter_add
// order).  The metric derivatives are analytic (shape: 2D |T|^2/(2 det T) - 1, 3D
// |T|^2 |T^{-1}|^2 / 9 - 1; size (det T + 1/det T)/2 - 1; composite = w_shape * shape +
// w_size * size); the Hessian is applied as the directional derivative of dmu along dT
// instead of forming the 4-tensor.
#pragma once

#include "hx_kernels.cuh"

namespace hx {

#ifndef TMOP_MINB
#define TMOP_MINB 4  // Hessian action 402 -> 361 us at 23^3 Q3 (127 regs, small spill) vs no bound
#endif

template <int DIM>
__device__ __forceinline__ double tm_ddot(const double (&a)[DIM][DIM], const double (&b)[DIM][DIM]) {
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < DIM; ++i)
#pragma unroll
    for (int j = 0; j < DIM; ++j) s = fma(a[i][j], b[i][j], s);
  return s;
}

// cofactor matrix (d det / dT) and determinant
template <int DIM>
__device__ __forceinline__ double tm_cof(const double (&T)[DIM][DIM], double (&C)[DIM][DIM]) {
  if constexpr (DIM == 2) {
    C[0][0] = T[1][1];
    C[0][1] = -T[1][0];
    C[1][0] = -T[0][1];
    C[1][1] = T[0][0];
    return T[0][0] * T[1][1] - T[0][1] * T[1][0];
  } else {
#pragma unroll
    for (int m = 0; m < 3; ++m)
#pragma unroll
      for (int n = 0; n < 3; ++n) {
        const int m1 = (m + 1) % 3, m2 = (m + 2) % 3, n1 = (n + 1) % 3, n2 = (n + 2) % 3;
        C[m][n] = T[m1][n1] * T[m2][n2] - T[m1][n2] * T[m2][n1];
      }
    return T[0][0] * C[0][0] + T[0][1] * C[0][1] + T[0][2] * C[0][2];
  }
}

// directional derivative of the cofactor matrix: dC = d cof(T)[dT]
template <int DIM>
__device__ __forceinline__ void tm_dcof(const double (&T)[DIM][DIM], const double (&dT)[DIM][DIM],
                                        double (&dC)[DIM][DIM]) {
  if constexpr (DIM == 2) {  // cof is linear in 2D
    dC[0][0] = dT[1][1];
    dC[0][1] = -dT[1][0];
    dC[1][0] = -dT[0][1];
    dC[1][1] = dT[0][0];
  } else {
#pragma unroll
    for (int m = 0; m < 3; ++m)
#pragma unroll
      for (int n = 0; n < 3; ++n) {
        const int m1 = (m + 1) % 3, m2 = (m + 2) % 3, n1 = (n + 1) % 3, n2 = (n + 2) % 3;
        dC[m][n] = (dT[m1][n1] * T[m2][n2] + T[m1][n1] * dT[m2][n2]) - (dT[m1][n2] * T[m2][n1] + T[m1][n2] * dT[m2][n1]);
      }
  }
}

struct TmopMetric {
  double ws, wz;  // weights of the shape and size parts
  int composite;  // 0: shape only (metric_for(d)), 1: ws * shape + wz * size
};

// mu, dmu (into D) and, with dT != null, the directional derivative d2mu[dT] (into H)
template <int DIM, bool DMU, bool DD>
__device__ __forceinline__ double tm_metric(const TmopMetric& mt, const double (&T)[DIM][DIM],
                                            const double (&dT)[DIM][DIM], double (&D)[DIM][DIM],
                                            double (&H)[DIM][DIM]) {
  double C[DIM][DIM];
  const double tau = tm_cof<DIM>(T, C);
  const double f = tm_ddot<DIM>(T, T);
  double mu_s, mu_z = 0.0;
  double Ds[DIM][DIM], Hs[DIM][DIM];
  if constexpr (DIM == 2) {
    mu_s = f / (2.0 * tau) - 1.0;
    const double it = 1.0 / tau, c2 = f / (2.0 * tau * tau);
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) Ds[i][j] = T[i][j] * it - c2 * C[i][j];
    if constexpr (DD) {
      const double cd = tm_ddot<2>(C, dT), td = tm_ddot<2>(T, dT);
      double dC[2][2];
      tm_dcof<2>(T, dT, dC);
      const double it2 = it * it, c3 = f * it2 * it;
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j)
          Hs[i][j] = dT[i][j] * it - (T[i][j] * cd + C[i][j] * td) * it2 + c3 * cd * C[i][j] - c2 * dC[i][j];
    }
  } else {
    // S = T^{-1} = C^T / tau; N = S^T S S^T
    double S[3][3];
    const double it = 1.0 / tau;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) S[i][j] = C[j][i] * it;
    const double g = tm_ddot<3>(S, S);
    double StS[3][3], SSt[3][3], N[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        double a = 0.0, b = 0.0;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          a = fma(S[k][i], S[k][j], a);
          b = fma(S[i][k], S[j][k], b);
        }
        StS[i][j] = a;
        SSt[i][j] = b;
      }
#pragma unroll
    for (int m = 0; m < 3; ++m)
#pragma unroll
      for (int z = 0; z < 3; ++z) {
        double a = 0.0;
#pragma unroll
        for (int k = 0; k < 3; ++k) a = fma(StS[m][k], S[z][k], a);
        N[m][z] = a;
      }
    mu_s = f * g / 9.0 - 1.0;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) Ds[i][j] = (2.0 * g * T[i][j] - 2.0 * f * N[i][j]) / 9.0;
    if constexpr (DD) {
      const double nd = tm_ddot<3>(N, dT), td = tm_ddot<3>(T, dT);
      // dN = -(S^T dT^T N + (S^T S) dT (S S^T) + N dT^T S^T)
      double A1[3][3], A2[3][3], A3[3][3], dN[3][3];
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          double u = 0.0, v = 0.0;
#pragma unroll
          for (int k = 0; k < 3; ++k) {
            u = fma(dT[k][i], N[k][j], u);   // (dT^T N)[i][j]
            v = fma(StS[i][k], dT[k][j], v);  // (S^T S dT)[i][j]
          }
          A1[i][j] = u;
          A2[i][j] = v;
        }
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          double u = 0.0;
#pragma unroll
          for (int k = 0; k < 3; ++k) u = fma(N[i][k], dT[j][k], u);  // (N dT^T)[i][j]
          A3[i][j] = u;
        }
#pragma unroll
      for (int m = 0; m < 3; ++m)
#pragma unroll
        for (int z = 0; z < 3; ++z) {
          double a = 0.0, b = 0.0, c = 0.0;
#pragma unroll
          for (int k = 0; k < 3; ++k) {
            a = fma(S[k][m], A1[k][z], a);   // S^T (dT^T N)
            b = fma(A2[m][k], SSt[k][z], b);  // (S^T S dT) S S^T
            c = fma(A3[m][k], S[z][k], c);    // (N dT^T) S^T
          }
          dN[m][z] = -(a + b + c);
        }
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j)
          Hs[i][j] = (2.0 * g * dT[i][j] - 4.0 * (nd * T[i][j] + td * N[i][j]) - 2.0 * f * dN[i][j]) / 9.0;
    }
  }
  if (!mt.composite) {
    if constexpr (DMU) {
#pragma unroll
      for (int i = 0; i < DIM; ++i)
#pragma unroll
        for (int j = 0; j < DIM; ++j) {
          D[i][j] = Ds[i][j];
          if constexpr (DD) H[i][j] = Hs[i][j];
        }
    }
    return mu_s;
  }
  // size part: mu = (tau + 1/tau)/2 - 1, dmu = (1 - 1/tau^2)/2 C,
  // d2mu[dT] = (C:dT)/tau^3 C + (1 - 1/tau^2)/2 dC[dT]
  mu_z = 0.5 * (tau + 1.0 / tau) - 1.0;
  const double h = 0.5 * (1.0 - 1.0 / (tau * tau));
  if constexpr (DMU) {
    double dC[DIM][DIM];
    double cd = 0.0;
    if constexpr (DD) {
      tm_dcof<DIM>(T, dT, dC);
      cd = tm_ddot<DIM>(C, dT);
    }
    const double it3 = 1.0 / (tau * tau * tau);
#pragma unroll
    for (int i = 0; i < DIM; ++i)
#pragma unroll
      for (int j = 0; j < DIM; ++j) {
        D[i][j] = mt.ws * Ds[i][j] + mt.wz * (h * C[i][j]);
        if constexpr (DD) H[i][j] = mt.ws * Hs[i][j] + mt.wz * (it3 * cd * C[i][j] + h * dC[i][j]);
      }
  }
  return mt.ws * mu_s + mt.wz * mu_z;
}

template <int DIM, int P>
struct TmopSmem {
  using D = Disc<DIM, P>;
  static constexpr int TAB = 5 * D::Q * D::D1;  // B, G, B o B, B o G, G o G
  // A also holds interp's 2D result (DIM x NQ) and the diagonal's first contraction
  static constexpr int A = cmax(cmax(DIM * D::NL, DIM * D::NQ), DIM == 3 ? 3 * DIM * D::Q * D::Q * D::D1 : 0);
  static constexpr int S = 2 * DIM * D::Q * ipow(D::D1, DIM - 1);
  static constexpr int OUT = DIM * (DIM + 1) * D::NQ;
  static constexpr int OUT2 = cmax(DIM * (DIM + 1) * D::NQ, DIM * DIM * DIM * D::NQ);
  static constexpr int R = DIM * D::NL;
  static constexpr int TOTAL = TAB + A + S + OUT + OUT2 + R;
  static constexpr size_t bytes = sizeof(double) * TOTAL;
};

struct TmopArgs {
  const double* x;      // (NN, d) positions (MODE 0-3), or the nodal limiting field r (MODE 4)
  const double* dx;     // (NN, d) Hessian-action direction (MODE 2)
  const double* winv;   // (NE, nq, d, d): W^{-1}[b][l]
  const double* wdetw;  // (NE, nq)
  const int* emap;
  const int* slot;
  const double* B;
  const double* G;
  TmopMetric mt;
  long long ne;
  double* evec;         // (NE*nl, NC) node-sorted element vectors (mu part)
  double* epart;        // (NE) per-element sums (MODE 0)
  int* bad;             // set when det A <= 0 at any point
  const double* x0;     // (NN, d) limiting anchor (LIM)
  const double* dlim;   // (NN) limiting radii (LIM)
  double* evec2;        // (NE*nl, NC) limiting element vectors (LIM, MODE 1-3)
  double* epart2;       // (NE) limiting per-element sums (LIM, MODE 0)
};

template <int DIM, int P, int NT, int MODE, bool LIM>
__global__ void __launch_bounds__(NT, TMOP_MINB) k_tmop(TmopArgs a) {  // persistent grid
  using D = Disc<DIM, P>;
  using SM = TmopSmem<DIM, P>;
  constexpr int D1 = D::D1, Q = D::Q, NL = D::NL, NQ = D::NQ, QD = Q * D1;
  constexpr int CS = (DIM + 1) * NQ;  // component stride of grad's output
  extern __shared__ double smem[];
  __shared__ double red[32];
  double* sB = smem;
  double* sG = sB + QD;
  double* sBB = sG + QD;
  double* sBG = sBB + QD;
  double* sGG = sBG + QD;
  double* rA = smem + SM::TAB;
  double* rS = rA + SM::A;
  double* rO = rS + SM::S;
  double* rO2 = rO + SM::OUT;
  double* rR = rO2 + SM::OUT2;
  const int tid = threadIdx.x;
  for (int i = tid; i < QD; i += NT) {
    const double b = a.B[i], g = a.G[i];
    sB[i] = b;
    sG[i] = g;
    sBB[i] = b * b;
    sBG[i] = b * g;
    sGG[i] = g * g;
  }
  __syncthreads();
  // persistent CTAs: the tables once, then one element at a time (grid-stride)
  auto element = [&](const long long e) {
  const int* em = a.emap + e * NL;
  const double* We = a.winv + e * NQ * DIM * DIM;
  const double* wd = a.wdetw + e * NQ;
  // the limiting term of this element (LIM): r = (x - x0)/d or dx/d at the nodes ->
  // the points -> sum w detW r^2 (MODE 0) or B^T (w detW r) into evec2 (MODE 1, 2); the
  // diagonal's (B o B)^T w detW (MODE 3).  Uses rA, rS, rO only.
  auto limiting = [&]() {
    if constexpr (MODE == 3) {
      for (int q = tid; q < NQ; q += NT) rA[q] = wd[q];
      __syncthreads();
      const double* res = interp_t<DIM, D1, Q, 1, NT>(sBB, rA, rS, tid);
      __syncthreads();
      for (int i = tid; i < NL; i += NT) a.evec2[a.slot[e * NL + i]] = res[i];
    } else {
      const double* src = MODE == 2 ? a.dx : a.x;
      for (int i = tid; i < NL * DIM; i += NT) {
        const int l = i / DIM, c = i - l * DIM;
        const long long n = em[l];
        const double d = a.dlim[n];
        rA[c * NL + l] = MODE == 2 ? src[n * DIM + c] / d : (src[n * DIM + c] - a.x0[n * DIM + c]) / d;
      }
      __syncthreads();
      double* rq = interp<DIM, D1, Q, DIM, NT>(sB, rA, rS, tid);
      __syncthreads();
      if constexpr (MODE == 0) {
        double acc = 0.0;
        for (int i = tid; i < DIM * NQ; i += NT) {
          const double v = rq[i];
          acc = fma(wd[i % NQ] * v, v, acc);
        }
        const double tot = block_sum<NT>(acc, red);
        if (tid == 0) a.epart2[e] = tot;
      } else {
        for (int i = tid; i < DIM * NQ; i += NT) rO[i] = wd[i % NQ] * rq[i];
        __syncthreads();
        const double* res = interp_t<DIM, D1, Q, DIM, NT>(sB, rO, rS, tid);
        __syncthreads();
        for (int i = tid; i < NL * DIM; i += NT) {
          const int l = i / DIM, c = i - l * DIM;
          a.evec2[(long long)a.slot[e * NL + l] * DIM + c] = res[c * NL + l];
        }
      }
    }
  };
  // gather the positions -> rA (component-major)
  for (int i = tid; i < NL * DIM; i += NT) {
    const int l = i / DIM, c = i - l * DIM;
    rA[c * NL + l] = a.x[(long long)em[l] * DIM + c];
  }
  __syncthreads();
  {
    grad<DIM, D1, Q, DIM, DIM + 1, NT>(sB, sG, rA, rS, rA, rO, tid);  // A[a][l] at the points
    __syncthreads();
    if constexpr (MODE == 2) {
      for (int i = tid; i < NL * DIM; i += NT) {
        const int l = i / DIM, c = i - l * DIM;
        rA[c * NL + l] = a.dx[(long long)em[l] * DIM + c];
      }
      __syncthreads();
      grad<DIM, D1, Q, DIM, DIM + 1, NT>(sB, sG, rA, rS, rA, rO2, tid);  // dA at the points
      __syncthreads();
    }
    double acc = 0.0;
    bool badq = false;
    for (int q = tid; q < NQ; q += NT) {
      double Am[DIM][DIM], T[DIM][DIM], Wi[DIM][DIM], dT[DIM][DIM], Dm[DIM][DIM], Hm[DIM][DIM];
#pragma unroll
      for (int i = 0; i < DIM; ++i)
#pragma unroll
        for (int j = 0; j < DIM; ++j) {
          Am[i][j] = rO[i * CS + j * NQ + q];
          Wi[i][j] = We[(q * DIM + i) * DIM + j];
        }
      double Cm[DIM][DIM];
      if (tm_cof<DIM>(Am, Cm) <= 0.0) badq = true;
#pragma unroll
      for (int i = 0; i < DIM; ++i)
#pragma unroll
        for (int l = 0; l < DIM; ++l) {
          double s = 0.0;
#pragma unroll
          for (int b = 0; b < DIM; ++b) s = fma(Am[i][b], Wi[b][l], s);
          T[i][l] = s;
        }
      if constexpr (MODE == 0) {
        const double mu = tm_metric<DIM, false, false>(a.mt, T, T, Dm, Hm);
        acc = fma(wd[q], mu, acc);
      } else if constexpr (MODE == 1 || MODE == 2) {
        if constexpr (MODE == 2) {
#pragma unroll
          for (int i = 0; i < DIM; ++i)
#pragma unroll
            for (int l = 0; l < DIM; ++l) {
              double s = 0.0;
#pragma unroll
              for (int b = 0; b < DIM; ++b) s = fma(rO2[i * CS + b * NQ + q], Wi[b][l], s);
              dT[i][l] = s;
            }
          tm_metric<DIM, true, true>(a.mt, T, dT, Dm, Hm);
        } else {
          tm_metric<DIM, true, false>(a.mt, T, T, Dm, Hm);
        }
        // P[c][l] = sum_n S[c][n] W^{-1}[l][n] w detW -> grad_t's input slots (in place)
#pragma unroll
        for (int c = 0; c < DIM; ++c)
#pragma unroll
          for (int l = 0; l < DIM; ++l) {
            double s = 0.0;
#pragma unroll
            for (int n = 0; n < DIM; ++n) s = fma(MODE == 2 ? Hm[c][n] : Dm[c][n], Wi[l][n], s);
            rO[c * CS + l * NQ + q] = s * wd[q];
          }
      } else {  // MODE 3: K_a[l1][l2] for every a, into rO2[(a*DIM + l1)*DIM + l2][q]
        double h4[DIM][DIM][DIM];  // h4[a][n][p] = d2mu[a,n,a,p]
#pragma unroll
        for (int pp = 0; pp < DIM; ++pp)
#pragma unroll
          for (int aa = 0; aa < DIM; ++aa) {
#pragma unroll
            for (int i = 0; i < DIM; ++i)
#pragma unroll
              for (int j = 0; j < DIM; ++j) dT[i][j] = (i == aa && j == pp) ? 1.0 : 0.0;
            tm_metric<DIM, true, true>(a.mt, T, dT, Dm, Hm);
#pragma unroll
            for (int n = 0; n < DIM; ++n) h4[aa][n][pp] = Hm[aa][n];
          }
#pragma unroll
        for (int aa = 0; aa < DIM; ++aa)
#pragma unroll
          for (int l1 = 0; l1 < DIM; ++l1)
#pragma unroll
            for (int l2 = 0; l2 < DIM; ++l2) {
              double s = 0.0;
#pragma unroll
              for (int n = 0; n < DIM; ++n) {
                double t = 0.0;
#pragma unroll
                for (int pp = 0; pp < DIM; ++pp) t = fma(h4[aa][n][pp], Wi[l2][pp], t);
                s = fma(Wi[l1][n], t, s);
              }
              rO2[((aa * DIM + l1) * DIM + l2) * NQ + q] = s * wd[q];
            }
      }
    }
    if (badq) *a.bad = 1;
    if constexpr (MODE == 0) {
      const double tot = block_sum<NT>(acc, red);
      if (tid == 0) a.epart[e] = tot;
      if constexpr (LIM) {
        __syncthreads();
        limiting();
      }
      return;
    }
    __syncthreads();
    if constexpr (MODE == 1 || MODE == 2) {
      grad_t<DIM, D1, Q, DIM, CS, NT>(sB, sG, rO, rA, rS, rR, tid);
      __syncthreads();
    } else {
      // diag[a][node] = sum_{l1,l2} prod_b (m1_b o m2_b)^T K_a[l1][l2], m = G on axis l else B
      for (int l1 = 0; l1 < DIM; ++l1)
        for (int l2 = 0; l2 < DIM; ++l2) {
          const double* Mb[3];
#pragma unroll
          for (int b = 0; b < DIM; ++b) {
            const int ng = (b == l1) + (b == l2);
            Mb[b] = ng == 0 ? sBB : (ng == 1 ? sBG : sGG);
          }
          // gather the DIM fields K_a[l1][l2] (a = 0..DIM-1) contiguously into rO
          for (int i = tid; i < DIM * NQ; i += NT) {
            const int aa = i / NQ, q = i - aa * NQ;
            rO[i] = rO2[((aa * DIM + l1) * DIM + l2) * NQ + q];
          }
          __syncthreads();
          const bool first = l1 == 0 && l2 == 0;
          if constexpr (DIM == 3) {
            contract<Q, Q, Q, 0, D1, true, DIM, NT>(Mb[0], rO, rA, tid);   // (D1, Q, Q)
            __syncthreads();
            contract<D1, Q, Q, 1, D1, true, DIM, NT>(Mb[1], rA, rS, tid);  // (D1, D1, Q)
            __syncthreads();
            if (first) contract<D1, D1, Q, 2, D1, true, DIM, NT>(Mb[2], rS, rR, tid);
            else contract<D1, D1, Q, 2, D1, true, DIM, NT, true>(Mb[2], rS, rR, tid);
          } else {
            contract<Q, Q, 1, 0, D1, true, DIM, NT>(Mb[0], rO, rA, tid);  // (D1, Q)
            __syncthreads();
            if (first) contract<D1, Q, 1, 1, D1, true, DIM, NT>(Mb[1], rA, rR, tid);
            else contract<D1, Q, 1, 1, D1, true, DIM, NT, true>(Mb[1], rA, rR, tid);
          }
          __syncthreads();
        }
    }
    for (int i = tid; i < NL * DIM; i += NT) {
      const int l = i / DIM, c = i - l * DIM;
      a.evec[(long long)a.slot[e * NL + l] * DIM + c] = rR[c * NL + l];
    }
    if constexpr (LIM) limiting();  // rA / rS / rO are free (grad_t / the diagonal are done)
  }
  };
  for (long long e = blockIdx.x; e < a.ne; e += gridDim.x) {
    element(e);
    __syncthreads();  // the element's images are dead before the next gather
  }
}

// node-level combine of the two assembled parts (elementwise, reference rounding):
//   mode 2  out = mu + (2 gamma s) / d   (gradient / Hessian action, meshopt.py:387-389, 422-424)
//   mode 3  out = mu + (2 gamma s) / d^2, s per node broadcast over components (meshopt.py:480-484)
__global__ void k_tmop_nodes(int mode, const double* x, const double* x0, const double* dlim, const double* mu,
                             const double* s, double gamma, int dim, long long nn, double* out) {
  const long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= nn * dim) return;
  const long long n = j / dim;
  const double d = dlim[n];
  if (mode == 2) out[j] = mu[j] + (2.0 * gamma * s[j]) / d;
  else out[j] = mu[j] + (2.0 * gamma * s[n]) / (d * d);
  (void)x;
  (void)x0;
}

}  // namespace hx
