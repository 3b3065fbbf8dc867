// hx_remap.cuh -- the remap-phase PA operators on the same contraction machinery:
// DiffusionPA (operators.py:143-185) and ConvectionPA (operators.py:188-236), scalar H1.
// One CTA per element: gather, reference gradients (grad), the point data combination,
// then grad_t (diffusion) or interp_t (convection); node-sorted E-vector out, scattered
// by the deterministic CSR node pass.
#pragma once

#include "hx_kernels.cuh"

namespace hx {

// D[a][c] = sum_b jinv[a][b] jinv[c][b] * wdetj (* nu)  ("abqe,cbqe,qe->acqe", operators.py:145-149)
template <int DIM>
__global__ void k_diff_D(const double* jinv, const double* wdetj, const double* nu, long long ne, int nq,
                         double* D /*(NE, d, d, nq)*/, double* D_ref /*(d, d, nq, NE) or null*/) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)nq * ne) return;
  const long long q = t / ne, e = t - q * ne;  // reference layout: element fastest
  const long long pe = q * ne + e;
  const long long stride = (long long)nq * ne;
  double scal = wdetj[pe];
  if (nu) scal *= nu[pe];
#pragma unroll
  for (int a = 0; a < DIM; ++a)
#pragma unroll
    for (int c = 0; c < DIM; ++c) {
      double s = 0.0;
#pragma unroll
      for (int b = 0; b < DIM; ++b) s = fma(jinv[(a * DIM + b) * stride + pe], jinv[(c * DIM + b) * stride + pe], s);
      const double v = s * scal;
      D[((e * DIM + a) * DIM + c) * nq + q] = v;
      if (D_ref) D_ref[(a * DIM + c) * stride + pe] = v;
    }
}

// D[l] = sum_b jinv[l][b] u[b] wdetj  ("lbqe,bqe,qe->lqe", operators.py:194-198)
template <int DIM>
__global__ void k_conv_D(const double* jinv, const double* u, const double* wdetj, long long ne, int nq,
                         double* D /*(NE, d, nq)*/, double* D_ref /*(d, nq, NE) or null*/) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)nq * ne) return;
  const long long q = t / ne, e = t - q * ne;
  const long long pe = q * ne + e;
  const long long stride = (long long)nq * ne;
#pragma unroll
  for (int l = 0; l < DIM; ++l) {
    double s = 0.0;
#pragma unroll
    for (int b = 0; b < DIM; ++b) s = fma(jinv[(l * DIM + b) * stride + pe], u[b * stride + pe], s);
    const double v = s * wdetj[pe];
    D[(e * DIM + l) * nq + q] = v;
    if (D_ref) D_ref[l * stride + pe] = v;
  }
}

template <int DIM, int P>
struct RemapSmem {
  using D = Disc<DIM, P>;
  static constexpr int A = cmax(D::NL, DIM == 3 ? 3 * D::Q * D::Q * D::D1 : D::NQ);
  static constexpr int S = 2 * D::Q * ipow(D::D1, DIM - 1);
  static constexpr int OUT = DIM * D::NQ;
  static constexpr int TOTAL = 2 * D::Q * D::D1 + A + S + OUT + D::NL;
  static constexpr size_t bytes = sizeof(double) * TOTAL;
};

struct RemapArgs {
  const double* x;    // (NN) scalar H1 field
  const double* D;    // diffusion (NE, d, d, nq) / convection (NE, d, nq)
  const int* emap;
  const int* slot;
  const double* B;
  const double* G;
  long long ne;
  double* evec;       // (NE*nl) node-sorted
};

// KIND 0: diffusion y = sum_a G_a^T (sum_b D[a][b] G_b x); KIND 1: convection y = B^T (sum_l D[l] G_l x)
template <int DIM, int P, int NT, int KIND>
__global__ void __launch_bounds__(NT) k_remap_op(RemapArgs a) {
  using D = Disc<DIM, P>;
  using SM = RemapSmem<DIM, P>;
  constexpr int D1 = D::D1, Q = D::Q, NL = D::NL, NQ = D::NQ;
  extern __shared__ double smem[];
  double* sB = smem;
  double* sG = sB + Q * D1;
  double* rA = sG + Q * D1;
  double* rS = rA + SM::A;
  double* rOut = rS + SM::S;
  double* rR = rOut + SM::OUT;
  const int tid = threadIdx.x;
  const long long e = blockIdx.x;
  for (int i = tid; i < Q * D1; i += NT) {
    sB[i] = a.B[i];
    sG[i] = a.G[i];
  }
  const int* em = a.emap + e * NL;
  for (int i = tid; i < NL; i += NT) rA[i] = a.x[em[i]];
  __syncthreads();
  grad<DIM, D1, Q, 1, DIM, NT>(sB, sG, rA, rS, rA, rOut, tid);
  __syncthreads();
  const double* De = a.D + e * (KIND == 0 ? DIM * DIM : DIM) * NQ;
  for (int q = tid; q < NQ; q += NT) {
    double g[DIM];
#pragma unroll
    for (int b = 0; b < DIM; ++b) g[b] = rOut[b * NQ + q];
    if constexpr (KIND == 0) {
#pragma unroll
      for (int c = 0; c < DIM; ++c) {
        double s = De[(c * DIM + 0) * NQ + q] * g[0];
#pragma unroll
        for (int b = 1; b < DIM; ++b) s += De[(c * DIM + b) * NQ + q] * g[b];
        rOut[c * NQ + q] = s;
      }
    } else {
      double s = De[q] * g[0];
#pragma unroll
      for (int l = 1; l < DIM; ++l) s += De[l * NQ + q] * g[l];
      rOut[q] = s;
    }
  }
  __syncthreads();
  const double* res;
  if constexpr (KIND == 0) {
    grad_t<DIM, D1, Q, 1, DIM * NQ, NT>(sB, sG, rOut, rA, rS, rR, tid);
    res = rR;
  } else {
    res = interp_t<DIM, D1, Q, 1, NT>(sB, rOut, rA, tid);
  }
  __syncthreads();
  for (int i = tid; i < NL; i += NT) a.evec[a.slot[e * NL + i]] = res[i];
}

}  // namespace hx
