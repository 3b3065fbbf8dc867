// hx_core.cuh -- element-tensor machinery for the sm_100a PA kernels.
//
// An element "team" (a warp, or a whole CTA) owns one element at a time.  Element
// tensors live in shared memory in the reference's tensor layout
// (n_{d-1}, ..., n_0) with x fastest (tensor_basis.py:7-13); components are
// stacked contiguously.  A 1D contraction along one axis is a small
// (m_out x m_in) matrix applied to every line of the tensor
// (contract_dim, tensor_basis.py:207-226): each team thread owns whole lines, keeps
// the m_in inputs of its line in registers and writes the m_out outputs, so a
// shared-memory load feeds m_out FMAs.  The basis matrices are read with
// warp-uniform addresses (shared-memory broadcast).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace hx {

__host__ __device__ constexpr int ipow(int b, int e) { return e == 0 ? 1 : b * ipow(b, e - 1); }
__host__ __device__ constexpr int cmax(int a, int b) { return a > b ? a : b; }

// Compile-time discretisation: DIM, kinematic nodes D1 = p+1, quadrature points
// Q = p+2, thermodynamic nodes DT = p (order p-1; order 0 has one node).
template <int DIM_, int P_>
struct Disc {
  static constexpr int DIM = DIM_, P = P_;
  static constexpr int D1 = P + 1, Q = P + 2, DT = P;
  static constexpr int NL = ipow(D1, DIM), NQ = ipow(Q, DIM), NT = ipow(DT, DIM);
};

// team barrier: a warp team uses __syncwarp, a CTA team __syncthreads
template <int T>
__device__ __forceinline__ void team_sync() {
  if constexpr (T <= 32) __syncwarp();
  else __syncthreads();
}

// out = M . in along axis AX of an (N0, N1, N2) tensor (N0 fastest), NC components.
// M is (MO x MI) row-major; TR: M is stored (MI x MO) and applied transposed.
// ACC: out += result instead of out = result.
template <int N0, int N1, int N2, int AX, int MO, bool TR, int NC, int T, bool ACC = false>
__device__ __forceinline__ void contract(const double* __restrict__ M, const double* in,
                                         double* out, int tid) {
  constexpr int MI = AX == 0 ? N0 : (AX == 1 ? N1 : N2);
  constexpr int O0 = AX == 0 ? MO : N0, O1 = AX == 1 ? MO : N1, O2 = AX == 2 ? MO : N2;
  constexpr int INSZ = N0 * N1 * N2, OUTSZ = O0 * O1 * O2;
  constexpr int NLN = INSZ / MI;
  constexpr int ISTR = AX == 0 ? 1 : (AX == 1 ? N0 : N0 * N1);
  constexpr int OSTR = AX == 0 ? 1 : (AX == 1 ? O0 : O0 * O1);
  for (int w = tid; w < NLN * NC; w += T) {
    const int c = w / NLN, l = w - c * NLN;
    int ib, ob;
    if constexpr (AX == 0) {
      ib = l * N0;
      ob = l * O0;
    } else if constexpr (AX == 1) {
      const int i0 = l % N0, i2 = l / N0;
      ib = i2 * N0 * N1 + i0;
      ob = i2 * O0 * O1 + i0;
    } else {
      ib = l;
      ob = l;
    }
    const double* src = in + c * INSZ + ib;
    double* dst = out + c * OUTSZ + ob;
    double xin[MI];
#pragma unroll
    for (int j = 0; j < MI; ++j) xin[j] = src[j * ISTR];
#pragma unroll
    for (int k = 0; k < MO; ++k) {
      double acc = 0.0;
#pragma unroll
      for (int j = 0; j < MI; ++j) acc = fma(TR ? M[j * MO + k] : M[k * MI + j], xin[j], acc);
      if constexpr (ACC) dst[k * OSTR] += acc;
      else dst[k * OSTR] = acc;
    }
    (void)O2;
  }
}

// Two matrices on the same input lines (e.g. B and G along x): out1 = M1.in, out2 = M2.in
template <int N0, int N1, int N2, int AX, int MO, bool TR, int NC, int T>
__device__ __forceinline__ void contract2(const double* __restrict__ M1, const double* __restrict__ M2,
                                          const double* in, double* out1, double* out2, int tid) {
  constexpr int MI = AX == 0 ? N0 : (AX == 1 ? N1 : N2);
  constexpr int O0 = AX == 0 ? MO : N0, O1 = AX == 1 ? MO : N1, O2 = AX == 2 ? MO : N2;
  constexpr int INSZ = N0 * N1 * N2, OUTSZ = O0 * O1 * O2;
  constexpr int NLN = INSZ / MI;
  constexpr int ISTR = AX == 0 ? 1 : (AX == 1 ? N0 : N0 * N1);
  constexpr int OSTR = AX == 0 ? 1 : (AX == 1 ? O0 : O0 * O1);
  for (int w = tid; w < NLN * NC; w += T) {
    const int c = w / NLN, l = w - c * NLN;
    int ib, ob;
    if constexpr (AX == 0) {
      ib = l * N0;
      ob = l * O0;
    } else if constexpr (AX == 1) {
      const int i0 = l % N0, i2 = l / N0;
      ib = i2 * N0 * N1 + i0;
      ob = i2 * O0 * O1 + i0;
    } else {
      ib = l;
      ob = l;
    }
    const double* src = in + c * INSZ + ib;
    double xin[MI];
#pragma unroll
    for (int j = 0; j < MI; ++j) xin[j] = src[j * ISTR];
#pragma unroll
    for (int k = 0; k < MO; ++k) {
      double a1 = 0.0, a2 = 0.0;
#pragma unroll
      for (int j = 0; j < MI; ++j) {
        a1 = fma(TR ? M1[j * MO + k] : M1[k * MI + j], xin[j], a1);
        a2 = fma(TR ? M2[j * MO + k] : M2[k * MI + j], xin[j], a2);
      }
      out1[c * OUTSZ + ob + k * OSTR] = a1;
      out2[c * OUTSZ + ob + k * OSTR] = a2;
    }
    (void)O2;
  }
}

// out = M1.in1 + M2.in2 (same shapes), used by the transposed gradients
template <int N0, int N1, int N2, int AX, int MO, bool TR, int NC, int T>
__device__ __forceinline__ void contract_sum2(const double* __restrict__ M1, const double* in1,
                                              const double* __restrict__ M2, const double* in2,
                                              double* out, int tid) {
  constexpr int MI = AX == 0 ? N0 : (AX == 1 ? N1 : N2);
  constexpr int O0 = AX == 0 ? MO : N0, O1 = AX == 1 ? MO : N1, O2 = AX == 2 ? MO : N2;
  constexpr int INSZ = N0 * N1 * N2, OUTSZ = O0 * O1 * O2;
  constexpr int NLN = INSZ / MI;
  constexpr int ISTR = AX == 0 ? 1 : (AX == 1 ? N0 : N0 * N1);
  constexpr int OSTR = AX == 0 ? 1 : (AX == 1 ? O0 : O0 * O1);
  for (int w = tid; w < NLN * NC; w += T) {
    const int c = w / NLN, l = w - c * NLN;
    int ib, ob;
    if constexpr (AX == 0) {
      ib = l * N0;
      ob = l * O0;
    } else if constexpr (AX == 1) {
      const int i0 = l % N0, i2 = l / N0;
      ib = i2 * N0 * N1 + i0;
      ob = i2 * O0 * O1 + i0;
    } else {
      ib = l;
      ob = l;
    }
    const double* s1 = in1 + c * INSZ + ib;
    const double* s2 = in2 + c * INSZ + ib;
    double x1[MI], x2[MI];
#pragma unroll
    for (int j = 0; j < MI; ++j) {
      x1[j] = s1[j * ISTR];
      x2[j] = s2[j * ISTR];
    }
#pragma unroll
    for (int k = 0; k < MO; ++k) {
      double a = 0.0;
#pragma unroll
      for (int j = 0; j < MI; ++j) {
        a = fma(TR ? M1[j * MO + k] : M1[k * MI + j], x1[j], a);
        a = fma(TR ? M2[j * MO + k] : M2[k * MI + j], x2[j], a);
      }
      out[c * OUTSZ + ob + k * OSTR] = a;
    }
    (void)O2;
  }
}

// ---------------------------------------------------------------------------
// Sum-factorised element operators built from the contractions.
// Sizes: ND = nodes per direction, NQD = points per direction.

// interpolation nodes -> points on every axis (tensor_interp, tensor_basis.py:234-238)
// in: NC x ND^DIM in A (clobbered); Bf: scratch. Returns the buffer holding the
// NC x NQD^DIM result (Bf in 3D, A in 2D).
template <int DIM, int ND, int NQD, int NC, int T>
__device__ __forceinline__ double* interp(const double* B, double* A, double* Bf, int tid) {
  if constexpr (DIM == 3) {
    contract<ND, ND, ND, 0, NQD, false, NC, T>(B, A, Bf, tid);  // (NQD, ND, ND)
    team_sync<T>();
    contract<NQD, ND, ND, 1, NQD, false, NC, T>(B, Bf, A, tid);  // (NQD, NQD, ND)
    team_sync<T>();
    contract<NQD, NQD, ND, 2, NQD, false, NC, T>(B, A, Bf, tid);  // (NQD^3)
    return Bf;
  } else {
    contract<ND, ND, 1, 0, NQD, false, NC, T>(B, A, Bf, tid);
    team_sync<T>();
    contract<NQD, ND, 1, 1, NQD, false, NC, T>(B, Bf, A, tid);
    return A;
  }
}

// transpose interpolation points -> nodes (tensor_interp_t, tensor_basis.py:241-245)
// in: NC x NQD^DIM in A (clobbered); returns the buffer with NC x ND^DIM (Bf in 3D, A in 2D)
template <int DIM, int ND, int NQD, int NC, int T>
__device__ __forceinline__ double* interp_t(const double* B, double* A, double* Bf, int tid) {
  if constexpr (DIM == 3) {
    contract<NQD, NQD, NQD, 2, ND, true, NC, T>(B, A, Bf, tid);  // (NQD,NQD,ND)
    team_sync<T>();
    contract<NQD, NQD, ND, 1, ND, true, NC, T>(B, Bf, A, tid);  // (NQD,ND,ND)
    team_sync<T>();
    contract<NQD, ND, ND, 0, ND, true, NC, T>(B, A, Bf, tid);  // (ND^3)
    return Bf;
  } else {
    contract<NQD, NQD, 1, 1, ND, true, NC, T>(B, A, Bf, tid);  // (NQD, ND)
    team_sync<T>();
    contract<NQD, ND, 1, 0, ND, true, NC, T>(B, Bf, A, tid);
    return A;
  }
}

// Reference-space gradients (and optionally the interpolant) of NC nodal fields
// (tensor_grad, tensor_basis.py:248-261).
// U: NC x D1^DIM (clobbered); S: scratch >= 2*NC*Q*D1^(DIM-1);
// Tm: scratch >= 3*NC*Q*Q*D1 (3D only; may alias U when sized for it);
// out: NC x NOUT x NQ with slot k = d/dxi_k (k < DIM) and slot DIM = interpolant.
template <int DIM, int D1, int Q, int NC, int NOUT, int T>
__device__ __forceinline__ void grad(const double* B, const double* G, double* U, double* S,
                                     double* Tm, double* out, int tid) {
  constexpr int NQ = ipow(Q, DIM);
  if constexpr (DIM == 3) {
    constexpr int SX = Q * D1 * D1;   // after x stage
    constexpr int SY = Q * Q * D1;    // after y stage
    double* Sb = S;                   // B_x u   : NC x (Q, D1, D1)
    double* Sg = S + NC * SX;         // G_x u
    contract2<D1, D1, D1, 0, Q, false, NC, T>(B, G, U, Sb, Sg, tid);
    team_sync<T>();
    double* Tbb = Tm;                 // B_y B_x u
    double* Tgb = Tm + NC * SY;       // G_y B_x u
    double* Tbg = Tm + 2 * NC * SY;   // B_y G_x u
    contract2<Q, D1, D1, 1, Q, false, NC, T>(B, G, Sb, Tbb, Tgb, tid);
    contract<Q, D1, D1, 1, Q, false, NC, T>(B, Sg, Tbg, tid);
    team_sync<T>();
    // z stage: per component c, write slots of out[c][k]
    for (int w = tid; w < NC * Q * Q; w += T) {
      const int c = w / (Q * Q), l = w - c * (Q * Q);
      const double* bb = Tbb + c * SY + l;
      const double* gb = Tgb + c * SY + l;
      const double* bg = Tbg + c * SY + l;
      double xbb[D1], xgb[D1], xbg[D1];
#pragma unroll
      for (int j = 0; j < D1; ++j) {
        xbb[j] = bb[j * Q * Q];
        xgb[j] = gb[j * Q * Q];
        xbg[j] = bg[j * Q * Q];
      }
      double* o = out + c * NOUT * NQ + l;
#pragma unroll
      for (int k = 0; k < Q; ++k) {
        double d0 = 0.0, d1 = 0.0, d2 = 0.0, it = 0.0;
#pragma unroll
        for (int j = 0; j < D1; ++j) {
          const double b = B[k * D1 + j], g = G[k * D1 + j];
          d0 = fma(b, xbg[j], d0);
          d1 = fma(b, xgb[j], d1);
          d2 = fma(g, xbb[j], d2);
          if constexpr (NOUT > 3) it = fma(b, xbb[j], it);
        }
        o[k * Q * Q] = d0;
        o[NQ + k * Q * Q] = d1;
        o[2 * NQ + k * Q * Q] = d2;
        if constexpr (NOUT > 3) o[3 * NQ + k * Q * Q] = it;
      }
    }
  } else {
    constexpr int SX = Q * D1;
    double* Sb = S;
    double* Sg = S + NC * SX;
    contract2<D1, D1, 1, 0, Q, false, NC, T>(B, G, U, Sb, Sg, tid);
    team_sync<T>();
    for (int w = tid; w < NC * Q; w += T) {
      const int c = w / Q, l = w - c * Q;  // l = qx
      double xb[D1], xg[D1];
#pragma unroll
      for (int j = 0; j < D1; ++j) {
        xb[j] = Sb[c * SX + j * Q + l];
        xg[j] = Sg[c * SX + j * Q + l];
      }
      double* o = out + c * NOUT * NQ + l;
#pragma unroll
      for (int k = 0; k < Q; ++k) {
        double d0 = 0.0, d1 = 0.0, it = 0.0;
#pragma unroll
        for (int j = 0; j < D1; ++j) {
          const double b = B[k * D1 + j], g = G[k * D1 + j];
          d0 = fma(b, xg[j], d0);
          d1 = fma(g, xb[j], d1);
          if constexpr (NOUT > 2) it = fma(b, xb[j], it);
        }
        o[k * Q] = d0;
        o[NQ + k * Q] = d1;
        if constexpr (NOUT > 2) o[2 * NQ + k * Q] = it;
      }
    }
    (void)Tm;
  }
}

// Transposed gradient: out[c] = sum_l G_l^T comps[c][l]  (tensor_grad_t, tensor_basis.py:264-273)
// Cin: NC x CSTRIDE-spaced component blocks, each with DIM slots of NQ;
// Z: scratch >= 3*NC*Q*Q*D1 (3D) ; Y: scratch >= 2*NC*Q*D1^(DIM-1); out: NC x D1^DIM.
template <int DIM, int D1, int Q, int NC, int CSTRIDE, int T>
__device__ __forceinline__ void grad_t(const double* B, const double* G, const double* Cin,
                                       double* Z, double* Y, double* out, int tid) {
  constexpr int NQ = ipow(Q, DIM);
  if constexpr (DIM == 3) {
    constexpr int SY = Q * Q * D1;
    constexpr int SX = Q * D1 * D1;
    // z stage (transposed): Z0 = B^T c0, Z1 = B^T c1, Z2 = G^T c2   -> (Q,Q,D1)
    for (int w = tid; w < NC * Q * Q; w += T) {
      const int c = w / (Q * Q), l = w - c * (Q * Q);
      const double* cc = Cin + c * CSTRIDE + l;
      double x0[Q], x1[Q], x2[Q];
#pragma unroll
      for (int j = 0; j < Q; ++j) {
        x0[j] = cc[j * Q * Q];
        x1[j] = cc[NQ + j * Q * Q];
        x2[j] = cc[2 * NQ + j * Q * Q];
      }
#pragma unroll
      for (int k = 0; k < D1; ++k) {
        double a0 = 0.0, a1 = 0.0, a2 = 0.0;
#pragma unroll
        for (int j = 0; j < Q; ++j) {
          const double b = B[j * D1 + k], g = G[j * D1 + k];
          a0 = fma(b, x0[j], a0);
          a1 = fma(b, x1[j], a1);
          a2 = fma(g, x2[j], a2);
        }
        Z[c * SY + k * Q * Q + l] = a0;
        Z[NC * SY + c * SY + k * Q * Q + l] = a1;
        Z[2 * NC * SY + c * SY + k * Q * Q + l] = a2;
      }
    }
    team_sync<T>();
    // y stage: YG = B_y^T Z0 (needs G_x^T), YB = G_y^T Z1 + B_y^T Z2 (needs B_x^T)
    double* YG = Y;
    double* YB = Y + NC * SX;
    contract<Q, Q, D1, 1, D1, true, NC, T>(B, Z, YG, tid);
    contract_sum2<Q, Q, D1, 1, D1, true, NC, T>(G, Z + NC * SY, B, Z + 2 * NC * SY, YB, tid);
    team_sync<T>();
    // x stage: out = G_x^T YG + B_x^T YB
    contract_sum2<Q, D1, D1, 0, D1, true, NC, T>(G, YG, B, YB, out, tid);
  } else {
    constexpr int SY = Q * D1;  // (Q, D1): x = Q, y = D1
    // y stage: Y0 = B_y^T c0 (then G_x^T), Y1 = G_y^T c1 (then B_x^T)
    for (int w = tid; w < NC * Q; w += T) {
      const int c = w / Q, l = w - c * Q;
      const double* cc = Cin + c * CSTRIDE + l;
      double x0[Q], x1[Q];
#pragma unroll
      for (int j = 0; j < Q; ++j) {
        x0[j] = cc[j * Q];
        x1[j] = cc[NQ + j * Q];
      }
#pragma unroll
      for (int k = 0; k < D1; ++k) {
        double a0 = 0.0, a1 = 0.0;
#pragma unroll
        for (int j = 0; j < Q; ++j) {
          a0 = fma(B[j * D1 + k], x0[j], a0);
          a1 = fma(G[j * D1 + k], x1[j], a1);
        }
        Y[c * SY + k * Q + l] = a0;
        Y[NC * SY + c * SY + k * Q + l] = a1;
      }
    }
    team_sync<T>();
    contract_sum2<Q, D1, 1, 0, D1, true, NC, T>(G, Y, B, Y + NC * SY, out, tid);
    (void)Z;
  }
}

// ---------------------------------------------------------------------------
// deterministic reductions

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ long long warp_sum_ll(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_down_sync(0xffffffffu, v, o));
  return v;
}

// block-wide sum in a fixed tree; result valid in thread 0. sbuf >= 32 doubles.
template <int NT>
__device__ __forceinline__ double block_sum(double v, double* sbuf) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) sbuf[w] = v;
  __syncthreads();
  double r = 0.0;
  if (w == 0) {
    r = lane < NT / 32 ? sbuf[lane] : 0.0;
    r = warp_sum(r);
  }
  return r;
}

// "last block" detection for single-pass grid reductions.  Thread 0 of every block
// has already written the block's partial; only it fences and bumps the counter
// (a fence in every thread costs an L1 invalidation per thread).  Returns true in
// exactly one block (all its threads), after an acquire fence.
__device__ __forceinline__ bool grid_last_block(unsigned int* counter, int* sflag) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned int prev = atomicAdd(counter, 1u);
    const int last = (prev == gridDim.x - 1) ? 1 : 0;
    if (last) __threadfence();
    *sflag = last;
  }
  __syncthreads();
  return *sflag != 0;
}

// fixed-order sum of n partials by one block of NT threads; result in thread 0
template <int NT>
__device__ __forceinline__ double reduce_partials(const double* partials, int n, double* sbuf) {
  // up to 8 strided partials per thread, all loads in flight before the (ordered) adds;
  // larger grids fall back to the loop
  double acc = 0.0;
  if (n <= 8 * NT) {
    double w[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int i = threadIdx.x + c * NT;
      w[c] = i < n ? __ldcg(partials + i) : 0.0;
    }
#pragma unroll
    for (int c = 0; c < 8; ++c) acc += w[c];
  } else {
    for (int i = threadIdx.x; i < n; i += NT) acc += __ldcg(partials + i);
  }
  return block_sum<NT>(acc, sbuf);
}

// order-preserving atomicMin for non-negative doubles (+inf allowed)
__device__ __forceinline__ void atomic_min_nonneg(double* addr, double v) {
  if (!(v >= 0.0)) return;  // NaN / negative never win (inverted stages are discarded)
  atomicMin(reinterpret_cast<unsigned long long*>(addr), __double_as_longlong(v));
}

}  // namespace hx
