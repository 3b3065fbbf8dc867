// hx_brick.cuh -- structured-brick fast path of the momentum CG (3D).
//
// When the dofmap is the lexicographic numbering of cartesian_mesh
// (fespace.py:352-385; node (i,j,k) = i + Nx (j + Ny k), element
// (ex,ey,ez) = ex + nx (ey + ny ez), local node (dx,dy,dz) x fastest) the
// restriction needs no index arrays: every E-vector position is arithmetic.
//   * E-vectors are stored ELEMENT-MAJOR (NE, nl, NC): the mass kernel writes each
//     element's block with coalesced stores instead of scattered slot writes.
//   * The node pass computes, for node (i,j,k), the (element, local) pairs that
//     touch it (1, 2, 4 or 8) in ascending element order and sums them from 0.0 --
//     the same sequential order as np.add.at over dofmap.T (fespace.py:227-234),
//     so the scatter stays bit-identical to the reference.
//   * The mass kernel loads each element's node rows (D1 nodes x NC components of
//     16-byte (z, p) pairs, contiguous) cooperatively into shared memory.
// The math per element is that of k_mass_pc (MassPA._apply_scalar operators.py:97-115).
#pragma once

#include "hx_kernels.cuh"

namespace hx {

// n / d for 0 <= n < 2^31 by multiply-high (d >= 1 fixed at setup)
struct FastDiv {
  unsigned d, m, s;
  __host__ __device__ __forceinline__ unsigned div(unsigned n) const {
#ifdef __CUDA_ARCH__
    return (__umulhi(n, m) + n) >> s;
#else
    return n / d;
#endif
  }
};

static inline FastDiv make_fastdiv(unsigned d) {
  unsigned s = 0;
  while ((1ull << s) < d) ++s;
  const unsigned long long m = ((1ull << 32) * ((1ull << s) - d)) / d + 1;
  return FastDiv{d, (unsigned)m, s};
}

struct Brick {
  int nx, ny, nz;  // elements per direction
  int Nx, Ny;      // nodes per direction (p*n + 1)
  long long NxNy;
  FastDiv fnx, fnxy, fNx, fNxNy;  // element / node coordinate splits
  int dX, dY, dZ;                 // element-major E offsets (in entries / NC) between the
                                  // lower and upper element of a shared node along x, y, z
};

// node coordinate i along an axis with n elements of order P: first (lowest) element
// coordinate e0, its local coordinate l0, and whether the next element shares the node
template <int P>
__device__ __forceinline__ void axis_first(int i, int n, int& e0, int& l0, int& two) {
  const int q = i / P, r = i - q * P;
  const bool face = (r == 0) && (q > 0);
  e0 = face ? q - 1 : q;
  l0 = face ? P : r;
  two = face && (q < n);
}

#ifndef NODE_ELD
#define NODE_ELD __ldg  // E-vector loads of the node pass: read-only path (598.8/600.4 vs 593.7/598.7 with __ldcg)
#endif
// deterministic node sum of an element-major E-vector (NE, nl, NC): ascending element
// order from 0.0, all (up to 8) loads issued before the adds
template <int P, int NC>
struct BrickSum {
  const double* E;
  Brick b;
  __device__ __forceinline__ double operator()(long long n, int c) const {
    constexpr int D1 = P + 1, NL = D1 * D1 * D1;
    const unsigned k = b.fNxNy.div((unsigned)n);
    const unsigned rem = (unsigned)n - k * (unsigned)b.NxNy;
    const unsigned j = b.fNx.div(rem);
    const int i = (int)(rem - j * (unsigned)b.Nx);
    int ex, lx, tx, ey, ly, ty, ez, lz, tz;
    axis_first<P>(i, b.nx, ex, lx, tx);
    axis_first<P>((int)j, b.ny, ey, ly, ty);
    axis_first<P>((int)k, b.nz, ez, lz, tz);
    const unsigned p0 = ((unsigned)((ez * b.ny + ey) * b.nx + ex) * NL + (lz * D1 + ly) * D1 + lx) * NC + c;
    double v[8];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int bb = 0; bb < 2; ++bb)
#pragma unroll
        for (int g = 0; g < 2; ++g) {
          const bool ok = a <= tz && bb <= ty && g <= tx;
          const unsigned pos = p0 + (unsigned)((a * b.dZ + bb * b.dY + g * b.dX) * NC);
          v[(a * 2 + bb) * 2 + g] = ok ? NODE_ELD(E + pos) : 0.0;
        }
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) s += v[q];  // absent entries are +0.0: sums unchanged
    return s;
  }
  // make the node's sum equal `total` (multi-GPU halo): the lowest element's entry takes
  // the total, the others become +0.0, so operator() returns exactly `total` afterwards
  __device__ __forceinline__ void patch(long long n, int c, double total) const {
    constexpr int D1 = P + 1, NL = D1 * D1 * D1;
    const unsigned k = b.fNxNy.div((unsigned)n);
    const unsigned rem = (unsigned)n - k * (unsigned)b.NxNy;
    const unsigned j = b.fNx.div(rem);
    const int i = (int)(rem - j * (unsigned)b.Nx);
    int ex, lx, tx, ey, ly, ty, ez, lz, tz;
    axis_first<P>(i, b.nx, ex, lx, tx);
    axis_first<P>((int)j, b.ny, ey, ly, ty);
    axis_first<P>((int)k, b.nz, ez, lz, tz);
    const unsigned p0 = ((unsigned)((ez * b.ny + ey) * b.nx + ex) * NL + (lz * D1 + ly) * D1 + lx) * NC + c;
    double* W = const_cast<double*>(E);
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int bb = 0; bb < 2; ++bb)
#pragma unroll
        for (int g = 0; g < 2; ++g)
          if (a <= tz && bb <= ty && g <= tx)
            W[p0 + (unsigned)((a * b.dZ + bb * b.dY + g * b.dX) * NC)] = (a | bb | g) ? 0.0 : total;
  }
};

__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async16d(double* dst, const double* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
// contiguous span of n doubles (dst 16-byte aligned): 16-byte copies when src allows
template <int NT>
__device__ __forceinline__ void cp_span(double* dst, const double* src, int n, int t) {
  if ((reinterpret_cast<unsigned long long>(src) & 15ull) == 0) {
    for (int i = t; i < n / 2; i += NT) cp_async16d(dst + 2 * i, src + 2 * i);
    if ((n & 1) && t == 0) cp_async8(dst + n - 1, src + n - 1);
  } else {
    for (int i = t; i < n; i += NT) cp_async8(dst + i, src + i);
  }
}

// generic (CSR, node-sorted E-vector) node sum as a functor
template <int NC>
struct CsrSum {
  const int* off;
  const double* E;
  __device__ __forceinline__ double operator()(long long n, int c) const { return node_sum1<NC>(off, E, n, c); }
  __device__ __forceinline__ void patch(long long n, int c, double total) const {
    double* W = const_cast<double*>(E);
    const int b = off[n], f = off[n + 1];
    for (int k = b; k < f; ++k) W[(long long)k * NC + c] = k == b ? total : 0.0;
  }
};

// ---------------------------------------------------------------------------
// CG mass action on a brick: p_k = z + beta p_{k-1} (pairs), y_e = B^T D B p_e,
// element-major E out, element-wise p.Ap partial -> alpha (last block).
// (Masked components of p are exactly 0 in this CG -- r, z start at 0 there and
// Ap := p keeps them 0 -- so p.Ap needs no wall term and p no mask.)

#ifndef MASS_BRICK_NT
#define MASS_BRICK_NT 128
#endif
#ifndef MASS_ALIAS
#define MASS_ALIAS 1
#endif
#ifndef MASS_ALIAS_PMIN
#define MASS_ALIAS_PMIN 3
#endif
#ifndef MASS_LD
#define MASS_LD __ldcg
#endif
#ifndef MASS_CMAJOR
#define MASS_CMAJOR 0
#endif
#ifndef MASS_P3COL
#define MASS_P3COL 0
#endif
#ifndef MASS_EBREG
#define MASS_EBREG 1  // measured 603 vs 592 Mdof*steps/s (mass 24.3 vs 25.6 us)
#endif
#ifndef MASS_DPF
#define MASS_DPF 0
#endif
#ifndef MASS_BAT
#define MASS_BAT 0
#endif
#ifndef MASS_BRICK_MINB
#define MASS_BRICK_MINB 5
#endif
template <int P, int NC>
struct MassBrickCfg {
  static constexpr int NT = MASS_BRICK_NT;   // threads per CTA
  static constexpr int D1 = P + 1, Q = P + 2, QQ = Q * Q, DD = D1 * D1, NL = D1 * DD, NQ = Q * QQ;
  static constexpr int PLN = NC * D1;          // planes per element
  static constexpr int EPC = NT / PLN;         // elements per pass
  // MASS_ALIAS (p >= 3, measured faster; p = 2 keeps separate images): the gather /
  // staging planes live inside the T planes -- each plane thread reads its own plane into
  // registers before it overwrites it (phases 1 and 3), so one image suffices
  static constexpr bool ALIAS = MASS_ALIAS && P >= MASS_ALIAS_PMIN;
  static constexpr int GP = ALIAS ? QQ : DD + 1;  // plane pitch of the gather / staging image
  static constexpr int GS = PLN * GP;             // gather doubles per element
  static constexpr int TS = PLN * QQ;             // T image doubles per element
  static constexpr size_t bytes = sizeof(double) * (size_t)EPC * ((ALIAS ? 0 : GS) + TS + (MASS_DPF ? NQ : 0));
};

struct MassBrickArgs {
  const double* pbuf0;  // interleaved (z, p) pairs, ping-pong (iteration k reads pbuf[(k-1)&1])
  const double* pbuf1;
  const double* D;      // (NE, nq)
  long long ne;
  double* evec;         // (NE, nl, NC) element-major, or node-sorted when slot is set
  const int* slot;      // null: element-major E; else node-sorted position of (e, l)
  CGDev* cg;
  double* partials;
  Brick b;
  PeerLite pl;          // multi-GPU prologue exchange (k_mass_brick<..., true>)
};

template <int P, int NC, bool PEER = false>
__global__ void __launch_bounds__(MASS_BRICK_NT, (P >= 4 ? 4 : MASS_BRICK_MINB) * 128 / MASS_BRICK_NT) k_mass_brick(MassBrickArgs a) {
  using M = MassBrickCfg<P, NC>;
  constexpr int D1 = M::D1, Q = M::Q, QQ = M::QQ, DD = M::DD, NL = M::NL, NQ = M::NQ;
  constexpr int PLN = M::PLN, EPC = M::EPC, GP = M::GP, GS = M::GS;
  const double* cB = c_B[P - 1];
  extern __shared__ __align__(16) double smem[];
  double* sG = smem;                 // gather image [el][c][dz][dy*D1+dx] (pitch GP); reused as staging
  double* sT = M::ALIAS ? smem : smem + EPC * GS;  // T image [el][c][dz][qy*Q+qx]
#if MASS_DPF
  double* sD = smem + EPC * (M::TS + (M::ALIAS ? 0 : GS));  // D of the pass (cp.async at pass start)
#endif
  __shared__ double red[32];
  double beta;
  int k;
  if (!cg_mass_begin<M::NT, PEER>(a.cg, red, beta, k, &a.pl)) return;
  const int t = threadIdx.x;
  const double* po = (k & 1) ? a.pbuf0 : a.pbuf1;
  double acc = 0.0;
  const int pe = t / PLN, pr = t - pe * PLN;
  __shared__ int sbase[EPC];  // first node of each element of the pass
  // per-thread gather / copy-out slots within an element (pass invariant)
  constexpr int ROWI = D1 * NC;                 // pairs per node row
  constexpr int ELI = DD * ROWI;                // pairs (= E entries) per element
  constexpr int SLOTS = (ELI + M::NT - 1) / M::NT;
  int soff[SLOTS], goff[SLOTS], eoff[SLOTS];
#pragma unroll
  for (int h = 0; h < SLOTS; ++h) {
    const int it = h * M::NT + t;
    const int row = it / ROWI, s = it - row * ROWI;  // row = dz*D1 + dy
#if MASS_CMAJOR
    // component-major within a node row: the 4 nodes of one component are consecutive
    // lanes (conflict-free shared stores / loads of a row); same 192-byte row in memory
    const int c = s / D1, dx = s - c * D1;
#else
    const int dx = s / NC, c = s - dx * NC;
#endif
    const int dz = row / D1, dy = row - dz * D1;
    soff[h] = (c * D1 + dz) * GP + dy * D1 + dx;
    goff[h] = (dx + dy * a.b.Nx + dz * (int)a.b.NxNy) * NC + c;
    eoff[h] = (row * D1 + dx) * NC + c;  // E entry (l, c) at l*NC + c
  }
  // balanced contiguous element range per CTA, walked in passes of up to EPC elements
  // (all CTAs finish within one pass of each other)
  const int ebeg = (int)(a.ne * blockIdx.x / gridDim.x);
  const int len = (int)(a.ne * (blockIdx.x + 1) / gridDim.x) - ebeg;
  const int npass = (len + EPC - 1) / EPC;
  for (int ps = 0; ps < npass; ++ps) {
    const int e0 = ebeg + len * ps / npass;
    const int nel = ebeg + len * (ps + 1) / npass - e0;
#if MASS_DPF
    // D of the pass lands in shared memory while the gather and phase 1 run
    cp_span<M::NT>(sD, a.D + (long long)e0 * NQ, nel * NQ, t);
    asm volatile("cp.async.commit_group;" ::: "memory");
#endif
#if MASS_EBREG
    // the pass's element base nodes (x NC) in registers, stepped along the element row
    // (no shared-memory table, no barrier): consecutive elements are P nodes apart except
    // where the row (or the layer) wraps
    int eb[EPC];
    {
      const unsigned e = (unsigned)e0;
      const unsigned ez = a.b.fnxy.div(e);
      const unsigned r2 = e - ez * (unsigned)(a.b.nx * a.b.ny);
      int ey = (int)a.b.fnx.div(r2), ex = (int)(r2 - (unsigned)ey * (unsigned)a.b.nx);
      int base = (ex * P + (ey * P) * a.b.Nx + ((int)ez * P) * (int)a.b.NxNy) * NC;
#pragma unroll
      for (int u = 0; u < EPC; ++u) {
        eb[u] = base;
        base += P * NC;
        if (++ex == a.b.nx) {
          ex = 0;
          base += (P * a.b.Nx - a.b.nx * P) * NC;
          if (++ey == a.b.ny) {
            ey = 0;
            base += (P * (int)a.b.NxNy - a.b.ny * P * a.b.Nx) * NC;
          }
        }
      }
    }
#define HX_EBASE(u) eb[u]
#else
    if (t < nel) {
      const unsigned e = (unsigned)(e0 + t);
      const unsigned ez = a.b.fnxy.div(e);
      const unsigned r2 = e - ez * (unsigned)(a.b.nx * a.b.ny);
      const unsigned ey = a.b.fnx.div(r2), ex = r2 - ey * (unsigned)a.b.nx;
      sbase[t] = (int)(ex * P + (ey * P) * (unsigned)a.b.Nx + (ez * P) * (unsigned)a.b.NxNy);
    }
    __syncthreads();
#define HX_EBASE(u) (sbase[u] * NC)
#endif
    // ---- phase 0: node rows (D1 nodes x NC pairs, contiguous) -> p image.  Thread t
    // owns the same (row, pair) slots of every element of the pass (offsets hoisted
    // out of the pass loop); all loads of a slot are issued before the first use.
#if MASS_BAT
    {
      // every (slot, element) load of the thread in flight together, BAT at a time
      constexpr int TOT = SLOTS * EPC, BAT = MASS_BAT < TOT ? MASS_BAT : TOT;
#pragma unroll
      for (int b0 = 0; b0 < TOT; b0 += BAT) {
        double2 q[BAT];
#pragma unroll
        for (int u = 0; u < BAT; ++u) {
          const int h = (b0 + u) / EPC, el = (b0 + u) - h * EPC;
          if (b0 + u < TOT && h * M::NT + t < ELI && el < nel)
            q[u] = __ldcg(reinterpret_cast<const double2*>(po) + (sbase[el] * NC + goff[h]));
        }
#pragma unroll
        for (int u = 0; u < BAT; ++u) {
          const int h = (b0 + u) / EPC, el = (b0 + u) - h * EPC;
          if (b0 + u < TOT && h * M::NT + t < ELI && el < nel)
            sG[el * GS + soff[h]] = __dadd_rn(q[u].x, __dmul_rn(beta, q[u].y));
        }
      }
    }
#else
#pragma unroll
    for (int h = 0; h < SLOTS; ++h) {
      if (h * M::NT + t < ELI) {
        constexpr int BAT = EPC < 6 ? EPC : 6;
#pragma unroll
        for (int e1 = 0; e1 < EPC; e1 += BAT) {
          double2 q[BAT];
#pragma unroll
          for (int u = 0; u < BAT; ++u)
            if (e1 + u < nel)
              q[u] = MASS_LD(reinterpret_cast<const double2*>(po) + (HX_EBASE(e1 + u) + goff[h]));
#pragma unroll
          for (int u = 0; u < BAT; ++u)
            if (e1 + u < nel) sG[(e1 + u) * GS + soff[h]] = __dadd_rn(q[u].x, __dmul_rn(beta, q[u].y));
        }
      }
    }
#endif
#undef HX_EBASE
    __syncthreads();
    // ---- phase 1 (planes): x and y contractions in registers -> T
    const bool pact = pe < nel;
    if (pact) {
      double u[DD];
      const double* g = sG + pe * GS + pr * GP;
#pragma unroll
      for (int k = 0; k < DD; ++k) u[k] = g[k];
      double v[D1][Q];
#pragma unroll
      for (int dy = 0; dy < D1; ++dy)
#pragma unroll
        for (int qx = 0; qx < Q; ++qx) {
          double s = 0.0;
#pragma unroll
          for (int dx = 0; dx < D1; ++dx) s = fma(cB[qx * D1 + dx], u[dy * D1 + dx], s);
          v[dy][qx] = s;
        }
      double* T = sT + pe * M::TS + pr * QQ;
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
#if MASS_DPF
    asm volatile("cp.async.wait_group 0;" ::: "memory");
#endif
    __syncthreads();
    // ---- phase 2 (columns): z, D, z^T for all components of a (qx, qy) column
    for (int it = t; it < nel * QQ; it += M::NT) {
      const int ce = it / QQ, l = it - ce * QQ;
      const long long ee = e0 + ce;
      double Dq[Q];
#pragma unroll
      for (int qz = 0; qz < Q; ++qz)
#if MASS_DPF
        Dq[qz] = sD[ce * NQ + qz * QQ + l];
#else
        Dq[qz] = __ldg(a.D + ee * NQ + qz * QQ + l);
#endif
      double* base = sT + ce * M::TS + l;
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
          acc = fma(du, s, acc);
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
    // ---- phase 3 (planes): y^T, x^T -> staging image (same layout as the gather image)
#if MASS_P3COL
    // column by column (qx): y^T of the column, then its x^T contribution accumulated into the
    // 16 outputs -- the same ascending sums as below (so bit-identical), with 25 instead of 45
    // doubles live
    if (pact) {
      const double* T = sT + pe * M::TS + pr * QQ;
      double o3[D1][D1];
#pragma unroll
      for (int dy = 0; dy < D1; ++dy)
#pragma unroll
        for (int dx = 0; dx < D1; ++dx) o3[dy][dx] = 0.0;
#pragma unroll
      for (int qx = 0; qx < Q; ++qx) {
        double tq[Q];
#pragma unroll
        for (int qy = 0; qy < Q; ++qy) tq[qy] = T[qy * Q + qx];
#pragma unroll
        for (int dy = 0; dy < D1; ++dy) {
          double v = 0.0;
#pragma unroll
          for (int qy = 0; qy < Q; ++qy) v = fma(cB[qy * D1 + dy], tq[qy], v);
#pragma unroll
          for (int dx = 0; dx < D1; ++dx) o3[dy][dx] = fma(cB[qx * D1 + dx], v, o3[dy][dx]);
        }
      }
      double* o = sG + pe * GS + pr * GP;
#pragma unroll
      for (int dy = 0; dy < D1; ++dy)
#pragma unroll
        for (int dx = 0; dx < D1; ++dx) o[dy * D1 + dx] = o3[dy][dx];
    }
    if (false)
#endif
    if (pact) {
      const double* T = sT + pe * M::TS + pr * QQ;
      double Tq[QQ];
#pragma unroll
      for (int k = 0; k < QQ; ++k) Tq[k] = T[k];
      double v[D1][Q];
#pragma unroll
      for (int dy = 0; dy < D1; ++dy)
#pragma unroll
        for (int qx = 0; qx < Q; ++qx) {
          double s = 0.0;
#pragma unroll
          for (int qy = 0; qy < Q; ++qy) s = fma(cB[qy * D1 + dy], Tq[qy * Q + qx], s);
          v[dy][qx] = s;
        }
      double* o = sG + pe * GS + pr * GP;
#pragma unroll
      for (int dy = 0; dy < D1; ++dy)
#pragma unroll
        for (int dx = 0; dx < D1; ++dx) {
          double s = 0.0;
#pragma unroll
          for (int qx = 0; qx < Q; ++qx) s = fma(cB[qx * D1 + dx], v[dy][qx], s);
          o[dy * D1 + dx] = s;
        }
    }
    __syncthreads();
    // ---- phase 4: copy-out of the pass: element-major (contiguous) or node-sorted
    // through the slot map (read contiguously, scattered 8-byte stores)
    if (a.slot) {
      const int* sl = a.slot + e0 * NL;
      for (int it = t; it < nel * NL; it += M::NT) {
        const int el = it / NL, l = it - el * NL;
        const int dz = l / DD, k = l - dz * DD;
        const long long pos = (long long)__ldg(sl + it) * NC;
#pragma unroll
        for (int c = 0; c < NC; ++c) __stcg(a.evec + pos + c, sG[el * GS + (c * D1 + dz) * GP + k]);
      }
    } else {
      // E entry (l, c) of an element sits at l*NC + c = (row*D1 + dx)*NC + c: the same
      // slot enumeration as the gather, so soff maps it to the staging image
      double* out = a.evec + e0 * (NL * NC);
#pragma unroll
      for (int h = 0; h < SLOTS; ++h) {
        const int it = h * M::NT + t;
        if (it < ELI) {
#pragma unroll
          for (int el = 0; el < EPC; ++el)
            if (el < nel) __stcg(out + el * ELI + eoff[h], sG[el * GS + soff[h]]);
        }
      }
    }
    __syncthreads();
  }
  cg_partial(a.partials, &a.cg->nparts_m, block_sum<M::NT>(acc, red));
  if constexpr (PEER) {  // a rank without neighbours posts p.Ap_k here (else the halo pack does)
    if ((a.pl.post & (PEER_POST_ON | PEER_POST_MASS)) == (PEER_POST_ON | PEER_POST_MASS))
      cg_post_last<M::NT>(a.pl, a.partials, gridDim.x, &a.cg->cnt[3], a.cg->seq0 + 2ull * k, red);
  }
}


// ---------------------------------------------------------------------------
// Pipelined variant (MASS_PIPE): the (z, p) pairs of a pass are staged raw into a
// separate shared pair image with cp.async (16-byte copies, no registers), one pass
// ahead: pass 0's copies are issued before the CG prologue (the r.z reduction and stop
// test of cg_mass_begin) and pass s+1's as soon as phase 1 of pass s has consumed the
// image, so the gather latency hides behind the prologue and phases 2-4.  Phase 1 forms
// p_k = z + beta p_{k-1} from the pair image.  The staging image aliases the T planes
// (each plane thread reads its own plane into registers before overwriting it).
#ifndef MASS_PIPE_NT
#define MASS_PIPE_NT 128
#endif
#ifndef MASS_PIPE_MINB
#define MASS_PIPE_MINB 4
#endif
#ifndef MASS_PIPE_D
#define MASS_PIPE_D 0
#endif
template <int P, int NC>
struct MassPipeCfg {
  static constexpr int NT = MASS_PIPE_NT;
  static constexpr int D1 = P + 1, Q = P + 2, QQ = Q * Q, DD = D1 * D1, NL = D1 * DD, NQ = Q * QQ;
  static constexpr int PLN = NC * D1;          // planes per element
  static constexpr int EPC = NT / PLN;         // elements per pass
  static constexpr int ROWI = D1 * NC;         // pairs per node row
  static constexpr int ELI = DD * ROWI;        // pairs per element (= E entries)
  static constexpr int GP = QQ, GS = PLN * GP; // staging (in the T planes)
  static constexpr int TS = PLN * QQ;
  // pair image padding (in pairs): phase 1's 16-byte reads of 8 consecutive plane lanes
  // (c, dz) hit distinct 16-byte bank groups when the dz stride is = ZM (mod 8) and the
  // element stride = 1 (mod 8)
  static constexpr int ZM = P == 2 ? 3 : (P == 3 ? 2 : 5);
  static constexpr int up8(int v, int m) { return v + (((m - v) % 8) + 8) % 8; }
  static constexpr int ZS = up8(D1 * ROWI, ZM);
  static constexpr int ELIP = up8(D1 * ZS, 1);
  static constexpr int DS = MASS_PIPE_D ? NQ : 0;  // D of the pass staged too
  static constexpr size_t bytes = sizeof(double) * ((size_t)EPC * (TS + 2 * ELIP) + (size_t)EPC * DS);
};

template <int P, int NC, bool PEER = false>
__global__ void __launch_bounds__(MASS_PIPE_NT, MASS_PIPE_MINB * 128 / MASS_PIPE_NT) k_mass_brick2(MassBrickArgs a) {
  using M = MassPipeCfg<P, NC>;
  constexpr int D1 = M::D1, Q = M::Q, QQ = M::QQ, DD = M::DD, NL = M::NL, NQ = M::NQ;
  constexpr int PLN = M::PLN, EPC = M::EPC, GP = M::GP, GS = M::GS, ROWI = M::ROWI, ELI = M::ELI;
  constexpr int ZS = M::ZS, ELIP = M::ELIP;
  constexpr int SLOTS = (ELI + M::NT - 1) / M::NT;
  const double* cB = c_B[P - 1];
  extern __shared__ __align__(16) double smem[];
  double* sT = smem;                                          // T image [el][c][dz][qy*Q+qx]
  double* sG = smem;                                          // staging (aliases T)
  double2* sP = reinterpret_cast<double2*>(smem + EPC * M::TS);  // pair image [el][dz][dy][dx][c]
#if MASS_PIPE_D
  double* sD = smem + EPC * (M::TS + 2 * ELIP);                     // D of the pass
#endif
  __shared__ double red[32];
  CGDev* g = a.cg;
  if (!g->active) return;
  const int t = threadIdx.x;
  const int k0 = g->it_m;
  const double2* po = reinterpret_cast<const double2*>((k0 & 1) ? a.pbuf0 : a.pbuf1);
  // per-thread slots (pass invariant): global pair offset from the element's first node,
  // and the element-major E offset of the same slot
  int goff[SLOTS], eoff[SLOTS], poff[SLOTS], soff[SLOTS];
#pragma unroll
  for (int h = 0; h < SLOTS; ++h) {
    const int it = h * M::NT + t;
    const int row = it / ROWI, s = it - row * ROWI;  // row = dz*D1 + dy
    const int dx = s / NC, c = s - dx * NC;
    const int dz = row / D1, dy = row - dz * D1;
    goff[h] = (dx + dy * a.b.Nx + dz * (int)a.b.NxNy) * NC + c;
    eoff[h] = (row * D1 + dx) * NC + c;
    poff[h] = dz * ZS + dy * ROWI + s;
    soff[h] = (c * D1 + dz) * GP + dy * D1 + dx;
  }
  const int ebeg = (int)(a.ne * blockIdx.x / gridDim.x);
  const int len = (int)(a.ne * (blockIdx.x + 1) / gridDim.x) - ebeg;
  const int npass = (len + EPC - 1) / EPC;
  auto pass_range = [&](int ps, int& e0, int& nel) {
    e0 = ebeg + len * ps / npass;
    nel = ebeg + len * (ps + 1) / npass - e0;
  };
  auto element_base = [&](unsigned e) {
    const unsigned ez = a.b.fnxy.div(e);
    const unsigned r2 = e - ez * (unsigned)(a.b.nx * a.b.ny);
    const unsigned ey = a.b.fnx.div(r2), ex = r2 - ey * (unsigned)a.b.nx;
    return (int)(ex * P + (ey * P) * (unsigned)a.b.Nx + (ez * P) * (unsigned)a.b.NxNy);
  };
  // cp.async of a pass's pairs (element bases computed per (slot, element): no barrier)
  auto issue = [&](int ps) {
    int e0, nel;
    pass_range(ps, e0, nel);
    for (int el = 0; el < nel; ++el) {
      const int base = element_base((unsigned)(e0 + el));
#pragma unroll
      for (int h = 0; h < SLOTS; ++h) {
        const int it = h * M::NT + t;
        if (it < ELI)
          cp_async16d(reinterpret_cast<double*>(sP + el * ELIP + poff[h]),
                      reinterpret_cast<const double*>(po + (base * NC + goff[h])));
      }
    }
#if MASS_PIPE_D
    cp_span<M::NT>(sD, a.D + (long long)e0 * NQ, nel * NQ, t);
#endif
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  if (npass > 0) issue(0);
  double beta;
  int k;
  if (!cg_mass_begin<M::NT, PEER>(g, red, beta, k, &a.pl)) {
    asm volatile("cp.async.wait_all;" ::: "memory");
    return;
  }
  double acc = 0.0;
  const int pe = t / PLN, pr = t - pe * PLN;
  const int pc = pr / D1, pz = pr - pc * D1;  // plane (c, dz)
  for (int ps = 0; ps < npass; ++ps) {
    int e0, nel;
    pass_range(ps, e0, nel);
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    // ---- phase 1 (planes): p = z + beta p_{k-1} from the pair image; x, y contractions
    const bool pact = pe < nel;
    if (pact) {
      double u[DD];
      const double2* pp = sP + pe * ELIP + pz * ZS + pc;
#pragma unroll
      for (int dy = 0; dy < D1; ++dy)
#pragma unroll
        for (int dx = 0; dx < D1; ++dx) {
          const double2 q = pp[dy * ROWI + dx * NC];
          u[dy * D1 + dx] = __dadd_rn(q.x, __dmul_rn(beta, q.y));
        }
      double v[D1][Q];
#pragma unroll
      for (int dy = 0; dy < D1; ++dy)
#pragma unroll
        for (int qx = 0; qx < Q; ++qx) {
          double s = 0.0;
#pragma unroll
          for (int dx = 0; dx < D1; ++dx) s = fma(cB[qx * D1 + dx], u[dy * D1 + dx], s);
          v[dy][qx] = s;
        }
      double* T = sT + pe * M::TS + pr * QQ;
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
#if !MASS_PIPE_D
    if (ps + 1 < npass) issue(ps + 1);  // the pair image is dead until the next pass
#endif
    // ---- phase 2 (columns): z, D, z^T for all components of a (qx, qy) column
    for (int it = t; it < nel * QQ; it += M::NT) {
      const int ce = it / QQ, l = it - ce * QQ;
      double Dq[Q];
#pragma unroll
      for (int qz = 0; qz < Q; ++qz)
#if MASS_PIPE_D
        Dq[qz] = sD[ce * NQ + qz * QQ + l];
#else
        Dq[qz] = __ldg(a.D + (long long)(e0 + ce) * NQ + qz * QQ + l);
#endif
      double* base = sT + ce * M::TS + l;
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
          acc = fma(du, s, acc);
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
#if MASS_PIPE_D
    if (ps + 1 < npass) issue(ps + 1);  // pair image and D of this pass are dead
#endif
    // ---- phase 3 (planes): y^T, x^T -> staging (own T plane, read into registers first)
    if (pact) {
      const double* T = sT + pe * M::TS + pr * QQ;
      double Tq[QQ];
#pragma unroll
      for (int kk = 0; kk < QQ; ++kk) Tq[kk] = T[kk];
      double v[D1][Q];
#pragma unroll
      for (int dy = 0; dy < D1; ++dy)
#pragma unroll
        for (int qx = 0; qx < Q; ++qx) {
          double s = 0.0;
#pragma unroll
          for (int qy = 0; qy < Q; ++qy) s = fma(cB[qy * D1 + dy], Tq[qy * Q + qx], s);
          v[dy][qx] = s;
        }
      double* o = sG + pe * GS + pr * GP;
#pragma unroll
      for (int dy = 0; dy < D1; ++dy)
#pragma unroll
        for (int dx = 0; dx < D1; ++dx) {
          double s = 0.0;
#pragma unroll
          for (int qx = 0; qx < Q; ++qx) s = fma(cB[qx * D1 + dx], v[dy][qx], s);
          o[dy * D1 + dx] = s;
        }
    }
    __syncthreads();
    // ---- phase 4: copy-out (element-major, or node-sorted through the slot map)
    if (a.slot) {
      const int* sl = a.slot + e0 * NL;
      for (int it = t; it < nel * NL; it += M::NT) {
        const int el = it / NL, l = it - el * NL;
        const int dz = l / DD, kk = l - dz * DD;
        const long long pos = (long long)__ldg(sl + it) * NC;
#pragma unroll
        for (int c = 0; c < NC; ++c) __stcg(a.evec + pos + c, sG[el * GS + (c * D1 + dz) * GP + kk]);
      }
    } else {
      double* out = a.evec + e0 * (NL * NC);
#pragma unroll
      for (int h = 0; h < SLOTS; ++h) {
        const int it = h * M::NT + t;
        if (it < ELI) {
#pragma unroll
          for (int el = 0; el < EPC; ++el)
            if (el < nel) __stcg(out + el * ELI + eoff[h], sG[el * GS + soff[h]]);
        }
      }
    }
  }
  cg_partial(a.partials, &g->nparts_m, block_sum<M::NT>(acc, red));
}

}  // namespace hx
