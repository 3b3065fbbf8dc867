// hx_tma.cuh -- TMA-staged CG mass action on a structured brick (3D, NC = 3).
//
// MassPA._apply_scalar (operators.py:97-115) inside cg_solve (operators.py:352-353),
// one launch per CG iteration like k_mass_brick, with every data movement of the
// element pass done by the copy engines instead of the threads:
//   * the pass is a run of up to EPC consecutive elements of one element row (fixed
//     ey, ez); its node box -- (EPC*P + 1) x (P+1) x (P+1) nodes of interleaved (z, p)
//     pairs -- is ONE 3D TMA tile load (cp.async.bulk.tensor, tensor map over the pair
//     array viewed as (Nx*NC*2, Ny, Nz) doubles).  Shared nodes of neighbouring
//     elements are fetched once; nothing is address-computed per node;
//   * the pass's D (point data, contiguous per element run) is a 1D bulk copy on the
//     same mbarrier;
//   * the element-major E block of the pass (contiguous) leaves shared memory as one
//     bulk store (cp.async.bulk.global.shared::cta);
//   * the next pass's box and D are issued as soon as phase 1 has consumed the box, so
//     the loads land while phases 2-3 of this pass run.
// The arithmetic per element (contraction order, p_k = z + beta p_{k-1} rounding, the
// p.Ap accumulation) is exactly k_mass_brick's, so E is bit-identical to it.
#pragma once

#include <cuda.h>  // CUtensorMap (type only; the encoder is fetched from the runtime)

#include "hx_async.cuh"
#include "hx_brick.cuh"

namespace hx {

#ifndef MASS_TMA_EPC3
#define MASS_TMA_EPC3 8
#endif
#ifndef MASS_TMA_NT3
#define MASS_TMA_NT3 128
#endif
#ifndef MASS_TMA_MINB3
#define MASS_TMA_MINB3 4
#endif
// per-order pass shape: EPC elements per pass, NT threads (>= NC*(P+1)*EPC planes)
template <int P>
struct MassTmaShape;
template <>
struct MassTmaShape<2> {
  static constexpr int EPC = 12, NT = 128, MINB = 5;
};
template <>
struct MassTmaShape<3> {
  static constexpr int EPC = MASS_TMA_EPC3, NT = MASS_TMA_NT3, MINB = MASS_TMA_MINB3;
};
template <>
struct MassTmaShape<4> {
  static constexpr int EPC = 4, NT = 96, MINB = 3;
};

template <int P, int NC>
struct MassTmaCfg {
  static constexpr int EPC = MassTmaShape<P>::EPC, NT = MassTmaShape<P>::NT, MINB = MassTmaShape<P>::MINB;
  static constexpr int D1 = P + 1, Q = P + 2, QQ = Q * Q, DD = D1 * D1, NL = D1 * DD, NQ = Q * QQ;
  static constexpr int PLN = NC * D1;         // planes (c, dz) per element
  static_assert(PLN * EPC <= NT, "one thread per plane");
  static constexpr int BX = EPC * P + 1;      // box nodes along x
  static constexpr int ROWD = BX * NC * 2;    // doubles per box node row (pairs)
  static constexpr int BOXD = ROWD * DD;      // box doubles
  static_assert(ROWD <= 256, "TMA box dimension");
  static constexpr int up16(int v) { return (v + 15) & ~15; }  // 128-byte multiples
  static constexpr int DSD = up16(EPC * NQ + 2);                // D buffer (1 double alignment slack)
  static constexpr int TS = PLN * QQ;         // T image doubles per element
  static constexpr int ELI = NL * NC;         // E entries per element
  static_assert(ELI <= TS, "E staging aliases the T image");
  static constexpr int OFF_D = up16(BOXD), OFF_T = OFF_D + 2 * DSD, OFF_BAR = OFF_T + up16(EPC * TS);
  // + 128 B: the kernel aligns the dynamic region to 128 bytes (TMA tile destination)
  static constexpr size_t bytes = sizeof(double) * (size_t)OFF_BAR + 2 * sizeof(unsigned long long) + 128;
  static constexpr unsigned BOX_BYTES = sizeof(double) * BOXD;
  // an element's E block is a whole number of 16-byte units (p = 3: 1536 B) -> one bulk
  // store per pass; otherwise (p = 2: 648 B, p = 4: 3000 B) the threads copy it out
  static constexpr bool BULK_OUT = (ELI * sizeof(double)) % 16 == 0;
};

template <int P, int NC, bool PEER = false>
__global__ void __launch_bounds__(MassTmaCfg<P, NC>::NT, MassTmaCfg<P, NC>::MINB)
    k_mass_tma(MassBrickArgs a, const __grid_constant__ CUtensorMap tm0, const __grid_constant__ CUtensorMap tm1,
               int nseg) {
  using M = MassTmaCfg<P, NC>;
  constexpr int D1 = M::D1, Q = M::Q, QQ = M::QQ, DD = M::DD, NQ = M::NQ, PLN = M::PLN, NT = M::NT;
  constexpr int ROWD = M::ROWD, TS = M::TS, ELI = M::ELI;
  const double* cB = c_B[P - 1];
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* smem = reinterpret_cast<double*>((reinterpret_cast<unsigned long long>(smem_raw) + 127) & ~127ull);
  double* sBox = smem;
  double* sD = smem + M::OFF_D;  // [2][DSD]
  double* sT = smem + M::OFF_T;  // T image [el][c][dz][qy*Q+qx]; E staging [el][l][c] once dead
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(smem + M::OFF_BAR);
  __shared__ double red[32];
  CGDev* g = a.cg;
  if (!g->active) return;
  const int t = threadIdx.x;
  const int k0 = g->it_m;
  const CUtensorMap* tm = (k0 & 1) ? &tm0 : &tm1;  // iteration k reads pbuf[(k-1)&1]
  // units: (row segment s, ey, ez), contiguous range per CTA
  const int nx = a.b.nx, ny = a.b.ny;
  const int units = nseg * ny * a.b.nz;
  const int u0 = (int)((long long)units * blockIdx.x / gridDim.x);
  const int u1 = (int)((long long)units * (blockIdx.x + 1) / gridDim.x);
  struct Unit {
    int ex0, len, ey, ez;
  };
  auto unit = [&](int u) {
    const int s = u % nseg, row = u / nseg;
    Unit w;
    w.ex0 = nx * s / nseg;
    w.len = nx * (s + 1) / nseg - w.ex0;
    w.ey = row % ny;
    w.ez = row / ny;
    return w;
  };
  auto issue = [&](int i) {  // unit u0 + i -> box, D buffer (i & 1), barrier (i & 1)
    const Unit w = unit(u0 + i);
    const long long e0 = w.ex0 + (long long)nx * (w.ey + (long long)ny * w.ez);
    const long long d0 = e0 * NQ, da = d0 & ~1ll;
    const unsigned dbytes = (unsigned)(((d0 - da + (long long)w.len * NQ) * 8 + 15) & ~15ll);
    unsigned long long* b = bar + (i & 1);
    mbar_expect_tx(b, M::BOX_BYTES + dbytes);
    tma_load_3d(sBox, tm, w.ex0 * P * NC * 2, w.ey * P, w.ez * P, b);
    bulk_load(sD + (i & 1) * M::DSD, a.D + da, dbytes, b);
  };
  if (t == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);
    mbar_fence_init();
  }
  __syncthreads();
  const int nu = u1 - u0;
  if (t == 0 && nu > 0) issue(0);  // lands while the prologue finishes the r.z reduction
  double beta;
  int k;
  if (!cg_mass_begin<NT, PEER>(g, red, beta, k, &a.pl)) {
    if (nu > 0) mbar_wait(bar, 0);  // no CTA exits with a tile in flight
    return;
  }
  double acc = 0.0;
  const int pe = t / PLN, pr = t - pe * PLN;
  const int pc = pr / D1, pz = pr - pc * D1;  // plane (c, dz)
  for (int i = 0; i < nu; ++i) {
    const Unit w = unit(u0 + i);
    const int nel = w.len;
    const long long e0 = w.ex0 + (long long)nx * (w.ey + (long long)ny * w.ez);
    if (t == 0) bulk_wait_read();  // the previous pass's E store has read the staging image
    __syncthreads();
    mbar_wait(bar + (i & 1), (i >> 1) & 1);
    // ---- phase 1 (planes): p = z + beta p_{k-1} from the box; x and y contractions -> T
    const bool pact = pe < nel;
    if (pact) {
      double u[DD];
      const double* bx = sBox + (pz * D1) * ROWD + (pe * P) * NC * 2 + pc * 2;
#pragma unroll
      for (int dy = 0; dy < D1; ++dy)
#pragma unroll
        for (int dx = 0; dx < D1; ++dx) {
          const double2 q = *reinterpret_cast<const double2*>(bx + dy * ROWD + dx * NC * 2);
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
      double* T = sT + pe * TS + pr * QQ;
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
    __syncthreads();  // the box is consumed: the next pass's tile may land in it
    if (t == 0 && i + 1 < nu) issue(i + 1);
    // ---- phase 2 (columns): z, D, z^T for all components of a (qx, qy) column
    const double* Dp = sD + (i & 1) * M::DSD + ((e0 * NQ) & 1);
    for (int it = t; it < nel * QQ; it += NT) {
      const int ce = it / QQ, l = it - ce * QQ;
      double Dq[Q];
#pragma unroll
      for (int qz = 0; qz < Q; ++qz) Dq[qz] = Dp[ce * NQ + qz * QQ + l];
      double* base = sT + ce * TS + l;
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        double col[D1];
#pragma unroll
        for (int dz = 0; dz < D1; ++dz) col[dz] = base[(c * D1 + dz) * QQ];
        double ww[Q];
#pragma unroll
        for (int qz = 0; qz < Q; ++qz) {
          double s = 0.0;
#pragma unroll
          for (int dz = 0; dz < D1; ++dz) s = fma(cB[qz * D1 + dz], col[dz], s);
          const double du = s * Dq[qz];
          acc = fma(du, s, acc);
          ww[qz] = du;
        }
#pragma unroll
        for (int dz = 0; dz < D1; ++dz) {
          double s = 0.0;
#pragma unroll
          for (int qz = 0; qz < Q; ++qz) s = fma(cB[qz * D1 + dz], ww[qz], s);
          base[(c * D1 + dz) * QQ] = s;
        }
      }
    }
    __syncthreads();
    // ---- phase 3 (planes): y^T, x^T -> E staging [el][l][c] (aliases the T image: every
    // plane is read into registers before any staging store)
    double Tq[QQ];
    if (pact) {
      const double* T = sT + pe * TS + pr * QQ;
#pragma unroll
      for (int kk = 0; kk < QQ; ++kk) Tq[kk] = T[kk];
    }
    __syncthreads();
    if (pact) {
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
      double* o = sT + pe * ELI + (pz * DD) * NC + pc;
#pragma unroll
      for (int dy = 0; dy < D1; ++dy)
#pragma unroll
        for (int dx = 0; dx < D1; ++dx) {
          double s = 0.0;
#pragma unroll
          for (int qx = 0; qx < Q; ++qx) s = fma(cB[qx * D1 + dx], v[dy][qx], s);
          o[(dy * D1 + dx) * NC] = s;
        }
      if constexpr (M::BULK_OUT) fence_proxy_async_smem();
    }
    __syncthreads();
    if constexpr (M::BULK_OUT) {
      if (t == 0) bulk_store(a.evec + e0 * ELI, sT, (unsigned)(nel * ELI * sizeof(double)));
    } else {
      double* out = a.evec + e0 * ELI;
      for (int it = t; it < nel * ELI; it += NT) __stcg(out + it, sT[it]);
    }
  }
  if (M::BULK_OUT && t == 0) bulk_wait_all();
  cg_partial(a.partials, &g->nparts_m, block_sum<NT>(acc, red));
}

}  // namespace hx

namespace hx {

// ---------------------------------------------------------------------------
// Warp-independent CG mass action on a brick (MASS_W2): every warp owns a contiguous
// range of element PAIRS and runs all phases of a pair on its own -- the gather of the
// pair's node rows into registers, the x/y plane stage, the z column stage and the
// transposed plane stage -- with __syncwarp between phases and no CTA-wide barrier
// (other warps of the SM keep the pipes busy while one waits on its gather).  Lane
// (el, c, dz) < 24 owns a plane of the pair; the column stage runs 50 columns over the
// 32 lanes.  Per-warp shared memory is the pair's T image (2 x NC*D1 planes of Q*Q),
// reused as the staging image for coalesced E stores.  Same per-element arithmetic as
// k_mass_brick (bit-identical E).
#ifndef MASS_W2_WARPS
#define MASS_W2_WARPS 4
#endif
#ifndef MASS_W2_MINB
#define MASS_W2_MINB 4
#endif
template <int P, int NC>
struct MassW2Cfg {
  static constexpr int D1 = P + 1, Q = P + 2, QQ = Q * Q, DD = D1 * D1, NL = D1 * DD, NQ = Q * QQ;
  static constexpr int PLN = NC * D1, EPW = 2;  // elements per warp pass
  static_assert(EPW * PLN <= 32, "one lane per plane");
  static constexpr int TP = QQ + (QQ % 2 == 0 ? 1 : 0);  // plane pitch (odd: conflict-free lanes)
  static constexpr int TS = PLN * TP;                     // T image doubles per element
  static constexpr int WS = EPW * TS;                     // per warp
  static constexpr int WARPS = MASS_W2_WARPS, NT = 32 * WARPS;
  // MASS_W2 prefetch variant: the next pair's node-row pairs (lane-private plane slots)
  // and point data land by cp.async while the current pair is contracted
  static constexpr int GB = EPW * PLN * DD * 2;     // gather buffer doubles ((z, p) pairs)
  static constexpr int DB = ((EPW * NQ + 1) & ~1);  // D buffer doubles
  static constexpr int WSP = WS + (WS & 1) + GB + DB;
  static constexpr size_t bytes = sizeof(double) * (size_t)WARPS * WS;
  static constexpr size_t bytes_pf = sizeof(double) * (size_t)WARPS * WSP;
};

template <int P, int NC, bool PEER = false, bool PF = false>
__global__ void __launch_bounds__(MassW2Cfg<P, NC>::NT, MASS_W2_MINB) k_mass_w2(MassBrickArgs a) {
  using M = MassW2Cfg<P, NC>;
  constexpr int D1 = M::D1, Q = M::Q, QQ = M::QQ, DD = M::DD, NL = M::NL, NQ = M::NQ, PLN = M::PLN;
  constexpr int TP = M::TP, TS = M::TS, EPW = M::EPW, NT = M::NT, ELI = NL * NC;
  const double* cB = c_B[P - 1];
  extern __shared__ __align__(16) double smem_w2[];
  __shared__ double red[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double* sT = smem_w2 + wid * (PF ? M::WSP : M::WS);
  double2* sG = reinterpret_cast<double2*>(sT + M::WS + (M::WS & 1));  // PF: [el][plane][DD] pairs
  double* sDb = sT + M::WS + (M::WS & 1) + M::GB;                       // PF: the pair's D
  const int gw = blockIdx.x * M::WARPS + wid, nw = gridDim.x * M::WARPS;
  const long long npairs = (a.ne + EPW - 1) / EPW;
  const long long pb = npairs * gw / nw, pe_ = npairs * (gw + 1) / nw;
  const int el = lane / PLN, pr = lane - el * PLN;
  const int pc = pr / D1, pz = pr - pc * D1;  // plane (c, dz)
  const bool lact = lane < EPW * PLN;
  // node-row pair source of this lane's plane for the pair starting at element e0
  auto plane_src = [&](const double* pbuf, long long e0) {
    const unsigned e = (unsigned)(e0 + el);
    const unsigned ez = a.b.fnxy.div(e);
    const unsigned r2 = e - ez * (unsigned)(a.b.nx * a.b.ny);
    const unsigned ey = a.b.fnx.div(r2), ex = r2 - ey * (unsigned)a.b.nx;
    const unsigned n0 = ex * P + (ey * P) * (unsigned)a.b.Nx + (ez * P + pz) * (unsigned)a.b.NxNy;
    return reinterpret_cast<const double2*>(pbuf) + (size_t)n0 * NC + pc;
  };
  auto nel_of = [&](long long e0) { return (int)(a.ne - e0 < EPW ? a.ne - e0 : EPW); };
  auto issue_gather = [&](const double* pbuf, long long pi) {  // PF: lane-private plane slots
    const long long e0 = pi * EPW;
    if (lact && el < nel_of(e0)) {
      const double2* src = plane_src(pbuf, e0);
      double2* dst = sG + (el * PLN + pr) * DD;
#pragma unroll
      for (int dy = 0; dy < D1; ++dy)
#pragma unroll
        for (int dx = 0; dx < D1; ++dx)
          cp_async16d(reinterpret_cast<double*>(dst + dy * D1 + dx),
                      reinterpret_cast<const double*>(src + (dy * a.b.Nx + dx) * NC));
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  auto issue_d = [&](long long pi) {  // PF: the pair's D (contiguous; 16-byte chunks when aligned)
    const long long e0 = pi * EPW;
    const int n = nel_of(e0) * NQ;
    cp_span<32>(sDb, a.D + e0 * NQ, n, lane);
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  if constexpr (PF) {
    if (!a.cg->active) return;
    const int k0 = a.cg->it_m;
    if (pb < pe_) {
      issue_gather((k0 & 1) ? a.pbuf0 : a.pbuf1, pb);  // lands during the prologue
      issue_d(pb);
    }
  }
  double beta;
  int k;
  if (!cg_mass_begin<NT, PEER>(a.cg, red, beta, k, &a.pl)) {
    if constexpr (PF) asm volatile("cp.async.wait_all;" ::: "memory");
    return;
  }
  const double* po = (k & 1) ? a.pbuf0 : a.pbuf1;
  double acc = 0.0;
  for (long long pi = pb; pi < pe_; ++pi) {
    const long long e0 = pi * EPW;
    const int nel = nel_of(e0);
    const bool pact = lact && el < nel;
    if constexpr (PF) {
      asm volatile("cp.async.wait_all;" ::: "memory");
      __syncwarp();
    }
    // ---- phase 1 (lane = plane): the plane's node row pairs, p = z + beta p_{k-1},
    // x and y contractions -> T
    if (pact) {
      double2 q[DD];
      if constexpr (PF) {
        const double2* g = sG + (el * PLN + pr) * DD;
#pragma unroll
        for (int i = 0; i < DD; ++i) q[i] = g[i];
      } else {
        const double2* src = plane_src(po, e0);
#pragma unroll
        for (int dy = 0; dy < D1; ++dy)
#pragma unroll
          for (int dx = 0; dx < D1; ++dx) q[dy * D1 + dx] = __ldcg(src + (dy * a.b.Nx + dx) * NC);
      }
      double u[DD];
#pragma unroll
      for (int i = 0; i < DD; ++i) u[i] = __dadd_rn(q[i].x, __dmul_rn(beta, q[i].y));
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
      double* T = sT + el * TS + pr * TP;
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
    __syncwarp();
    if constexpr (PF) {
      if (pi + 1 < pe_) issue_gather(po, pi + 1);  // the gather slots are consumed
    }
    // ---- phase 2 (lane = column): z, D, z^T for all components of a (qx, qy) column
    for (int it = lane; it < nel * QQ; it += 32) {
      const int ce = it / QQ, l = it - ce * QQ;
      double Dq[Q];
      if constexpr (PF) {
#pragma unroll
        for (int qz = 0; qz < Q; ++qz) Dq[qz] = sDb[ce * NQ + qz * QQ + l];
      } else {
        const double* Dp = a.D + (e0 + ce) * NQ + l;
#pragma unroll
        for (int qz = 0; qz < Q; ++qz) Dq[qz] = __ldg(Dp + qz * QQ);
      }
      double* base = sT + ce * TS + l;
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        double col[D1];
#pragma unroll
        for (int dz = 0; dz < D1; ++dz) col[dz] = base[(c * D1 + dz) * TP];
        double ww[Q];
#pragma unroll
        for (int qz = 0; qz < Q; ++qz) {
          double s = 0.0;
#pragma unroll
          for (int dz = 0; dz < D1; ++dz) s = fma(cB[qz * D1 + dz], col[dz], s);
          const double du = s * Dq[qz];
          acc = fma(du, s, acc);
          ww[qz] = du;
        }
#pragma unroll
        for (int dz = 0; dz < D1; ++dz) {
          double s = 0.0;
#pragma unroll
          for (int qz = 0; qz < Q; ++qz) s = fma(cB[qz * D1 + dz], ww[qz], s);
          base[(c * D1 + dz) * TP] = s;
        }
      }
    }
    __syncwarp();
    if constexpr (PF) {
      if (pi + 1 < pe_) issue_d(pi + 1);  // the D buffer is consumed
    }
    // ---- phase 3 (lane = plane): y^T, x^T -> staging over the lane's own plane
    if (pact) {
      double* T = sT + el * TS + pr * TP;
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
#pragma unroll
      for (int dy = 0; dy < D1; ++dy)
#pragma unroll
        for (int dx = 0; dx < D1; ++dx) {
          double s = 0.0;
#pragma unroll
          for (int qx = 0; qx < Q; ++qx) s = fma(cB[qx * D1 + dx], v[dy][qx], s);
          T[dy * D1 + dx] = s;
        }
    }
    __syncwarp();
    // ---- copy-out: the pair's E block (element-major [e][l][c], contiguous) from the
    // plane images, coalesced stores
    double* out = a.evec + e0 * ELI;
    for (int it = lane; it < nel * ELI; it += 32) {
      const int ce = it / ELI, r = it - ce * ELI;
      const int l = r / NC, c = r - l * NC;
      const int dz = l / DD, kk = l - dz * DD;
      __stcg(out + it, sT[ce * TS + (c * D1 + dz) * TP + kk]);
    }
    __syncwarp();
  }
  cg_partial(a.partials, &a.cg->nparts_m, block_sum<NT>(acc, red));
}

}  // namespace hx
