// hx_node.cuh -- CG node pass on a structured brick, one warp per node-row segment.
//
// The tail of a cg_solve iteration (operators.py:352-365) for the brick layout:
// Ap = G^T E (the deterministic ascending-element node sum of the element-major
// E-vector, BrickSum), identity on masked rows, x += alpha p (every second iteration),
// r -= alpha Ap, z = D^{-1} r, the (z, p) pair for the next mass launch and the r.z
// partial -- the same arithmetic as k_cg_node, mapped so that the index work is
// amortised:
//   * a warp owns a segment of one node row (fixed j, k): the y / z parts of every
//     node's element coordinates (first element, local index, second sharer) are
//     warp-uniform and computed once per segment;
//   * lane l handles the entries l, l + 32, ... of the segment's (node, comp) range, so
//     its in-row offsets (node, component) are per-lane constants of the launch and every
//     vector access of the warp is contiguous;
//   * the loads of GRP entries per lane are issued before the first use.
#pragma once

#include "hx_brick.cuh"

namespace hx {

#ifndef NODE_ROW_MINB
#define NODE_ROW_MINB 3
#endif
#ifndef NODE_ROW_GRP
#define NODE_ROW_GRP 2
#endif

// MS = entry slots per lane (ceil(NC * seg / 32)), processed GRP at a time
template <int P, int NC, int MS>
__global__ void __launch_bounds__(256, NODE_ROW_MINB) k_cg_node_row(NodeArgs a, Brick b, int seg, int nseg_row) {
  constexpr int D1 = P + 1, NL = D1 * D1 * D1, GRP = NODE_ROW_GRP;
  __shared__ double red[32];
  CGDev* g = a.cg;
  double alpha, alpha_prev;
  int k;
  if (!cg_node_begin<256, false>(g, red, alpha, alpha_prev, k)) return;
  const double beta = g->beta;
  const double* po = (k & 1) ? a.pbuf0 : a.pbuf1;
  double* pn = (k & 1) ? a.pbuf1 : a.pbuf0;
  const bool xk = (k & 1) == 0;  // x stored every second iteration (see k_cg_node)
  const int lane = threadIdx.x & 31;
  const int warp = (int)((blockIdx.x * 256u + threadIdx.x) >> 5), nwarps = (int)((gridDim.x * 256u) >> 5);
  const int Nx = b.Nx;
  const int nrows = b.Ny * (b.nz * P + 1);
  const unsigned oz = (unsigned)(b.dZ * NC), oy = (unsigned)(b.dY * NC), ox = (unsigned)(b.dX * NC);
  double rz = 0.0;
  for (int s = warp; s < nrows * nseg_row; s += nwarps) {
    const int row = s / nseg_row, part = s - row * nseg_row;
    const int jy = row % b.Ny, kz = row / b.Ny;
    const int i0 = part * seg;
    const int ne_seg = NC * min(seg, Nx - i0);  // entries of the segment
    // warp-uniform y / z element coordinates of the row
    int ey, ly, ty, ez, lz, tz;
    axis_first<P>(jy, b.ny, ey, ly, ty);
    axis_first<P>(kz, b.nz, ez, lz, tz);
    const unsigned ebase = (unsigned)((ez * b.ny + ey) * b.nx) * NL + (unsigned)((lz * D1 + ly) * D1);
    const unsigned j0 = (unsigned)(row * Nx + i0) * NC;  // first entry of the segment
#pragma unroll
    for (int m0 = 0; m0 < MS; m0 += GRP) {
      double2 zp[GRP];
      double xj[GRP], rj[GRP], dj[GRP], v[GRP][8];
      bool msk[GRP], act[GRP];
#pragma unroll
      for (int u = 0; u < GRP; ++u) {
        const int idx = lane + 32 * (m0 + u);
        act[u] = (m0 + u < MS) && idx < ne_seg;
        if (act[u]) {
          const int dn = idx / NC, c = idx - dn * NC;
          const unsigned j = j0 + (unsigned)idx;
          zp[u] = __ldcg(reinterpret_cast<const double2*>(po) + j);
          if (xk) xj[u] = __ldcg(a.x + j);
          rj[u] = __ldcg(a.r + j);
          msk[u] = a.mask && a.mask[j];
          dj[u] = a.invdn ? (msk[u] ? 1.0 : __ldg(a.invdn + (j0 / NC + dn))) : __ldg(a.invd + j);
          int ex, lx, tx;
          axis_first<P>(i0 + dn, b.nx, ex, lx, tx);
          const unsigned p0 = (ebase + (unsigned)ex * NL + (unsigned)lx) * NC + (unsigned)c;
          // BrickSum order: (z, y, x) pairs ascending = ascending element
#pragma unroll
          for (int az = 0; az < 2; ++az)
#pragma unroll
            for (int by = 0; by < 2; ++by) {
              const bool okq = az <= tz && by <= ty;
              const unsigned pq = p0 + (az ? oz : 0u) + (by ? oy : 0u);
              v[u][(az * 2 + by) * 2] = okq ? __ldcg(a.evec + pq) : 0.0;
              v[u][(az * 2 + by) * 2 + 1] = (okq && tx) ? __ldcg(a.evec + pq + ox) : 0.0;
            }
        }
      }
#pragma unroll
      for (int u = 0; u < GRP; ++u) {
        if (act[u]) {
          double ssum = 0.0;
#pragma unroll
          for (int q = 0; q < 8; ++q) ssum += v[u][q];  // absent entries are +0.0
          const unsigned j = j0 + (unsigned)(lane + 32 * (m0 + u));
          const double p = __dadd_rn(zp[u].x, __dmul_rn(beta, zp[u].y));
          const double ap = msk[u] ? p : ssum;
          if (xk) a.x[j] = __dadd_rn(__dadd_rn(xj[u], __dmul_rn(alpha_prev, zp[u].y)), __dmul_rn(alpha, p));
          const double r = __dsub_rn(rj[u], __dmul_rn(alpha, ap));
          a.r[j] = r;
          const double z = __dmul_rn(dj[u], r);
          reinterpret_cast<double2*>(pn)[j] = make_double2(z, p);
          rz = fma(r, z, rz);
        }
      }
    }
  }
  cg_partial(a.partials, &g->nparts_n, block_sum<256>(rz, red));
}

// ---------------------------------------------------------------------------
// Asynchronous node pass (HX_NODE_ASYNC): the same iteration tail as k_cg_node over tiles
// of TN consecutive (node, comp) entries, staged in shared memory one tile ahead by
// cp.async (LDGSTS) so that no register holds an in-flight load:
//   * the tile's contiguous streams -- (z, p) pairs, r, x (every second iteration), the
//     mask bytes and the per-node 1/diag -- as 16 / 8 / 4-byte copies;
//   * its E entries (BrickSum order: up to 8 per entry, ascending element) as 8-byte copies
//     of the present entries only, slot-major ([slot][entry]: conflict-free reads), with a
//     presence byte per entry;
//   * the first two tiles are issued BEFORE the prologue that finishes M(k)'s p.Ap
//     reduction, so that reduction's latency overlaps the first loads.
// Arithmetic and rounding per entry are k_cg_node's (same sum order, same x / r / z / p
// expressions); only the per-CTA r.z partial groups entries differently.
#ifndef NODE_ASYNC_TN
#define NODE_ASYNC_TN 512
#endif
#ifndef NODE_ASYNC_MINB
#define NODE_ASYNC_MINB 2
#endif
template <int NC>
struct NodeAsyncCfg {
  static constexpr int NT = 256, TN = NODE_ASYNC_TN, PER = TN / NT;
  static constexpr int TNODES = TN / NC + 2;  // nodes a tile can touch
  // stage layout (doubles): pairs 2 TN | r TN | x TN | E 8 TN | invdn TNODES | mask TN bytes | presence TN bytes
  static constexpr int OP = 0, OR = 2 * TN, OX = 3 * TN, OE = 4 * TN, OD = 12 * TN;
  static constexpr int OM = OD + ((TNODES + 1) & ~1);  // byte regions start here (in doubles)
  static constexpr int SD = OM + (2 * TN) / 8;         // stage size in doubles
  static constexpr size_t bytes = sizeof(double) * 2 * (size_t)SD;
};

__device__ __forceinline__ void cp_async_z(void* dst, const void* src, int bytes, int src_bytes) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  if (bytes == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(src_bytes) : "memory");
  else if (bytes == 8)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(src), "r"(src_bytes) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(d), "l"(src), "r"(src_bytes) : "memory");
}

template <int P, int NC>
__global__ void __launch_bounds__(256, NODE_ASYNC_MINB) k_cg_node_async(NodeArgs a, Brick b) {
  using C = NodeAsyncCfg<NC>;
  constexpr int NT = C::NT, TN = C::TN, PER = C::PER, D1 = P + 1, NL = D1 * D1 * D1;
  extern __shared__ __align__(16) double smem[];
  __shared__ double red[32];
  CGDev* g = a.cg;
  if (!g->active) return;
  const int k = g->it_n;  // the iteration cg_node_begin finishes
  const double* po = (k & 1) ? a.pbuf0 : a.pbuf1;
  double* pn = (k & 1) ? a.pbuf1 : a.pbuf0;
  const bool xk = (k & 1) == 0;  // x stored every second iteration (see k_cg_node)
  const long long N = a.nn * NC;
  const long long ntiles = (N + TN - 1) / TN;
  const int t = threadIdx.x;
  const unsigned oz = (unsigned)(b.dZ * NC), oy = (unsigned)(b.dY * NC), ox = (unsigned)(b.dX * NC);
  auto issue = [&](int st, long long tile) {
    if (tile < ntiles) {
      double* S = smem + st * C::SD;
      const long long j0 = tile * TN;
      const int nt = (int)((N - j0) < TN ? (N - j0) : TN);
      // pairs (16 B per entry), r and x (8 B, 16-B chunks), mask (4-B chunks), 1/diag per node
      for (int i = t; i < nt; i += NT)
        cp_async_z(S + C::OP + 2 * i, po + 2 * (j0 + i), 16, 16);
      for (int i = t; 2 * i < nt; i += NT) {
        const int sb = (nt - 2 * i) >= 2 ? 16 : 8;
        cp_async_z(S + C::OR + 2 * i, a.r + j0 + 2 * i, 16, sb);
        if (xk) cp_async_z(S + C::OX + 2 * i, a.x + j0 + 2 * i, 16, sb);
      }
      if (a.mask)
        for (int i = t; 4 * i < nt; i += NT) {
          const int rem = nt - 4 * i;
          cp_async_z(reinterpret_cast<unsigned char*>(S + C::OM) + 4 * i, a.mask + j0 + 4 * i, 4, rem >= 4 ? 4 : rem);
        }
      const long long n0 = j0 / NC, n1 = (j0 + nt - 1) / NC;
      for (int i = t; i <= (int)(n1 - n0); i += NT) cp_async_z(S + C::OD + i, a.invdn + n0 + i, 8, 8);
      // E entries present for each (node, comp) entry, in BrickSum's ascending order
      unsigned char* pres = reinterpret_cast<unsigned char*>(S + C::OM) + TN;
#pragma unroll
      for (int u = 0; u < PER; ++u) {
        const int i = t + u * NT;
        if (i < nt) {
          const long long j = j0 + i;
          const unsigned n = (unsigned)(j / NC);
          const int c = (int)(j - (long long)n * NC);
          const unsigned kk = b.fNxNy.div(n);
          const unsigned rem = n - kk * (unsigned)b.NxNy;
          const unsigned jj = b.fNx.div(rem);
          const int ii = (int)(rem - jj * (unsigned)b.Nx);
          int ex, lx, tx, ey, ly, ty, ez, lz, tz;
          axis_first<P>(ii, b.nx, ex, lx, tx);
          axis_first<P>((int)jj, b.ny, ey, ly, ty);
          axis_first<P>((int)kk, b.nz, ez, lz, tz);
          const unsigned p0 = ((unsigned)((ez * b.ny + ey) * b.nx + ex) * NL + (lz * D1 + ly) * D1 + lx) * NC + c;
          unsigned char pm = 0;
#pragma unroll
          for (int az = 0; az < 2; ++az)
#pragma unroll
            for (int by = 0; by < 2; ++by)
#pragma unroll
              for (int gx = 0; gx < 2; ++gx)
                if (az <= tz && by <= ty && gx <= tx) {
                  const int q = (az * 2 + by) * 2 + gx;
                  pm |= (unsigned char)(1u << q);
                  cp_async_z(S + C::OE + q * TN + i, a.evec + p0 + (az ? oz : 0u) + (by ? oy : 0u) + (gx ? ox : 0u),
                             8, 8);
                }
          pres[i] = pm;
        }
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  long long tile = blockIdx.x;
  const long long tstride = gridDim.x;
  issue(0, tile);
  issue(1, tile + tstride);
  double alpha, alpha_prev;
  int kk;
  if (!cg_node_begin<256, false>(g, red, alpha, alpha_prev, kk)) {
    asm volatile("cp.async.wait_all;" ::: "memory");
    return;
  }
  const double beta = g->beta;
  double rz = 0.0;
  for (int st = 0; tile < ntiles; tile += tstride, st ^= 1) {
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    __syncthreads();  // this tile's copies (every thread's) have landed
    const double* S = smem + st * C::SD;
    const unsigned char* msk = reinterpret_cast<const unsigned char*>(S + C::OM);
    const unsigned char* pres = msk + TN;
    const long long j0 = tile * TN;
    const int nt = (int)((N - j0) < TN ? (N - j0) : TN);
    const long long n0 = j0 / NC;
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int i = t + u * NT;
      if (i < nt) {
        const long long j = j0 + i;
        const unsigned pm = pres[i];
        double s = 0.0;
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (pm & (1u << q)) s += S[C::OE + q * TN + i];  // ascending element, from 0.0
        const double2 zp = reinterpret_cast<const double2*>(S + C::OP)[i];
        const bool m = a.mask && msk[i];
        const double dj = m ? 1.0 : S[C::OD + (int)(j / NC - n0)];
        const double p = __dadd_rn(zp.x, __dmul_rn(beta, zp.y));
        const double ap = m ? p : s;
        if (xk) __stcg(a.x + j, __dadd_rn(__dadd_rn(S[C::OX + i], __dmul_rn(alpha_prev, zp.y)), __dmul_rn(alpha, p)));
        const double r = __dsub_rn(S[C::OR + i], __dmul_rn(alpha, ap));
        __stcg(a.r + j, r);
        const double z = __dmul_rn(dj, r);
        __stcg(reinterpret_cast<double2*>(pn) + j, make_double2(z, p));
        rz = fma(r, z, rz);
      }
    }
    __syncthreads();  // every thread is done with this stage before it is refilled
    issue(st, tile + 2 * tstride);
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  cg_partial(a.partials, &g->nparts_n, block_sum<256>(rz, red));
}

}  // namespace hx
