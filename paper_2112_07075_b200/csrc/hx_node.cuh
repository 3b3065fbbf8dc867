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

}  // namespace hx
