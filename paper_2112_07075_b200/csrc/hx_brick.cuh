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

// (element coordinate, local coordinate) pairs touching node coordinate i along one
// axis with n elements of order P, ascending element order.  Returns the count.
template <int P>
__device__ __forceinline__ int axis_pairs(int i, int n, int (&ec)[2], int (&lc)[2]) {
  const int q = i / P, r = i - q * P;
  if (r != 0) {
    ec[0] = q;
    lc[0] = r;
    return 1;
  }
  if (q == 0) {
    ec[0] = 0;
    lc[0] = 0;
    return 1;
  }
  if (q == n) {
    ec[0] = n - 1;
    lc[0] = P;
    return 1;
  }
  ec[0] = q - 1;
  lc[0] = P;
  ec[1] = q;
  lc[1] = 0;
  return 2;
}

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
          v[(a * 2 + bb) * 2 + g] = ok ? __ldcg(E + pos) : 0.0;
        }
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) s += v[q];  // absent entries are +0.0: sums unchanged
    return s;
  }
};

// generic (CSR, node-sorted E-vector) node sum as a functor
template <int NC>
struct CsrSum {
  const int* off;
  const double* E;
  __device__ __forceinline__ double operator()(long long n, int c) const { return node_sum1<NC>(off, E, n, c); }
};

// ---------------------------------------------------------------------------
// CG mass action on a brick: p_k = z + beta p_{k-1} (pairs), y_e = B^T D B p_e,
// element-major E out, element-wise p.Ap partial -> alpha (last block).
// (Masked components of p are exactly 0 in this CG -- r, z start at 0 there and
// Ap := p keeps them 0 -- so p.Ap needs no wall term and p no mask.)

template <int P, int NC>
struct MassBrickCfg {
  static constexpr int D1 = P + 1, Q = P + 2, QQ = Q * Q, DD = D1 * D1, NL = D1 * DD, NQ = Q * QQ;
  static constexpr int PLN = NC * D1;          // planes per element
  static constexpr int EPC = 128 / PLN;        // elements per pass
  static constexpr int GP = DD + 1;            // padded plane pitch of the gather / staging image
  static constexpr int GS = PLN * GP;          // gather doubles per element
  static constexpr int TS = PLN * QQ;          // T image doubles per element
  static constexpr size_t bytes = sizeof(double) * (size_t)EPC * (GS + TS);
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
};

template <int P, int NC>
__global__ void __launch_bounds__(128, 4) k_mass_brick(MassBrickArgs a) {
  using M = MassBrickCfg<P, NC>;
  constexpr int D1 = M::D1, Q = M::Q, QQ = M::QQ, DD = M::DD, NL = M::NL, NQ = M::NQ;
  constexpr int PLN = M::PLN, EPC = M::EPC, GP = M::GP, GS = M::GS;
  const double* cB = c_B[P - 1];
  extern __shared__ double smem[];
  double* sG = smem;                 // gather image [el][c][dz][dy*D1+dx] (pitch GP); reused as staging
  double* sT = smem + EPC * GS;      // T image [el][c][dz][qy*Q+qx]
  __shared__ double red[32];
  __shared__ int sflag;
  if (!a.cg->active) return;
  const int t = threadIdx.x;
  const double beta = a.cg->beta;
  const double* po = (a.cg->it & 1) ? a.pbuf0 : a.pbuf1;
  double acc = 0.0;
  const int pe = t / PLN, pr = t - pe * PLN;
  __shared__ int sbase[EPC];  // first node of each element of the pass
  // per-thread gather / copy-out slots within an element (pass invariant)
  constexpr int ROWI = D1 * NC;                 // pairs per node row
  constexpr int ELI = DD * ROWI;                // pairs (= E entries) per element
  constexpr int SLOTS = (ELI + 127) / 128;
  int soff[SLOTS], goff[SLOTS];
#pragma unroll
  for (int h = 0; h < SLOTS; ++h) {
    const int it = h * 128 + t;
    const int row = it / ROWI, s = it - row * ROWI;  // row = dz*D1 + dy
    const int dz = row / D1, dy = row - dz * D1, dx = s / NC, c = s - dx * NC;
    soff[h] = (c * D1 + dz) * GP + dy * D1 + dx;
    goff[h] = (dx + dy * a.b.Nx + dz * (int)a.b.NxNy) * NC + c;
  }
  for (long long e0 = (long long)blockIdx.x * EPC; e0 < a.ne; e0 += (long long)gridDim.x * EPC) {
    const int nel = (int)((a.ne - e0) < EPC ? (a.ne - e0) : EPC);
    if (t < nel) {
      const unsigned e = (unsigned)(e0 + t);
      const unsigned ez = a.b.fnxy.div(e);
      const unsigned r2 = e - ez * (unsigned)(a.b.nx * a.b.ny);
      const unsigned ey = a.b.fnx.div(r2), ex = r2 - ey * (unsigned)a.b.nx;
      sbase[t] = (int)(ex * P + (ey * P) * (unsigned)a.b.Nx + (ez * P) * (unsigned)a.b.NxNy);
    }
    __syncthreads();
    // ---- phase 0: node rows (D1 nodes x NC pairs, contiguous) -> p image.  Thread t
    // owns the same (row, pair) slots of every element of the pass (offsets hoisted
    // out of the pass loop); all loads of a slot are issued before the first use.
#pragma unroll
    for (int h = 0; h < SLOTS; ++h) {
      if (h * 128 + t < ELI) {
        double2 q[EPC];
#pragma unroll
        for (int el = 0; el < EPC; ++el)
          if (el < nel) q[el] = __ldcg(reinterpret_cast<const double2*>(po) + (long long)sbase[el] * NC + goff[h]);
#pragma unroll
        for (int el = 0; el < EPC; ++el)
          if (el < nel) sG[el * GS + soff[h]] = __dadd_rn(q[el].x, __dmul_rn(beta, q[el].y));
      }
    }
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
    __syncthreads();
    // ---- phase 2 (columns): z, D, z^T for all components of a (qx, qy) column
    for (int it = t; it < nel * QQ; it += 128) {
      const int ce = it / QQ, l = it - ce * QQ;
      const long long ee = e0 + ce;
      double Dq[Q];
#pragma unroll
      for (int qz = 0; qz < Q; ++qz) Dq[qz] = __ldg(a.D + ee * NQ + qz * QQ + l);
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
      for (int it = t; it < nel * NL; it += 128) {
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
        const int it = h * 128 + t;
        if (it < ELI) {
#pragma unroll
          for (int el = 0; el < EPC; ++el)
            if (el < nel) __stcg(out + el * ELI + it, sG[el * GS + soff[h]]);
        }
      }
    }
    __syncthreads();
  }
  const double bs = block_sum<128>(acc, red);
  if (threadIdx.x == 0) a.partials[blockIdx.x] = bs;
  if (grid_last_block(&a.cg->cnt[0], &sflag)) {
    const double pAp = reduce_partials<128>(a.partials, gridDim.x, red);
    if (threadIdx.x == 0) {
      a.cg->cnt[0] = 0;
      if (pAp <= 0.0) {
        a.cg->code = 3;
        a.cg->active = 0;
      } else {
        a.cg->alpha = a.cg->rz / pAp;
      }
    }
  }
}

}  // namespace hx

namespace hx {

// entries of node n in an element-major E-vector: up to 8 (element, local) positions in
// ascending element order (absent ones: -1)
template <int P, int NC>
__device__ __forceinline__ void brick_entries(const Brick& b, unsigned n, long long (&pos)[8]) {
  constexpr int D1 = P + 1, NL = D1 * D1 * D1;
  const unsigned k = b.fNxNy.div(n);
  const unsigned rem = n - k * (unsigned)b.NxNy;
  const unsigned j = b.fNx.div(rem);
  const int i = (int)(rem - j * (unsigned)b.Nx);
  int ex[2], lx[2], ey[2], ly[2], ez[2], lz[2];
  const int cx = axis_pairs<P>(i, b.nx, ex, lx);
  const int cy = axis_pairs<P>((int)j, b.ny, ey, ly);
  const int cz = axis_pairs<P>((int)k, b.nz, ez, lz);
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int bb = 0; bb < 2; ++bb)
#pragma unroll
      for (int g = 0; g < 2; ++g) {
        const bool ok = a < cz && bb < cy && g < cx;
        const long long e = ((long long)ez[a] * b.ny + ey[bb]) * b.nx + ex[g];
        const int l = (lz[a] * D1 + ly[bb]) * D1 + lx[g];
        pos[(a * 2 + bb) * 2 + g] = ok ? (e * NL + l) * NC : -1;
      }
}

// all NC components of node n from an element-major E-vector, ascending element order
template <int P, int NC>
__device__ __forceinline__ void brick_node_sum(const Brick& b, const double* E, unsigned n, double (&s)[NC]) {
  long long pos[8];
  brick_entries<P, NC>(b, n, pos);
  double v[8][NC];
#pragma unroll
  for (int q = 0; q < 8; ++q)
#pragma unroll
    for (int c = 0; c < NC; ++c) v[q][c] = pos[q] >= 0 ? __ldcg(E + pos[q] + c) : 0.0;
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    double t = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) t += v[q][c];  // absent entries are +0.0: sums unchanged
    s[c] = t;
  }
}

// CG iteration tail on a brick, one thread per node (all components): the same
// recurrence and rounding as k_cg_node (operators.py:352-365).
template <int P, int NC>
__global__ void __launch_bounds__(256, 3) k_cg_node_brick(NodeArgs a, Brick b) {
  __shared__ double red[32];
  __shared__ int sflag;
  CGDev* g = a.cg;
  if (!g->active) return;
  const int k = g->it;
  const double alpha = g->alpha, beta = g->beta;
  const double* po = (k & 1) ? a.pbuf0 : a.pbuf1;
  double* pn = (k & 1) ? a.pbuf1 : a.pbuf0;
  double rz = 0.0;
  const unsigned nn = (unsigned)a.nn;
  for (unsigned n = blockIdx.x * blockDim.x + threadIdx.x; n < nn; n += gridDim.x * blockDim.x) {
    double s[NC];
    brick_node_sum<P, NC>(b, a.evec, n, s);
    double2 zp[NC];
    double xj[NC], rj[NC], dj[NC];
    bool m[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const long long j = (long long)n * NC + c;
      zp[c] = __ldcg(reinterpret_cast<const double2*>(po) + j);
      xj[c] = __ldcg(a.x + j);
      rj[c] = __ldcg(a.r + j);
      dj[c] = __ldg(a.invd + j);
      m[c] = a.mask && a.mask[j];
    }
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const long long j = (long long)n * NC + c;
      const double p = __dadd_rn(zp[c].x, __dmul_rn(beta, zp[c].y));
      const double ap = m[c] ? p : s[c];
      a.x[j] = __dadd_rn(xj[c], __dmul_rn(alpha, p));
      const double r = __dsub_rn(rj[c], __dmul_rn(alpha, ap));
      a.r[j] = r;
      const double z = __dmul_rn(dj[c], r);
      reinterpret_cast<double2*>(pn)[j] = make_double2(z, p);
      rz = fma(r, z, rz);
    }
  }
  const double brz = block_sum<256>(rz, red);
  if (threadIdx.x == 0) a.partials[blockIdx.x] = brz;
  if (grid_last_block(&g->cnt[1], &sflag)) {
    const double rzn = reduce_partials<256>(a.partials, gridDim.x, red);
    if (threadIdx.x == 0) {
      g->cnt[1] = 0;
      const double res = sqrt(fmax(rzn, 0.0));
      if (a.hist) a.hist[k] = res;
      g->nres = k + 1;
      if (res <= g->tol * g->norm0) {
        g->iters = k;
        g->active = 0;
      } else if (k >= g->max_iter) {
        g->code = 4;
        g->iters = k;
        g->active = 0;
      } else {
        g->beta = rzn / g->rz;
        g->rz = rzn;
        g->it = k + 1;
      }
      cg_publish(g);
    }
  }
}

}  // namespace hx
