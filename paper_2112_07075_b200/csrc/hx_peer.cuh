// hx_peer.cuh -- device-resident exchange of the multi-GPU momentum CG over peer memory.
//
// The mesh is split into bricks, one per rank (paper_2112_07075_b200/partition.py; the
// paper's P operator, identity in the reference).  Inside the CG
// (cg_solve operators.py:333-366 on the PA mass) two things cross subdomains:
//   * the H1 node sums at interface nodes (halo): every sharer needs the sum of all
//     ranks' element contributions;
//   * the scalars p.Ap and r.z (and r.z, nnz(b) at the start): world sums.
// Both move through a per-rank MAILBOX in device memory that every rank maps (CUDA IPC
// across processes over NVLink, plain pointers when several ranks share a process):
//   [flag[src] u64 x HX_MAXR | slot[parity][src][SLOTW] doubles | recv[src][maxh][nc] doubles]
// A sender writes its data straight into the receivers' mailboxes (P2P stores), then
// publishes a sequence number with a system-scope release store; a receiver spins on
// its own flags with acquire loads.  Sequence numbers come from a per-rank device
// counter that every rank advances identically (all ranks run the same launches and
// take the same CG decisions, because they see the same world scalars), so the whole
// loop stays on the device: no host round trip, no NCCL call inside the iteration.
// Combination order is fixed (ascending rank, from 0.0), so every sharer of a node
// holds bit-identical values -- deterministic, though not bit-identical to one GPU.
// The spin-waits assume every rank's launch gets to run: true with one GPU per rank, and
// for ranks sharing a GPU only while their launches fit on it together (the in-process
// tests use small meshes); a rank that never arrives ends the spin after a bound (code 6).
#pragma once

#include "hx_brick.cuh"

namespace hx {

// CG world scalar: fixed-order sum of this launch's per-CTA partials (NV values each,
// stride NV), posted to every rank; after all ranks posted, the ascending-rank sum
// replaces partial 0 and the partial count becomes 1, so the consuming CG kernel
// (cg_mass_begin / cg_node_begin) reads the world value unchanged.  Halo data written
// by k_halo_pack before this launch is published by the same flag.
template <int NV>
__global__ void __launch_bounds__(256) k_peer_sync(PeerDev pd, CGDev* g, double* parts, int* nparts) {
  __shared__ double red[32];
  if (g && !g->active) return;
  double v[NV > 0 ? NV : 1];
  if constexpr (NV > 0) {
    const int n = *nparts;
#pragma unroll
    for (int t = 0; t < NV; ++t) {
      double acc = 0.0;
      for (int i = threadIdx.x; i < n; i += 256) acc += __ldcg(parts + (long long)i * NV + t);
      v[t] = block_sum<256>(acc, red);
    }
  }
  if (threadIdx.x == 0) {
    const unsigned long long seq = *pd.seq + 1;
    *pd.seq = seq;
    const int par = (int)(seq & 1);
    if constexpr (NV > 0)
      for (int q = 0; q < pd.nranks; ++q) {
        double* s = pd.mb[q] + MB_SLOT + (par * HX_MAXR + pd.rank) * SLOTW;
#pragma unroll
        for (int t = 0; t < NV; ++t) s[t] = v[t];
      }
    __threadfence_system();
    for (int q = 0; q < pd.nranks; ++q) st_release_sys(mb_flag(pd.mb[q], pd.rank), seq);
    if (peer_wait(pd, nullptr, pd.nranks, seq)) {
      if constexpr (NV > 0) {
        const double* s = pd.mb[pd.rank] + MB_SLOT + par * HX_MAXR * SLOTW;
#pragma unroll
        for (int t = 0; t < NV; ++t) {
          double tot = 0.0;
          for (int q = 0; q < pd.nranks; ++q) tot += __ldcg(s + q * SLOTW + t);
          parts[t] = tot;
        }
        *nparts = 1;
      }
    } else {
      *pd.err = 1;
      if (g) {
        g->code = 6;
        g->active = 0;
        cg_publish(g);
      }
    }
  }
}

// world step status (timestep_estimate / rk2_step decisions, hydro.py:364-405): for each
// of n StatusDev records, min of the CFL ratio, sum of the clamp counts, min of the
// inversion key (a rank-local key: any inversion anywhere makes every rank retry)
__global__ void k_peer_status(PeerDev pd, StatusDev* st, int n) {
  if (threadIdx.x != 0) return;
  const unsigned long long seq = *pd.seq + 1;
  *pd.seq = seq;
  const int par = (int)(seq & 1);
  for (int q = 0; q < pd.nranks; ++q) {
    double* s = pd.mb[q] + MB_SLOT + (par * HX_MAXR + pd.rank) * SLOTW;
    for (int i = 0; i < n; ++i) {
      s[3 * i] = __longlong_as_double((long long)st[i].inv_key);
      s[3 * i + 1] = __longlong_as_double((long long)st[i].clamps);
      s[3 * i + 2] = st[i].min_ratio;
    }
  }
  __threadfence_system();
  for (int q = 0; q < pd.nranks; ++q) st_release_sys(mb_flag(pd.mb[q], pd.rank), seq);
  if (!peer_wait(pd, nullptr, pd.nranks, seq)) {
    *pd.err = 1;
    for (int i = 0; i < n; ++i) st[i].inv_key = 0;  // report a failure: every rank stops
    return;
  }
  const double* s = pd.mb[pd.rank] + MB_SLOT + par * HX_MAXR * SLOTW;
  for (int i = 0; i < n; ++i) {
    unsigned long long key = ~0ull, cl = 0;
    double r = __longlong_as_double(0x7ff0000000000000ll);
    for (int q = 0; q < pd.nranks; ++q) {
      const unsigned long long k = (unsigned long long)__double_as_longlong(__ldcg(s + q * SLOTW + 3 * i));
      key = k < key ? k : key;
      cl += (unsigned long long)__double_as_longlong(__ldcg(s + q * SLOTW + 3 * i + 1));
      r = fmin(r, __ldcg(s + q * SLOTW + 3 * i + 2));
    }
    st[i].inv_key = key;
    st[i].clamps = cl;
    st[i].min_ratio = r;
  }
}

// node-vector view for halo sums of assembled node data (the mass diagonal)
template <int NC>
struct NodeVec {
  double* v;
  __device__ __forceinline__ double operator()(long long n, int c) const { return v[n * NC + c]; }
  __device__ __forceinline__ void patch(long long n, int c, double total) const { v[n * NC + c] = total; }
};

// halo, part 1: this rank's node sums at the nodes it shares, stored into each
// neighbour's recv block (published by the following k_peer_sync)
template <int NC, class SUM>
__global__ void __launch_bounds__(256) k_halo_pack(PeerDev pd, CGDev* g, SUM sum, PeerLite pl) {
  __shared__ double red[32];
  if (g && !g->active) return;
  const long long N = (long long)pd.nsh * NC;
  bool wrote = false;
  for (long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x; j < N; j += (long long)gridDim.x * blockDim.x) {
    const int e = (int)(j / NC), c = (int)(j - (long long)e * NC);
    const int n = __ldg(pd.snode + e), q = __ldg(pd.sdst + e), i = __ldg(pd.sidx + e);
    pd.mb[q][MB_RECV + ((long long)pd.rank * pd.maxh + i) * NC + c] = sum(n, c);
    wrote = true;
  }
  if (wrote) __threadfence_system();
  // in the CG: post this rank's p.Ap_k behind the halo (the flag publishes both)
  if (g && (pl.post & PEER_POST_ON)) cg_post_last<256>(pl, g->parts_m, g->nparts_m, &g->cnt[3], g->seq0 + 2ull * g->it_n, red);
}

// halo, part 2 (after the flags): total = sum over the sharers in ascending rank order
// from 0.0 (own partial from the local E-vector), written back into the E-vector so the
// node pass's sum yields exactly the total
template <int NC, class SUM>
__global__ void __launch_bounds__(256) k_halo_combine(PeerDev pd, const CGDev* g, SUM sum) {
  if (g && !g->active) return;
  if (*pd.err) return;
  const long long N = (long long)pd.nh * NC;
  const double* recv = pd.mb[pd.rank] + MB_RECV;
  for (long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x; j < N; j += (long long)gridDim.x * blockDim.x) {
    const int h = (int)(j / NC), c = (int)(j - (long long)h * NC);
    const int n = __ldg(pd.hnode + h);
    const double own = sum(n, c);
    double tot = 0.0;
    for (int s = __ldg(pd.hoff + h); s < __ldg(pd.hoff + h + 1); ++s) {
      const int src = __ldg(pd.hsrc + s);
      tot += src < 0 ? own : __ldcg(recv + ((long long)(src >> 24) * pd.maxh + (src & 0xffffff)) * NC + c);
    }
    sum.patch(n, c, tot);
  }
}

}  // namespace hx
