// hx_api.cu -- C-ABI of libb200hydro.so (declared in include/b200hydro.h).
//
// Host orchestration of the sm_100a kernels in hx_kernels.cuh: context setup
// (restriction maps, basis tables), operator handles, the device-resident
// momentum CG and the Lagrange step driver.  Every entry point cites the
// reference call it replaces in the header.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <type_traits>
#include <utility>
#include <memory>
#include <vector>

#include "../../include/b200hydro.h"
#include "hx_kernels.cuh"
#include "hx_brick.cuh"
#include "hx_rates.cuh"
#include "hx_remap.cuh"
#include "hx_tmop.cuh"
#include "hx_peer.cuh"
#include "hx_tma.cuh"
#include "hx_node.cuh"

using namespace hx;

struct hx_ctx {
  int dim, p, Q, D1, DT, nl, nq, nt;
  long long ne, nn;
  int device;
  bool brick = false;  // dofmap is a lexicographic brick (cartesian_mesh): structured CG path
  bool elem_major = false;  // brick CG E-vectors element-major (else node-sorted, CSR node pass)
  Brick bk{};
  cudaStream_t stream = 0;
  std::string err;
  long long launches = 0;
  // tables
  double *B = nullptr, *G = nullptr, *Bt = nullptr, *wnd = nullptr, *psi1 = nullptr;
  // restriction
  int *emap = nullptr, *off = nullptr, *idx = nullptr, *slot = nullptr;
  int* emapf = nullptr;      // packed CG element map (node | owner | mask) of the phase mask
  int* emapf_api = nullptr;  // the same for hx_mass_cg calls (rebuilt per call)
  uint8_t* own = nullptr;
  // workspaces
  double* evec = nullptr;     // (NE, nl, d)
  double* evec2 = nullptr;    // second E buffer (API scatter staging)
  double *r = nullptr, *z = nullptr, *p0 = nullptr, *p1 = nullptr;
  double* gamma_e = nullptr;  // per-element adiabatic index override (hx_set_material) or null
  char* arena = nullptr;      // CG working set: pairs, r, 1/diag, mask, x (dv0, dv1), E-vector, D_M
  size_t arena_bytes = 0;
  double* partials = nullptr; // reduction partials: two regions of preg doubles
  long long preg = 0;
  double* hist = nullptr;     // CG residual history
  int hist_len = 0;
  CGDev* cg = nullptr;        // [2]: stage-1 and stage-2 momentum solves
  StatusDev* st = nullptr;    // [4]: S, mid, new, scratch
  double* dt = nullptr;       // [2]
  double* scal = nullptr;     // small scalars
  // phase data
  bool phase = false;
  double* Dm = nullptr;       // (NE, nq)
  double* qd0 = nullptr;      // (NE, nq)
  double* minv = nullptr;     // (NE, nt, nt), or packed lower triangles (NE, nt (nt + 1) / 2)
  int minv_packed = 0;        // minv_packed<dim, p>(): the packed symmetric layout
  double* mdiag = nullptr;    // (NN)
  double* invd = nullptr;     // (NN, d)
  double* invdn = nullptr;    // (NN) 1/mass-diagonal per node (node passes read it with the mask)
  uint8_t* mask = nullptr;    // (NN, d) phase mask
  bool has_mask = false;
  // stage buffers for the step driver
  double *xm = nullptr, *vm = nullptr, *em = nullptr;
  double *dv0 = nullptr, *dv1 = nullptr, *de0 = nullptr, *de1 = nullptr;
  // TMA tensor maps over the CG pair buffers (p0, p1) per component count (k_mass_tma)
  CUtensorMap tm_pair[4][2];
  int tm_state[4] = {0, 0, 0, 0};  // 0 not built, 1 ok, -1 unavailable
  // host mirrors
  CGDev* h_cg = nullptr;
  StatusDev* h_st = nullptr;
  int* h_perr = nullptr;  // pinned copy of the peer-exchange error flag (pd.err)
  double* h_dt = nullptr;
  // live per-kernel-class timing (hx_prof_*): event pairs around instrumented launches
  bool prof_on = false;
  std::vector<cudaEvent_t> prof_ev;
  std::vector<int> prof_cls;
  int prof_used = 0;
  int prof_pending = 0;
  // graph-mode kernel timing by duplication (hx_prof_dup): a step graph in which every
  // launch of one kernel class is followed by a second, equivalent launch (the same
  // node; for the non-idempotent CG node pass a dry copy whose stores go to scratch).
  // The class's cost in the step is then (T_dup - T_plain) / (working duplicates),
  // measured with events around whole steps.  Each duplicate is tagged with its
  // (CG stage, iteration) so launches past convergence are not counted.
  struct GProf {
    std::vector<int> stage, iter;
  };
  bool prof_capture = false;
  int dup_class = -1;               // class duplicated in graphs captured now (-1: none)
  int prof_tag_stage = -1, prof_tag_iter = 0;
  GProf* gp = nullptr;              // the duplicating graph being captured
  double* dup_scratch = nullptr;    // dry node-pass outputs (x, r, pairs x2, partials)
  double prof_tot[8] = {0};
  long long prof_cnt[8] = {0};
  // CUDA-graph step path (one graph per buffer/parameter set)
  struct StepGraph {
    const void* key[6];
    double dt_fixed;
    hx_params prm;
    int seen = 0;
    int dup = -1;  // duplicated kernel class (hx_prof_dup), -1 for the plain graph
    std::shared_ptr<GProf> gprof;
    cudaGraphExec_t exec = nullptr;
  };
  std::vector<StepGraph> graphs;
  bool step_warm = false;
  cudaStream_t gstream = nullptr, gstream2 = nullptr;
  // single-GPU step graphs: external events marking x' and e' complete inside the graph, so
  // hx_step_host reads them back on its copy stream (created on first use) while stage 2 runs
  cudaStream_t cstream = nullptr;
  cudaEvent_t ev_x = nullptr, ev_e = nullptr, ev_v = nullptr;
  double* early_xh = nullptr;  // hx_step_host: host x', e' read back early (null: off)
  double* early_eh = nullptr;
  double* early_vh = nullptr;
  bool early_done = false;     // the last graph launch queued those reads
  double* t_dev = nullptr;
  double* h_t = nullptr;
  // host-buffer entry scratch (device state)
  double *hx_x = nullptr, *hx_v = nullptr, *hx_e = nullptr, *hx_xo = nullptr, *hx_vo = nullptr, *hx_eo = nullptr;
  // hx_step_host streamed inputs (brick, single GPU): x, v, e are copied in z-slabs on the
  // copy stream, each slab followed by a flag copy (= the call's epoch); the stage-1 rates
  // kernel waits per pass for the slab its elements need, so the H2D overlaps it
  unsigned long long* in_flag = nullptr;  // device: [in_ns] slab epochs, [in_ns] required epoch
  unsigned long long* h_in = nullptr;     // pinned: the epoch values copied
  unsigned long long* in_err_dev = nullptr;  // device view of h_in[HX_MAX_SLABS] (mapped): wait timed out
  unsigned long long in_epoch = 0;
  int in_ns = 0, in_ez = 0;               // slabs, layer-count key (-1: halving counts)
  std::vector<long long> in_node_end, in_elem_end;
  cudaStream_t istream = nullptr;        // the slab copies (own stream: independent of cstream's
                                        // read-backs, which wait on the step's events)
  const double *in_xh = nullptr, *in_vh = nullptr, *in_eh = nullptr;  // slabs still to enqueue
  // multi-GPU exchange (hx_peer_*): plan arrays + own mailbox; active once connected
  bool peer = false;
  PeerDev pd{};
  double* mailbox = nullptr;
  int* peer_plan = nullptr;      // snode|sdst|sidx|hnode|hoff|hsrc (one allocation)
  uint8_t* peer_owned = nullptr;
  unsigned long long* peer_ctr = nullptr;  // [0] seq, [1] err (as int)
  int* peer_ifx = nullptr;       // (NN) interface index
  PeerDev* pd_dev = nullptr;     // device copy read by the CG kernels
  PeerLite pl{};                 // prologue essentials passed by value
  int last_iters[2] = {0, 0};    // CG iterations of the last plain step's two solves (graph unroll)
};

static int issue_inputs(hx_ctx* ctx);

struct hx_mass {
  hx_ctx* ctx;
  double* D;  // (NE, nq)
};

struct hx_op {
  hx_ctx* ctx;
  int kind;   // 0 diffusion, 1 convection
  double* D;  // (NE, d, d, nq) / (NE, d, nq)
};

struct hx_force {
  hx_ctx* ctx;
  double* DF;  // (NE, d*d, nq)
};

struct hx_tmop {
  hx_ctx* ctx;
  double* winv = nullptr;   // (NE, nq, d, d)
  double* wdetw = nullptr;  // (NE, nq)
  double* x0 = nullptr;     // (NN, d)
  double* dlim = nullptr;   // (NN)
  double* nb0 = nullptr;    // (NN, d) node scratch: the mu part
  double* nb1 = nullptr;    // (NN, d) node scratch: limiting field / its assembled part
  double* epart = nullptr;  // (NE) per-element sums
  double* sums = nullptr;   // (2) device scalars
  int* bad = nullptr;       // det A <= 0 seen
  TmopMetric mt{1.0, 0.0, 0};
  double gamma = 0.0;
};

// ---------------------------------------------------------------------------
// helpers

static int fail(hx_ctx* c, int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (c) c->err = buf;
  return code;
}

#define CK(call)                                                                          \
  do {                                                                                    \
    cudaError_t _e = (call);                                                              \
    if (_e != cudaSuccess)                                                                \
      return fail(ctx, HX_ECUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(_e), \
                  __FILE__, __LINE__);                                                    \
  } while (0)

#define CKL()                                                                            \
  do {                                                                                   \
    ++ctx->launches;                                                                     \
    cudaError_t _e = cudaGetLastError();                                                 \
    if (_e != cudaSuccess)                                                               \
      return fail(ctx, HX_ECUDA, "kernel launch failed: %s (%s:%d)", cudaGetErrorString(_e), \
                  __FILE__, __LINE__);                                                   \
  } while (0)

template <typename T>
static cudaError_t dalloc(T** p, size_t n) {
  return cudaMalloc((void**)p, std::max<size_t>(n, 1) * sizeof(T));
}

static inline unsigned gblocks(long long n, int nt) { return (unsigned)((n + nt - 1) / nt); }

enum { K_RATES = 0, K_MASS = 1, K_CGNODE = 2, K_CGINIT = 3, K_AXPY = 4, K_VALID = 5, K_OTHER = 6 };

static void prof_collect(hx_ctx* c) {
  if (c->prof_used == 0) return;
  cudaEventSynchronize(c->prof_ev[2 * c->prof_used - 1]);
  for (int i = 0; i < c->prof_used; ++i) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, c->prof_ev[2 * i], c->prof_ev[2 * i + 1]);
    c->prof_tot[c->prof_cls[i]] += ms;
    c->prof_cnt[c->prof_cls[i]] += 1;
  }
  c->prof_used = 0;
}

static int dup_last_node(hx_ctx* c, int cls);

// after a duplicating graph's launch: count the duplicates that did work (CG launches of
// iteration k > the stage's iteration count exit at once)
static void gprof_collect(hx_ctx* c, const hx_ctx::GProf* g, const int* stage_iters) {
  for (size_t i = 0; i < g->stage.size(); ++i) {
    const int st = g->stage[i], k = g->iter[i];
    if (st >= 0 && k > 0 && k > stage_iters[st]) continue;
    c->prof_cnt[c->dup_class] += 1;
  }
}

static void prof_begin(hx_ctx* c, int cls) {
  if (c->prof_capture) {
    c->prof_pending = cls;
    return;
  }
  if (!c->prof_on) return;
  if ((size_t)(2 * c->prof_used + 2) > c->prof_ev.size()) prof_collect(c);
  cudaEventRecord(c->prof_ev[2 * c->prof_used], c->stream);
  c->prof_pending = cls;
}

static void prof_end(hx_ctx* c) {
  if (c->prof_capture) {
    // duplicate on the outer capture stream only (a WHILE body takes no duplicates)
    if (c->prof_pending == c->dup_class && c->stream == c->gstream && c->gp &&
        dup_last_node(c, c->prof_pending) == HX_OK) {
      c->gp->stage.push_back(c->prof_tag_stage);
      c->gp->iter.push_back(c->prof_tag_iter);
    }
    return;
  }
  if (!c->prof_on) return;
  cudaEventRecord(c->prof_ev[2 * c->prof_used + 1], c->stream);
  c->prof_cls[c->prof_used] = c->prof_pending;
  ++c->prof_used;
}

// HX_GRID_CAP=n caps every persistent grid at n CTAs (test hook: small meshes then take
// the multi-pass paths of the persistent kernels that production sizes take)
static long long grid_cap() {
  static long long cap = -1;
  if (cap < 0) {
    const char* v = getenv("HX_GRID_CAP");
    cap = v ? std::max(0ll, atoll(v)) : 0;
  }
  return cap;
}

static unsigned capg(unsigned g) {
  return grid_cap() > 0 ? (unsigned)std::max(1ll, std::min<long long>(g, grid_cap())) : g;
}

// resident-capacity grid for persistent kernels (SMs x max resident blocks)
template <typename K>
static unsigned persistent_grid(K kernel, int threads, size_t smem, long long work_blocks) {
  static int sms = 0;
  if (!sms) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int per = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kernel, threads, smem);
  long long g = (long long)std::max(per, 1) * sms;
  if (grid_cap() > 0) g = std::min(g, grid_cap());
  return (unsigned)std::max<long long>(1, std::min<long long>(g, work_blocks));
}

static Tables tables(const hx_ctx* c) { return Tables{c->B, c->G, c->Bt, c->wnd, c->psi1}; }

template <typename K>
static cudaError_t smem_attr(K kernel, size_t bytes) {
  if (bytes > 48 * 1024) return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  return cudaSuccess;
}

// run a functor templated on <DIM, P> for the context's discretisation
template <template <int, int> class F, typename... Args>
static int dispatch(hx_ctx* ctx, Args&&... args) {
  switch (ctx->dim * 10 + ctx->p) {
    case 21: return F<2, 1>::run(ctx, args...);
    case 22: return F<2, 2>::run(ctx, args...);
    case 23: return F<2, 3>::run(ctx, args...);
    case 24: return F<2, 4>::run(ctx, args...);
    case 31: return F<3, 1>::run(ctx, args...);
    case 32: return F<3, 2>::run(ctx, args...);
    case 33: return F<3, 3>::run(ctx, args...);
    case 34: return F<3, 4>::run(ctx, args...);
  }
  return fail(ctx, HX_EINVAL, "unsupported discretisation dim=%d p=%d", ctx->dim, ctx->p);
}

static constexpr int RATES_NT = 128;

// ---------------------------------------------------------------------------
// launchers

static int g_rates_kernel = -1;  // HX_RATES=cta: the CTA-per-element rates kernel for 3D

template <int P, int MODE>
static int launch_rates_pc(hx_ctx* ctx, const RatesPCArgs& a) {
  using R = RatesPC<P>;
  auto k = k_rates_pc<P, MODE>;
  static bool attr = false;
  if (!attr) {
    CK(smem_attr(k, R::bytes));
    attr = true;
  }
  static unsigned grid = 0;
  if (!grid) grid = persistent_grid(k, R::THREADS, R::bytes, 1ll << 40);
  prof_begin(ctx, MODE == 0 ? K_RATES : (MODE == 2 ? K_OTHER : K_VALID));
  k<<<std::min(grid, gblocks(ctx->ne, R::EPC)), R::THREADS, R::bytes, ctx->stream>>>(a);
  prof_end(ctx);
  CKL();
  return HX_OK;
}

template <int P>
static int launch_valid(hx_ctx* ctx, const RatesPCArgs& a) {
  using V = ValidCfg<P>;
  auto k = k_valid<P>;
  static bool attr = false;
  if (!attr) {
    CK(smem_attr(k, V::bytes));
    attr = true;
  }
  static unsigned grid = 0;
  if (!grid) grid = persistent_grid(k, V::NT, V::bytes, 1ll << 40);
  prof_begin(ctx, K_VALID);
  k<<<std::min(grid, gblocks(ctx->ne, V::EPC)), V::NT, V::bytes, ctx->stream>>>(a);
  prof_end(ctx);
  CKL();
  return HX_OK;
}

template <int DIM, int P>
struct LaunchRates {
  static int run(hx_ctx* ctx, const double* x, const double* v, const double* e, double* evec, double* de,
                 StatusDev* st, int mode, double gamma, double q1, double q2) {
    if (g_rates_kernel < 0) {
      const char* s = getenv("HX_RATES");
      g_rates_kernel = (s && strcmp(s, "cta") == 0) ? 0 : 1;
    }
    if constexpr (DIM == 3 && P >= 2) {
      if (g_rates_kernel == 1) {
        RatesPCArgs a{x, v, e, ctx->qd0, ctx->emap, ctx->elem_major ? nullptr : ctx->slot, ctx->minv, ctx->wnd,
                      ctx->psi1, gamma, q1, q2, ctx->gamma_e, ctx->ne, evec, de, st, ctx->bk, ctx->brick ? 1 : 0};
        if (mode == 0 && ctx->in_ns > 0 && x == ctx->hx_x && ctx->brick && !ctx->peer) {
          a.inflag = ctx->in_flag;  // hx_step_host's streamed inputs (a no-op wait otherwise)
          a.inerr = ctx->in_err_dev;
          a.in_ns = ctx->in_ns;
        }
        // the lean validity kernel is measured faster for p <= 3 (p = 2: 44 vs 51 us,
        // p = 3: 35 vs 40); at p = 4 its images cap it at 2 CTAs/SM and the rates kernel's
        // geometry-only mode wins (54 vs 89 us)
        if (mode == 0) return launch_rates_pc<P, 0>(ctx, a);
        if (mode == 2) return launch_rates_pc<P, 2>(ctx, a);
        return P <= 3 ? launch_valid<P>(ctx, a) : launch_rates_pc<P, 1>(ctx, a);
      }
    }
    using SM = RatesSmem<DIM, P>;
    auto kern = k_rates<DIM, P, RATES_NT>;
    static bool attr = false;
    if (!attr) {
      CK(smem_attr(kern, SM::bytes));
      attr = true;
    }
    RatesArgs a{x, v, e, ctx->qd0, ctx->emap, ctx->elem_major ? nullptr : ctx->slot, ctx->minv, tables(ctx), gamma, q1, q2,
                ctx->gamma_e, ctx->ne, evec, de, st, mode};
    prof_begin(ctx, mode == 0 ? K_RATES : K_VALID);
    kern<<<(unsigned)ctx->ne, RATES_NT, SM::bytes, ctx->stream>>>(a);
    prof_end(ctx);
    CKL();
    return HX_OK;
  }
};

template <int P, int NC, int MINB>
static int launch_mass3w_b(hx_ctx* ctx, bool cgmode, const MassArgs& a) {
  using M = Mass3W<P, NC>;
  if (cgmode) {
    auto k = k_mass3w<P, NC, true, MINB>;
    CK(smem_attr(k, M::bytes));
    static unsigned grid = 0;
    if (!grid) grid = persistent_grid(k, 32 * M::WPB, M::bytes, 1ll << 40);
    prof_begin(ctx, K_MASS);
    k<<<std::min<unsigned>(grid, gblocks(ctx->ne, M::WPB)), 32 * M::WPB, M::bytes, ctx->stream>>>(a);
    prof_end(ctx);
  } else {
    auto k = k_mass3w<P, NC, false, MINB>;
    CK(smem_attr(k, M::bytes));
    static unsigned grid = 0;
    if (!grid) grid = persistent_grid(k, 32 * M::WPB, M::bytes, 1ll << 40);
    k<<<std::min<unsigned>(grid, gblocks(ctx->ne, M::WPB)), 32 * M::WPB, M::bytes, ctx->stream>>>(a);
  }
  CKL();
  return HX_OK;
}

static int g_mass_minb = -1;  // HX_MASS_MINB: resident-block target of k_mass3w (register cap)

template <int P, int NC>
static int launch_mass3w(hx_ctx* ctx, bool cgmode, const MassArgs& a) {
  if (g_mass_minb < 0) {
    const char* v = getenv("HX_MASS_MINB");
    g_mass_minb = v ? atoi(v) : 4;
  }
  if (g_mass_minb >= 5 && P <= 3) return launch_mass3w_b<P, NC, 5>(ctx, cgmode, a);
  if (g_mass_minb <= 3 || P >= 4) return launch_mass3w_b<P, NC, 3>(ctx, cgmode, a);
  return launch_mass3w_b<P, NC, 4>(ctx, cgmode, a);
}

template <int P, int NC>
static int launch_mass_pc(hx_ctx* ctx, bool cgmode, const MassArgs& a) {
  using M = MassPC<P, NC>;
  const unsigned work = gblocks(ctx->ne, M::EPC);
  if (cgmode) {
    auto k = k_mass_pc<P, NC, true>;
    CK(smem_attr(k, M::bytes));
    static unsigned grid = 0;
    if (!grid) grid = persistent_grid(k, 128, M::bytes, 1ll << 40);
    prof_begin(ctx, K_MASS);
    k<<<std::min(grid, work), 128, M::bytes, ctx->stream>>>(a);
    prof_end(ctx);
  } else {
    auto k = k_mass_pc<P, NC, false>;
    CK(smem_attr(k, M::bytes));
    static unsigned grid = 0;
    if (!grid) grid = persistent_grid(k, 128, M::bytes, 1ll << 40);
    k<<<std::min(grid, work), 128, M::bytes, ctx->stream>>>(a);
  }
  CKL();
  return HX_OK;
}

static int g_mass_variant = -1;  // HX_MASS_KERNEL=line|pc (generic 3D meshes; default pc for p<=3)

template <int P, int NC>
static int launch_mass3d(hx_ctx* ctx, bool cgmode, const MassArgs& a) {
  if (g_mass_variant < 0) {
    const char* v = getenv("HX_MASS_KERNEL");
    g_mass_variant = 2;
    if (v && strcmp(v, "line") == 0) g_mass_variant = 1;
  }
  if (g_mass_variant >= 2 && P <= 3) return launch_mass_pc<P, NC>(ctx, cgmode, a);
  return launch_mass3w<P, NC>(ctx, cgmode, a);
}

template <int DIM, int P>
struct LaunchMass {
  static int run(hx_ctx* ctx, int nc, bool cgmode, const MassArgs& a) {
    using D = Disc<DIM, P>;
    if constexpr (DIM == 3) {
      if (nc == 1) return launch_mass3d<P, 1>(ctx, cgmode, a);
      if (nc == 2) return launch_mass3d<P, 2>(ctx, cgmode, a);
      if (nc == 3) return launch_mass3d<P, 3>(ctx, cgmode, a);
    }
    const unsigned grid = gblocks(ctx->ne, 4);
    const size_t bytes = sizeof(double) * (D::Q * D::D1 + 4 * 2 * nc * D::NQ);
#define HX_MASS_CASE(NC)                                                              \
  if (nc == NC) {                                                                     \
    if (cgmode) {                                                                     \
      auto k = k_mass<DIM, P, NC, true>;                                              \
      CK(smem_attr(k, bytes));                                                        \
      prof_begin(ctx, K_MASS);                                                        \
      k<<<grid, 128, bytes, ctx->stream>>>(a);                                        \
      prof_end(ctx);                                                                  \
    } else {                                                                          \
      auto k = k_mass<DIM, P, NC, false>;                                             \
      CK(smem_attr(k, bytes));                                                        \
      k<<<grid, 128, bytes, ctx->stream>>>(a);                                        \
    }                                                                                 \
    CKL();                                                                            \
    return HX_OK;                                                                     \
  }
    HX_MASS_CASE(1)
    HX_MASS_CASE(2)
    HX_MASS_CASE(3)
#undef HX_MASS_CASE
    return fail(ctx, HX_EINVAL, "ncomp must be 1..3");
  }
};

template <int DIM, int P>
struct LaunchMassDiag {
  static int run(hx_ctx* ctx, const double* D, double* evec) {
    k_mass_diag<DIM, P><<<gblocks(ctx->ne, 4), 128, 0, ctx->stream>>>(D, ctx->B, ctx->slot, ctx->ne, evec);
    CKL();
    return HX_OK;
  }
};

template <int DIM, int P>
struct LaunchGeom {
  static int run(hx_ctx* ctx, const GeomArgs& a) {
    using SM = GeomSmem<DIM, P>;
    auto k = k_geom<DIM, P, 128>;
    CK(smem_attr(k, SM::bytes));
    k<<<(unsigned)ctx->ne, 128, SM::bytes, ctx->stream>>>(a);
    CKL();
    return HX_OK;
  }
};

template <int DIM, int P>
struct LaunchStress {
  static int run(hx_ctx* ctx, const StressArgs& a) {
    using SM = RatesSmem<DIM, P>;
    auto k = k_stress<DIM, P, 128>;
    CK(smem_attr(k, SM::bytes));
    k<<<(unsigned)ctx->ne, 128, SM::bytes, ctx->stream>>>(a);
    CKL();
    return HX_OK;
  }
};

template <int DIM, int P>
struct LaunchForce {
  static int run(hx_ctx* ctx, const ForceArgs& a, bool trans) {
    using SM = ForceSmem<DIM, P>;
    if (trans) {
      auto k = k_force<DIM, P, 128, true>;
      CK(smem_attr(k, SM::bytes));
      k<<<(unsigned)ctx->ne, 128, SM::bytes, ctx->stream>>>(a);
    } else {
      auto k = k_force<DIM, P, 128, false>;
      CK(smem_attr(k, SM::bytes));
      k<<<(unsigned)ctx->ne, 128, SM::bytes, ctx->stream>>>(a);
    }
    CKL();
    return HX_OK;
  }
};

template <int DIM, int P>
struct LaunchMinv {
  static int run(hx_ctx* ctx, double* minv_ref) {
    using D = Disc<DIM, P>;
    if constexpr (minv_packed<DIM, P>()) {  // k_minv_warp writes the packed layout
      constexpr int Q = P + 2, DT = P;
      const size_t wb = sizeof(double) * 8 * (D::NQ + DT * DT * Q * Q + DT * DT * DT * DT * Q);
      auto kw = k_minv_warp<P>;
      CK(smem_attr(kw, wb));
      kw<<<capg(std::min<unsigned>(gblocks(ctx->ne, 8), 148 * 8)), 256, wb, ctx->stream>>>(ctx->Dm, ctx->ne, ctx->minv,
                                                                                     minv_ref);
      CKL();
      return HX_OK;
    }
    const size_t bytes = sizeof(double) * (D::NT * 2 * D::NT + D::NQ * D::NT);
    auto k = k_minv<DIM, P>;
    CK(smem_attr(k, bytes));
    k<<<(unsigned)ctx->ne, 128, bytes, ctx->stream>>>(ctx->Dm, ctx->Bt, ctx->ne, ctx->minv, minv_ref);
    CKL();
    return HX_OK;
  }
};

template <int DIM, int P>
struct LaunchIE {
  static int run(hx_ctx* ctx, const double* e, const double* qd0, double* per_elem) {
    k_internal_energy<DIM, P><<<gblocks(ctx->ne, 4), 128, 0, ctx->stream>>>(e, qd0, ctx->Bt, ctx->wnd, ctx->ne,
                                                                            per_elem);
    CKL();
    return HX_OK;
  }
};

// scatter (internal E layout) with 1..3 comps
static int launch_scatter(hx_ctx* ctx, const double* evec, int nc, double* out) {
  NodeArgs a{};
  a.off = ctx->off;
  a.idx = ctx->idx;
  a.evec = evec;
  a.out = out;
  a.nn = ctx->nn;
  const unsigned g = gblocks(ctx->nn, 256);
  if (nc == 1) k_scatter<1><<<g, 256, 0, ctx->stream>>>(a);
  else if (nc == 2) k_scatter<2><<<g, 256, 0, ctx->stream>>>(a);
  else k_scatter<3><<<g, 256, 0, ctx->stream>>>(a);
  CKL();
  return HX_OK;
}

static int status_reset(hx_ctx* ctx, StatusDev* st, int n = 1) {
  k_status_reset<<<1, 32, 0, ctx->stream>>>(st, n);
  CKL();
  return HX_OK;
}

// host-side pinned staging for StatusDev resets (cudaMemcpyAsync from stack memory
// is synchronous for pageable memory, which is fine for correctness)

static void decode_inv(const hx_ctx* ctx, unsigned long long key, hx_inverted* inv) {
  if (!inv) return;
  if (key == ~0ull) {
    inv->inverted = 0;
    return;
  }
  inv->inverted = 1;
  inv->point = (int64_t)(key / (unsigned long long)ctx->ne);
  inv->element = (int64_t)(key % (unsigned long long)ctx->ne);
  inv->detj = NAN;
}

// ---------------------------------------------------------------------------
// context

extern "C" int hx_create(const hx_mesh_desc* d, hx_ctx** out) {
  hx_ctx* ctx = nullptr;
  if (!d || !out) return HX_EINVAL;
  *out = nullptr;
  if (d->dim != 2 && d->dim != 3) return HX_EINVAL;
  if (d->order < 1 || d->order > 4) return HX_EINVAL;
  if (d->q1d != d->order + 2) return HX_EINVAL;
  if (d->thermo_order != std::max(d->order - 1, 0)) return HX_EINVAL;
  if (d->num_elements < 1 || d->num_nodes < 1) return HX_EINVAL;
  ctx = new hx_ctx();
  ctx->dim = d->dim;
  ctx->p = d->order;
  ctx->D1 = d->order + 1;
  ctx->Q = d->q1d;
  ctx->DT = std::max(d->order, 1);
  ctx->nl = (int)std::pow(ctx->D1, ctx->dim);
  ctx->nq = (int)std::pow(ctx->Q, ctx->dim);
  ctx->nt = (int)std::pow(ctx->DT, ctx->dim);
  ctx->ne = d->num_elements;
  ctx->nn = d->num_nodes;
  ctx->device = d->device;
  if (ctx->nn >= (1ll << 27) || (long long)ctx->ne * ctx->nl >= (1ll << 31)) {
    int rc = fail(ctx, HX_EINVAL, "mesh too large for 27-bit node ids / 32-bit E-vector indices (split it across ranks)");
    delete ctx;
    return rc;
  }
  cudaError_t ce = cudaSetDevice(d->device);
  if (ce != cudaSuccess) {
    delete ctx;
    return HX_ECUDA;
  }
  const int nl = ctx->nl, nq = ctx->nq, Q = ctx->Q, D1 = ctx->D1, DT = ctx->DT;
  const long long ne = ctx->ne, nn = ctx->nn;
  // restriction maps
  std::vector<int> emap((size_t)ne * nl);
  std::vector<int> cnt(nn + 1, 0);
  for (long long e = 0; e < ne; ++e)
    for (int l = 0; l < nl; ++l) {
      const long long n = d->dofmap_host[(long long)l * ne + e];
      if (n < 0 || n >= nn) {
        int rc = fail(ctx, HX_EINVAL, "dofmap entry %lld out of range", n);
        delete ctx;
        return rc;
      }
      emap[e * nl + l] = (int)n;
      cnt[n + 1]++;
    }
  // structured brick? (cartesian_mesh numbering, fespace.py:352-385)
  if (ctx->dim == 3 && ctx->p >= 2) {
    const int p = ctx->p;
    const long long n1 = emap[p], n2 = emap[p * D1], n3 = emap[p * D1 * D1];
    bool ok = emap[0] == 0 && n1 == p && n2 % p == 0 && n3 % p == 0 && n2 > 0 && n3 > 0;
    long long Nx = ok ? n2 / p : 0, NxNy = ok ? n3 / p : 0;
    ok = ok && Nx > 1 && NxNy % Nx == 0 && (Nx - 1) % p == 0;
    long long Ny = ok ? NxNy / Nx : 0;
    ok = ok && Ny > 1 && (Ny - 1) % p == 0;
    const long long bx = ok ? (Nx - 1) / p : 1, by = ok ? (Ny - 1) / p : 1;
    ok = ok && ne % (bx * by) == 0;
    const long long bz = ok ? ne / (bx * by) : 1;
    ok = ok && nn == NxNy * (bz * p + 1);
    for (long long e = 0; ok && e < ne; ++e) {
      const long long ez = e / (bx * by), ey = (e / bx) % by, ex = e % bx;
      for (int l = 0; l < nl; ++l) {
        const int dx = l % D1, dy = (l / D1) % D1, dz = l / (D1 * D1);
        const long long want = (ex * p + dx) + Nx * (ey * p + dy) + NxNy * (ez * p + dz);
        if (emap[e * nl + l] != want) {
          ok = false;
          break;
        }
      }
    }
    ok = ok && (long long)ne * nl * 3 < (1ll << 31);  // 32-bit element-major E offsets
    const char* env = getenv("HX_BRICK");
    if (env && env[0] == '0') ok = false;
    if (ok) {
      ctx->brick = true;
      const char* ev = getenv("HX_EVEC");  // HX_EVEC=sorted: node-sorted E with the brick mass kernel
      ctx->elem_major = !(ev && strcmp(ev, "sorted") == 0);
      ctx->bk = Brick{(int)bx, (int)by, (int)bz, (int)Nx, (int)Ny, NxNy, make_fastdiv((unsigned)bx),
                      make_fastdiv((unsigned)(bx * by)), make_fastdiv((unsigned)Nx), make_fastdiv((unsigned)NxNy),
                      nl - p, (int)bx * nl - p * D1, (int)(bx * by) * nl - p * D1 * D1};
    }
  }
  std::vector<int> off(nn + 1, 0);
  for (long long n = 0; n < nn; ++n) off[n + 1] = off[n] + cnt[n + 1];
  std::vector<int> fill(off.begin(), off.end() - 1);
  std::vector<int> idx((size_t)ne * nl);
  std::vector<uint8_t> own((size_t)ne * nl, 0);
  std::vector<int> slot((size_t)ne * nl);
  for (long long e = 0; e < ne; ++e)  // ascending element => deterministic accumulation order
    for (int l = 0; l < nl; ++l) {
      const int n = emap[e * nl + l];
      if (fill[n] == off[n]) own[e * nl + l] = 1;
      slot[e * nl + l] = fill[n];
      idx[fill[n]++] = (int)(e * nl + l);
    }
  // tables: tensor weights (x fastest) and the thermodynamic interpolant of 1
  std::vector<double> wnd(nq), psi1(nq);
  for (int q = 0; q < nq; ++q) {
    int qq = q;
    double w = 1.0;
    std::vector<int> dig(ctx->dim);
    for (int a = 0; a < ctx->dim; ++a) {
      dig[a] = qq % Q;
      qq /= Q;
    }
    // weights: np.multiply.outer chain -> w[q_slowest] * ... * w[q_fastest]
    w = d->qweights_host[dig[ctx->dim - 1]];
    for (int a = ctx->dim - 2; a >= 0; --a) w *= d->qweights_host[dig[a]];
    wnd[q] = w;
  }
  {
    // psi1 = tensor_interp(Bt, ones): per axis sum_j Bt[q, j]
    std::vector<double> rowsum(Q);
    for (int q = 0; q < Q; ++q) {
      double s = 0.0;
      for (int j = 0; j < DT; ++j) s += d->Bt_host[q * DT + j];
      rowsum[q] = s;
    }
    for (int q = 0; q < nq; ++q) {
      int qq = q;
      double v = 1.0;
      for (int a = 0; a < ctx->dim; ++a) {
        v *= rowsum[qq % Q];
        qq /= Q;
      }
      psi1[q] = v;
    }
  }
  const int dd = ctx->dim;
  const size_t nv = (size_t)nn * dd;
  bool ok = true;
  ok &= dalloc(&ctx->B, Q * D1) == cudaSuccess;
  ok &= dalloc(&ctx->G, Q * D1) == cudaSuccess;
  ok &= dalloc(&ctx->Bt, Q * DT) == cudaSuccess;
  ok &= dalloc(&ctx->wnd, nq) == cudaSuccess;
  ok &= dalloc(&ctx->psi1, nq) == cudaSuccess;
  ok &= dalloc(&ctx->emap, (size_t)ne * nl) == cudaSuccess;
  ok &= dalloc(&ctx->off, nn + 1) == cudaSuccess;
  ok &= dalloc(&ctx->idx, (size_t)ne * nl) == cudaSuccess;
  ok &= dalloc(&ctx->own, (size_t)ne * nl) == cudaSuccess;
  ok &= dalloc(&ctx->slot, (size_t)ne * nl + 8) == cudaSuccess;
  {
    // CG working set in one arena (L2 persisting access window over it, see l2_window)
    auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
    const size_t sizes[] = {al(16 * nv), al(16 * nv), al(8 * nv), al(8 * nv), al(nv), al(8 * nv), al(8 * nv),
                            al(8 * (size_t)ne * nl * dd), al(8 * ((size_t)ne * nq + 8))};
    size_t tot = 0;
    for (size_t s : sizes) tot += s;
    char* base = nullptr;
    ok &= cudaMalloc(&base, tot) == cudaSuccess;
    ctx->arena = base;
    ctx->arena_bytes = tot;
    if (base) {
      char* q = base;
      ctx->p0 = (double*)q; q += sizes[0];
      ctx->p1 = (double*)q; q += sizes[1];
      ctx->r = (double*)q; q += sizes[2];
      ctx->invd = (double*)q; q += sizes[3];
      ctx->mask = (uint8_t*)q; q += sizes[4];
      ctx->dv0 = (double*)q; q += sizes[5];
      ctx->dv1 = (double*)q; q += sizes[6];
      ctx->evec = (double*)q; q += sizes[7];
      ctx->Dm = (double*)q;
    }
  }
  ok &= dalloc(&ctx->evec2, (size_t)ne * std::max(nl * dd, nq)) == cudaSuccess;
  ok &= dalloc(&ctx->z, nv) == cudaSuccess;
  ok &= dalloc(&ctx->emapf, (size_t)ne * nl + 8) == cudaSuccess;
  ok &= dalloc(&ctx->emapf_api, (size_t)ne * nl + 8) == cudaSuccess;
  ctx->preg = 2 * std::max<long long>(gblocks(3 * nn, 256), gblocks(ne, 1)) + 64;
  ok &= dalloc(&ctx->partials, 2 * (size_t)ctx->preg) == cudaSuccess;
  ok &= dalloc(&ctx->cg, 2) == cudaSuccess;
  ok &= dalloc(&ctx->t_dev, 2) == cudaSuccess;  // {t, caller-given dt} for the step graphs
  ok &= cudaMallocHost((void**)&ctx->h_t, 2 * sizeof(double)) == cudaSuccess;
  ok &= cudaStreamCreateWithFlags(&ctx->gstream, cudaStreamNonBlocking) == cudaSuccess;
  ok &= cudaStreamCreateWithFlags(&ctx->gstream2, cudaStreamNonBlocking) == cudaSuccess;
  for (cudaEvent_t* ev : {&ctx->ev_x, &ctx->ev_e, &ctx->ev_v})
    ok &= cudaEventCreateWithFlags(ev, cudaEventDisableTiming) == cudaSuccess;
  ok &= dalloc(&ctx->st, 4) == cudaSuccess;
  ok &= dalloc(&ctx->dt, 2) == cudaSuccess;
  ok &= dalloc(&ctx->scal, 16) == cudaSuccess;
  ok &= dalloc(&ctx->qd0, (size_t)ne * nq) == cudaSuccess;
  ctx->minv_packed = (ctx->dim == 3 && ctx->p <= 3) ? 1 : 0;  // == minv_packed<DIM, P>()
  ok &= dalloc(&ctx->minv, (size_t)ne * (ctx->minv_packed ? tri(ctx->nt) : ctx->nt * ctx->nt)) == cudaSuccess;
  ok &= dalloc(&ctx->mdiag, nn) == cudaSuccess;
  ok &= dalloc(&ctx->invdn, nn) == cudaSuccess;
  ok &= dalloc(&ctx->xm, nv) == cudaSuccess;
  ok &= dalloc(&ctx->vm, nv) == cudaSuccess;
  ok &= dalloc(&ctx->em, (size_t)ne * ctx->nt) == cudaSuccess;
  ok &= dalloc(&ctx->de0, (size_t)ne * ctx->nt) == cudaSuccess;
  ok &= dalloc(&ctx->de1, (size_t)ne * ctx->nt) == cudaSuccess;
  ok &= cudaMallocHost((void**)&ctx->h_cg, 2 * sizeof(CGDev)) == cudaSuccess;
  ok &= cudaMallocHost((void**)&ctx->h_st, 4 * sizeof(StatusDev)) == cudaSuccess;
  ok &= cudaMallocHost((void**)&ctx->h_dt, 2 * sizeof(double)) == cudaSuccess;
  ok &= cudaMallocHost((void**)&ctx->h_perr, sizeof(int)) == cudaSuccess;
  if (ok) *ctx->h_perr = 0;
  if (!ok) {
    int rc = fail(ctx, HX_ECUDA, "device allocation failed");
    hx_destroy(ctx);
    return rc;
  }
  ok &= cudaMemcpy(ctx->B, d->B_host, sizeof(double) * Q * D1, cudaMemcpyHostToDevice) == cudaSuccess;
  ok &= cudaMemcpy(ctx->G, d->G_host, sizeof(double) * Q * D1, cudaMemcpyHostToDevice) == cudaSuccess;
  ok &= cudaMemcpy(ctx->Bt, d->Bt_host, sizeof(double) * Q * DT, cudaMemcpyHostToDevice) == cudaSuccess;
  ok &= cudaMemcpy(ctx->wnd, wnd.data(), sizeof(double) * nq, cudaMemcpyHostToDevice) == cudaSuccess;
  ok &= cudaMemcpy(ctx->psi1, psi1.data(), sizeof(double) * nq, cudaMemcpyHostToDevice) == cudaSuccess;
  ok &= cudaMemcpy(ctx->emap, emap.data(), sizeof(int) * emap.size(), cudaMemcpyHostToDevice) == cudaSuccess;
  ok &= cudaMemcpy(ctx->off, off.data(), sizeof(int) * off.size(), cudaMemcpyHostToDevice) == cudaSuccess;
  ok &= cudaMemcpy(ctx->idx, idx.data(), sizeof(int) * idx.size(), cudaMemcpyHostToDevice) == cudaSuccess;
  ok &= cudaMemcpy(ctx->own, own.data(), own.size(), cudaMemcpyHostToDevice) == cudaSuccess;
  ok &= cudaMemcpy(ctx->slot, slot.data(), sizeof(int) * slot.size(), cudaMemcpyHostToDevice) == cudaSuccess;
  ok &= cudaMemset(ctx->cg, 0, 2 * sizeof(CGDev)) == cudaSuccess;
  ok &= cudaMemset(ctx->mask, 0, nv) == cudaSuccess;
  {
    // fixed per-order tables in the constant bank (k_mass3d); all contexts of one
    // order must agree on them
    static std::vector<double> seen[4];
    std::vector<double> tb(d->B_host, d->B_host + Q * D1);
    if (!seen[ctx->p - 1].empty() && seen[ctx->p - 1] != tb) {
      int rc = fail(ctx, HX_EINVAL, "basis tables for order %d differ from an existing context", ctx->p);
      hx_destroy(ctx);
      return rc;
    }
    seen[ctx->p - 1] = tb;
    ok &= cudaMemcpyToSymbol(c_B, tb.data(), sizeof(double) * tb.size(), sizeof(double) * 30 * (ctx->p - 1)) ==
          cudaSuccess;
    ok &= cudaMemcpyToSymbol(c_Bt, d->Bt_host, sizeof(double) * Q * DT, sizeof(double) * 30 * (ctx->p - 1)) ==
          cudaSuccess;
    ok &= cudaMemcpyToSymbol(c_G, d->G_host, sizeof(double) * Q * D1, sizeof(double) * 30 * (ctx->p - 1)) ==
          cudaSuccess;
  }
  if (!ok) {
    int rc = fail(ctx, HX_ECUDA, "device upload failed");
    hx_destroy(ctx);
    return rc;
  }
  *out = ctx;
  return HX_OK;
}

extern "C" int hx_destroy(hx_ctx* ctx) {
  if (!ctx) return HX_OK;
  cudaSetDevice(ctx->device);
  void* dev[] = {ctx->B,  ctx->G,    ctx->Bt,   ctx->wnd,  ctx->psi1, ctx->emap, ctx->off,   ctx->idx,
                 ctx->own, ctx->slot, ctx->emapf, ctx->emapf_api, ctx->arena, ctx->evec2, ctx->z, ctx->partials,
                 ctx->hist, ctx->cg,  ctx->st,   ctx->dt,   ctx->scal, ctx->qd0,   ctx->minv, ctx->invdn,
                 ctx->mdiag, ctx->xm, ctx->vm,   ctx->em, ctx->gamma_e,
                 ctx->de0, ctx->de1, ctx->hx_x, ctx->hx_v, ctx->hx_e, ctx->hx_xo, ctx->hx_vo, ctx->hx_eo,
                 ctx->in_flag};
  for (void* p : dev)
    if (p) cudaFree(p);
  if (ctx->h_cg) cudaFreeHost(ctx->h_cg);
  if (ctx->h_st) cudaFreeHost(ctx->h_st);
  if (ctx->h_perr) cudaFreeHost(ctx->h_perr);
  if (ctx->dup_scratch) cudaFree(ctx->dup_scratch);
  if (ctx->h_dt) cudaFreeHost(ctx->h_dt);
  if (ctx->h_t) cudaFreeHost(ctx->h_t);
  if (ctx->h_in) cudaFreeHost(ctx->h_in);
  if (ctx->t_dev) cudaFree(ctx->t_dev);
  for (auto& g : ctx->graphs)
    if (g.exec) cudaGraphExecDestroy(g.exec);
  if (ctx->gstream) cudaStreamDestroy(ctx->gstream);
  if (ctx->gstream2) cudaStreamDestroy(ctx->gstream2);
  if (ctx->cstream) cudaStreamDestroy(ctx->cstream);
  if (ctx->istream) cudaStreamDestroy(ctx->istream);
  for (cudaEvent_t ev : {ctx->ev_x, ctx->ev_e, ctx->ev_v})
    if (ev) cudaEventDestroy(ev);
  for (auto& e : ctx->prof_ev) cudaEventDestroy(e);
  if (ctx->mailbox) cudaFree(ctx->mailbox);
  if (ctx->peer_plan) cudaFree(ctx->peer_plan);
  if (ctx->peer_owned) cudaFree(ctx->peer_owned);
  if (ctx->peer_ctr) cudaFree(ctx->peer_ctr);
  if (ctx->peer_ifx) cudaFree(ctx->peer_ifx);
  if (ctx->pd_dev) cudaFree(ctx->pd_dev);
  delete ctx;
  return HX_OK;
}

extern "C" int hx_set_stream(hx_ctx* ctx, void* stream) {
  if (!ctx) return HX_EINVAL;
  ctx->stream = (cudaStream_t)stream;
  return HX_OK;
}

extern "C" const char* hx_last_error(hx_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }
extern "C" int64_t hx_kernel_launches(hx_ctx* ctx) { return ctx ? ctx->launches : 0; }
extern "C" int hx_layout(hx_ctx* ctx) { return ctx && ctx->brick ? 1 : 0; }

extern "C" int hx_set_material(hx_ctx* ctx, const double* gamma_e) {
  if (!ctx) return HX_EINVAL;
  CK(cudaSetDevice(ctx->device));
  if (!gamma_e) {
    if (ctx->gamma_e) cudaFree(ctx->gamma_e);
    ctx->gamma_e = nullptr;
  } else {
    if (!ctx->gamma_e) CK(dalloc(&ctx->gamma_e, (size_t)ctx->ne));
    CK(cudaMemcpyAsync(ctx->gamma_e, gamma_e, sizeof(double) * ctx->ne, cudaMemcpyDeviceToDevice, ctx->stream));
  }
  for (auto& g : ctx->graphs)  // captured steps bake the material pointer in
    if (g.exec) cudaGraphExecDestroy(g.exec);
  ctx->graphs.clear();
  return HX_OK;
}

// ---------------------------------------------------------------------------
// restriction

extern "C" int hx_gather(hx_ctx* ctx, int space, const double* L, int ncomp, double* E) {
  if (!ctx || !L || !E || ncomp < 1) return HX_EINVAL;
  CK(cudaSetDevice(ctx->device));
  if (space == HX_SPACE_H1) {
    const long long tot = (long long)ctx->nl * ctx->ne * ncomp;
    k_gather_ref<<<gblocks(tot, 256), 256, 0, ctx->stream>>>(L, ctx->emap, ctx->nl, ctx->ne, ncomp, E);
  } else {
    const long long tot = (long long)ctx->nt * ctx->ne * ncomp;
    k_l2_gather<<<gblocks(tot, 256), 256, 0, ctx->stream>>>(L, ctx->nt, ctx->ne, ncomp, E, 0);
  }
  CKL();
  return HX_OK;
}

extern "C" int hx_scatter_add(hx_ctx* ctx, int space, const double* E, int ncomp, double* L) {
  if (!ctx || !L || !E || ncomp < 1) return HX_EINVAL;
  CK(cudaSetDevice(ctx->device));
  if (space == HX_SPACE_H1) {
    k_scatter_ref<<<gblocks(ctx->nn * ncomp, 256), 256, 0, ctx->stream>>>(E, ctx->off, ctx->idx, ctx->nl, ctx->ne,
                                                                         ctx->nn, ncomp, L);
  } else {
    const long long tot = (long long)ctx->nt * ctx->ne * ncomp;
    k_l2_gather<<<gblocks(tot, 256), 256, 0, ctx->stream>>>(E, ctx->nt, ctx->ne, ncomp, L, 1);
  }
  CKL();
  return HX_OK;
}

// ---------------------------------------------------------------------------
// geometry

// queue the copy of the peer-exchange error flag (a timed-out peer wait anywhere in the
// work queued so far); checked by peer_check after the next stream sync
static int peer_err_fetch(hx_ctx* ctx) {
  if (!ctx->peer || !ctx->peer_ctr) return HX_OK;
  CK(cudaMemcpyAsync(ctx->h_perr, ctx->peer_ctr + 1, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  return HX_OK;
}

static int peer_check(hx_ctx* ctx) {
  if (ctx->peer && ctx->peer_ctr && *ctx->h_perr)
    return fail(ctx, HX_ENCCL, "peer exchange timed out (a rank did not arrive)");
  return HX_OK;
}

static int read_status(hx_ctx* ctx, StatusDev* st, StatusDev* h) {
  CK(cudaMemcpyAsync(h, st, sizeof(StatusDev), cudaMemcpyDeviceToHost, ctx->stream));
  int rc = peer_err_fetch(ctx);
  if (rc) return rc;
  CK(cudaStreamSynchronize(ctx->stream));
  return peer_check(ctx);
}

extern "C" int hx_geometry(hx_ctx* ctx, const double* x, double* jac, double* detj, double* jinv, double* wdetj,
                           hx_inverted* inv) {
  if (!ctx || !x) return HX_EINVAL;
  CK(cudaSetDevice(ctx->device));
  StatusDev* st = ctx->st + 3;
  int rc = status_reset(ctx, st);
  if (rc) return rc;
  GeomArgs a{x, ctx->emap, tables(ctx), ctx->ne, jac, detj, jinv, wdetj, nullptr, nullptr, nullptr, st};
  rc = dispatch<LaunchGeom>(ctx, a);
  if (rc) return rc;
  rc = read_status(ctx, st, ctx->h_st + 3);
  if (rc) return rc;
  decode_inv(ctx, ctx->h_st[3].inv_key, inv);
  if (ctx->h_st[3].inv_key != ~0ull) {
    // fetch det J at the offending point for the message (fespace.py:39)
    if (detj && inv) {
      const long long pe = inv->point * ctx->ne + inv->element;
      CK(cudaMemcpy(&inv->detj, detj + pe, sizeof(double), cudaMemcpyDeviceToHost));
    }
    return HX_EINVERTED;
  }
  return HX_OK;
}

// ---------------------------------------------------------------------------
// mass

__global__ void k_recip(const double* in, long long n, double* out);
__global__ void k_invdiag(const double* diag, const uint8_t* mask, int nc, long long nn, double* invd) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nn * nc) return;
  const long long n = t / nc;
  invd[t] = 1.0 / ((mask && mask[t]) ? 1.0 : diag[n]);
}


extern "C" int hx_mass_create(hx_ctx* ctx, const double* D, hx_mass** out) {
  if (!ctx || !D || !out) return HX_EINVAL;
  CK(cudaSetDevice(ctx->device));
  hx_mass* m = new hx_mass{ctx, nullptr};
  if (dalloc(&m->D, (size_t)ctx->ne * ctx->nq + 8) != cudaSuccess) {  // +pad: bulk copies read 16-B spans
    delete m;
    return fail(ctx, HX_ECUDA, "alloc");
  }
  const long long n = (long long)ctx->nq * ctx->ne;
  k_transpose<<<gblocks(n, 256), 256, 0, ctx->stream>>>(D, ctx->nq, ctx->ne, m->D);
  CKL();
  *out = m;
  return HX_OK;
}

extern "C" int hx_mass_destroy(hx_mass* m) {
  if (!m) return HX_OK;
  cudaFree(m->D);
  delete m;
  return HX_OK;
}

static int mass_evec(hx_ctx* ctx, const double* D, const double* x, int nc, double* evec) {
  MassArgs a{};
  a.x = x;
  a.D = D;
  a.emap = ctx->emap;
  a.slot = ctx->slot;
  a.B = ctx->B;
  a.ne = ctx->ne;
  a.evec = evec;
  a.own = ctx->own;
  return dispatch<LaunchMass>(ctx, nc, false, a);
}

extern "C" int hx_mass_apply(hx_mass* m, const double* x, int ncomp, double* y) {
  if (!m || !x || !y || ncomp < 1 || ncomp > 3) return m ? fail(m->ctx, HX_EINVAL, "bad arguments") : HX_EINVAL;
  hx_ctx* ctx = m->ctx;
  CK(cudaSetDevice(ctx->device));
  int rc = mass_evec(ctx, m->D, x, ncomp, ctx->evec2);
  if (rc) return rc;
  return launch_scatter(ctx, ctx->evec2, ncomp, y);
}

extern "C" int hx_mass_diagonal(hx_mass* m, double* diag) {
  if (!m || !diag) return HX_EINVAL;
  hx_ctx* ctx = m->ctx;
  CK(cudaSetDevice(ctx->device));
  int rc = dispatch<LaunchMassDiag>(ctx, (const double*)m->D, ctx->evec2);
  if (rc) return rc;
  return launch_scatter(ctx, ctx->evec2, 1, diag);
}

// Device CG on the PA mass.  k_cg_init, then iterations of (k_mass*, k_cg_node);
// the stop test runs on the device (k_cg_node's last block).  Outside a graph the
// host polls a pinned copy of the CG state once per chunk of iterations (kernels
// past convergence exit at once); inside a graph the iterations sit in a
// conditional WHILE node driven by the same flag (cudaGraphSetConditional).
struct CGLaunch {
  NodeArgs na;
  MassArgs ma;
  MassBrickArgs mb;  // structured-brick mass (ctx->brick)
  int nc;
};

// node-sum functor for the context's E-vector layout: element-major brick sums or
// the node-sorted CSR sums; f(sum, integral_constant<NC>)
template <int N>
using IC = std::integral_constant<int, N>;

template <class F>
static int with_node_sum(hx_ctx* ctx, int nc, const double* evec, F&& f) {
  if (ctx->elem_major) {
    switch (ctx->p * 10 + nc) {
      case 21: return f(BrickSum<2, 1>{evec, ctx->bk}, IC<1>());
      case 22: return f(BrickSum<2, 2>{evec, ctx->bk}, IC<2>());
      case 23: return f(BrickSum<2, 3>{evec, ctx->bk}, IC<3>());
      case 31: return f(BrickSum<3, 1>{evec, ctx->bk}, IC<1>());
      case 32: return f(BrickSum<3, 2>{evec, ctx->bk}, IC<2>());
      case 33: return f(BrickSum<3, 3>{evec, ctx->bk}, IC<3>());
      case 41: return f(BrickSum<4, 1>{evec, ctx->bk}, IC<1>());
      case 42: return f(BrickSum<4, 2>{evec, ctx->bk}, IC<2>());
      case 43: return f(BrickSum<4, 3>{evec, ctx->bk}, IC<3>());
    }
    return fail(ctx, HX_EINVAL, "brick node sum: unsupported p=%d nc=%d", ctx->p, nc);
  }
  if (nc == 1) return f(CsrSum<1>{ctx->off, evec}, IC<1>());
  if (nc == 2) return f(CsrSum<2>{ctx->off, evec}, IC<2>());
  return f(CsrSum<3>{ctx->off, evec}, IC<3>());
}

template <class S>
struct BrickOrder {
  static constexpr int value = 0;
};
template <int P, int NC>
struct BrickOrder<BrickSum<P, NC>> {
  static constexpr int value = P;
};

// HX_NODE_ROW=1: the warp-per-row-segment brick node pass (k_cg_node_row).  Measured on the
// 3D Sedov Q3 bench: 20.0 us vs 16.5 us for k_cg_node (same instruction count, fewer loads
// in flight per thread), so opt-in
static int g_node_row = -1;

// single-GPU brick node pass, one warp per node-row segment (hx_node.cuh)
template <int P, int NC>
static bool launch_node_row(hx_ctx* ctx, const NodeArgs& na, int* rc) {
  if (g_node_row < 0) {
    const char* v = getenv("HX_NODE_ROW");
    g_node_row = (v && v[0] == '1') ? 1 : 0;
  }
  constexpr int MS = 4;
  constexpr int SEGMAX = 32 * MS / NC;
  if (!g_node_row || ctx->peer) return false;
  const int Nx = ctx->bk.Nx;
  const int nseg_row = (Nx + SEGMAX - 1) / SEGMAX;
  const int seg = (Nx + nseg_row - 1) / nseg_row;
  auto k = k_cg_node_row<P, NC, MS>;
  static unsigned cap = 0;
  if (!cap) cap = persistent_grid(k, 256, 0, 1ll << 40);
  const long long nrows = (long long)ctx->bk.Ny * (ctx->bk.nz * P + 1);
  const unsigned need = gblocks(nrows * nseg_row, 8);
  prof_begin(ctx, K_CGNODE);
  k<<<std::min(need, cap), 256, 0, ctx->stream>>>(na, ctx->bk, seg, nseg_row);
  prof_end(ctx);
  const cudaError_t e = cudaGetLastError();
  *rc = e == cudaSuccess ? HX_OK : fail(ctx, HX_ECUDA, "k_cg_node_row launch: %s", cudaGetErrorString(e));
  ++ctx->launches;
  return true;
}

// HX_NODE_ASYNC=1: the cp.async-staged brick node pass (k_cg_node_async)
static int g_node_async = -1;

template <int P, int NC>
static bool launch_node_async(hx_ctx* ctx, const NodeArgs& na, int* rc) {
  if (g_node_async < 0) {
    const char* v = getenv("HX_NODE_ASYNC");
    g_node_async = v ? atoi(v) : 0;
  }
  if (!g_node_async || ctx->peer || !na.invdn) return false;
  using C = NodeAsyncCfg<NC>;
  auto k = k_cg_node_async<P, NC>;
  static bool attr = false;
  if (!attr) {
    *rc = smem_attr(k, C::bytes) == cudaSuccess ? HX_OK : HX_ECUDA;
    if (*rc) return true;
    attr = true;
  }
  static unsigned cap = 0;
  if (!cap) cap = persistent_grid(k, C::NT, C::bytes, 1ll << 40);
  const long long ntiles = (ctx->nn * NC + C::TN - 1) / C::TN;
  prof_begin(ctx, K_CGNODE);
  k<<<(unsigned)std::min<long long>(cap, ntiles), C::NT, C::bytes, ctx->stream>>>(na, ctx->bk);
  prof_end(ctx);
  const cudaError_t e = cudaGetLastError();
  *rc = e == cudaSuccess ? HX_OK : fail(ctx, HX_ECUDA, "k_cg_node_async launch: %s", cudaGetErrorString(e));
  ++ctx->launches;
  return true;
}

template <int NC, class SUM>
static int launch_cg_nodes(hx_ctx* ctx, const NodeArgs& na, SUM sum, bool init) {
  if constexpr (BrickOrder<SUM>::value > 0) {
    int rc = HX_OK;
    if (!init && launch_node_async<BrickOrder<SUM>::value, NC>(ctx, na, &rc)) return rc;
    if (!init && launch_node_row<BrickOrder<SUM>::value, NC>(ctx, na, &rc)) return rc;
  }
#ifndef NODE_PF
#define NODE_PF 0
#endif
  auto kn = ctx->peer ? k_cg_node_peer<NC, SUM, true> : (NODE_PF ? k_cg_node_peer<NC, SUM, false> : k_cg_node<NC, SUM>);
  auto ki = k_cg_init<NC, SUM>;
  static unsigned caps_n[2] = {0, 0}, cap_i = 0;
  unsigned& cap_n = caps_n[ctx->peer ? 1 : 0];
  if (!cap_n) cap_n = persistent_grid(kn, 256, 0, 1ll << 40);
  if (!cap_i) cap_i = persistent_grid(ki, 256, 0, 1ll << 40);
  const unsigned need = gblocks(ctx->nn * NC, 256);
  if (init) {
    prof_begin(ctx, K_CGINIT);
    ki<<<std::min(need, cap_i), 256, 0, ctx->stream>>>(na, sum);
  } else {
    prof_begin(ctx, K_CGNODE);
    kn<<<std::min(need, cap_n), 256, 0, ctx->stream>>>(na, sum);
  }
  prof_end(ctx);
  CKL();
  return HX_OK;
}

#ifndef MASS_PIPE
#define MASS_PIPE 0
#endif
template <int P, int NC>
static bool launch_mass_tma(hx_ctx* ctx, const MassBrickArgs& a, int* rc);

template <int P, int NC>
static int launch_mass_brick(hx_ctx* ctx, const MassBrickArgs& a) {
  {
    int rc = HX_OK;
    if (launch_mass_tma<P, NC>(ctx, a, &rc)) return rc;
  }
  {
    static int w2 = -1;  // HX_MASS_W2=1: warp-independent pair kernel (k_mass_w2)
    if (w2 < 0) {
      const char* v = getenv("HX_MASS_W2");
      w2 = v ? atoi(v) : 0;
    }
    if (w2 && !a.slot && NC * (P + 1) * 2 <= 32) {
      using M = MassW2Cfg<P, NC>;
      const bool pf = w2 == 2;  // HX_MASS_W2=2: with the cp.async prefetch of the next pair
      auto k = pf ? (ctx->peer ? k_mass_w2<P, NC, true, true> : k_mass_w2<P, NC, false, true>)
                  : (ctx->peer ? k_mass_w2<P, NC, true> : k_mass_w2<P, NC, false>);
      const size_t bytes = pf ? M::bytes_pf : M::bytes;
      CK(smem_attr(k, bytes));
      static unsigned grids[4] = {0, 0, 0, 0};
      unsigned& grid = grids[(ctx->peer ? 1 : 0) + (pf ? 2 : 0)];
      if (!grid) grid = persistent_grid(k, M::NT, bytes, 1ll << 40);
      const long long pairs = (ctx->ne + 1) / 2;
      prof_begin(ctx, K_MASS);
      k<<<(unsigned)std::min<long long>(grid, (pairs + M::WARPS - 1) / M::WARPS), M::NT, bytes, ctx->stream>>>(a);
      prof_end(ctx);
      CKL();
      return HX_OK;
    }
  }
  if (MASS_PIPE) {
    using M = MassPipeCfg<P, NC>;
    auto k = ctx->peer ? k_mass_brick2<P, NC, true> : k_mass_brick2<P, NC, false>;
    CK(smem_attr(k, M::bytes));
    static unsigned grids[2] = {0, 0};
    unsigned& grid = grids[ctx->peer ? 1 : 0];
    if (!grid) grid = persistent_grid(k, M::NT, M::bytes, 1ll << 40);
    prof_begin(ctx, K_MASS);
    k<<<std::min(grid, gblocks(ctx->ne, M::EPC)), M::NT, M::bytes, ctx->stream>>>(a);
    prof_end(ctx);
    CKL();
    return HX_OK;
  }
  using M = MassBrickCfg<P, NC>;
  auto k = ctx->peer ? k_mass_brick<P, NC, true> : k_mass_brick<P, NC, false>;
  CK(smem_attr(k, M::bytes));
  static unsigned grids[2] = {0, 0};
  unsigned& grid = grids[ctx->peer ? 1 : 0];
  if (!grid) grid = persistent_grid(k, M::NT, M::bytes, 1ll << 40);
  prof_begin(ctx, K_MASS);
  k<<<std::min(grid, gblocks(ctx->ne, M::EPC)), M::NT, M::bytes, ctx->stream>>>(a);
  prof_end(ctx);
  CKL();
  return HX_OK;
}

// ---- TMA-staged brick mass (hx_tma.cuh): tensor maps over the (z, p) pair buffers
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &f, 12000, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiledFn)f;
    cudaGetLastError();
  }
  return fn;
}

// pair array (NN, NC, 2) doubles viewed as (Nx*NC*2, Ny, Nz); box = one pass's node box
template <int P, int NC>
static bool pair_maps(hx_ctx* ctx) {
  int& stt = ctx->tm_state[NC];
  if (stt) return stt > 0;
  stt = -1;
  EncodeTiledFn enc = encode_tiled();
  if (!enc) return false;
  using M = MassTmaCfg<P, NC>;
  const cuuint64_t row = (cuuint64_t)ctx->bk.Nx * NC * 2;
  const cuuint64_t gdim[3] = {row, (cuuint64_t)ctx->bk.Ny, (cuuint64_t)(ctx->bk.nz * P + 1)};
  const cuuint64_t gstr[2] = {row * 8, row * 8 * (cuuint64_t)ctx->bk.Ny};
  const cuuint32_t box[3] = {(cuuint32_t)M::ROWD, (cuuint32_t)M::D1, (cuuint32_t)M::D1};
  const cuuint32_t est[3] = {1, 1, 1};
  double* bufs[2] = {ctx->p0, ctx->p1};
  for (int b = 0; b < 2; ++b)
    if (enc(&ctx->tm_pair[NC][b], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, bufs[b], gdim, gstr, box, est,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return false;
  stt = 1;
  return true;
}

// HX_MASS_TMA=1: the TMA-staged brick mass kernel (k_mass_tma).  Measured on the 3D Sedov
// Q3 bench (profiles/r2/r2f_*, r2g_*): 27.4 us vs 26.0 us for k_mass_brick, so opt-in
static int g_mass_tma = -1;

template <int P, int NC>
static bool launch_mass_tma(hx_ctx* ctx, const MassBrickArgs& a, int* rc) {
  if (g_mass_tma < 0) {
    const char* v = getenv("HX_MASS_TMA");
    g_mass_tma = (v && v[0] == '1') ? 1 : 0;
  }
  if constexpr (NC != 3) {
    return false;
  } else {
  if (!g_mass_tma || a.slot || ((unsigned long long)a.D & 15ull)) return false;
  if (!pair_maps<P, NC>(ctx)) return false;
  using M = MassTmaCfg<P, NC>;
  auto k = ctx->peer ? k_mass_tma<P, NC, true> : k_mass_tma<P, NC, false>;
  *rc = HX_OK;
  if (smem_attr(k, M::bytes) != cudaSuccess) {
    *rc = fail(ctx, HX_ECUDA, "k_mass_tma: shared memory attribute");
    return true;
  }
  static unsigned grids[2] = {0, 0};
  unsigned& grid = grids[ctx->peer ? 1 : 0];
  if (!grid) grid = persistent_grid(k, M::NT, M::bytes, 1ll << 40);
  const int nseg = (ctx->bk.nx + M::EPC - 1) / M::EPC;
  const long long units = (long long)nseg * ctx->bk.ny * ctx->bk.nz;
  prof_begin(ctx, K_MASS);
  k<<<(unsigned)std::min<long long>(grid, units), M::NT, M::bytes, ctx->stream>>>(a, ctx->tm_pair[NC][0],
      a.pbuf1 == a.pbuf0 ? ctx->tm_pair[NC][0] : ctx->tm_pair[NC][1], nseg);
  prof_end(ctx);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) *rc = fail(ctx, HX_ECUDA, "k_mass_tma launch: %s", cudaGetErrorString(e));
  else ++ctx->launches;
  return true;
  }
}

static int mass_brick(hx_ctx* ctx, int nc, const MassBrickArgs& a) {
  switch (ctx->p * 10 + nc) {
    case 21: return launch_mass_brick<2, 1>(ctx, a);
    case 22: return launch_mass_brick<2, 2>(ctx, a);
    case 23: return launch_mass_brick<2, 3>(ctx, a);
    case 31: return launch_mass_brick<3, 1>(ctx, a);
    case 32: return launch_mass_brick<3, 2>(ctx, a);
    case 33: return launch_mass_brick<3, 3>(ctx, a);
    case 41: return launch_mass_brick<4, 1>(ctx, a);
    case 42: return launch_mass_brick<4, 2>(ctx, a);
    case 43: return launch_mass_brick<4, 3>(ctx, a);
  }
  return fail(ctx, HX_EINVAL, "brick mass: unsupported p=%d nc=%d", ctx->p, nc);
}

static int build_emapf(hx_ctx* ctx, const uint8_t* mask, int nc, int* out) {
  const long long n = ctx->ne * ctx->nl;
  k_build_emapf<<<gblocks(n, 256), 256, 0, ctx->stream>>>(ctx->emap, ctx->own, mask, nc, n, out);
  CKL();
  return HX_OK;
}

static int cg_prepare(hx_ctx* ctx, CGDev* cg, const double* D, const double* rhs, const double* evec_rhs, int negate,
                      const uint8_t* mask, const double* invd, double rel_tol, int max_iter, double* x, int nc,
                      double* hist, CGLaunch& L, const int* emapf) {
  if (hist == nullptr) {
    if (ctx->hist_len < max_iter + 1) {
      if (ctx->hist) cudaFree(ctx->hist);
      ctx->hist = nullptr;
      CK(dalloc(&ctx->hist, (size_t)max_iter + 1));
      ctx->hist_len = max_iter + 1;
    }
    hist = ctx->hist;
  }
  NodeArgs& na = L.na;
  na = NodeArgs{};
  na.off = ctx->off;
  na.idx = ctx->idx;
  na.evec = evec_rhs ? evec_rhs : ctx->evec;
  na.mask = mask;
  na.invd = invd;
  // the phase's momentum solve: per-node 1/diag (bit-identical z; a third of the bytes)
  static int inode = -1, inplace = -1;
  if (inode < 0) {
    const char* v = getenv("HX_INVD_NODE");
    inode = (v && v[0] == '0') ? 0 : 1;
    const char* w = getenv("HX_PAIRS_INPLACE");
    inplace = (w && w[0] == '0') ? 0 : 1;
  }
  na.invdn = (inode && invd == ctx->invd && nc == ctx->dim) ? ctx->invdn : nullptr;
  na.x = x;
  na.r = ctx->r;
  na.z = ctx->z;
  na.pbuf0 = ctx->p0;
  na.pbuf1 = ctx->p1;
  na.rhs = rhs;
  na.nn = ctx->nn;
  na.cg = cg;
  const size_t preg = (size_t)ctx->preg;  // partial regions: [node / init | mass]
  na.partials = ctx->partials;
  na.pm = ctx->partials + preg;
  na.hist = hist;
  na.negate = negate;
  na.tol = rel_tol;
  na.max_iter = max_iter;
  na.owned = ctx->peer ? ctx->peer_owned : nullptr;
  na.peer = ctx->peer ? ctx->pd_dev : nullptr;
  na.pl = ctx->pl;
  MassArgs& ma = L.ma;
  ma = MassArgs{};
  ma.x = ctx->z;
  ma.pbuf0 = ctx->p0;
  ma.pbuf1 = ctx->p1;
  ma.mask = mask;
  ma.own = ctx->own;
  ma.D = D;
  ma.emap = ctx->emap;
  ma.emapf = emapf;
  ma.slot = ctx->slot;
  ma.B = ctx->B;
  ma.ne = ctx->ne;
  ma.evec = ctx->evec;
  ma.cg = cg;
  ma.partials = ctx->partials + preg;
  L.nc = nc;
  L.mb = MassBrickArgs{ctx->p0, ctx->p1, D, ctx->ne, ctx->evec, ctx->elem_major ? nullptr : ctx->slot, cg,
                       ctx->partials + preg, ctx->bk, ctx->pl};
  // (z, p) pairs updated in place (HX_PAIRS_INPLACE=0: ping-pong): within a node launch
  // every pair is read and rewritten by the same thread, and the mass launches read them
  // only between node launches -- one 16 B/dof buffer less in the L2 working set
  if (inplace) {
    na.pbuf1 = na.pbuf0;
    ma.pbuf1 = ma.pbuf0;
    L.mb.pbuf1 = L.mb.pbuf0;
  }
  return HX_OK;
}

// multi-GPU: world sum of a CG launch's partials (k_peer_sync), see hx_peer.cuh
template <int NV>
static int peer_sync(hx_ctx* ctx, CGDev* g, double* parts, int* nparts) {
  k_peer_sync<NV><<<1, 256, 0, ctx->stream>>>(ctx->pd, g, parts, nparts);
  CKL();
  return HX_OK;
}

// multi-GPU, after a mass launch: this rank's interface partials into the neighbours'
// receive blocks; the node launch's prologue publishes them with the world p.Ap and
// sums the interface nodes itself (peer_node_sum)
static int peer_halo(hx_ctx* ctx, CGLaunch& L) {
  if (ctx->pd.nsh == 0) return HX_OK;  // no neighbours: nothing to send
  const unsigned gp = capg(std::max(1u, std::min<unsigned>(gblocks((long long)ctx->pd.nsh * L.nc, 256), 592)));
  int rc = with_node_sum(ctx, L.nc, ctx->evec, [&](auto sum, auto ncc) {
    k_halo_pack<decltype(ncc)::value><<<gp, 256, 0, ctx->stream>>>(ctx->pd, L.na.cg, sum, ctx->pl);
    return HX_OK;
  });
  if (rc) return rc;
  CKL();
  return HX_OK;
}

// multi-GPU halo of an E-vector's interface nodes outside the CG (F.1 before the CG init)
static int peer_evec_halo(hx_ctx* ctx, double* evec, int nc) {
  const unsigned gp = capg(std::max(1u, std::min<unsigned>(gblocks((long long)ctx->pd.nsh * nc, 256), 592)));
  const unsigned gc = capg(std::max(1u, std::min<unsigned>(gblocks((long long)ctx->pd.nh * nc, 256), 592)));
  int rc = with_node_sum(ctx, nc, evec, [&](auto sum, auto ncc) {
    k_halo_pack<decltype(ncc)::value><<<gp, 256, 0, ctx->stream>>>(ctx->pd, nullptr, sum, ctx->pl);
    return HX_OK;
  });
  if (rc) return rc;
  CKL();
  rc = peer_sync<0>(ctx, nullptr, nullptr, nullptr);
  if (rc) return rc;
  rc = with_node_sum(ctx, nc, evec, [&](auto sum, auto ncc) {
    k_halo_combine<decltype(ncc)::value><<<gc, 256, 0, ctx->stream>>>(ctx->pd, nullptr, sum);
    return HX_OK;
  });
  CKL();
  return rc;
}

// multi-GPU world status (CFL ratio min, clamp sum, inversion) of n records
static int peer_status(hx_ctx* ctx, StatusDev* st, int n) {
  k_peer_status<<<1, 32, 0, ctx->stream>>>(ctx->pd, st, n);
  CKL();
  return HX_OK;
}

// fused rates (+ multi-GPU: world status, F.1 interface sums)
static int rates_launch(hx_ctx* ctx, const hx_params* prm, const double* x, const double* v, const double* e,
                        double* de, StatusDev* st) {
  int rc = dispatch<LaunchRates>(ctx, x, v, e, ctx->evec, de, st, 0, prm->gamma, prm->q1, prm->q2);
  if (rc || !ctx->peer) return rc;
  rc = peer_status(ctx, st, 1);
  if (rc) return rc;
  return peer_evec_halo(ctx, ctx->evec, ctx->dim);
}

// geometry validity of a new state (+ multi-GPU: world inversion)
static int validity_launch(hx_ctx* ctx, const double* x, StatusDev* st) {
  int rc = dispatch<LaunchRates>(ctx, x, (const double*)nullptr, (const double*)nullptr, (double*)nullptr,
                                 (double*)nullptr, st, 1, 0.0, 0.0, 0.0);
  if (rc || !ctx->peer) return rc;
  return peer_status(ctx, st, 1);
}

static int cg_launch_init(hx_ctx* ctx, CGLaunch& L) {
  int rc = with_node_sum(ctx, L.nc, L.na.evec, [&](auto sum, auto ncc) {
    return launch_cg_nodes<decltype(ncc)::value>(ctx, L.na, sum, true);
  });
  if (rc) return rc;

  L.na.evec = ctx->evec;
  L.na.rhs = nullptr;
  return HX_OK;
}

static int cg_launch_iter(hx_ctx* ctx, CGLaunch& L) {
  int rc = ctx->brick ? mass_brick(ctx, L.nc, L.mb) : dispatch<LaunchMass>(ctx, L.nc, true, L.ma);
  if (rc) return rc;
  if (ctx->peer) {
    rc = peer_halo(ctx, L);
    if (rc) return rc;
  }
  // world scalars: p.Ap in the node launch's prologue, r.z in the next mass launch's
  return with_node_sum(ctx, L.nc, ctx->evec, [&](auto sum, auto ncc) {
    return launch_cg_nodes<decltype(ncc)::value>(ctx, L.na, sum, false);
  });
}

static int cg_launch_finish(hx_ctx* ctx, CGLaunch& L) {
  const long long n = ctx->nn * L.nc;
  k_cg_finish<<<capg(std::min<unsigned>(gblocks(n, 256), 1184)), 256, 0, ctx->stream>>>(L.na.cg, L.na.pbuf0,
                                                                                  L.na.pbuf1, L.na.x, n);
  CKL();
  return HX_OK;
}

// device CG code -> C-ABI status (3 breakdown, 6 peer timeout, else max_iter)
static int cg_code(int c) {
  return c == 0 ? HX_OK : (c == 3 ? HX_ECG_BREAKDOWN : (c == 6 ? HX_ENCCL : HX_ECG_MAXITER));
}

static void cg_info_from(const CGDev& g, hx_cg_info* info) {
  if (!info) return;
  info->code = cg_code(g.code);
  info->iterations = g.iters;
  info->n_residuals = g.nres;
}

static int run_cg(hx_ctx* ctx, const double* D, const double* rhs, const double* evec_rhs, int negate,
                  const uint8_t* mask, const double* invd, double rel_tol, int max_iter, double* x, int nc,
                  double* hist, hx_cg_info* info, CGDev* cg = nullptr, const int* emapf = nullptr) {
  if (!cg) cg = ctx->cg;
  if (!emapf) emapf = ctx->emapf;
  CGLaunch L;
  int rc = cg_prepare(ctx, cg, D, rhs, evec_rhs, negate, mask, invd, rel_tol, max_iter, x, nc, hist, L, emapf);
  if (rc) return rc;
  rc = cg_launch_init(ctx, L);
  if (rc) return rc;
  int done_iters = 0;
  // profiling (hx_prof_enable): one iteration per poll, so that no launch past
  // convergence (an early-exit launch) enters the per-kernel averages
  int chunk = ctx->prof_on ? 1 : 8;
  while (true) {
    for (int i = 0; i < chunk; ++i) {
      rc = cg_launch_iter(ctx, L);
      if (rc) return rc;
    }
    done_iters += chunk;
    CK(cudaMemcpyAsync(ctx->h_cg, cg, sizeof(CGDev), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    if (!ctx->h_cg->active) break;
    if (done_iters > max_iter + 1) break;
    if (!ctx->prof_on) chunk = std::min(chunk * 2, 64);
  }
  rc = cg_launch_finish(ctx, L);
  if (rc) return rc;
  cg_info_from(*ctx->h_cg, info);
  return HX_OK;
}

// capture the CG of one stage into the graph being captured on ctx->stream
static int cg_capture(hx_ctx* ctx, CGLaunch& L, int iters_hint = 0) {
  cudaStreamCaptureStatus cs;
  cudaGraph_t g;
  const cudaGraphNode_t* deps = nullptr;
  size_t nd = 0;
  CK(cudaStreamGetCaptureInfo(ctx->stream, &cs, nullptr, &g, &deps, &nd));
  cudaGraphConditionalHandle h;
  CK(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
  L.na.cond = (unsigned long long)h;
  L.na.use_cond = 1;
  int rc = cg_launch_init(ctx, L);
  if (rc) return rc;
  // graph shape: the expected iterations (previous plain solve of this stage + 1) as plain
  // kernel nodes ahead of a WHILE node with a 2-iteration body, which then usually
  // evaluates once and skips (578 vs 573 Mdof*steps/s with two half-length bodies,
  // HX_CG_SHAPE=halves)
  static int shape = -1;
  if (shape < 0) {
    const char* v = getenv("HX_CG_SHAPE");
    shape = (v && strcmp(v, "halves") == 0) ? 0 : 1;
  }
  const bool prefix = shape == 1 && iters_hint > 0;
  if (prefix)
    for (int u = 0; u < iters_hint + 1 && rc == HX_OK; ++u) {
      ctx->prof_tag_iter = u + 1;  // iteration k = u + 1 (profiling graphs only)
      rc = cg_launch_iter(ctx, L);
    }
  ctx->prof_tag_iter = 0;
  if (rc) return rc;
  CK(cudaStreamGetCaptureInfo(ctx->stream, &cs, nullptr, &g, &deps, &nd));
  cudaGraphNodeParams p = {};
  p.type = cudaGraphNodeTypeConditional;
  p.conditional.handle = h;
  p.conditional.type = cudaGraphCondTypeWhile;
  p.conditional.size = 1;
  cudaGraphNode_t node;
  CK(cudaGraphAddNode(&node, g, deps, nd, &p));
  CK(cudaStreamUpdateCaptureDependencies(ctx->stream, &node, 1, cudaStreamSetCaptureDependencies));
  cudaGraph_t body = p.conditional.phGraph_out[0];
  cudaStream_t outer = ctx->stream;
  CK(cudaStreamBeginCaptureToGraph(ctx->gstream2, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
  ctx->stream = ctx->gstream2;
  // iterations per WHILE body (launches past convergence exit at once).  Measured on the
  // 3D Sedov Q3 bench: a body evaluation costs ~5.8 us, an iteration launched past
  // convergence ~2.3 us, so the body holds about half of the iterations the previous plain
  // solve of this stage needed (two bodies; drift of +-2 iterations stays cheap);
  // HX_CG_UNROLL overrides
  static int unroll_env = -2;
  if (unroll_env == -2) {
    const char* v = getenv("HX_CG_UNROLL");
    unroll_env = v ? std::max(1, atoi(v)) : -1;
  }
  const int unroll = prefix ? 2
                   : unroll_env > 0 ? unroll_env
                                    : (iters_hint > 0 ? std::min(32, std::max(2, (iters_hint + 3) / 2)) : 4);
  for (int u = 0; u < unroll && rc == HX_OK; ++u) rc = cg_launch_iter(ctx, L);
  ctx->stream = outer;
  if (rc) return rc;
  CK(cudaStreamEndCapture(ctx->gstream2, &body));
  return cg_launch_finish(ctx, L);
}

__global__ void k_recip(const double* in, long long n, double* out) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  out[t] = in ? 1.0 / in[t] : 1.0;
}

extern "C" int hx_mass_cg(hx_mass* m, const double* rhs, int ncomp, const uint8_t* bcmask,
                          const double* precond_diag, double rel_tol, int max_iter, double* x,
                          double* residuals, hx_cg_info* info) {
  if (!m || !rhs || !x || max_iter < 0 || ncomp < 1 || ncomp > 3) return HX_EINVAL;
  hx_ctx* ctx = m->ctx;
  CK(cudaSetDevice(ctx->device));
  // inv_diag = 1 / precond_diag (operators.py:344); none -> identity
  double* invd = ctx->vm;  // scratch (NN, d) >= (NN, ncomp)
  const long long nv = ctx->nn * ncomp;
  k_recip<<<gblocks(nv, 256), 256, 0, ctx->stream>>>(precond_diag, nv, invd);
  CKL();
  int rc = build_emapf(ctx, bcmask, ncomp, ctx->emapf_api);
  if (rc) return rc;
  hx_cg_info ci{};
  rc = run_cg(ctx, m->D, rhs, nullptr, 0, bcmask, invd, rel_tol, max_iter, x, ncomp, residuals, &ci, ctx->cg,
              ctx->emapf_api);
  if (rc) return rc;
  CK(cudaStreamSynchronize(ctx->stream));
  if (info) *info = ci;
  return ci.code;
}

// ---------------------------------------------------------------------------
// force

extern "C" int hx_force_create(hx_ctx* ctx, const double* sigma, const double* jinv, const double* wdetj,
                               double* D_out, hx_force** out) {
  if (!ctx || !sigma || !jinv || !wdetj || !out) return HX_EINVAL;
  CK(cudaSetDevice(ctx->device));
  hx_force* f = new hx_force{ctx, nullptr};
  if (dalloc(&f->DF, (size_t)ctx->ne * ctx->dim * ctx->dim * ctx->nq) != cudaSuccess) {
    delete f;
    return fail(ctx, HX_ECUDA, "alloc");
  }
  const long long n = (long long)ctx->nq * ctx->ne;
  if (ctx->dim == 2) k_force_D<2><<<gblocks(n, 256), 256, 0, ctx->stream>>>(sigma, jinv, wdetj, ctx->ne, ctx->nq, f->DF, D_out);
  else k_force_D<3><<<gblocks(n, 256), 256, 0, ctx->stream>>>(sigma, jinv, wdetj, ctx->ne, ctx->nq, f->DF, D_out);
  CKL();
  *out = f;
  return HX_OK;
}

extern "C" int hx_force_destroy(hx_force* f) {
  if (!f) return HX_OK;
  cudaFree(f->DF);
  delete f;
  return HX_OK;
}

extern "C" int hx_force_apply(hx_force* f, const double* e, double* y) {
  if (!f || !e || !y) return HX_EINVAL;
  hx_ctx* ctx = f->ctx;
  CK(cudaSetDevice(ctx->device));
  ForceArgs a{e, f->DF, ctx->emap, ctx->slot, tables(ctx), ctx->ne, ctx->evec2, nullptr};
  int rc = dispatch<LaunchForce>(ctx, a, false);
  if (rc) return rc;
  return launch_scatter(ctx, ctx->evec2, ctx->dim, y);
}

extern "C" int hx_force_apply_t(hx_force* f, const double* v, double* y) {
  if (!f || !v || !y) return HX_EINVAL;
  hx_ctx* ctx = f->ctx;
  CK(cudaSetDevice(ctx->device));
  ForceArgs a{v, f->DF, ctx->emap, ctx->slot, tables(ctx), ctx->ne, nullptr, y};
  return dispatch<LaunchForce>(ctx, a, true);
}

// ---------------------------------------------------------------------------
// remap-phase operators: DiffusionPA / ConvectionPA (operators.py:143-236)

template <int DIM, int P>
struct LaunchRemap {
  static int run(hx_ctx* ctx, const hx_op* op, const double* x) {
    using SM = RemapSmem<DIM, P>;
    RemapArgs a{x, op->D, ctx->emap, ctx->slot, ctx->B, ctx->G, ctx->ne, ctx->evec2};
    if (op->kind == 0) {
      auto k = k_remap_op<DIM, P, 128, 0>;
      CK(smem_attr(k, SM::bytes));
      k<<<(unsigned)ctx->ne, 128, SM::bytes, ctx->stream>>>(a);
    } else {
      auto k = k_remap_op<DIM, P, 128, 1>;
      CK(smem_attr(k, SM::bytes));
      k<<<(unsigned)ctx->ne, 128, SM::bytes, ctx->stream>>>(a);
    }
    CKL();
    return HX_OK;
  }
};

static int remap_create(hx_ctx* ctx, int kind, const double* jinv, const double* wdetj, const double* nu,
                        const double* u, double* D_out, hx_op** out) {
  if (!ctx || !jinv || !wdetj || !out || (kind == 1 && !u)) return HX_EINVAL;
  CK(cudaSetDevice(ctx->device));
  const int d = ctx->dim;
  hx_op* op = new hx_op{ctx, kind, nullptr};
  const size_t n = (size_t)ctx->ne * (kind == 0 ? d * d : d) * ctx->nq;
  if (dalloc(&op->D, n) != cudaSuccess) {
    delete op;
    return fail(ctx, HX_ECUDA, "alloc");
  }
  const long long np = (long long)ctx->nq * ctx->ne;
  if (kind == 0) {
    if (d == 2) k_diff_D<2><<<gblocks(np, 256), 256, 0, ctx->stream>>>(jinv, wdetj, nu, ctx->ne, ctx->nq, op->D, D_out);
    else k_diff_D<3><<<gblocks(np, 256), 256, 0, ctx->stream>>>(jinv, wdetj, nu, ctx->ne, ctx->nq, op->D, D_out);
  } else {
    if (d == 2) k_conv_D<2><<<gblocks(np, 256), 256, 0, ctx->stream>>>(jinv, u, wdetj, ctx->ne, ctx->nq, op->D, D_out);
    else k_conv_D<3><<<gblocks(np, 256), 256, 0, ctx->stream>>>(jinv, u, wdetj, ctx->ne, ctx->nq, op->D, D_out);
  }
  CKL();
  *out = op;
  return HX_OK;
}

extern "C" int hx_diffusion_create(hx_ctx* ctx, const double* jinv, const double* wdetj, const double* nu,
                                   double* D_out, hx_op** out) {
  return remap_create(ctx, 0, jinv, wdetj, nu, nullptr, D_out, out);
}

extern "C" int hx_convection_create(hx_ctx* ctx, const double* jinv, const double* u_points, const double* wdetj,
                                    double* D_out, hx_op** out) {
  return remap_create(ctx, 1, jinv, wdetj, nullptr, u_points, D_out, out);
}

extern "C" int hx_op_apply(hx_op* op, const double* x, double* y) {
  if (!op || !x || !y) return HX_EINVAL;
  hx_ctx* ctx = op->ctx;
  CK(cudaSetDevice(ctx->device));
  int rc = dispatch<LaunchRemap>(ctx, (const hx_op*)op, x);
  if (rc) return rc;
  return launch_scatter(ctx, ctx->evec2, 1, y);
}

extern "C" int hx_op_destroy(hx_op* op) {
  if (!op) return HX_OK;
  cudaFree(op->D);
  delete op;
  return HX_OK;
}

// ---------------------------------------------------------------------------
// TMOP mesh-optimisation operator (meshopt.py:248-486)

template <int DIM, int P>
struct LaunchTmop {
  static int run(hx_ctx* ctx, const hx_tmop* op, int mode, bool lim, const double* x, const double* dx) {
    using SM = TmopSmem<DIM, P>;
    TmopArgs a{x, dx, op->winv, op->wdetw, ctx->emap, ctx->slot, ctx->B, ctx->G, op->mt, ctx->ne, ctx->evec2,
               op->epart, op->bad, op->x0, op->dlim, ctx->evec, op->epart + ctx->ne};
    constexpr int NT = 128;
    switch (mode * 2 + (lim ? 1 : 0)) {
#define HX_TMOP_MODE(M, L)                                       \
  case M * 2 + L: {                                              \
    auto k = k_tmop<DIM, P, NT, M, L>;                           \
    CK(smem_attr(k, SM::bytes));                                 \
    static unsigned grid = 0;                                    \
    if (!grid) grid = persistent_grid(k, NT, SM::bytes, 1ll << 40); \
    k<<<std::min<unsigned>(grid, gblocks(ctx->ne, 1)), NT, SM::bytes, ctx->stream>>>(a); \
    break;                                                       \
  }
      HX_TMOP_MODE(0, false)
      HX_TMOP_MODE(0, true)
      HX_TMOP_MODE(1, false)
      HX_TMOP_MODE(1, true)
      HX_TMOP_MODE(2, false)
      HX_TMOP_MODE(2, true)
      HX_TMOP_MODE(3, false)
      HX_TMOP_MODE(3, true)
#undef HX_TMOP_MODE
      default:
        return HX_EINVAL;
    }
    CKL();
    return HX_OK;
  }
};

__global__ void k_tmop_winv(const double* winv_ref /*(d,d,nq,NE)*/, int d, int nq, long long ne, double* winv) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)d * d * nq * ne) return;
  const long long e = t % ne, r = t / ne;
  const int q = (int)(r % nq), bl = (int)(r / nq);
  winv[(e * nq + q) * d * d + bl] = winv_ref[t];
}

extern "C" int hx_tmop_create(hx_ctx* ctx, const double* winv, const double* wdetw, const double* x0,
                              const double* dlim, int composite, double w_shape, double w_size, double gamma,
                              hx_tmop** out) {
  if (!ctx || !winv || !wdetw || !x0 || !dlim || !out) return HX_EINVAL;
  CK(cudaSetDevice(ctx->device));
  const int d = ctx->dim;
  hx_tmop* op = new hx_tmop();
  op->ctx = ctx;
  op->mt = TmopMetric{w_shape, w_size, composite ? 1 : 0};
  op->gamma = gamma;
  const size_t nv = (size_t)ctx->nn * d, npq = (size_t)ctx->ne * ctx->nq;
  bool ok = dalloc(&op->winv, npq * d * d) == cudaSuccess;
  ok &= dalloc(&op->wdetw, npq) == cudaSuccess;
  ok &= dalloc(&op->x0, nv) == cudaSuccess;
  ok &= dalloc(&op->dlim, ctx->nn) == cudaSuccess;
  ok &= dalloc(&op->nb0, nv) == cudaSuccess;
  ok &= dalloc(&op->nb1, nv) == cudaSuccess;
  ok &= dalloc(&op->epart, 2 * (size_t)ctx->ne) == cudaSuccess;  // mu, limiting
  ok &= dalloc(&op->sums, 2) == cudaSuccess;
  ok &= cudaMalloc(&op->bad, sizeof(int)) == cudaSuccess;
  if (!ok) {
    hx_tmop_destroy(op);
    return fail(ctx, HX_ECUDA, "hx_tmop_create: alloc");
  }
  const long long nw = (long long)npq * d * d;
  k_tmop_winv<<<gblocks(nw, 256), 256, 0, ctx->stream>>>(winv, d, ctx->nq, ctx->ne, op->winv);
  CKL();
  k_transpose<<<gblocks((long long)npq, 256), 256, 0, ctx->stream>>>(wdetw, ctx->nq, ctx->ne, op->wdetw);
  CKL();
  CK(cudaMemcpyAsync(op->x0, x0, sizeof(double) * nv, cudaMemcpyDeviceToDevice, ctx->stream));
  CK(cudaMemcpyAsync(op->dlim, dlim, sizeof(double) * ctx->nn, cudaMemcpyDeviceToDevice, ctx->stream));
  *out = op;
  return HX_OK;
}

extern "C" int hx_tmop_set_gamma(hx_tmop* op, double gamma) {
  if (!op) return HX_EINVAL;
  op->gamma = gamma;
  return HX_OK;
}

static int tmop_bad_reset(hx_tmop* op) {
  hx_ctx* ctx = op->ctx;
  CK(cudaMemsetAsync(op->bad, 0, sizeof(int), ctx->stream));
  return HX_OK;
}

static int tmop_bad_read(hx_tmop* op, int* bad) {
  hx_ctx* ctx = op->ctx;
  CK(cudaMemcpyAsync(ctx->h_t, op->bad, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  *bad = *reinterpret_cast<int*>(ctx->h_t);
  return HX_OK;
}

static int tmop_sum(hx_tmop* op, int slot, double* host) {
  hx_ctx* ctx = op->ctx;
  k_sum<<<1, 256, 0, ctx->stream>>>(op->epart + slot * ctx->ne, ctx->ne, op->sums + slot);
  CKL();
  CK(cudaMemcpyAsync(host, op->sums + slot, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  return HX_OK;
}

// the two integrals of the objective (meshopt.py:335-356): mu_sum = sum w detW mu(T) at x
// (valid = 0 when det A <= 0 anywhere: the caller's +inf sentinel, meshopt.py:322-326,
// 357-362) and, when want_limit, lim_sum = sum_a sum_q w detW ((x - x0)/d)_a^2 (without gamma)
extern "C" int hx_tmop_terms(hx_tmop* op, const double* x, int want_limit, double* mu_sum, double* lim_sum,
                             int* valid) {
  if (!op || !x || !mu_sum || !valid) return HX_EINVAL;
  hx_ctx* ctx = op->ctx;
  CK(cudaSetDevice(ctx->device));
  int rc = tmop_bad_reset(op);
  if (rc) return rc;
  rc = dispatch<LaunchTmop>(ctx, (const hx_tmop*)op, 0, want_limit != 0, x, (const double*)nullptr);
  if (rc) return rc;
  double h[2] = {0.0, 0.0};
  rc = tmop_sum(op, 0, &h[0]);
  if (rc) return rc;
  if (want_limit) {
    rc = tmop_sum(op, 1, &h[1]);
    if (rc) return rc;
  }
  int bad = 0;
  rc = tmop_bad_read(op, &bad);  // synchronises the stream (the sums landed too)
  if (rc) return rc;
  *valid = bad ? 0 : 1;
  *mu_sum = h[0];
  if (lim_sum) *lim_sum = h[1];
  return HX_OK;
}

// kind 1 gradient (x), 2 Hessian action (x, dx), 3 Hessian diagonal (x): the mu part
// assembled, plus gamma's limiting part (meshopt.py:376-486).  HX_EINVERTED when det A <= 0
// anywhere (the reference raises ValueError).
static int tmop_derivative(hx_tmop* op, int kind, const double* x, const double* dx, double* out) {
  hx_ctx* ctx = op->ctx;
  CK(cudaSetDevice(ctx->device));
  const int d = ctx->dim;
  const long long nv = ctx->nn * d;
  int rc = tmop_bad_reset(op);
  if (rc) return rc;
  const bool lim = op->gamma != 0.0;
  rc = dispatch<LaunchTmop>(ctx, (const hx_tmop*)op, kind, lim, x, dx);
  if (rc) return rc;
  rc = launch_scatter(ctx, ctx->evec2, d, lim ? op->nb0 : out);
  if (rc) return rc;
  if (lim) {  // the limiting element vectors (same launch) -> nodes, then the reference's combine
    rc = launch_scatter(ctx, ctx->evec, kind == 3 ? 1 : d, op->nb1);
    if (rc) return rc;
    k_tmop_nodes<<<gblocks(nv, 256), 256, 0, ctx->stream>>>(kind == 3 ? 3 : 2, nullptr, nullptr, op->dlim, op->nb0,
                                                            op->nb1, op->gamma, d, ctx->nn, out);
    CKL();
  }
  int bad = 0;
  rc = tmop_bad_read(op, &bad);
  if (rc) return rc;
  if (bad) return fail(ctx, HX_EINVERTED, "TMOP: mesh has non-positive Jacobians");
  return HX_OK;
}

extern "C" int hx_tmop_gradient(hx_tmop* op, const double* x, double* grad) {
  if (!op || !x || !grad) return HX_EINVAL;
  return tmop_derivative(op, 1, x, nullptr, grad);
}

extern "C" int hx_tmop_hessian_action(hx_tmop* op, const double* x, const double* dx, double* out) {
  if (!op || !x || !dx || !out) return HX_EINVAL;
  return tmop_derivative(op, 2, x, dx, out);
}

extern "C" int hx_tmop_hessian_diagonal(hx_tmop* op, const double* x, double* diag) {
  if (!op || !x || !diag) return HX_EINVAL;
  return tmop_derivative(op, 3, x, nullptr, diag);
}

extern "C" int hx_tmop_destroy(hx_tmop* op) {
  if (!op) return HX_OK;
  cudaFree(op->winv);
  cudaFree(op->wdetw);
  cudaFree(op->x0);
  cudaFree(op->dlim);
  cudaFree(op->nb0);
  cudaFree(op->nb1);
  cudaFree(op->epart);
  cudaFree(op->sums);
  cudaFree(op->bad);
  delete op;
  return HX_OK;
}

// ---------------------------------------------------------------------------
// phase

extern "C" int hx_phase_begin(hx_ctx* ctx, const double* x, const double* qdata0, const uint8_t* bcmask,
                              double* mass_D_out, double* mass_diag_out, double* minv_out) {
  if (!ctx || !x || !qdata0) return HX_EINVAL;
  CK(cudaSetDevice(ctx->device));
  StatusDev* st = ctx->st + 3;
  int rc = status_reset(ctx, st);
  if (rc) return rc;
  GeomArgs a{x, ctx->emap, tables(ctx), ctx->ne, nullptr, nullptr, nullptr, nullptr, ctx->Dm, mass_D_out, qdata0, st};
  rc = dispatch<LaunchGeom>(ctx, a);
  if (rc) return rc;
  const long long n = (long long)ctx->nq * ctx->ne;
  k_transpose<<<gblocks(n, 256), 256, 0, ctx->stream>>>(qdata0, ctx->nq, ctx->ne, ctx->qd0);
  CKL();
  rc = dispatch<LaunchMassDiag>(ctx, (const double*)ctx->Dm, ctx->evec2);
  if (rc) return rc;
  rc = launch_scatter(ctx, ctx->evec2, 1, ctx->mdiag);
  if (rc) return rc;
  if (ctx->peer) {  // multi-GPU: interface sums of the assembled diagonal
    const unsigned gp = capg(std::max(1u, std::min<unsigned>(gblocks(ctx->pd.nsh, 256), 592)));
    const unsigned gc = capg(std::max(1u, std::min<unsigned>(gblocks(ctx->pd.nh, 256), 592)));
    k_halo_pack<1><<<gp, 256, 0, ctx->stream>>>(ctx->pd, nullptr, NodeVec<1>{ctx->mdiag}, ctx->pl);
    CKL();
    rc = peer_sync<0>(ctx, nullptr, nullptr, nullptr);
    if (rc) return rc;
    k_halo_combine<1><<<gc, 256, 0, ctx->stream>>>(ctx->pd, nullptr, NodeVec<1>{ctx->mdiag});
    CKL();
  }
  const long long nv = ctx->nn * ctx->dim;
  if (bcmask) CK(cudaMemcpyAsync(ctx->mask, bcmask, nv, cudaMemcpyDeviceToDevice, ctx->stream));
  else CK(cudaMemsetAsync(ctx->mask, 0, nv, ctx->stream));
  ctx->has_mask = bcmask != nullptr;
  k_invdiag<<<gblocks(nv, 256), 256, 0, ctx->stream>>>(ctx->mdiag, ctx->mask, ctx->dim, ctx->nn, ctx->invd);
  CKL();
  k_recip<<<gblocks(ctx->nn, 256), 256, 0, ctx->stream>>>(ctx->mdiag, ctx->nn, ctx->invdn);
  CKL();
  rc = build_emapf(ctx, ctx->has_mask ? ctx->mask : nullptr, ctx->dim, ctx->emapf);
  if (rc) return rc;
  for (auto& g : ctx->graphs)  // graphs captured against the previous phase are stale
    if (g.exec) cudaGraphExecDestroy(g.exec);
  ctx->graphs.clear();
  rc = dispatch<LaunchMinv>(ctx, minv_out);
  if (rc) return rc;
  if (mass_diag_out) CK(cudaMemcpyAsync(mass_diag_out, ctx->mdiag, sizeof(double) * ctx->nn, cudaMemcpyDeviceToDevice, ctx->stream));
  rc = read_status(ctx, st, ctx->h_st + 3);
  if (rc) return rc;
  if (ctx->h_st[3].inv_key != ~0ull) return fail(ctx, HX_EINVERTED, "inverted element in begin_phase");
  ctx->phase = true;
  return HX_OK;
}

extern "C" int hx_stress(hx_ctx* ctx, const hx_params* prm, const double* x, const double* v, const double* e,
                         const double* qdata0, double* sigma, double* min_ratio, int64_t* clamped,
                         hx_inverted* inv) {
  if (!ctx || !prm || !x || !v || !e || !qdata0) return HX_EINVAL;
  CK(cudaSetDevice(ctx->device));
  StatusDev* st = ctx->st + 3;
  int rc = status_reset(ctx, st);
  if (rc) return rc;
  StressArgs a{x, v, e, qdata0, ctx->emap, tables(ctx), prm->gamma, prm->q1, prm->q2, ctx->gamma_e, ctx->ne, sigma, st};
  rc = dispatch<LaunchStress>(ctx, a);
  if (rc) return rc;
  rc = read_status(ctx, st, ctx->h_st + 3);
  if (rc) return rc;
  const StatusDev& h = ctx->h_st[3];
  if (min_ratio) *min_ratio = h.min_ratio;
  if (clamped) *clamped = (int64_t)h.clamps;
  decode_inv(ctx, h.inv_key, inv);
  return h.inv_key != ~0ull ? HX_EINVERTED : HX_OK;
}

// timestep_estimate's CFL ratio (hydro.py:364-367): compute_geometric_factors' inversion
// check + stress_qdata's min h/(c_s+|v|) and clamp count, without materialising the
// geometry or sigma -- one fused point-physics launch (k_rates_pc MODE 2) on the phase's
// qdata0.  3D, p >= 2 (the fused kernels' range); other discretisations keep the
// reference's geometry + stress calls (hx_geometry, hx_stress).
extern "C" int hx_timestep_ratio(hx_ctx* ctx, const hx_params* prm, const double* x, const double* v,
                                 const double* e, double* min_ratio, int64_t* clamped, hx_inverted* inv) {
  if (!ctx || !prm || !x || !v || !e || !ctx->phase) return HX_EINVAL;
  if (ctx->dim != 3 || ctx->p < 2) return fail(ctx, HX_EINVAL, "hx_timestep_ratio: 3D, p >= 2 only");
  CK(cudaSetDevice(ctx->device));
  StatusDev* st = ctx->st + 3;
  int rc = status_reset(ctx, st);
  if (rc) return rc;
  rc = dispatch<LaunchRates>(ctx, x, v, e, (double*)nullptr, (double*)nullptr, st, 2, prm->gamma, prm->q1, prm->q2);
  if (!rc && ctx->peer) rc = peer_status(ctx, st, 1);
  if (rc) return rc;
  rc = read_status(ctx, st, ctx->h_st + 3);
  if (rc) return rc;
  const StatusDev& h = ctx->h_st[3];
  if (min_ratio) *min_ratio = h.min_ratio;
  if (clamped) *clamped = (int64_t)h.clamps;
  decode_inv(ctx, h.inv_key, inv);
  return h.inv_key != ~0ull ? HX_EINVERTED : HX_OK;
}

extern "C" int hx_energy_solve(hx_ctx* ctx, const double* rhs, double* out) {
  if (!ctx || !rhs || !out || !ctx->phase) return HX_EINVAL;
  CK(cudaSetDevice(ctx->device));
  const long long n = ctx->ne * ctx->nt;
  k_energy_solve<<<gblocks(n, 256), 256, 0, ctx->stream>>>(ctx->minv, rhs, ctx->nt, ctx->ne, out, ctx->minv_packed);
  CKL();
  return HX_OK;
}

// One rates() evaluation on device: fused qpoint/force kernel then the masked CG.
// Status lands in st; CG info in *cgi.  No host sync except inside the CG poll.
static int rates_device(hx_ctx* ctx, const hx_params* prm, const double* x, const double* v, const double* e,
                        double* dv, double* de, StatusDev* st, hx_cg_info* cgi, CGDev* cg = nullptr) {
  int rc = status_reset(ctx, st);
  if (rc) return rc;
  rc = rates_launch(ctx, prm, x, v, e, de, st);
  if (rc) return rc;
  // rhs = where(mask, 0, -F.1) built inside k_cg_init from the element vectors
  return run_cg(ctx, ctx->Dm, nullptr, ctx->evec, 1, ctx->has_mask ? ctx->mask : nullptr, ctx->invd,
                prm->rel_tol, prm->max_iter, dv, ctx->dim, nullptr, cgi, cg);
}

extern "C" int hx_rates(hx_ctx* ctx, const hx_params* prm, const double* x, const double* v, const double* e,
                        double* dv, double* de, hx_step_info* info) {
  if (!ctx || !prm || !x || !v || !e || !dv || !de || !ctx->phase) return HX_EINVAL;
  CK(cudaSetDevice(ctx->device));
  hx_cg_info ci{};
  StatusDev* st = ctx->st + 0;
  int rc = rates_device(ctx, prm, x, v, e, dv, de, st, &ci);
  if (rc) return rc;
  rc = read_status(ctx, st, ctx->h_st);
  if (rc) return rc;
  const StatusDev& h = ctx->h_st[0];
  hx_step_info out{};
  out.cg_iterations[0] = ci.iterations;
  out.clamped = (int64_t)h.clamps;
  out.min_h_over_speed = h.min_ratio;
  decode_inv(ctx, h.inv_key, &out.inv);
  out.code = out.inv.inverted ? HX_EINVERTED : ci.code;
  if (info) *info = out;
  return out.code;
}

// timestep_estimate (dt_fixed < 0) + rk2_step on device (hydro.py:364-405)
static int step_impl(hx_ctx* ctx, const hx_params* prm, double t, double dt_fixed, const double* x,
                     const double* v, const double* e, double* x_out, double* v_out, double* e_out,
                     hx_step_info* info, int attempt0 = 0, const hx_step_info* carry = nullptr) {
  if (!ctx || !prm || !x || !v || !e || !x_out || !v_out || !e_out || !ctx->phase) return HX_EINVAL;
  {
    const int irc = issue_inputs(ctx);  // plain launches may sync mid-step: copies first
    if (irc) return irc;
  }
  CK(cudaSetDevice(ctx->device));
  const bool estimate = dt_fixed < 0.0;
  hx_step_info out{};
  if (carry) out = *carry;
  const long long nv = ctx->nn * ctx->dim, nte = ctx->ne * ctx->nt;
  const unsigned ga = gblocks((std::max(nv, nte) + 1) / 2, 256);  // 2 entries per thread
  long long clamps_total = carry ? carry->clamped : 0;
  for (int attempt = attempt0; attempt <= prm->max_retries; ++attempt) {
    // stage 1: rates(S) -- its ratio is also timestep_estimate's (same state)
    hx_cg_info c0{}, c1{};
    int rc = rates_device(ctx, prm, x, v, e, ctx->dv0, ctx->de0, ctx->st + 0, &c0, ctx->cg);
    if (rc) return rc;
    DtArgs da{ctx->st + 0, ctx->dt, prm->cfl, prm->dt_max, prm->t_final, t, dt_fixed, attempt, nullptr};
    k_dt<<<1, 1, 0, ctx->stream>>>(da);
    CKL();
    AxpyArgs m{x, v, e, v, ctx->dv0, ctx->de0, ctx->xm, ctx->vm, ctx->em, ctx->dt + 1, 0.5, nv, nte};
    prof_begin(ctx, K_AXPY);
    k_axpy_state<<<ga, 256, 0, ctx->stream>>>(m);
    prof_end(ctx);
    CKL();
    rc = read_status(ctx, ctx->st + 0, ctx->h_st + 0);
    if (rc) return rc;
    const StatusDev s0 = ctx->h_st[0];
    CK(cudaMemcpy(ctx->h_dt, ctx->dt, 2 * sizeof(double), cudaMemcpyDeviceToHost));
    if (!estimate && s0.inv_key != ~0ull) {  // rates(state) raised inside rk2_step: retry
      out.failed_stage = 0;
      decode_inv(ctx, s0.inv_key, &out.inv);
      out.retries = attempt + 1;
      continue;
    }
    if (estimate && attempt == 0) {
      if (s0.inv_key != ~0ull) {  // timestep_estimate on an inverted state raises
        out.code = HX_EINVERTED;
        out.failed_stage = 0;
        decode_inv(ctx, s0.inv_key, &out.inv);
        if (info) *info = out;
        return out.code;
      }
      clamps_total += (long long)s0.clamps;  // timestep_estimate's stress_qdata call
      out.dt = ctx->h_dt[0];
      if (ctx->h_dt[0] < prm->dt_min) {
        out.code = HX_EUNDERFLOW;
        out.failed_stage = 0;
        if (info) *info = out;
        return out.code;
      }
    }
    clamps_total += (long long)s0.clamps;  // rates(state)
    if (c0.code) {
      out.code = c0.code;
      if (info) *info = out;
      return out.code;
    }
    // stage 2: rates(mid)
    rc = rates_device(ctx, prm, ctx->xm, ctx->vm, ctx->em, ctx->dv1, ctx->de1, ctx->st + 1, &c1, ctx->cg + 1);
    if (rc) return rc;
    AxpyArgs n{x, v, e, ctx->vm, ctx->dv1, ctx->de1, x_out, v_out, e_out, ctx->dt + 1, 1.0, nv, nte};
    prof_begin(ctx, K_AXPY);
    k_axpy_state<<<ga, 256, 0, ctx->stream>>>(n);
    prof_end(ctx);
    CKL();
    // validity of the new geometry (hydro.py:400-401)
    rc = status_reset(ctx, ctx->st + 2);
    if (rc) return rc;
    rc = validity_launch(ctx, x_out, ctx->st + 2);
    if (rc) return rc;
    CK(cudaMemcpyAsync(ctx->h_st + 1, ctx->st + 1, 2 * sizeof(StatusDev), cudaMemcpyDeviceToHost, ctx->stream));
    rc = peer_err_fetch(ctx);
    if (rc) return rc;
    CK(cudaStreamSynchronize(ctx->stream));
    rc = peer_check(ctx);
    if (rc) return rc;
    const StatusDev s1 = ctx->h_st[1], s2 = ctx->h_st[2];
    out.cg_iterations[0] = c0.iterations;
    out.cg_iterations[1] = c1.iterations;
    if (s1.inv_key != ~0ull) {  // rates(mid) raised before stress_qdata
      out.failed_stage = 1;
      decode_inv(ctx, s1.inv_key, &out.inv);
      out.retries = attempt + 1;
      continue;
    }
    clamps_total += (long long)s1.clamps;
    if (c1.code) {
      out.code = c1.code;
      if (info) *info = out;
      return out.code;
    }
    if (s2.inv_key != ~0ull) {
      out.failed_stage = 2;
      decode_inv(ctx, s2.inv_key, &out.inv);
      out.retries = attempt + 1;
      continue;
    }
    out.code = HX_OK;
    out.retries = attempt;
    ctx->last_iters[0] = c0.iterations;
    ctx->last_iters[1] = c1.iterations;
    out.dt = ctx->h_dt[1];
    out.min_h_over_speed = s1.min_ratio;
    out.t_new = t + ctx->h_dt[1];
    out.clamped = clamps_total;
    out.inv.inverted = 0;
    if (info) *info = out;
    return HX_OK;
  }
  out.code = HX_EUNDERFLOW;
  out.clamped = clamps_total;
  if (info) *info = out;
  return out.code;
}

// ---- the same step as ONE CUDA graph (attempt 0; retries fall back to step_impl)

// Mark the CG working set (arena) as L2-persisting on a stream (HX_L2PERSIST=0 disables):
// the ~21 iterations of a momentum solve re-read it while the rates kernels stream
// through M_e^{-1} and the point data.  Captured into the step graph's kernel nodes.
static void l2_window(hx_ctx* ctx, cudaStream_t s) {
  static int on = -1;
  if (on < 0) {
    const char* v = getenv("HX_L2PERSIST");
    on = (v && v[0] == '0') ? 0 : 1;
  }
  if (!on || !ctx->arena) return;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, ctx->device) != cudaSuccess) return;
  if (prop.persistingL2CacheMaxSize <= 0 || prop.accessPolicyMaxWindowSize <= 0) return;
  // only when the working set fits in L2: on a larger one (a 30^3 Q3 brick, 180 MB) the
  // persisting window measured 2-4x slower CG kernels; on a 23^3 brick (81 MB) +1%
  if (ctx->arena_bytes > (size_t)prop.l2CacheSize) return;
  const size_t persist = std::min<size_t>(prop.persistingL2CacheMaxSize, ctx->arena_bytes);
  cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, persist);
  cudaStreamAttrValue v = {};
  v.accessPolicyWindow.base_ptr = ctx->arena;
  v.accessPolicyWindow.num_bytes = std::min<size_t>(ctx->arena_bytes, (size_t)prop.accessPolicyMaxWindowSize);
  v.accessPolicyWindow.hitRatio = std::min(1.0f, (float)persist / (float)v.accessPolicyWindow.num_bytes);
  v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
  v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
  cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &v);
  cudaGetLastError();
}

static bool same_params(const hx_params& a, const hx_params& b) { return memcmp(&a, &b, sizeof a) == 0; }

static int g_early = -1;  // HX_EARLY=0: the serial step graph (x', e', validity at the end)

// end of a captured step: status / CG state / dt words into the pinned host copies
struct StatusOut {
  const unsigned long long* src[3];
  unsigned long long* dst[3];
  int n[3];
};
static_assert(sizeof(StatusDev) % 8 == 0 && sizeof(CGDev) % 8 == 0, "word copies");
__global__ void k_status_out(StatusOut so) {
#pragma unroll
  for (int r = 0; r < 3; ++r)
    for (int i = threadIdx.x; i < so.n[r]; i += blockDim.x) so.dst[r][i] = __ldcg(so.src[r] + i);
}
static int g_status_kernel = -1;  // HX_STATUS_KERNEL=0: three D2H copy nodes instead

static int capture_step(hx_ctx* ctx, const hx_params* prm, double dt_fixed, const double* x, const double* v,
                        const double* e, double* x_out, double* v_out, double* e_out, cudaGraphExec_t* exec,
                        hx_ctx::GProf* gprof = nullptr) {
  const long long nv = ctx->nn * ctx->dim, nte = ctx->ne * ctx->nt;
  const unsigned ga = gblocks((std::max(nv, nte) + 1) / 2, 256);  // 2 entries per thread
  if (g_early < 0) {
    const char* ge = getenv("HX_EARLY");
    g_early = (ge && ge[0] == '0') ? 0 : 1;
  }
  cudaStream_t user = ctx->stream;
  const bool prof = ctx->prof_on;
  const long long launches = ctx->launches;
  ctx->prof_on = false;
  ctx->stream = ctx->gstream;
  if (gprof) {
    gprof->stage.clear();
    gprof->iter.clear();
    ctx->gp = gprof;
    ctx->prof_capture = true;
  }
  cudaGraph_t graph = nullptr;
  int rc = HX_OK;
  l2_window(ctx, ctx->gstream);
  l2_window(ctx, ctx->gstream2);
  auto body = [&]() -> int {
    CK(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
    int r = status_reset(ctx, ctx->st, 3);
    if (r) return r;
    const uint8_t* mask = ctx->has_mask ? ctx->mask : nullptr;
    // stage 1: rates(S); its CFL ratio is timestep_estimate's
    ctx->prof_tag_stage = -1;
    r = rates_launch(ctx, prm, x, v, e, ctx->de0, ctx->st + 0);
    if (r) return r;
    ctx->prof_tag_stage = 0;
    CGLaunch L0;
    r = cg_prepare(ctx, ctx->cg, ctx->Dm, nullptr, ctx->evec, 1, mask, ctx->invd, prm->rel_tol, prm->max_iter,
                   ctx->dv0, ctx->dim, nullptr, L0, ctx->emapf);
    if (r) return r;
    r = cg_capture(ctx, L0, ctx->last_iters[0]);
    if (r) return r;
    ctx->prof_tag_stage = -1;
    DtArgs da{ctx->st + 0, ctx->dt, prm->cfl, prm->dt_max, prm->t_final, 0.0, dt_fixed, 0, ctx->t_dev};
    k_dt<<<1, 1, 0, ctx->stream>>>(da);
    CKL();
    // single GPU: x' = x + dt v_half is known as soon as v_half is, and e' = e + dt de1 after
    // stage 2's rates, so both are written early; external events mark them for the host
    // read-back of hx_step_host, which then overlaps stage 2.  (A side branch running the
    // validity check of x' concurrently with stage 2 measured neutral and costs two more
    // streams per context, so the check stays at the end.)
    const bool early = !ctx->peer && g_early != 0;
    AxpyArgs m{x, v, e, v, ctx->dv0, ctx->de0, ctx->xm, ctx->vm, ctx->em, ctx->dt + 1, 0.5, nv, nte};
    if (early) m.xf = x_out;
    prof_begin(ctx, K_AXPY);
    k_axpy_state<<<ga, 256, 0, ctx->stream>>>(m);
    prof_end(ctx);
    CKL();
    cudaStream_t main_s = ctx->stream;
    if (early) CK(cudaEventRecordWithFlags(ctx->ev_x, main_s, cudaEventRecordExternal));
    // stage 2: rates(mid)
    r = rates_launch(ctx, prm, ctx->xm, ctx->vm, ctx->em, ctx->de1, ctx->st + 1);
    if (r) return r;
    if (early) {
      AxpyArgs ee{x, v, e, nullptr, nullptr, ctx->de1, nullptr, nullptr, e_out, ctx->dt + 1, 1.0, 0, nte};
      k_axpy_state<<<gblocks((nte + 1) / 2, 256), 256, 0, ctx->stream>>>(ee);
      CKL();
      CK(cudaEventRecordWithFlags(ctx->ev_e, main_s, cudaEventRecordExternal));
    }
    ctx->prof_tag_stage = 1;
    CGLaunch L1;
    r = cg_prepare(ctx, ctx->cg + 1, ctx->Dm, nullptr, ctx->evec, 1, mask, ctx->invd, prm->rel_tol,
                   prm->max_iter, ctx->dv1, ctx->dim, nullptr, L1, ctx->emapf);
    if (r) return r;
    r = cg_capture(ctx, L1, ctx->last_iters[1]);
    if (r) return r;
    ctx->prof_tag_stage = -1;
    AxpyArgs n{x, v, e, ctx->vm, ctx->dv1, ctx->de1, early ? nullptr : x_out, v_out, early ? nullptr : e_out,
               ctx->dt + 1, 1.0, nv, early ? 0 : nte};
    prof_begin(ctx, K_AXPY);
    k_axpy_state<<<ga, 256, 0, ctx->stream>>>(n);
    prof_end(ctx);
    CKL();
    if (early) CK(cudaEventRecordWithFlags(ctx->ev_v, main_s, cudaEventRecordExternal));  // v' read back during the check
    // validity of the new geometry
    r = validity_launch(ctx, x_out, ctx->st + 2);
    if (r) return r;
    if (g_status_kernel < 0) {
      const char* sk = getenv("HX_STATUS_KERNEL");
      g_status_kernel = (sk && sk[0] == '0') ? 0 : 1;
    }
    if (g_status_kernel) {
      // one kernel node writes the step's status, CG states and dt straight into the pinned
      // (UVA-mapped) host copies instead of three small D2H copy nodes
      StatusOut so{{reinterpret_cast<const unsigned long long*>(ctx->st),
                    reinterpret_cast<const unsigned long long*>(ctx->cg),
                    reinterpret_cast<const unsigned long long*>(ctx->dt)},
                   {reinterpret_cast<unsigned long long*>(ctx->h_st), reinterpret_cast<unsigned long long*>(ctx->h_cg),
                    reinterpret_cast<unsigned long long*>(ctx->h_dt)},
                   {(int)(3 * sizeof(StatusDev) / 8), (int)(2 * sizeof(CGDev) / 8), 2}};
      k_status_out<<<1, 128, 0, ctx->stream>>>(so);
      CKL();
    } else {
      CK(cudaMemcpyAsync(ctx->h_st, ctx->st, 3 * sizeof(StatusDev), cudaMemcpyDeviceToHost, ctx->stream));
      CK(cudaMemcpyAsync(ctx->h_cg, ctx->cg, 2 * sizeof(CGDev), cudaMemcpyDeviceToHost, ctx->stream));
      CK(cudaMemcpyAsync(ctx->h_dt, ctx->dt, 2 * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    }
    r = peer_err_fetch(ctx);
    if (r) return r;
    CK(cudaStreamEndCapture(ctx->stream, &graph));
    return HX_OK;
  };
  rc = body();
  if (rc) {
    cudaStreamCaptureStatus cs;
    if (cudaStreamIsCapturing(ctx->stream, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone) {
      cudaGraph_t junk;
      cudaStreamEndCapture(ctx->stream, &junk);
      if (junk) cudaGraphDestroy(junk);
    }
    cudaGetLastError();
  }
  ctx->stream = user;
  ctx->prof_on = prof;
  ctx->prof_capture = false;
  ctx->gp = nullptr;
  ctx->prof_tag_stage = -1;
  ctx->launches = launches;
  if (rc) return rc;
  cudaError_t ce = cudaGraphInstantiate(exec, graph, 0);
  cudaGraphDestroy(graph);
  if (ce != cudaSuccess) return fail(ctx, HX_ECUDA, "cudaGraphInstantiate: %s", cudaGetErrorString(ce));
  return HX_OK;
}

static int g_use_graph = -1;  // HX_GRAPH=0 disables the graph path

// the context's own state buffers (host-buffer entry hx_step_host, staged steps)
static int ensure_stage(hx_ctx* ctx) {
  if (!ctx->cstream) CK(cudaStreamCreateWithFlags(&ctx->cstream, cudaStreamNonBlocking));
  if (ctx->hx_x) return HX_OK;
  const size_t nvb = sizeof(double) * ctx->nn * ctx->dim, neb = sizeof(double) * ctx->ne * ctx->nt;
  CK(cudaMalloc(&ctx->hx_x, nvb));
  CK(cudaMalloc(&ctx->hx_v, nvb));
  CK(cudaMalloc(&ctx->hx_e, neb));
  CK(cudaMalloc(&ctx->hx_xo, nvb));
  CK(cudaMalloc(&ctx->hx_vo, nvb));
  CK(cudaMalloc(&ctx->hx_eo, neb));
  return HX_OK;
}

static int step_dispatch(hx_ctx* ctx, const hx_params* prm, double t, double dt_fixed, const double* x,
                         const double* v, const double* e, double* x_out, double* v_out, double* e_out,
                         hx_step_info* info) {
  if (!ctx || !prm || !x || !v || !e || !x_out || !v_out || !e_out || !ctx->phase) return HX_EINVAL;
  if (g_use_graph < 0) {
    const char* s = getenv("HX_GRAPH");
    g_use_graph = (s && s[0] == '0') ? 0 : 1;
  }
  if (!g_use_graph || ctx->prof_on) return step_impl(ctx, prm, t, dt_fixed, x, v, e, x_out, v_out, e_out, info);
  CK(cudaSetDevice(ctx->device));
  const void* key[6] = {x, v, e, x_out, v_out, e_out};
  hx_ctx::StepGraph* sg = nullptr;
  const int dup = ctx->dup_class;
  for (auto& g : ctx->graphs)
    // a caller-given dt (rk2_step) is a graph input like t, not part of the graph
    if (!memcmp(g.key, key, sizeof key) && (g.dt_fixed >= 0.0) == (dt_fixed >= 0.0) && same_params(g.prm, *prm) &&
        g.dup == dup)
      sg = &g;
  if (!sg) {
    // buffers churning (a reference-API caller gets fresh output arrays every call, so the
    // keys keep changing): after two graphs of this configuration, stage through the
    // context's own buffers (D2D copies in and out, ~13 us at 1M dofs) instead of capturing
    // and instantiating a graph per new buffer set
    int same = 0;
    for (auto& g : ctx->graphs)
      if ((g.dt_fixed >= 0.0) == (dt_fixed >= 0.0) && same_params(g.prm, *prm) && g.dup == dup) ++same;
    if (same >= 2 && ctx->step_warm && x != ctx->hx_x) {
      int rc = ensure_stage(ctx);
      if (rc) return rc;
      const size_t nvb = sizeof(double) * ctx->nn * ctx->dim, neb = sizeof(double) * ctx->ne * ctx->nt;
      CK(cudaMemcpyAsync(ctx->hx_x, x, nvb, cudaMemcpyDeviceToDevice, ctx->stream));
      CK(cudaMemcpyAsync(ctx->hx_v, v, nvb, cudaMemcpyDeviceToDevice, ctx->stream));
      CK(cudaMemcpyAsync(ctx->hx_e, e, neb, cudaMemcpyDeviceToDevice, ctx->stream));
      rc = step_dispatch(ctx, prm, t, dt_fixed, ctx->hx_x, ctx->hx_v, ctx->hx_e, ctx->hx_xo, ctx->hx_vo, ctx->hx_eo,
                         info);
      if (rc) return rc;
      CK(cudaMemcpyAsync(x_out, ctx->hx_xo, nvb, cudaMemcpyDeviceToDevice, ctx->stream));
      CK(cudaMemcpyAsync(v_out, ctx->hx_vo, nvb, cudaMemcpyDeviceToDevice, ctx->stream));
      CK(cudaMemcpyAsync(e_out, ctx->hx_eo, neb, cudaMemcpyDeviceToDevice, ctx->stream));
      CK(cudaStreamSynchronize(ctx->stream));
      return HX_OK;
    }
    if (ctx->graphs.size() >= 16) {
      for (auto& g : ctx->graphs)
        if (g.exec) cudaGraphExecDestroy(g.exec);
      ctx->graphs.clear();
    }
    ctx->graphs.emplace_back();
    sg = &ctx->graphs.back();
    memcpy(sg->key, key, sizeof key);
    sg->dt_fixed = dt_fixed;
    sg->prm = *prm;
    sg->dup = dup;
  }
  // the context's very first step runs as plain launches (warms every lazy init: kernel
  // attributes, occupancy queries, workspace sizes); every later new buffer/parameter set is
  // captured on first use
  if (!ctx->step_warm) {
    ctx->step_warm = true;
    return step_impl(ctx, prm, t, dt_fixed, x, v, e, x_out, v_out, e_out, info);
  }
  ++sg->seen;
  if (!sg->exec) {
    if (dup >= 0) sg->gprof = std::make_shared<hx_ctx::GProf>();
    int rc = capture_step(ctx, prm, dt_fixed, x, v, e, x_out, v_out, e_out, &sg->exec, sg->gprof.get());
    if (rc) return rc;
  }
  ctx->h_t[0] = t;
  ctx->h_t[1] = dt_fixed;
  CK(cudaMemcpyAsync(ctx->t_dev, ctx->h_t, 2 * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaGraphLaunch(sg->exec, ctx->stream));
  {
    const int irc = issue_inputs(ctx);  // hx_step_host's slab copies, behind the launch
    if (irc) return irc;
  }
  ctx->early_done = false;
  if (ctx->early_xh && !ctx->peer && g_early == 1) {
    // hx_step_host: read x' and e' back while stage 2 still runs (the graph's external
    // events mark them written); a retried step rewrites them and is read again after
    const size_t nvb = sizeof(double) * ctx->nn * ctx->dim, neb = sizeof(double) * ctx->ne * ctx->nt;
    CK(cudaStreamWaitEvent(ctx->cstream, ctx->ev_x, 0));
    CK(cudaMemcpyAsync(ctx->early_xh, x_out, nvb, cudaMemcpyDeviceToHost, ctx->cstream));
    CK(cudaStreamWaitEvent(ctx->cstream, ctx->ev_e, 0));
    CK(cudaMemcpyAsync(ctx->early_eh, e_out, neb, cudaMemcpyDeviceToHost, ctx->cstream));
    CK(cudaStreamWaitEvent(ctx->cstream, ctx->ev_v, 0));
    CK(cudaMemcpyAsync(ctx->early_vh, v_out, nvb, cudaMemcpyDeviceToHost, ctx->cstream));
    ctx->early_done = true;
  }
  CK(cudaStreamSynchronize(ctx->stream));
  {
    const int prc = peer_check(ctx);  // before the status: a timed-out status exchange reads as an inversion
    if (prc) {
      if (info) info->code = prc;
      return prc;
    }
  }
  const StatusDev s0 = ctx->h_st[0], s1 = ctx->h_st[1], s2 = ctx->h_st[2];
  const CGDev c0 = ctx->h_cg[0], c1 = ctx->h_cg[1];
  ctx->launches += 11 + (g_status_kernel > 0 ? 1 : 0) + 2 * (long long)(c0.iters + c1.iters);
  if (dup >= 0 && sg->gprof) {
    const int it[2] = {c0.iters, c1.iters};
    gprof_collect(ctx, sg->gprof.get(), it);
  }
  hx_step_info out{};
  const bool estimate = dt_fixed < 0.0;
  long long clamps = 0;
  out.cg_iterations[0] = c0.iters;
  out.cg_iterations[1] = c1.iters;
  // interpretation identical to step_impl's first attempt
  if (s0.inv_key != ~0ull) {
    if (estimate) {
      out.code = HX_EINVERTED;
      out.failed_stage = 0;
      decode_inv(ctx, s0.inv_key, &out.inv);
      if (info) *info = out;
      return out.code;
    }
    out.failed_stage = 0;
    decode_inv(ctx, s0.inv_key, &out.inv);
    out.retries = 1;
    return step_impl(ctx, prm, t, dt_fixed, x, v, e, x_out, v_out, e_out, info, 1, &out);
  }
  if (estimate) {
    clamps += (long long)s0.clamps;
    out.dt = ctx->h_dt[0];
    if (ctx->h_dt[0] < prm->dt_min) {
      out.code = HX_EUNDERFLOW;
      out.failed_stage = 0;
      out.clamped = clamps;
      if (info) *info = out;
      return out.code;
    }
  }
  clamps += (long long)s0.clamps;
  if (c0.code) {
    out.code = cg_code(c0.code);
    if (info) *info = out;
    return out.code;
  }
  if (s1.inv_key != ~0ull) {
    out.failed_stage = 1;
    decode_inv(ctx, s1.inv_key, &out.inv);
    out.retries = 1;
    out.clamped = clamps;
    return step_impl(ctx, prm, t, dt_fixed, x, v, e, x_out, v_out, e_out, info, 1, &out);
  }
  clamps += (long long)s1.clamps;
  if (c1.code) {
    out.code = cg_code(c1.code);
    if (info) *info = out;
    return out.code;
  }
  if (s2.inv_key != ~0ull) {
    out.failed_stage = 2;
    decode_inv(ctx, s2.inv_key, &out.inv);
    out.retries = 1;
    out.clamped = clamps;
    return step_impl(ctx, prm, t, dt_fixed, x, v, e, x_out, v_out, e_out, info, 1, &out);
  }
  out.code = HX_OK;
  out.retries = 0;
  out.dt = ctx->h_dt[1];
  out.min_h_over_speed = s1.min_ratio;
  out.t_new = t + ctx->h_dt[1];
  out.clamped = clamps;
  out.inv.inverted = 0;
  if (info) *info = out;
  return HX_OK;
}

extern "C" int hx_step(hx_ctx* ctx, const hx_params* prm, double t, const double* x, const double* v,
                       const double* e, double* x_out, double* v_out, double* e_out, hx_step_info* info) {
  return step_dispatch(ctx, prm, t, -1.0, x, v, e, x_out, v_out, e_out, info);
}

extern "C" int hx_rk2_step(hx_ctx* ctx, const hx_params* prm, double t, double dt, const double* x,
                           const double* v, const double* e, double* x_out, double* v_out, double* e_out,
                           hx_step_info* info) {
  if (!(dt >= 0.0)) return fail(ctx, HX_EINVAL, "dt must be >= 0");
  return step_dispatch(ctx, prm, t, dt, x, v, e, x_out, v_out, e_out, info);
}

// hx_step_host's slab copies + flags on istream (once per call; a no-op when none are pending).
// Called right after the step graph's launch, before a plain-launch step (which may sync the
// stream mid-step), and on hx_step_host's way out (error paths), so every waiting rates launch
// is always followed by its copies.
typedef int (*StreamWrite64Fn)(cudaStream_t, unsigned long long, unsigned long long, unsigned);
static StreamWrite64Fn g_write64 = nullptr;  // cuStreamWriteValue64 (driver entry point), or null

static int issue_inputs(hx_ctx* ctx) {
  if (!ctx->in_xh) return HX_OK;
  const double *x_host = ctx->in_xh, *v_host = ctx->in_vh, *e_host = ctx->in_eh;
  ctx->in_xh = ctx->in_vh = ctx->in_eh = nullptr;
  long long n0 = 0, e0 = 0;
  const int d = ctx->dim, nt = ctx->nt;
  for (int s = 0; s < ctx->in_ns; ++s) {
    const long long n1 = ctx->in_node_end[s], e1 = ctx->in_elem_end[s];
    if (n1 > n0) {
      CK(cudaMemcpyAsync(ctx->hx_x + n0 * d, x_host + n0 * d, sizeof(double) * (n1 - n0) * d,
                         cudaMemcpyHostToDevice, ctx->istream));
      CK(cudaMemcpyAsync(ctx->hx_v + n0 * d, v_host + n0 * d, sizeof(double) * (n1 - n0) * d,
                         cudaMemcpyHostToDevice, ctx->istream));
    }
    if (e1 > e0)
      CK(cudaMemcpyAsync(ctx->hx_e + e0 * nt, e_host + e0 * nt, sizeof(double) * (e1 - e0) * nt,
                         cudaMemcpyHostToDevice, ctx->istream));
    // the flag: a stream memory operation (front end, no DMA: a small H2D copy costs ~13 us)
    if (g_write64) {
      if (g_write64(ctx->istream, (unsigned long long)(uintptr_t)(ctx->in_flag + s), ctx->h_in[s], 0) != 0)
        return fail(ctx, HX_ECUDA, "cuStreamWriteValue64 failed");
    } else {
      CK(cudaMemcpyAsync(ctx->in_flag + s, ctx->h_in + s, sizeof(unsigned long long), cudaMemcpyHostToDevice,
                         ctx->istream));
    }
    n0 = n1;
    e0 = e1;
  }
  return HX_OK;
}

static int g_stream_in = -1;
static constexpr int HX_MAX_SLABS = 64;

// slab boundaries of the streamed inputs: slab s holds the elements of element layers
// [zend(s-1), zend(s)) (e) and every node they touch (x, v: node layers up to P*zend(s)), each
// end rounded up to 16 nodes / 16 elements so that no 128-byte line of x, v or e spans two
// slabs (16 * 24 B = 3 lines, 16 * nt * 8 B = nt lines).  Layer counts halve from slab to slab
// (HX_STREAM_UNIFORM=1: equal): the rates kernel's work left after the last slab lands is
// then small.  The device table zend[] sits behind the flags: in_flag[ns + 1 + s].
static int stream_in_setup(hx_ctx* ctx, int slabs) {
  const int nz = ctx->bk.nz;
  const int ns = std::min(std::min(slabs, nz), HX_MAX_SLABS);
  const char* su = getenv("HX_STREAM_UNIFORM");
  const int geo = (su && su[0] == '1') ? 0 : 1;
  std::vector<int> cnt(ns, 1);
  {
    double wsum = 0.0;
    for (int q = 0; q < ns; ++q) wsum += geo ? std::ldexp(1.0, std::min(ns - 1 - q, 30)) : 1.0;
    int tot = 0;
    for (int q = 0; q < ns; ++q) {
      const double w = geo ? std::ldexp(1.0, std::min(ns - 1 - q, 30)) : 1.0;
      cnt[q] = std::max(1, (int)std::lround(nz * w / wsum));
      tot += cnt[q];
    }
    while (tot > nz) {  // take back from the largest slab
      int m = 0;
      for (int q = 1; q < ns; ++q)
        if (cnt[q] > cnt[m]) m = q;
      --cnt[m];
      --tot;
    }
    for (; tot < nz; ++tot) ++cnt[0];
  }
  const int ez = geo ? -1 : cnt[0];  // cache key (with ns)
  if (!ctx->istream) CK(cudaStreamCreateWithFlags(&ctx->istream, cudaStreamNonBlocking));
  static bool looked = false;
  if (!looked) {
    looked = true;
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue64", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess && !getenv("HX_STREAM_IN_MEMCPY"))
      g_write64 = (StreamWrite64Fn)fn;
    cudaGetLastError();
  }
  if (ctx->in_flag && ctx->in_ns == ns && ctx->in_ez == ez) return HX_OK;
  if (ctx->in_flag) {
    CK(cudaStreamSynchronize(ctx->stream));
    cudaFree(ctx->in_flag);
    ctx->in_flag = nullptr;
  }
  if (!ctx->h_in) {
    CK(cudaHostAlloc(&ctx->h_in, sizeof(unsigned long long) * (HX_MAX_SLABS + 1), cudaHostAllocMapped));
    void* dp = nullptr;
    CK(cudaHostGetDevicePointer(&dp, ctx->h_in, 0));
    ctx->in_err_dev = (unsigned long long*)dp + HX_MAX_SLABS;
  }
  if (ns > HX_MAX_SLABS) return fail(ctx, HX_EINVAL, "streamed inputs: %d slabs > %d", ns, HX_MAX_SLABS);
  CK(cudaMalloc(&ctx->in_flag, sizeof(unsigned long long) * (2 * ns + 1)));
  CK(cudaMemset(ctx->in_flag, 0, sizeof(unsigned long long) * (ns + 1)));
  ctx->in_epoch = 0;
  ctx->in_node_end.assign(ns, 0);
  ctx->in_elem_end.assign(ns, 0);
  const long long lay = (long long)ctx->bk.nx * ctx->bk.ny;
  std::vector<unsigned long long> zt(ns);
  long long zacc = 0;
  for (int s = 0; s < ns; ++s) {
    zacc += cnt[s];
    const long long zend = std::min<long long>(zacc, nz);
    zt[s] = (unsigned long long)zend;
    long long n1 = (zend * ctx->p + 1) * ctx->bk.NxNy, e1 = zend * lay;
    n1 = (n1 + 15) / 16 * 16;
    e1 = (e1 + 15) / 16 * 16;
    ctx->in_node_end[s] = s == ns - 1 ? ctx->nn : std::min(n1, ctx->nn);
    ctx->in_elem_end[s] = s == ns - 1 ? ctx->ne : std::min(e1, ctx->ne);
  }
  CK(cudaMemcpy(ctx->in_flag + ns + 1, zt.data(), sizeof(unsigned long long) * ns, cudaMemcpyHostToDevice));
  ctx->in_ez = ez;
  ctx->in_ns = ns;
  // graphs captured before the slabs existed launch the rates kernel without the wait
  for (auto& g : ctx->graphs)
    if (g.exec) cudaGraphExecDestroy(g.exec);
  ctx->graphs.clear();
  return HX_OK;
}

extern "C" int hx_step_host(hx_ctx* ctx, const hx_params* prm, double t, double* x_host, double* v_host,
                            double* e_host, hx_step_info* info) {
  if (!ctx || !prm || !x_host || !v_host || !e_host) return HX_EINVAL;
  CK(cudaSetDevice(ctx->device));
  const size_t nvb = sizeof(double) * ctx->nn * ctx->dim, neb = sizeof(double) * ctx->ne * ctx->nt;
  int src = ensure_stage(ctx);
  if (src) return src;
  {
    const char* se = getenv("HX_STREAM_IN");  // slabs of the streamed H2D (0: one up-front copy)
    g_stream_in = se ? atoi(se) : 3;  // measured: 2-4 slabs best (per-slab DMA setup ~10 us)
  }
  if (g_rates_kernel < 0) {
    const char* sr = getenv("HX_RATES");
    g_rates_kernel = (sr && strcmp(sr, "cta") == 0) ? 0 : 1;
  }
  const bool streamed = g_stream_in > 0 && ctx->dim == 3 && ctx->p >= 2 && ctx->brick && !ctx->peer &&
                        g_rates_kernel != 0 && ctx->bk.nz >= 2;
  if (streamed) {
    src = stream_in_setup(ctx, g_stream_in);
    if (src) return src;
    // required epoch first (stream-ordered before the step's first rates launch), then the
    // slabs on the copy stream, each followed by its flag; the copies depend on nothing the
    // step does, so the waiting rates kernel cannot block them
    const unsigned long long ep = ++ctx->in_epoch;
    for (int s = 0; s <= ctx->in_ns; ++s) ctx->h_in[s] = ep;
    ctx->h_in[HX_MAX_SLABS] = 0;
    CK(cudaMemcpyAsync(ctx->in_flag + ctx->in_ns, ctx->h_in + ctx->in_ns, sizeof(unsigned long long),
                       cudaMemcpyHostToDevice, ctx->stream));
    ctx->in_xh = x_host;  // enqueued right after the step's launch (issue_inputs): the host's
    ctx->in_vh = v_host;  // enqueue time then overlaps the GPU instead of delaying the launch
    ctx->in_eh = e_host;
  } else {
    CK(cudaMemcpyAsync(ctx->hx_x, x_host, nvb, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(ctx->hx_v, v_host, nvb, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(ctx->hx_e, e_host, neb, cudaMemcpyHostToDevice, ctx->stream));
  }
  // x' and e' may be read back by the step itself while its stage 2 runs (step_dispatch)
  ctx->early_xh = x_host;
  ctx->early_eh = e_host;
  ctx->early_vh = v_host;
  ctx->early_done = false;
  hx_step_info local{};
  hx_step_info* inf = info ? info : &local;
  int rc = hx_step(ctx, prm, t, ctx->hx_x, ctx->hx_v, ctx->hx_e, ctx->hx_xo, ctx->hx_vo, ctx->hx_eo, inf);
  {
    const int irc = issue_inputs(ctx);  // (error paths that launched nothing: keep the flags whole)
    if (streamed) CK(cudaStreamSynchronize(ctx->istream));
    if (irc && !rc) rc = irc;
    if (streamed && !rc && *(volatile unsigned long long*)(ctx->h_in + HX_MAX_SLABS))
      rc = fail(ctx, HX_ECUDA, "hx_step_host: streamed input slab did not land within the wait bound");
  }
  ctx->early_xh = ctx->early_eh = ctx->early_vh = nullptr;
  const bool early = ctx->early_done && inf->retries == 0;
  CK(cudaStreamSynchronize(ctx->cstream));
  if (rc) {
    if (ctx->early_done) {  // a failed step leaves the caller's state as it was
      CK(cudaMemcpyAsync(x_host, ctx->hx_x, nvb, cudaMemcpyDeviceToHost, ctx->stream));
      CK(cudaMemcpyAsync(v_host, ctx->hx_v, nvb, cudaMemcpyDeviceToHost, ctx->stream));
      CK(cudaMemcpyAsync(e_host, ctx->hx_e, neb, cudaMemcpyDeviceToHost, ctx->stream));
      CK(cudaStreamSynchronize(ctx->stream));
    }
    return rc;
  }
  if (!early) {
    CK(cudaMemcpyAsync(x_host, ctx->hx_xo, nvb, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaMemcpyAsync(v_host, ctx->hx_vo, nvb, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaMemcpyAsync(e_host, ctx->hx_eo, neb, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
  }
  return HX_OK;
}

extern "C" int hx_energies(hx_ctx* ctx, const double* v, const double* e, const double* qdata0, double* kinetic,
                           double* internal) {
  if (!ctx || !v || !e || !qdata0 || !ctx->phase) return HX_EINVAL;
  CK(cudaSetDevice(ctx->device));
  // KE = 0.5 v . (M v)  (hydro.py:409-411)
  int rc = mass_evec(ctx, ctx->Dm, v, ctx->dim, ctx->evec2);
  if (rc) return rc;
  rc = launch_scatter(ctx, ctx->evec2, ctx->dim, ctx->xm);
  if (rc) return rc;
  k_dot<<<1, 256, 0, ctx->stream>>>(v, ctx->xm, ctx->nn * ctx->dim, ctx->scal);
  CKL();
  // IE = sum w qdata0 e_q (hydro.py:413-420); qdata0 given in reference layout
  const long long n = (long long)ctx->nq * ctx->ne;
  k_transpose<<<gblocks(n, 256), 256, 0, ctx->stream>>>(qdata0, ctx->nq, ctx->ne, ctx->evec2);
  CKL();
  rc = dispatch<LaunchIE>(ctx, e, (const double*)ctx->evec2, ctx->vm);
  if (rc) return rc;
  k_sum<<<1, 256, 0, ctx->stream>>>(ctx->vm, ctx->ne, ctx->scal + 1);
  CKL();
  double h[2];
  CK(cudaMemcpyAsync(h, ctx->scal, sizeof h, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  if (kinetic) *kinetic = 0.5 * h[0];
  if (internal) *internal = h[1];
  return HX_OK;
}

// ---------------------------------------------------------------------------
// ---------------------------------------------------------------------------
// multi-GPU exchange over peer memory (hx_peer.cuh)

static constexpr size_t mailbox_doubles(int maxh) { return (size_t)MB_RECV + (size_t)HX_MAXR * maxh * 3; }

extern "C" int hx_peer_setup(hx_ctx* ctx, int rank, int nranks, int maxh, int nsh, const int32_t* snode,
                             const int32_t* sdst, const int32_t* sidx, int nh, const int32_t* hnode,
                             const int32_t* hoff, const int32_t* hsrc, int nnbr, const int32_t* nbr,
                             const uint8_t* owned, void** mailbox) {
  if (!ctx || !mailbox || nranks < 1 || nranks > HX_MAXR || rank < 0 || rank >= nranks || maxh < 0 || nsh < 0 ||
      nh < 0 || nnbr < 0 || nnbr > HX_MAXR || !owned || (nsh && (!snode || !sdst || !sidx)) ||
      (nh && (!hnode || !hoff || !hsrc)) || (nnbr && !nbr))
    return fail(ctx, HX_EINVAL, "hx_peer_setup: bad arguments");
  if (maxh >= (1 << 24)) return fail(ctx, HX_EINVAL, "hx_peer_setup: halo too large");
  CK(cudaSetDevice(ctx->device));
  const long long nhs = nh ? hoff[nh] : 0;
  for (int j = 0; j < nsh; ++j)
    if (sdst[j] < 0 || sdst[j] >= nranks || sidx[j] < 0 || sidx[j] >= maxh || snode[j] < 0 || snode[j] >= ctx->nn)
      return fail(ctx, HX_EINVAL, "hx_peer_setup: shared entry %d out of range", j);
  for (int h = 0; h < nh; ++h)
    if (hnode[h] < 0 || hnode[h] >= ctx->nn || hoff[h + 1] < hoff[h])
      return fail(ctx, HX_EINVAL, "hx_peer_setup: interface node %d out of range", h);
  for (long long s = 0; s < nhs; ++s)
    if (hsrc[s] >= 0 && ((hsrc[s] >> 24) >= nranks || (hsrc[s] & 0xffffff) >= maxh))
      return fail(ctx, HX_EINVAL, "hx_peer_setup: sharer entry %lld out of range", s);
  if (ctx->mailbox) cudaFree(ctx->mailbox);
  if (ctx->peer_plan) cudaFree(ctx->peer_plan);
  if (ctx->peer_owned) cudaFree(ctx->peer_owned);
  if (ctx->peer_ctr) cudaFree(ctx->peer_ctr);
  ctx->mailbox = nullptr;
  ctx->peer_plan = nullptr;
  ctx->peer_owned = nullptr;
  ctx->peer_ctr = nullptr;
  ctx->peer = false;
  for (auto& g : ctx->graphs)  // graphs captured with the previous exchange state
    if (g.exec) cudaGraphExecDestroy(g.exec);
  ctx->graphs.clear();
  ctx->step_warm = false;
  const size_t nmb = mailbox_doubles(maxh);
  CK(dalloc(&ctx->mailbox, nmb));
  CK(cudaMemset(ctx->mailbox, 0, nmb * sizeof(double)));
  const size_t nplan = 3 * (size_t)nsh + (size_t)nh + (size_t)nh + 1 + (size_t)nhs;
  std::vector<int> plan(std::max<size_t>(nplan, 1));
  size_t o = 0;
  for (int j = 0; j < nsh; ++j) plan[o + j] = snode[j];
  o += nsh;
  for (int j = 0; j < nsh; ++j) plan[o + j] = sdst[j];
  o += nsh;
  for (int j = 0; j < nsh; ++j) plan[o + j] = sidx[j];
  o += nsh;
  for (int h = 0; h < nh; ++h) plan[o + h] = hnode[h];
  o += nh;
  for (int h = 0; h <= nh; ++h) plan[o + h] = nh ? hoff[h] : 0;
  o += nh + 1;
  for (long long q = 0; q < nhs; ++q) plan[o + q] = hsrc[q];
  CK(dalloc(&ctx->peer_plan, plan.size()));
  CK(cudaMemcpy(ctx->peer_plan, plan.data(), plan.size() * sizeof(int), cudaMemcpyHostToDevice));
  CK(dalloc(&ctx->peer_owned, (size_t)ctx->nn));
  CK(cudaMemcpy(ctx->peer_owned, owned, (size_t)ctx->nn, cudaMemcpyHostToDevice));
  {
    std::vector<int> ifx((size_t)ctx->nn, -1);
    for (int h = 0; h < nh; ++h) ifx[hnode[h]] = h;
    if (ctx->peer_ifx) cudaFree(ctx->peer_ifx);
    CK(dalloc(&ctx->peer_ifx, (size_t)ctx->nn));
    CK(cudaMemcpy(ctx->peer_ifx, ifx.data(), ifx.size() * sizeof(int), cudaMemcpyHostToDevice));
  }
  CK(dalloc(&ctx->peer_ctr, 2));
  CK(cudaMemset(ctx->peer_ctr, 0, 2 * sizeof(unsigned long long)));
  PeerDev& pd = ctx->pd;
  pd = PeerDev{};
  pd.rank = rank;
  pd.nranks = nranks;
  pd.maxh = maxh;
  pd.nsh = nsh;
  pd.nh = nh;
  pd.nnbr = nnbr;
  pd.seq = ctx->peer_ctr;
  pd.err = reinterpret_cast<int*>(ctx->peer_ctr + 1);
  for (int q = 0; q < nnbr; ++q) pd.nbr[q] = nbr[q];
  const int* P = ctx->peer_plan;
  pd.snode = P;
  pd.sdst = P + nsh;
  pd.sidx = P + 2 * nsh;
  pd.hnode = P + 3 * nsh;
  pd.hoff = P + 3 * nsh + nh;
  pd.hsrc = P + 3 * nsh + 2 * nh + 1;
  pd.owned = ctx->peer_owned;
  pd.ifx = ctx->peer_ifx;
  *mailbox = ctx->mailbox;
  return HX_OK;
}

extern "C" int hx_peer_connect(hx_ctx* ctx, void* const* mailboxes) {
  if (!ctx || !mailboxes || !ctx->mailbox) return fail(ctx, HX_EINVAL, "hx_peer_connect: call hx_peer_setup first");
  for (int q = 0; q < ctx->pd.nranks; ++q) {
    if (!mailboxes[q] && q != ctx->pd.rank) return fail(ctx, HX_EINVAL, "hx_peer_connect: mailbox of rank %d missing", q);
    ctx->pd.mb[q] = q == ctx->pd.rank ? ctx->mailbox : static_cast<double*>(mailboxes[q]);
  }
  // load the exchange kernels now: with lazy module loading a first launch may wait for
  // the context's running kernels -- a peer's spin-wait when ranks share a process
  for (int nc = 1; nc <= 3; ++nc) {
    int rc = with_node_sum(ctx, nc, ctx->evec, [&](auto sum, auto ncc) -> int {
      cudaFuncAttributes fa;
      CK(cudaFuncGetAttributes(&fa, k_halo_pack<decltype(ncc)::value, decltype(sum)>));
      CK(cudaFuncGetAttributes(&fa, k_halo_combine<decltype(ncc)::value, decltype(sum)>));
      return HX_OK;
    });
    if (rc) return rc;
  }
  cudaFuncAttributes fa;
  CK(cudaFuncGetAttributes(&fa, k_peer_sync<0>));
  CK(cudaFuncGetAttributes(&fa, k_peer_status));
  if (!ctx->pd_dev) CK(dalloc(&ctx->pd_dev, 1));
  CK(cudaMemcpy(ctx->pd_dev, &ctx->pd, sizeof(PeerDev), cudaMemcpyHostToDevice));
  // step graphs captured before the exchange was connected lack its launches
  for (auto& g : ctx->graphs)
    if (g.exec) cudaGraphExecDestroy(g.exec);
  ctx->graphs.clear();
  ctx->step_warm = false;
  // HX_PEER_POST=1: the CG's world scalars posted by their producer launches (PeerLite::post).
  // Opt-in: on the one-rank proxy the producers' last-CTA tail (740 arrivals on one counter,
  // then the reduction) costs more than the consumer-side handshake it replaces (2.23 vs 2.11
  // ms/step, profiles/r2/r2g_variants.md); the opt-in mass-kernel variants never post
  auto envon = [](const char* n) {
    const char* v = getenv(n);
    return v && v[0] && v[0] != '0';
  };
  int post = 0;
  if (envon("HX_PEER_POST") && !envon("HX_MASS_TMA") && !envon("HX_MASS_W2") && !MASS_PIPE && ctx->brick &&
      ctx->elem_major)
    post = PEER_POST_ON | (ctx->pd.nsh == 0 ? PEER_POST_MASS : 0);
  ctx->pl = PeerLite{ctx->mailbox, reinterpret_cast<double* const*>(reinterpret_cast<char*>(ctx->pd_dev) +
                                                                     offsetof(PeerDev, mb)),
                     ctx->peer_ctr, ctx->pd.rank, ctx->pd.nranks, post};
  ctx->peer = true;
  return HX_OK;
}

// detach the context from the exchange: waits for its queued work, drops the peer
// pointers and every step graph that contains exchange launches.  Phase data built with
// interface sums (mass diagonal) stay; call hx_phase_begin again before solo steps.
extern "C" int hx_peer_disconnect(hx_ctx* ctx) {
  if (!ctx) return HX_EINVAL;
  CK(cudaSetDevice(ctx->device));
  CK(cudaStreamSynchronize(ctx->stream));
  CK(cudaStreamSynchronize(ctx->gstream));
  for (auto& g : ctx->graphs)
    if (g.exec) cudaGraphExecDestroy(g.exec);
  ctx->graphs.clear();
  ctx->step_warm = false;
  ctx->peer = false;
  for (int q = 0; q < HX_MAXR; ++q) ctx->pd.mb[q] = nullptr;
  if (ctx->pd_dev) CK(cudaMemcpy(ctx->pd_dev, &ctx->pd, sizeof(PeerDev), cudaMemcpyHostToDevice));
  return HX_OK;
}

extern "C" int hx_peer_ipc_handle(const void* mailbox, void* handle_out) {
  if (!mailbox || !handle_out) return HX_EINVAL;
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, const_cast<void*>(mailbox)) != cudaSuccess) return HX_ECUDA;
  memcpy(handle_out, &h, sizeof h);
  return HX_OK;
}

extern "C" int hx_peer_ipc_open(const void* handle, void** ptr_out) {
  if (!handle || !ptr_out) return HX_EINVAL;
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof h);
  if (cudaIpcOpenMemHandle(ptr_out, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) return HX_ECUDA;
  return HX_OK;
}

extern "C" int hx_peer_ipc_close(void* ptr) {
  return cudaIpcCloseMemHandle(ptr) == cudaSuccess ? HX_OK : HX_ECUDA;
}

extern "C" int hx_comm_active(hx_ctx* ctx) { return ctx && ctx->peer ? 1 : 0; }

extern "C" int hx_peer_state(hx_ctx* ctx, uint64_t* out) {
  if (!ctx || !out || !ctx->mailbox) return HX_EINVAL;
  CK(cudaMemcpy(out, ctx->peer_ctr, 2 * sizeof(uint64_t), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(out + 2, ctx->mailbox, HX_MAXR * sizeof(uint64_t), cudaMemcpyDeviceToHost));
  return HX_OK;
}

// ---------------------------------------------------------------------------
// live kernel timing

// fp64 FMA peak probe: 8 independent DFMA chains per thread, full occupancy
__global__ void __launch_bounds__(256) k_fp64_probe(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) x[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < 8; ++c) x[c] = fma(x[c], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += x[c];
  if (s == 12345.678) out[threadIdx.x] = s;  // keeps the chains live
}

extern "C" int hx_fp64_peak(double* tflops) {
  if (!tflops) return HX_EINVAL;
  int dev = 0, sms = 0, occ = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return HX_ECUDA;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_fp64_probe, 256, 0);
  double* out = nullptr;
  cudaStream_t st = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  int rc = HX_OK;
  const unsigned blocks = (unsigned)(sms * occ);
  const int iters = 20000;
  float best = 1e30f;
  if (cudaMalloc(&out, 256 * sizeof(double)) != cudaSuccess || cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreate(&e0) != cudaSuccess || cudaEventCreate(&e1) != cudaSuccess) {
    rc = HX_ECUDA;
  } else {
    k_fp64_probe<<<blocks, 256, 0, st>>>(out, 100, 0.999999, 1e-7);
    for (int r = 0; r < 5 && rc == HX_OK; ++r) {
      cudaEventRecord(e0, st);
      k_fp64_probe<<<blocks, 256, 0, st>>>(out, iters, 0.999999, 1e-7);
      cudaEventRecord(e1, st);
      if (cudaEventSynchronize(e1) != cudaSuccess) rc = HX_ECUDA;
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms > 0.f && ms < best) best = ms;
    }
  }
  if (rc == HX_OK) *tflops = 2.0 * (double)blocks * 256.0 * iters * 8.0 / (best * 1e-3) / 1e12;
  if (e0) cudaEventDestroy(e0);
  if (e1) cudaEventDestroy(e1);
  if (st) cudaStreamDestroy(st);
  if (out) cudaFree(out);
  return rc;
}

// duplicate the kernel node just captured on ctx->stream and make it the capture's new
// tail.  The node pass (K_CGNODE) is not idempotent (r -= alpha Ap): its duplicate is a
// dry copy whose outputs (x, r, (z, p) pairs, r.z partials) go to scratch buffers -- the
// same loads, arithmetic and store volume; its CG-state writes repeat the original's.
static int dup_last_node(hx_ctx* c, int cls) {
  cudaStreamCaptureStatus cs;
  cudaGraph_t g;
  const cudaGraphNode_t* deps = nullptr;
  size_t nd = 0;
  if (cudaStreamGetCaptureInfo(c->stream, &cs, nullptr, &g, &deps, &nd) != cudaSuccess || nd != 1)
    return HX_ECUDA;
  cudaGraphNode_t last = deps[0];
  cudaGraphNodeType ty;
  if (cudaGraphNodeGetType(last, &ty) != cudaSuccess || ty != cudaGraphNodeTypeKernel) return HX_ECUDA;
  cudaKernelNodeParams kp;
  if (cudaGraphKernelNodeGetParams(last, &kp) != cudaSuccess) return HX_ECUDA;
  NodeArgs dry;
  void* args2[2];
  if (cls == K_CGNODE) {
    const long long nv = c->nn * 3;
    if (!c->dup_scratch) return HX_ECUDA;  // allocated by hx_prof_dup (no cudaMalloc while capturing)
    memcpy(&dry, kp.kernelParams[0], sizeof dry);
    dry.x = c->dup_scratch;
    dry.r = c->dup_scratch + nv;
    dry.pbuf0 = c->dup_scratch + 2 * nv;
    dry.pbuf1 = c->dup_scratch + 4 * nv;
    dry.partials = c->dup_scratch + 6 * nv;
    args2[0] = &dry;
    args2[1] = kp.kernelParams[1];
    kp.kernelParams = args2;
  }
  cudaGraphNode_t node;
  if (cudaGraphAddKernelNode(&node, g, &last, 1, &kp) != cudaSuccess) return HX_ECUDA;
  cudaGraphKernelNodeCopyAttributes(node, last);  // L2 access-policy window of the original
  cudaGetLastError();
  if (cudaStreamUpdateCaptureDependencies(c->stream, &node, 1, cudaStreamSetCaptureDependencies) != cudaSuccess)
    return HX_ECUDA;
  return HX_OK;
}

// step graphs captured from now on duplicate every launch of kernel class `cls`
// (-1: plain graphs); hx_prof_read(cls) then counts the duplicates that did work
extern "C" int hx_prof_dup(hx_ctx* ctx, int cls) {
  if (!ctx || cls < -1 || cls > K_OTHER) return HX_EINVAL;
  if (cls == K_CGNODE && !ctx->dup_scratch) {
    CK(cudaSetDevice(ctx->device));
    CK(dalloc(&ctx->dup_scratch, (size_t)6 * ctx->nn * 3 + 2 * (size_t)ctx->preg));
  }
  ctx->dup_class = cls;
  return HX_OK;
}

extern "C" int hx_prof_enable(hx_ctx* ctx, int on) {
  if (!ctx) return HX_EINVAL;
  CK(cudaSetDevice(ctx->device));
  if (on && ctx->prof_ev.empty()) {
    ctx->prof_ev.resize(8192);
    ctx->prof_cls.resize(4096);
    for (auto& e : ctx->prof_ev) CK(cudaEventCreate(&e));
  }
  ctx->prof_on = on != 0;
  return HX_OK;
}

extern "C" int hx_prof_read(hx_ctx* ctx, int kclass, double* total_ms, int64_t* count) {
  if (!ctx || kclass < 0 || kclass > 7) return HX_EINVAL;
  prof_collect(ctx);
  if (total_ms) *total_ms = ctx->prof_tot[kclass];
  if (count) *count = ctx->prof_cnt[kclass];
  return HX_OK;
}

extern "C" int hx_prof_reset(hx_ctx* ctx) {
  if (!ctx) return HX_EINVAL;
  prof_collect(ctx);
  for (int i = 0; i < 8; ++i) {
    ctx->prof_tot[i] = 0;
    ctx->prof_cnt[i] = 0;
  }
  return HX_OK;
}
