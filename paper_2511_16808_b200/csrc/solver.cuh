// solver.cuh -- the templated solver (host orchestration of one hierarchy) shared by the
// per-precision translation units solver_c64.cu / solver_c128.cu (compiled in parallel);
// hmg.cu holds the extern "C" boundary and the process-wide launch / profiling state.
//
//
// Hot path: FGMRES(m) right-preconditioned by one
// multigrid cycle (Alg. 2.1) on the shifted operator H_s (Eq. 2.6)
// with additive Vanka smoothing (Eq. 3.8), Galerkin coarse operators
// and level-dependent intergrid (Eqs. 3.3-3.4).  Every arithmetic
// step runs in the kernels of k_*.cuh; this file only sequences launches.
#pragma once
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <array>
#include <atomic>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <memory>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "../../include/hmg.h"
#include "common.cuh"
#include "runtime.cuh"
#include "k_krylov.cuh"
#include "k_operator.cuh"
#include "k_setup.cuh"
#include "k_transfer.cuh"
#include "k_vanka.cuh"
#include "k_uniform.cuh"
#include "k_stage3d.cuh"
#include "k_tail.cuh"
#include "k_dict.cuh"

namespace hmg {

struct DBuf {
  void *p = nullptr;
  size_t bytes = 0;
  bool own = true;   // false: a view of another DBuf's memory (per-stream workspaces share coefficients)
  DBuf() = default;
  DBuf(const DBuf &) = delete;
  DBuf &operator=(const DBuf &) = delete;
  DBuf(DBuf &&o) noexcept : p(o.p), bytes(o.bytes), own(o.own) { o.p = nullptr; o.bytes = 0; o.own = true; }
  DBuf &operator=(DBuf &&o) noexcept {
    if (this != &o) { release(); p = o.p; bytes = o.bytes; own = o.own; o.p = nullptr; o.bytes = 0; o.own = true; }
    return *this;
  }
  ~DBuf() { release(); }
  static DBuf view(const DBuf &o) {
    DBuf v;
    v.p = o.p;
    v.bytes = o.bytes;
    v.own = false;
    return v;
  }
  void release() {
    if (p && own) cudaFree(p);
    p = nullptr;
    bytes = 0;
    own = true;
  }
  void alloc(size_t n, cudaStream_t s) {
    release();
    if (n == 0) n = 16;
    CK(cudaMalloc(&p, n));
    bytes = n;
    CK(cudaMemsetAsync(p, 0, n, s));
  }
  template <typename X> X *as() const { return reinterpret_cast<X *>(p); }
};

// transfer radii for level l -> l+1
static void level_scheme(int scheme, int l, int &rR, int &rP) {
  switch (scheme) {
    case HMG_LEVDEP: rR = l == 0 ? 2 : 1; rP = 2; break;
    case HMG_LINEAR: rR = 1; rP = 1; break;
    case HMG_CUBIC: rR = 2; rP = 2; break;
    case HMG_MIXED: rR = 1; rP = 2; break;
    default: throw HmgError(HMG_EINVAL, "unknown intergrid scheme");
  }
}

// TMA tensor map over a padded level box (k_stage3d.cuh): 8-byte words, dims
// (x words incl. ghosts, rows incl. ghosts, planes incl. ghosts), box
// (bx elements, by rows, 1 plane); out-of-range box parts are zero-filled.
// cuTensorMapEncodeTiled comes from the driver through the runtime's entry-point
// query (no libcuda link dependency).
static CUtensorMap make_tmap(const void *base, int esz, const Geo &g, int bx, int by) {
  static const PFN_cuTensorMapEncodeTiled_v12000 enc = [] {   // thread-safe one-time lookup
    cudaDriverEntryPointQueryResult q;
    void *fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }();
  if (!enc) throw HmgError(HMG_ECUDA, "cuTensorMapEncodeTiled unavailable");
  CUtensorMap m;
  const int w = esz / 8;
  const int nz = g.dim == 3 ? g.n[2] + 2 * g.G : 1;
  cuuint64_t dims[3] = {(cuuint64_t)g.px * w, (cuuint64_t)(g.n[1] + 2 * g.G), (cuuint64_t)nz};
  cuuint64_t strides[2] = {(cuuint64_t)g.px * esz, (cuuint64_t)g.pxy * esz};
  cuuint32_t box[3] = {(cuuint32_t)(bx * w), (cuuint32_t)by, 1};
  cuuint32_t es[3] = {1, 1, 1};
  const CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, const_cast<void *>(base), dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw HmgError(HMG_ECUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return m;
}

static TransferW transfer_weights(int rR, int rP) {
  TransferW t{};
  t.rR = rR;
  t.rP = rP;
  const double lin[3] = {0.25, 0.5, 0.25};
  const double cub[5] = {1.0 / 16, 4.0 / 16, 6.0 / 16, 4.0 / 16, 1.0 / 16};
  for (int k = 0; k < 2 * rR + 1; ++k) t.wR[k] = rR == 1 ? lin[k] : cub[k];
  for (int k = 0; k < 2 * rP + 1; ++k) t.wP[k] = rP == 1 ? lin[k] : cub[k];
  return t;
}

static int patch_size(int dim, int kind) {
  switch (kind) {
    case HMG_JACOBI: return 1;
    case HMG_VANKA_ELEMENT: return 1 << dim;
    case HMG_VANKA_PLUS: return 2 * dim + 1;
    case HMG_VANKA_RB: return 5;
  }
  return 0;
}

static __global__ void k_identity(int N, double2 *__restrict__ A) {
  HMG_PDL_PROLOGUE();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < (int64_t)N * N) A[i] = make_double2((i / N) == (i % N) ? 1.0 : 0.0, 0.0);
}

// e = A_L^{-1} r for nr right-hand sides at a stride of bs (one warp per row; each
// row of the inverse is read once for all of them)
template <typename T, int NR = 1>
__global__ void k_coarse_gemv(Geo g, const double2 *__restrict__ Ainv, const cplx<T> *__restrict__ r,
                              cplx<T> *__restrict__ e, int64_t bs = 0) {
  HMG_PDL_PROLOGUE();
  const int N = (int)g.nodes();
  const int row = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= N) return;
  double ax[NR], ay[NR];
#pragma unroll
  for (int q = 0; q < NR; ++q) ax[q] = ay[q] = 0;
  for (int col = lane; col < N; col += 32) {
    const int cx = col % g.n[0], cy = (col / g.n[0]) % g.n[1], cz = col / (g.n[0] * g.n[1]);
    const int64_t ci = g.idx(cx, cy, cz);
    const double2 a = Ainv[(int64_t)row * N + col];
#pragma unroll
    for (int q = 0; q < NR; ++q) {
      const cplx<T> v = r[q * bs + ci];
      ax[q] = fma(a.x, (double)v.x, fma(-a.y, (double)v.y, ax[q]));
      ay[q] = fma(a.x, (double)v.y, fma(a.y, (double)v.x, ay[q]));
    }
  }
#pragma unroll
  for (int q = 0; q < NR; ++q) {
    const double sx = warp_sum(ax[q]), sy = warp_sum(ay[q]);
    if (lane == 0) {
      const int rx = row % g.n[0], ry = (row / g.n[0]) % g.n[1], rz = row / (g.n[0] * g.n[1]);
      e[q * bs + g.idx(rx, ry, rz)] = mkc<T>((T)sx, (T)sy);
    }
  }
}

struct SolverBase {
  virtual ~SolverBase() = default;
  hmg_options opt{};
  std::vector<double> damping;
  int L = 0;
  Comm *comm = nullptr;   // not owned; nullptr or size 1 = single GPU
  virtual void build(const double *kappa, double omega, const double *gamma, double alpha, cudaStream_t s) = 0;
  virtual void api_apply(int level, int shifted, const void *x, void *y, cudaStream_t s) = 0;
  virtual void api_residual(int level, int shifted, const void *f, const void *x, void *r, cudaStream_t s) = 0;
  virtual void api_smooth(int level, const void *f, void *u, cudaStream_t s) = 0;
  virtual void api_restrict(int level, const void *r, void *fc, cudaStream_t s) = 0;
  virtual void api_prolong(int level, const void *ec, void *u, cudaStream_t s) = 0;
  virtual void api_coarse(const void *r, void *e, cudaStream_t s) = 0;
  virtual void api_vcycle(const void *f, void *x, int zero, cudaStream_t s) = 0;
  virtual hmg_status api_fgmres(const void *q, void *x, int host, int restart, double tol, int maxiter,
                                cudaStream_t s, hmg_report *rep) = 0;
  virtual hmg_status api_fgmres_batch(int nrhs, const void *q, void *x, int host, int restart, double tol,
                                      int maxiter, cudaStream_t s, hmg_report *reps) = 0;
  virtual int64_t level_nodes(int level, int64_t n[3]) const = 0;
  virtual int radius(int level) const = 0;
  virtual int copy_stencil(int level, double *out, int64_t cap) = 0;
  virtual void level_rows(int level, int64_t *lo, int64_t *hi) const = 0;
  virtual int64_t uniform_box(int level, int64_t *lo, int64_t *hi) const = 0;
  virtual int dict_classes(int level, int *cn, int *bn) const = 0;
  // a solver sharing this one's (immutable) hierarchy with a workspace of its own
  virtual std::unique_ptr<SolverBase> clone_workspace(cudaStream_t s) const = 0;
};

// Slab partition: level-0 rows of the slowest axis split
// evenly; coarse node I belongs to the rank owning fine node 2I, i.e.
// [ceil(lo/2), ceil(hi/2)); a level is distributed while every rank holds at
// least 2 G rows (so a halo of depth <= G comes from the adjacent rank only)
// and all finer levels are distributed; the coarsest level is always
// replicated.  lo/hi/dist are [levels * nranks] / [levels].
static void slab_partition(const std::vector<int64_t> &Nl, int nranks, int G, std::vector<int64_t> &lo,
                           std::vector<int64_t> &hi, std::vector<int> &dist) {
  const int L = (int)Nl.size();
  lo.assign((size_t)L * nranks, 0);
  hi.assign((size_t)L * nranks, 0);
  dist.assign(L, 0);
  for (int r = 0; r < nranks; ++r) {
    lo[r] = Nl[0] * r / nranks;
    hi[r] = Nl[0] * (r + 1) / nranks;
  }
  for (int l = 1; l < L; ++l)
    for (int r = 0; r < nranks; ++r) {
      lo[(size_t)l * nranks + r] = (lo[(size_t)(l - 1) * nranks + r] + 1) / 2;
      hi[(size_t)l * nranks + r] = (hi[(size_t)(l - 1) * nranks + r] + 1) / 2;
    }
  for (int l = 0; l < L - 1; ++l) {
    if (nranks < 2 || (l > 0 && !dist[l - 1])) break;
    bool ok = true;
    for (int r = 0; r < nranks; ++r) ok = ok && hi[(size_t)l * nranks + r] - lo[(size_t)l * nranks + r] >= 2 * G;
    if (!ok) break;
    dist[l] = 1;
  }
}

// Setup windows of the partitioned build: for every slab-partitioned
// level l the global slab-axis rows [wlo, whi) on which this rank computes the
// level's fp64 setup arrays.  They must cover (coarse to fine):
//   - the rows the rank keeps, [lo - G, hi + G), and the patch support around them
//     (2 rows: patch inverses of the anchors within 1 row, each reading its patch's
//     nodes within 1 more; the RB closed form on level 0 reads sigma 1 row away);
//   - the fine rows the next level's Galerkin product R A P (rows 2I -+ rR) -- or the
//     REDISCRETIZE full-weighting average (2I -+ 1) -- reads for that level's window,
//     and for the first replicated level for the rank's own share of its rows
//     (computed here, then allgathered).
// Replicated levels use the whole grid.  Every value a rank keeps is computed from the
// same inputs by the same arithmetic as in the replicated build (bit-identical).
static void plan_windows(const std::vector<int64_t> &Nl, const std::vector<int64_t> &lo,
                         const std::vector<int64_t> &hi, const std::vector<int> &dist, int nranks, int me, int G,
                         const std::vector<int> &rR, bool rediscretize, bool rb_fine, std::vector<int64_t> &wlo,
                         std::vector<int64_t> &whi) {
  const int L = (int)Nl.size();
  wlo.assign(L, 0);
  whi = Nl;
  for (int l = L - 1; l >= 0; --l) {
    if (!dist[l]) continue;
    const int64_t plo = lo[(size_t)l * nranks + me], phi = hi[(size_t)l * nranks + me];
    const int reach = (l == 0 && rb_fine) ? 1 : 2;
    int64_t a = plo - G - reach, b = phi + G + reach;
    if (l + 1 < L) {
      const int64_t na = dist[l + 1] ? wlo[l + 1] : lo[(size_t)(l + 1) * nranks + me];
      const int64_t nb = dist[l + 1] ? whi[l + 1] : hi[(size_t)(l + 1) * nranks + me];
      const int rr = rediscretize ? 1 : rR[l];
      if (nb > na) {
        a = std::min(a, 2 * na - rr);
        b = std::max(b, 2 * (nb - 1) + rr + 1);
      }
    }
    wlo[l] = std::max<int64_t>(0, a);
    whi[l] = std::min<int64_t>(Nl[l], b);
  }
}

constexpr double kReorthEta2 = 0.01;  // ||w'||^2 < eta^2 ||w||^2 triggers a second CGS pass

template <typename T> struct Solver : SolverBase {
  using C = cplx<T>;
  using D = double2;
  struct Level {
    Geo geo;
    double h = 0;
    int r = 1;      // stored stencil radius
    int rR = 0, rP = 0;
    DBuf coef;      // C [K][total] (levels > 0)
    DBuf bop;       // C [NB][total]: the assembled additive Vanka operator B (Eq. 3.8)
    DBuf u, f, r_, y;
    bool dist = false;          // slab-partitioned (else replicated on every rank)
    int64_t lo = 0, hi = 0;     // this rank's global rows on the slab axis
    bool gather_in = false;     // first replicated level: filled by allgather
    Geo view;                   // (gather_in) this rank's owned rows inside the replicated buffer
    // uniform-box compression (k_uniform.cuh): nodes in ub take their coefficients
    // from the centre node's copies below instead of the stored planes
    UBox ub = ubox_empty();
    std::vector<C> ucoef, ubop;
    // coefficient dictionaries (k_dict.cuh): class index per node (uint16, padded box) and
    // the class table [class][k]; cn / bn = number of classes (0: the planes are read)
    DBuf ccls, ctab, bcls, btab;
    int cn = 0, bn = 0;
    std::vector<size_t> goff, glen;   // (gather_in) per-rank byte ranges for the allgather (per element size 1)
  };
  std::vector<Level> lev;
  int G = 2;
  // slab partition [level * nranks + rank] and the setup windows (partitioned build)
  std::vector<int64_t> plo, phi, wlo, whi;
  std::vector<int> pdist;
  bool part_setup = false;
  double omega = 0, alpha = 0;
  DBuf sig, w2k2, gq;     // fine-level coefficients
  DBuf sigd;              // fine-level sigma in fp64 (restart residual of FGMRES)
  DBuf ainv;              // coarsest inverse, double2 N_L x N_L
  bool rb_closed = false; // fine level uses the closed-form RB patch solve
  bool stage3d = true;    // 3D fine operator: z-marching staged kernel (HMG_NO_STAGE3D=1 at build: the gather)
  bool fmarch = true;     // 2D c64 fine operator: warp-marching kernel (HMG_NO_FMARCH=1 at build: node-parallel)
  bool rbfast = true;     // RB sweep: constant-coefficient interior warps (HMG_NO_RB_FAST=1 at build: generic)
  bool flat3d = true;     // register-blocked 3D stencils with flat (x, y) thread indexing (HMG_NO_FLAT3D=1 at build: off)
  int vanka_bz = 2;       // assembled-Vanka stencil: nodes per thread along the slow axis (HMG_VANKA_BZ at build)
  int smarch = 0;         // 2D c64 stored stencil: warp-marching kernel on large levels, segment height
                          // (HMG_SMARCH=8|16 at build; off by default: measured slower than the blocked gather)
  bool rrfuse = true;     // 2D c64 fine residual + restriction fused (HMG_NO_RRFUSE=1 at build)
  bool zblock3 = true;    // 3D transfers with 4 coarse planes per thread (HMG_NO_ZBLOCK3=1 at build)
  // persistent coarse tail (k_tail.cuh): levels >= tail_l0 of a V(1,1) cycle in one launch
  int tail_l0 = -1;
  DBuf tail_lv, tail_uc, tail_bar;
  int tail_grid = 0;
  DBuf rb_ia, rb_id;      // its sigma-only factors 1/a_j and 1/(a_c - e^2 sum 1/a_l), stored in T
  C usig{}, uia{}, uid{};  // level-0 uniform-box values of sig, rb_ia, rb_id
  D usigd{};
  // FGMRES workspace
  int ws_m = 0;
  DBuf V, Z, partial, dres, io;
  // address ranges of the solver-owned basis (whole-cycle graphs are captured only for
  // these: per-call batch states are freed when the call returns)
  std::pair<const char *, const char *> ownV{nullptr, nullptr}, ownZ{nullptr, nullptr};
  DBuf qd, xd, rd;        // fp64 right-hand side, iterate and restart residual
  int reorth = 0;         // second Gram-Schmidt passes in the last solve
  // CUDA graph of the coarse part of the cycle (levels >= 1 run on fixed
  // buffers, so one capture serves every call); single-rank runs only
  std::map<int, cudaGraphExec_t> cgraphs;   // coarse-cycle graph per batch width
  std::map<int, long long> cgraph_kernels_nr;
  // whole zero-guess V-cycles (level 0 included) per (f, u) buffer pair: FGMRES feeds the
  // same m pairs (V_j, Z_j) every restart, so each pair's graph is captured once
  std::map<std::pair<const void *, void *>, std::pair<cudaGraphExec_t, long long>> fgraphs;
  // multi-RHS batches: levels >= 1 hold nrb right-hand sides at a stride of one
  // padded box (capacity nrb_cap); the fine level runs per right-hand side
  int nrb = 1, nrb_cap = 1;
  cudaStream_t gstream = nullptr;
  // side stream for the border instance of a split kernel pair (fork / join by events,
  // also inside graph capture): both halves write disjoint nodes and read the same inputs
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  bool split_conc = true;   // HMG_NO_SPLIT_CONC=1 at build: the two halves back to back
  // 2D Galerkin levels: the stored stencil from a shared-memory tile of x (HMG_NO_TILE2D=1 at
  // build: the gather).  Measured at N = 4096: level-1 residual 134 -> 122 ms per solve; the
  // same tiling of the Vanka operator was slower (92 -> 116 ms) and was dropped.
  bool tile2d = true;
  // c64: the V-cycle's fine-level residuals in fp32 arithmetic (config 3 keeps its
  // 70 iterations, 2.52 -> 2.40 ms per iteration; config 1 N = 4096 its 872, 1.440 -> 1.412 s;
  // HMG_F64RES=1 at build: fp64 as before).  The FGMRES matvec and restart residual stay fp64.
  bool f32res = true;
  cudaEvent_t gev_in = nullptr, gev_out = nullptr;
  int nblk = 0;
  double *hpin = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  cudaEvent_t ev_dots = nullptr;   // the Arnoldi dots have reached the host (pipelined FGMRES)

  ~Solver() override {
    for (auto &kv : cgraphs) cudaGraphExecDestroy(kv.second);
    for (auto &kv : fgraphs) cudaGraphExecDestroy(kv.second.first);
    if (gev_in) cudaEventDestroy(gev_in);
    if (gev_out) cudaEventDestroy(gev_out);
    if (gstream) cudaStreamDestroy(gstream);
    if (side) cudaStreamDestroy(side);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    if (hpin) cudaFreeHost(hpin);
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
    if (ev_dots) cudaEventDestroy(ev_dots);
  }

  const Geo &g0() const { return lev[0].geo; }
  double damp(int l) const { return damping[std::min<size_t>(l, damping.size() - 1)]; }

  // ------------------------------------------------------------------ build
  void build(const double *kappa, double omega_, const double *gamma, double alpha_, cudaStream_t s) override {
    omega = omega_;
    alpha = alpha_;
    const int dim = opt.dim;
    L = opt.levels;
    G = opt.intergrid == HMG_CUBIC ? 3 : 2;
    stage3d = std::getenv("HMG_NO_STAGE3D") == nullptr;
    fmarch = std::getenv("HMG_NO_FMARCH") == nullptr;
    rbfast = std::getenv("HMG_NO_RB_FAST") == nullptr;
    smarch = std::getenv("HMG_SMARCH") ? std::atoi(std::getenv("HMG_SMARCH")) : 0;
    rrfuse = std::getenv("HMG_NO_RRFUSE") == nullptr;
    zblock3 = std::getenv("HMG_NO_ZBLOCK3") == nullptr;
    // measured: BZ = 2 helps the 3D element operator (config 3 level 0: 53 -> 50 ms per solve)
    // and hurts the 2D RB one (level 1 at N = 4096: 103 -> 117 ms)
    split_conc = std::getenv("HMG_NO_SPLIT_CONC") == nullptr;
    tile2d = std::getenv("HMG_NO_TILE2D") == nullptr;
    flat3d = std::getenv("HMG_NO_FLAT3D") == nullptr;
    f32res = std::getenv("HMG_F64RES") == nullptr;
    vanka_bz = std::getenv("HMG_VANKA_BZ") ? std::atoi(std::getenv("HMG_VANKA_BZ")) : (opt.dim == 3 ? 2 : 1);
    if (comm && comm->size > 1) G = opt.intergrid == HMG_CUBIC ? 5 : 4;   // halo depth of the fused sweeps (u: 2 + r)
    lev.resize(L);
    int64_t nodes[3] = {opt.cells[0] + 1, opt.cells[1] + 1, dim == 3 ? opt.cells[2] + 1 : 1};
    double h = opt.h;
    for (int l = 0; l < L; ++l) {
      lev[l].geo = make_geo(dim, nodes, G);
      lev[l].h = h;
      lev[l].lo = 0;
      lev[l].hi = nodes[dim == 3 ? 2 : 1];
      for (int a = 0; a < dim; ++a) nodes[a] = (nodes[a] - 1) / 2 + 1;
      h *= 2;
    }
    for (int l = 0; l + 1 < L; ++l) level_scheme(opt.intergrid, l, lev[l].rR, lev[l].rP);
    rb_closed = (dim == 2 && opt.smoother == HMG_VANKA_RB);
    // slab partition and setup windows: with a communicator every rank computes the
    // partitioned levels only on its window of rows (HMG_REPLICATED_SETUP=1: the whole
    // grid, then sliced -- the round-1 build, kept for comparison)
    const int ax = slab_axis();
    const int64_t N0 = lev[0].geo.nodes();   // global fine nodes
    {
      std::vector<int64_t> Nl(L);
      std::vector<int> rR(L, 1);
      for (int l = 0; l < L; ++l) Nl[l] = lev[l].geo.N[ax];
      for (int l = 0; l + 1 < L; ++l) rR[l] = lev[l].rR;
      wlo.assign(L, 0);
      whi = Nl;
      if (comm && comm->size > 1) {
        slab_partition(Nl, comm->size, G, plo, phi, pdist);
        part_setup = std::getenv("HMG_REPLICATED_SETUP") == nullptr;
        if (part_setup)
          plan_windows(Nl, plo, phi, pdist, comm->size, comm->rank, G, rR, opt.coarse_op == HMG_REDISCRETIZE,
                       rb_closed, wlo, whi);
      }
      for (int l = 0; l < L; ++l) lev[l].geo = rows_geo(lev[l].geo, wlo[l], whi[l]);
    }
    const Geo &f0 = lev[0].geo;
    const int64_t Nw = f0.nodes();           // nodes of the level-0 window
    // a1: coefficients (the window's rows of the host arrays)
    {
      const int64_t row_nodes = dim == 3 ? (int64_t)f0.n[0] * f0.n[1] : f0.n[0];
      DBuf dk, dg;
      dk.alloc(Nw * sizeof(double), s);
      dg.alloc(Nw * sizeof(double), s);
      CK(cudaMemcpyAsync(dk.p, kappa + wlo[0] * row_nodes, Nw * sizeof(double), cudaMemcpyHostToDevice, s));
      CK(cudaMemcpyAsync(dg.p, gamma + wlo[0] * row_nodes, Nw * sizeof(double), cudaMemcpyHostToDevice, s));
      w2k2.alloc(f0.total * sizeof(double), s);
      gq.alloc(f0.total * sizeof(double), s);
      sig.alloc(f0.total * sizeof(C), s);
      sigd.alloc(f0.total * sizeof(double2), s);
      auto nl = node_launch(f0);
      launch(k_sigma<T>, nl.grid, nl.block, 0, s, f0, dk.template as<double>(), dg.template as<double>(), omega, w2k2.template as<double>(),
             gq.template as<double>(), sig.template as<C>(), sigd.template as<double2>());
      CK(cudaStreamSynchronize(s));
    }
    if (L == 1) {   // operator-only hierarchy: the matrix-free fine operator, no cycle
      if (comm && comm->size > 1) distribute(s);
      lev[0].u.alloc(f0.total * sizeof(C), s);
      lev[0].f.alloc(f0.total * sizeof(C), s);
      lev[0].r_.alloc(f0.total * sizeof(C), s);
      io.alloc((size_t)N0 * sizeof(C), s);
      CK(cudaEventCreate(&ev0));
      CK(cudaEventCreate(&ev1));
    CK(cudaEventCreateWithFlags(&ev_dots, cudaEventDisableTiming));
      CK(cudaMallocHost((void **)&hpin, 4096 * sizeof(double)));
      CK(cudaStreamSynchronize(s));
      return;
    }
    // level operators in fp64
    std::vector<DBuf> cd(L);
    lev[0].r = 1;
    materialize(lev[0].geo, lev[0].h, w2k2.template as<double>(), gq.template as<double>(), cd[0], s);
    DBuf cw, cg;  // REDISCRETIZE coarse fields
    const double *pw = w2k2.template as<double>(), *pg = gq.template as<double>();
    for (int l = 0; l + 1 < L; ++l) {
      Level &F = lev[l], &Cc = lev[l + 1];
      // the first replicated level of a partitioned build: this rank computes its share
      // of the rows (cview), then every plane is allgathered
      const bool share = part_setup && pdist[l] && !pdist[l + 1];
      const Geo cview = share ? rows_view(Cc.geo, plo[(size_t)(l + 1) * comm->size + comm->rank],
                                          phi[(size_t)(l + 1) * comm->size + comm->rank])
                              : Cc.geo;
      if (opt.coarse_op == HMG_GALERKIN) {
        const int rc = (F.rR + F.r + F.rP) / 2;
        if (rc > G) throw HmgError(HMG_EINVAL, "coarse stencil radius exceeds ghost width");
        if (dim == 3 && rc > 2) throw HmgError(HMG_EINVAL, "CUBIC intergrid is supported in 2D only");
        Cc.r = rc;
        const int K = kcount(dim, rc);
        cd[l + 1].alloc((size_t)K * Cc.geo.total * sizeof(double2), s);
        TransferW tw = transfer_weights(F.rR, F.rP);
        auto nl = node_launch(cview);
        const Geo &cg2 = cview;
        if (dim == 2) {
          if (rc == 1) launch(k_galerkin<2, 1>, nl.grid, nl.block, 0, s, F.geo, cg2, cd[l].template as<double2>(), F.r, tw, cd[l + 1].template as<double2>());
          else if (rc == 2) launch(k_galerkin<2, 2>, nl.grid, nl.block, 0, s, F.geo, cg2, cd[l].template as<double2>(), F.r, tw, cd[l + 1].template as<double2>());
          else launch(k_galerkin<2, 3>, nl.grid, nl.block, 0, s, F.geo, cg2, cd[l].template as<double2>(), F.r, tw, cd[l + 1].template as<double2>());
        } else {
          if (rc == 1) launch(k_galerkin<3, 1>, nl.grid, nl.block, 0, s, F.geo, cg2, cd[l].template as<double2>(), F.r, tw, cd[l + 1].template as<double2>());
          else launch(k_galerkin<3, 2>, nl.grid, nl.block, 0, s, F.geo, cg2, cd[l].template as<double2>(), F.r, tw, cd[l + 1].template as<double2>());
        }
        if (share) gather_rows(l + 1, cd[l + 1], K, sizeof(double2), s);
      } else {
        DBuf nw, ng;
        nw.alloc(Cc.geo.total * sizeof(double), s);
        ng.alloc(Cc.geo.total * sizeof(double), s);
        auto nl = node_launch(cview);
        launch(k_fw_average, nl.grid, nl.block, 0, s, F.geo, cview, pw, nw.template as<double>());
        launch(k_fw_average, nl.grid, nl.block, 0, s, F.geo, cview, pg, ng.template as<double>());
        if (share) {
          gather_rows(l + 1, nw, 1, sizeof(double), s);
          gather_rows(l + 1, ng, 1, sizeof(double), s);
        }
        CK(cudaStreamSynchronize(s));
        cw = std::move(nw);
        cg = std::move(ng);
        pw = cw.template as<double>();
        pg = cg.template as<double>();
        Cc.r = 1;
        materialize(Cc.geo, Cc.h, pw, pg, cd[l + 1], s);
      }
      CK(cudaStreamSynchronize(s));
    }
    // stored stencils in the working precision (levels > 0)
    for (int l = 1; l < L; ++l) {
      Level &Lv = lev[l];
      const int64_t n = (int64_t)kcount(dim, Lv.r) * Lv.geo.total;
      Lv.coef.alloc(n * sizeof(C), s);
      launch(k_cast<T>, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, s, cd[l].template as<double2>(), Lv.coef.template as<C>(), n);
    }
    // Vanka patch factors (on a partitioned level only for the rows the rank keeps)
    DBuf errb;
    errb.alloc(sizeof(unsigned long long), s);
    for (int l = 0; l + 1 < L; ++l) {
      Level &Lv = lev[l];
      const int k = patch_size(dim, opt.smoother);
      if (l == 0 && rb_closed) {   // fused closed-form sweep: two factor planes, no inverses, no y planes
        rb_ia.alloc(Lv.geo.total * sizeof(C), s);
        rb_id.alloc(Lv.geo.total * sizeof(C), s);
        auto nl = node_launch(Lv.geo);
        const bool c4 = opt.fine_stencil == HMG_COMPACT4;
        const double Lc = c4 ? FineW<2, ST_COMPACT4>::Lc : FineW<2, ST_FD2>::Lc;
        const double Mc = c4 ? FineW<2, ST_COMPACT4>::Mc : FineW<2, ST_FD2>::Mc;
        const double Le = c4 ? FineW<2, ST_COMPACT4>::Le : FineW<2, ST_FD2>::Le;
        const double ih2 = 1.0 / (Lv.h * Lv.h);
        const Geo kv = keep_view(l);
        nl = node_launch(kv);
        launch(k_rb_factors<T>, nl.grid, nl.block, 0, s, kv, (const double2 *)sigd.template as<double2>(), alpha,
               ih2, Lc, Mc, Le * ih2, rb_ia.template as<C>(), rb_id.template as<C>());
        continue;
      }
      DBuf hv;   // fp64 patch inverses (setup scratch)
      hv.alloc((size_t)k * k * Lv.geo.total * sizeof(double2), s);
      CK(cudaMemsetAsync(errb.p, 0xff, sizeof(unsigned long long), s));
      patch_inverse(keep_view(l, 1), cd[l], Lv.r, hv.template as<double2>(), errb.template as<unsigned long long>(), s);
      unsigned long long bad = 0;
      CK(cudaMemcpyAsync(&bad, errb.p, sizeof(bad), cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      if (bad != ~0ull) {
        const int64_t nx = Lv.geo.N[0], ny = Lv.geo.N[1];   // the kernel reports GLOBAL indices
        char buf[160];
        snprintf(buf, sizeof buf, "singular Vanka patch at level %d, anchor node (%lld, %lld, %lld)", l,
                 (long long)(bad % nx), (long long)((bad / nx) % ny), (long long)(bad / (nx * ny)));
        throw HmgError(HMG_ESINGULAR_PATCH, buf);
      }
      // assemble B = sum_i V_i^T W_i H_i^{-1} V_i as an NB-point stencil (fp64 sums, stored in T)
      const int nb = bstencil_planes();
      Lv.bop.alloc((size_t)nb * Lv.geo.total * sizeof(C), s);
      assemble_vanka(keep_view(l), Lv.bop.template as<C>(), hv.template as<double2>(), s);
      CK(cudaStreamSynchronize(s));
    }
    // coarsest dense inverse (fp64)
    {
      Level &Lc = lev[L - 1];
      const int N = (int)Lc.geo.nodes();
      if ((int64_t)N * N * 16 > (int64_t)8 << 30) throw HmgError(HMG_EINVAL, "coarsest level too large for a dense inverse");
      DBuf A, fcol, err;
      A.alloc((size_t)N * N * sizeof(double2), s);
      ainv.alloc((size_t)N * N * sizeof(double2), s);
      fcol.alloc((size_t)N * sizeof(double2), s);
      err.alloc(sizeof(int), s);
      auto nl = node_launch(Lc.geo);
      launch(k_dense_assemble, nl.grid, nl.block, 0, s, Lc.geo, cd[L - 1].template as<double2>(), Lc.r, A.template as<double2>());
      launch(k_identity, dim3((unsigned)(((int64_t)N * N + 255) / 256)), dim3(256), 0, s, N, ainv.template as<double2>());
      for (int k = 0; k < N; ++k) {
        launch(k_gj_pivot, dim3(1), dim3(1024), 0, s, N, k, A.template as<double2>(), ainv.template as<double2>(), fcol.template as<double2>(), err.template as<int>());
        launch(k_gj_eliminate, dim3((N + 255) / 256, N), dim3(256), 0, s, N, k, A.template as<double2>(), ainv.template as<double2>(),
               fcol.template as<double2>());
      }
      int bad = 0;
      CK(cudaMemcpyAsync(&bad, err.p, sizeof(int), cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      if (bad) throw HmgError(HMG_ESINGULAR_COARSE, "coarsest Galerkin matrix is singular");
    }
    if (comm && comm->size > 1) distribute(s);
    // cycle workspace
    for (int l = 0; l < L; ++l) {
      Level &Lv = lev[l];

      Lv.u.alloc(Lv.geo.total * vsize(l), s);
      Lv.f.alloc(Lv.geo.total * vsize(l), s);
      Lv.r_.alloc(Lv.geo.total * vsize(l), s);
    }
    io.alloc((size_t)N0 * sizeof(C), s);
    CK(cudaEventCreate(&ev0));
    CK(cudaEventCreate(&ev1));
    CK(cudaEventCreateWithFlags(&ev_dots, cudaEventDisableTiming));
    CK(cudaMallocHost((void **)&hpin, 4096 * sizeof(double)));
    find_uniform(s);
    find_dicts(s);
    setup_tail(s);
    CK(cudaStreamSynchronize(s));
  }

  // ------------------------------------------------------ persistent coarse tail
  // The levels below HMG_TAIL_NODES nodes of a one-rank V(1,1) cycle run as ONE persistent
  // kernel (k_coarse_tail; HMG_TAIL_NODES=0 disables; default below).  Device table of
  // TailLevel + the uniform-box copies in fp64 + a grid-barrier word pair, own per solver
  // (per-stream clones build their own: concurrent launches must not share the barrier).
  // blocks per SM the tail is compiled for (HMG_TAIL_MINB=2 at build: a 128-register cap; measured
  // 22.9 vs 22.1 ms per config-3 solve for the uncapped 1)
  int tail_minb = 1;
  // cluster tail: cluster size (0: the cooperative grid-barrier tail).  One thread-block cluster
  // of 16 (8) blocks x TAIL_CL_NT threads runs the levels below HMG_TAIL_CLUSTER_NODES nodes with
  // the hardware cluster barrier between passes.  Opt-in: bit-identical, but measured slower than
  // the per-kernel graph (N = 4096 c64: levels >= 4 on a 16-block cluster 1.681 vs 1.604 ms per
  // iteration, levels >= 5 1.616; 8 blocks 1.779): 16 SMs are too few for the passes themselves
  int tail_cluster = 0;
  int tail_kind() const {
    switch (opt.smoother) {
      case HMG_VANKA_RB: return PK_RB;
      case HMG_VANKA_ELEMENT: return PK_ELEMENT;
      case HMG_JACOBI: return PK_JACOBI;
      default: return PK_PLUS;
    }
  }
  template <int DIM, int KIND> void *tail_kernel() const {
    return tail_minb == 1 ? (void *)k_coarse_tail<T, DIM, KIND, 1> : (void *)k_coarse_tail<T, DIM, KIND, 2>;
  }
  void *tail_fn() const {
    const int d = opt.dim;
    if (tail_cluster) return tail_cluster_fn(sizeof(T) == 8, d, tail_kind());
    switch (opt.smoother) {
      case HMG_VANKA_RB: return tail_kernel<2, PK_RB>();
      case HMG_VANKA_ELEMENT: return d == 2 ? tail_kernel<2, PK_ELEMENT>() : tail_kernel<3, PK_ELEMENT>();
      case HMG_JACOBI: return d == 2 ? tail_kernel<2, PK_JACOBI>() : tail_kernel<3, PK_JACOBI>();
      case HMG_VANKA_PLUS: return d == 2 ? tail_kernel<2, PK_PLUS>() : tail_kernel<3, PK_PLUS>();
    }
    return nullptr;
  }
  void setup_tail(cudaStream_t s) {
    tail_l0 = -1;
    tail_minb = std::getenv("HMG_TAIL_MINB") ? std::atoi(std::getenv("HMG_TAIL_MINB")) : 1;
    // default: 3D only (config 3: 3.50 -> 3.40 ms per iteration); in 2D the per-kernel graph is
    // faster (N = 4096: levels >= 4 in one tail launch 177 us per cycle, the solve 1.505 -> 1.543 s)
    const int64_t thr = std::getenv("HMG_TAIL_NODES") ? std::atoll(std::getenv("HMG_TAIL_NODES"))
                                                      : (opt.dim == 3 ? 300000 : 0);
    const int64_t cthr = std::getenv("HMG_TAIL_CLUSTER_NODES") ? std::atoll(std::getenv("HMG_TAIL_CLUSTER_NODES"))
                                                               : 0;
    tail_cluster = 0;
    if (L < 3 || (comm && comm->size > 1) || opt.cycle != 0 || opt.nu1 != 1 || opt.nu2 != 1) return;
    int l0 = -1;
    for (int l = 1; l + 1 < L && thr > 0; ++l)
      if (lev[l].geo.nodes() <= thr) { l0 = l; break; }
    if (l0 < 0 && cthr > 0) {   // no grid-barrier tail: the cluster tail on the smaller levels
      for (int l = 1; l + 1 < L; ++l)
        if (lev[l].geo.nodes() <= cthr) { l0 = l; break; }
      if (l0 >= 0) {
        void *fn = tail_cluster_fn(sizeof(T) == 8, opt.dim, tail_kind());
        const int want = std::getenv("HMG_TAIL_CLUSTER") ? std::atoi(std::getenv("HMG_TAIL_CLUSTER")) : 16;
        for (int cs = want; fn && cs >= 2 && !tail_cluster; cs /= 2) {
          if (cs > 8 && cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
            (void)cudaGetLastError();
            continue;
          }
          cudaLaunchConfig_t cfg = {};
          cfg.gridDim = dim3(cs);
          cfg.blockDim = dim3(TAIL_CL_NT);
          cudaLaunchAttribute at[1];
          at[0].id = cudaLaunchAttributeClusterDimension;
          at[0].val.clusterDim.x = cs;
          at[0].val.clusterDim.y = 1;
          at[0].val.clusterDim.z = 1;
          cfg.attrs = at;
          cfg.numAttrs = 1;
          int nc = 0;
          if (cudaOccupancyMaxActiveClusters(&nc, fn, &cfg) == cudaSuccess && nc >= 1) tail_cluster = cs;
          else (void)cudaGetLastError();
        }
        if (!tail_cluster) l0 = -1;
      }
    }
    if (l0 < 0) return;
    std::vector<TailLevel> tl(L);
    std::vector<double2> uc;   // all uniform copies, offsets recorded per level
    std::vector<size_t> oc(L, 0), ob(L, 0);
    for (int l = l0; l < L; ++l) {
      oc[l] = uc.size();
      for (const C &c : lev[l].ucoef) uc.push_back(make_double2((double)c.x, (double)c.y));
      ob[l] = uc.size();
      for (const C &c : lev[l].ubop) uc.push_back(make_double2((double)c.x, (double)c.y));
    }
    tail_uc.alloc(std::max<size_t>(1, uc.size()) * sizeof(double2), s);
    if (!uc.empty()) CK(cudaMemcpyAsync(tail_uc.p, uc.data(), uc.size() * sizeof(double2), cudaMemcpyHostToDevice, s));
    for (int l = l0; l < L; ++l) {
      TailLevel &t = tl[l];
      const Level &Lv = lev[l];
      t.geo = Lv.geo;
      t.r = Lv.r;
      t.rR = Lv.rR;
      t.rP = Lv.rP;
      t.w = damp(l);
      t.coef = Lv.coef.p;
      t.bop = Lv.bop.p;
      t.ccls = coef_cls(Lv);
      t.bcls = bop_cls(Lv);
      t.ctab = coef_tab(Lv);
      t.btab = bop_tab(Lv);
      t.ub = Lv.ub;
      t.ucoef = tail_uc.template as<double2>() + oc[l];
      t.ubop = tail_uc.template as<double2>() + ob[l];
      t.u = Lv.u.template as<double2>();
      t.f = Lv.f.template as<double2>();
      t.r_ = Lv.r_.template as<double2>();
    }
    tail_lv.alloc(L * sizeof(TailLevel), s);
    CK(cudaMemcpyAsync(tail_lv.p, tl.data(), L * sizeof(TailLevel), cudaMemcpyHostToDevice, s));
    tail_bar.alloc(2 * sizeof(unsigned), s);
    if (tail_cluster) {
      tail_grid = tail_cluster;
    } else {
      int per_sm = 0, dev = 0, sms = 0;
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tail_fn(), 256, 0));
      CK(cudaGetDevice(&dev));
      CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
      tail_grid = std::max(1, std::min(per_sm, tail_minb)) * sms;   // co-resident (cooperative launch, launch_tail)
    }
    CK(cudaStreamSynchronize(s));
    tail_l0 = l0;
  }
  void launch_tail(cudaStream_t s) {
    const TailLevel *tl = tail_lv.template as<TailLevel>();
    const D *ai = ainv.template as<D>();
    unsigned *bar = tail_bar.template as<unsigned>();
    tag("coarse_tail", tail_l0, 0.0);
    // cooperative launch: the driver guarantees every block is resident at once (the software
    // grid barrier needs it, also when other streams run tails concurrently); capturable
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(tail_grid);
    cfg.blockDim = dim3(tail_cluster ? TAIL_CL_NT : 256);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    if (tail_cluster) {   // one cluster: the hardware co-schedules its blocks (no cooperative launch)
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = tail_cluster;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
    } else {
      at[0].id = cudaLaunchAttributeCooperative;
      at[0].val.cooperative = 1;
    }
    cfg.attrs = at;
    cfg.numAttrs = 1;
    const int pi = prof_before(s);
    void *args[] = {(void *)&tl, (void *)&tail_l0, (void *)&L, (void *)&ai, (void *)&bar};
    CK(cudaLaunchKernelExC(&cfg, tail_fn(), args));
    count_launch();
    prof_after(s, pi);
  }

  // ------------------------------------------------------ uniform-box compression
  // Per level: the largest box around the centre node in which every stored
  // coefficient equals the centre node's bit for bit (k_uniform.cuh).  Greedy
  // growth, one face at a time; every face added is checked whole, so the box
  // is exact (a valid box, maximal for box-shaped uniform regions such as the
  // interior of a sponge-bordered homogeneous medium).  HMG_NO_UNIFORM=1 (read
  // at build) keeps every box empty: the stored path everywhere.
  template <typename E> void flag_planes(const Geo &g, const DBuf &b, int nplanes, int64_t ref, DBuf &flags,
                                         cudaStream_t s) {
    if (!b.p || nplanes <= 0) return;
    auto nl = node_launch(g);
    launch(k_uniform_flags<E>, nl.grid, nl.block, 0, s, g, b.template as<E>(), nplanes, ref,
           flags.template as<unsigned char>());
  }
  static UBox grow_box(const std::vector<unsigned char> &f, const int n[3], int dim) {
    UBox b = ubox_empty();
    int c[3] = {n[0] / 2, n[1] / 2, dim == 3 ? n[2] / 2 : 0};
    auto at = [&](int x, int y, int z) { return f[((size_t)z * n[1] + y) * n[0] + x] != 0; };
    if (!at(c[0], c[1], c[2])) return b;
    for (int a = 0; a < 3; ++a) { b.lo[a] = c[a]; b.hi[a] = c[a] + 1; }
    auto face_ok = [&](int a, int v) {   // all nodes of the box's cross-section at coordinate v on axis a
      int lo[3] = {b.lo[0], b.lo[1], b.lo[2]}, hi[3] = {b.hi[0], b.hi[1], b.hi[2]};
      lo[a] = v;
      hi[a] = v + 1;
      for (int z = lo[2]; z < hi[2]; ++z)
        for (int y = lo[1]; y < hi[1]; ++y)
          for (int x = lo[0]; x < hi[0]; ++x)
            if (!at(x, y, z)) return false;
      return true;
    };
    for (bool grew = true; grew;) {
      grew = false;
      for (int a = 0; a < dim; ++a) {
        if (b.lo[a] > 0 && face_ok(a, b.lo[a] - 1)) { --b.lo[a]; grew = true; }
        if (b.hi[a] < n[a] && face_ok(a, b.hi[a])) { ++b.hi[a]; grew = true; }
      }
    }
    return b;
  }
  void find_uniform(cudaStream_t s) {
    static_assert(sizeof(C) % 8 == 0, "flag comparison in 8-byte words");
    const bool off = std::getenv("HMG_NO_UNIFORM") != nullptr;
    for (int l = 0; l < L; ++l) {
      Level &Lv = lev[l];
      Lv.ub = ubox_empty();
      Lv.ucoef.clear();
      Lv.ubop.clear();
      if (off || l == L - 1) continue;   // the coarsest level is a dense inverse
      const Geo &g = Lv.geo;
      const int64_t N = g.nodes();
      const int cx = g.n[0] / 2, cy = g.n[1] / 2, cz = opt.dim == 3 ? g.n[2] / 2 : 0;
      const int64_t ref = g.idx(cx, cy, cz);
      DBuf flags;
      flags.alloc((size_t)N, s);
      CK(cudaMemsetAsync(flags.p, 1, (size_t)N, s));
      const int nb = Lv.bop.p ? bstencil_planes() : 0;
      const int K = l > 0 ? kcount(opt.dim, Lv.r) : 0;
      if (l == 0) {
        flag_planes<C>(g, sig, 1, ref, flags, s);
        flag_planes<D>(g, sigd, 1, ref, flags, s);
        flag_planes<C>(g, rb_ia, 1, ref, flags, s);
        flag_planes<C>(g, rb_id, 1, ref, flags, s);
      } else {
        flag_planes<C>(g, Lv.coef, K, ref, flags, s);
      }
      flag_planes<C>(g, Lv.bop, nb, ref, flags, s);
      std::vector<unsigned char> hf((size_t)N);
      CK(cudaMemcpyAsync(hf.data(), flags.p, (size_t)N, cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      Lv.ub = grow_box(hf, g.n, opt.dim);
      if (Lv.ub.nodes() < 64) { Lv.ub = ubox_empty(); continue; }   // not worth a branch
      auto fetch = [&](const DBuf &b, int nplanes, size_t es, void *dst) {
        for (int k = 0; k < nplanes; ++k)
          CK(cudaMemcpyAsync((char *)dst + k * es, (const char *)b.p + ((size_t)k * g.total + ref) * es, es,
                             cudaMemcpyDeviceToHost, s));
      };
      if (l == 0) {
        fetch(sig, 1, sizeof(C), &usig);
        fetch(sigd, 1, sizeof(D), &usigd);
        if (rb_ia.p) fetch(rb_ia, 1, sizeof(C), &uia);
        if (rb_id.p) fetch(rb_id, 1, sizeof(C), &uid);
      } else {
        Lv.ucoef.resize(K);
        fetch(Lv.coef, K, sizeof(C), Lv.ucoef.data());
      }
      if (nb) {
        Lv.ubop.resize(nb);
        fetch(Lv.bop, nb, sizeof(C), Lv.ubop.data());
      }
      CK(cudaStreamSynchronize(s));
    }
  }
  // ------------------------------------------------------ coefficient dictionary
  // Distinct coefficient vectors of a level's planes (k_dict.cuh): returns the number of
  // classes, 0 when the level keeps its planes (more than 65535 classes, a table not
  // much smaller than the planes, a hash-probe overflow or a failed bitwise check).
  int build_dict(const Geo &g, const DBuf &planes, int nplanes, DBuf &cls, DBuf &tab, cudaStream_t s) {
    typedef unsigned long long ull;
    if (!planes.p || nplanes <= 0) return 0;
    const int64_t N = g.nodes();
    constexpr int W = (int)(sizeof(C) / 8);
    constexpr int kMaxCls = 65535;
    unsigned S = 1024;
    while ((int64_t)S < 4 * std::min<int64_t>(N, kMaxCls)) S <<= 1;
    DBuf keys, slot, flag;
    keys.alloc((size_t)S * sizeof(ull), s);
    slot.alloc((size_t)N * sizeof(int), s);
    flag.alloc(2 * sizeof(int), s);
    auto nl = node_launch(g);
    launch(k_dict_insert, nl.grid, nl.block, 0, s, g, planes.template as<ull>(), nplanes, W, keys.template as<ull>(),
           S - 1, slot.template as<int>(), flag.template as<int>(), kMaxCls);
    std::vector<ull> hk(S);
    int hf[2] = {0, 0};
    CK(cudaMemcpyAsync(hk.data(), keys.p, (size_t)S * sizeof(ull), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(hf, flag.p, 2 * sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (hf[0]) return 0;
    std::vector<int> remap(S, 0);
    int n = 0;
    for (unsigned i = 0; i < S; ++i)
      if (hk[i] != kDictEmpty) remap[i] = n++;
    if (n == 0 || n > kMaxCls || (double)n * nplanes * sizeof(C) > 0.25 * (double)nplanes * g.total * sizeof(C)) return 0;
    DBuf dremap, rep;
    dremap.alloc((size_t)S * sizeof(int), s);
    CK(cudaMemcpyAsync(dremap.p, remap.data(), (size_t)S * sizeof(int), cudaMemcpyHostToDevice, s));
    rep.alloc((size_t)n * sizeof(int), s);
    CK(cudaMemsetAsync(rep.p, 0x7f, (size_t)n * sizeof(int), s));
    cls.alloc((size_t)g.total * sizeof(unsigned short), s);
    launch(k_dict_assign, nl.grid, nl.block, 0, s, g, (const int *)slot.template as<int>(),
           (const int *)dremap.template as<int>(), cls.template as<unsigned short>(), rep.template as<int>());
    tab.alloc((size_t)n * nplanes * sizeof(C), s);
    const int64_t nt = (int64_t)n * nplanes;
    launch(k_dict_fill, dim3((unsigned)((nt + 255) / 256)), dim3(256), 0, s, g, planes.template as<ull>(), nplanes, W,
           (const int *)rep.template as<int>(), n, tab.template as<ull>());
    CK(cudaMemsetAsync(flag.p, 0, sizeof(int), s));
    launch(k_dict_verify, nl.grid, nl.block, 0, s, g, planes.template as<ull>(), nplanes, W,
           (const unsigned short *)cls.template as<unsigned short>(), (const ull *)tab.template as<ull>(),
           flag.template as<int>());
    CK(cudaMemcpyAsync(hf, flag.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (hf[0]) {
      cls.release();
      tab.release();
      return 0;
    }
    return n;
  }
  void find_dicts(cudaStream_t s) {
    const bool off = std::getenv("HMG_NO_DICT") != nullptr;   // read at build
    for (int l = 0; l < L; ++l) {
      Level &Lv = lev[l];
      Lv.ccls.release(); Lv.ctab.release(); Lv.bcls.release(); Lv.btab.release();
      Lv.cn = Lv.bn = 0;
      if (off || l == L - 1 || outside(l) == 0) continue;
      // tables in the storage precision T (converted in the kernels like the planes: an fp64
      // table measured slower, its 16-byte loads outweigh the conversions)
      if (l > 0) Lv.cn = build_dict(Lv.geo, Lv.coef, kcount(opt.dim, Lv.r), Lv.ccls, Lv.ctab, s);
      if (Lv.bop.p) Lv.bn = build_dict(Lv.geo, Lv.bop, bstencil_planes(), Lv.bcls, Lv.btab, s);
    }
  }
  // what a kernel reads for level l's stencil / Vanka operator: the class table and the
  // class index when the level has a dictionary, else the planes (and null)
  const unsigned short *coef_cls(const Level &Lv) const { return Lv.cn ? Lv.ccls.template as<unsigned short>() : nullptr; }
  const C *coef_tab(const Level &Lv) const { return Lv.cn ? Lv.ctab.template as<C>() : nullptr; }
  const unsigned short *bop_cls(const Level &Lv) const { return Lv.bn ? Lv.bcls.template as<unsigned short>() : nullptr; }
  const C *bop_tab(const Level &Lv) const { return Lv.bn ? Lv.btab.template as<C>() : nullptr; }
  // algorithmic coefficient bytes per launch outside the uniform box: K planes, or the 2-byte index
  double coef_bytes(int l, int K) const { return lev[l].cn ? 2.0 * outside(l) : (double)K * sizeof(C) * outside(l); }
  double bop_bytes(int l, int NB) const { return lev[l].bn ? 2.0 * outside(l) : (double)NB * sizeof(C) * outside(l); }

  // kernel-parameter copy of n coefficients (unused entries zero)
  // kernel-parameter copy in the kernel's ARITHMETIC precision E (exact widening of
  // the stored values: the same numbers the stored path converts per node)
  template <int K, typename E = T> static UCoef<K, E> ucopy(const std::vector<C> &v) {
    UCoef<K, E> u{};
    for (int k = 0; k < K && k < (int)v.size(); ++k) u.c[k] = mkc<E>((E)v[k].x, (E)v[k].y);
    return u;
  }
  static D widen(const C &c) { return make_double2((double)c.x, (double)c.y); }
  // coefficient-plane bytes a launch over level l really streams (nodes outside the box)
  double outside(int l) const { return (double)(lev[l].geo.nodes() - lev[l].ub.nodes()); }

  // ---------------------------------------------------------- distribution
  int slab_axis() const { return opt.dim == 3 ? 2 : 1; }
  int64_t rowsize(const Geo &g) const { return opt.dim == 3 ? g.pxy : g.px; }

  // the box of global slab-axis rows [a, b) of the full level box `full` (setup window)
  Geo rows_geo(const Geo &full, int64_t a, int64_t b) const {
    const int ax = slab_axis();
    Geo g = full;
    g.n[ax] = (int)(b - a);
    g.o[ax] = (int)a;
    g.total = rowsize(full) * (g.n[ax] + 2 * G);
    if (opt.dim == 2) g.pxy = g.total;
    g.slab_len = (int64_t)g.n[ax] * rowsize(full);
    return g;
  }
  // global rows [a, b) of the box g addressed in g's own memory layout (kernel launch view)
  Geo rows_view(const Geo &g, int64_t a, int64_t b) const {
    const int ax = slab_axis();
    Geo v = g;
    a = std::max<int64_t>(a, g.o[ax]);
    b = std::min<int64_t>(b, (int64_t)g.o[ax] + g.n[ax]);
    v.n[ax] = (int)std::max<int64_t>(0, b - a);
    v.base = g.base + (a - g.o[ax]) * rowsize(g);
    v.o[ax] = (int)a;
    return v;
  }
  // rows of level l the rank keeps (its slab +- G), widened by `extra` (patch anchors);
  // the whole box on replicated levels / one rank
  Geo keep_view(int l, int extra = 0) const {
    const Geo &g = lev[l].geo;
    if (!part_setup || !pdist[l]) return g;
    const int P = comm->size, me = comm->rank;
    return rows_view(g, plo[(size_t)l * P + me] - G - extra, phi[(size_t)l * P + me] + G + extra);
  }
  // allgather `planes` planes of a per-node array of the (replicated) level l: rank q
  // contributes its partition rows [plo_q, phi_q) of every plane
  void gather_rows(int l, DBuf &b, int planes, size_t esize, cudaStream_t s) {
    const Geo &g = lev[l].geo;
    const int P = comm->size;
    std::vector<size_t> off(P), len(P);
    for (int k = 0; k < planes; ++k) {
      for (int q = 0; q < P; ++q) {
        off[q] = ((size_t)k * g.total + (size_t)(G + plo[(size_t)l * P + q]) * rowsize(g)) * esize;
        len[q] = (size_t)(phi[(size_t)l * P + q] - plo[(size_t)l * P + q]) * rowsize(g) * esize;
      }
      comm->allgatherv(b.p, off, len, s);
    }
    CK(cudaStreamSynchronize(s));
  }

  // keep only this rank's slab (+ G ghost rows) of a per-node array of the
  // replicated setup: rows [lo - G, hi + G) are contiguous in the padded box
  void slice(DBuf &b, size_t esize, const Geo &gG, const Geo &gL, int64_t lo, cudaStream_t s) {
    if (!b.p) return;
    const size_t planes = b.bytes / (esize * gG.total);
    DBuf nb;
    nb.alloc(planes * gL.total * esize, s);
    for (size_t k = 0; k < planes; ++k)
      CK(cudaMemcpyAsync((char *)nb.p + k * gL.total * esize, (const char *)b.p + (k * gG.total + lo * rowsize(gG)) * esize,
                         gL.total * esize, cudaMemcpyDeviceToDevice, s));
    CK(cudaStreamSynchronize(s));
    b = std::move(nb);
  }

  void distribute(cudaStream_t s) {
    const int ax = slab_axis(), P = comm->size, me = comm->rank;
    std::vector<int64_t> Nl(L);
    const std::vector<int64_t> &lo = plo, &hi = phi;
    const std::vector<int> &dist = pdist;
    for (int l = 0; l < L; ++l) Nl[l] = lev[l].geo.N[ax];
    for (int l = 0; l < L; ++l) {
      Level &Lv = lev[l];
      Lv.lo = 0;
      Lv.hi = Nl[l];
      if (!dist[l]) {
        if (l > 0 && dist[l - 1]) {   // first replicated level: restricted rows are allgathered
          Lv.gather_in = true;
          Lv.view = Lv.geo;
          const int64_t a = lo[(size_t)l * P + me], b = hi[(size_t)l * P + me];
          Lv.view.n[ax] = (int)(b - a);
          Lv.view.o[ax] = (int)a;
          Lv.view.base += a * rowsize(Lv.geo);
          Lv.goff.resize(P);
          Lv.glen.resize(P);
          for (int q = 0; q < P; ++q) {
            Lv.goff[q] = (size_t)(G + lo[(size_t)l * P + q]) * rowsize(Lv.geo);
            Lv.glen[q] = (size_t)(hi[(size_t)l * P + q] - lo[(size_t)l * P + q]) * rowsize(Lv.geo);
          }
        }
        continue;
      }
      Lv.dist = true;
      Lv.lo = lo[(size_t)l * P + me];
      Lv.hi = hi[(size_t)l * P + me];
      const Geo gG = Lv.geo;   // the setup window (the whole level in a replicated build)
      const Geo gL = rows_geo(gG, Lv.lo, Lv.hi);
      const int64_t r0 = Lv.lo - gG.o[ax];   // padded row of global row lo - G in the window
      slice(Lv.coef, sizeof(C), gG, gL, r0, s);
      slice(Lv.bop, sizeof(C), gG, gL, r0, s);
      if (l == 0) {
        slice(sig, sizeof(C), gG, gL, r0, s);
        slice(sigd, sizeof(D), gG, gL, r0, s);
        slice(rb_ia, sizeof(C), gG, gL, r0, s);
        slice(rb_id, sizeof(C), gG, gL, r0, s);
        slice(w2k2, sizeof(double), gG, gL, r0, s);
        slice(gq, sizeof(double), gG, gL, r0, s);
      }
      Lv.geo = gL;
    }
  }

  // fill `depth` slab-axis ghost rows of `nplanes` planes of a level vector
  // from the neighbouring ranks (no-op on replicated levels / one GPU)
  void halo(int l, const void *vec, int depth, cudaStream_t s, int nplanes = 1, size_t esize = 0) {
    halos(l, {{vec, depth}}, s, nplanes, esize);
  }
  // the halos of several vectors of level l exchanged as ONE communication step
  void halos(int l, std::initializer_list<std::pair<const void *, int>> vd, cudaStream_t s, int nplanes = 1,
             size_t esize = 0) {
    const Level &Lv = lev[l];
    if (!Lv.dist) return;
    if (!esize) esize = vsize(l);
    const Geo &g = Lv.geo;
    const int n = g.n[slab_axis()];
    const size_t row = (size_t)rowsize(g) * esize;
    std::vector<Comm::HaloReq> rq;
    for (const auto &v : vd) {
      if (!v.first || v.second <= 0) continue;
      const int depth = v.second;
      for (int k = 0; k < nplanes; ++k) {
        char *b = (char *)v.first + (size_t)k * g.total * esize;
        rq.push_back({b + (size_t)G * row, b + (size_t)(G - depth) * row, b + (size_t)(G + n - depth) * row,
                      b + (size_t)(G + n) * row, (size_t)depth * row});
      }
    }
    if (!rq.empty()) comm->halo_multi(rq, s);
  }
  void allreduce(double2 *d, int n, cudaStream_t s) {
    if (comm && comm->size > 1) comm->allreduce_sum(reinterpret_cast<double *>(d), 2 * n, s);
  }

  // level 1 of a 2D Galerkin hierarchy: residual/apply through the fine grid
  // (opt-in, HMG_MF1=1: measured 0.33 ms vs 0.19 ms for the stored stencil at
  // N = 4096, shared-memory-wavefront bound).
  // Slabs: the coarse slab's R P support, fine rows [2 lo - rR - 1, 2 (hi - 1) + rR + 1],
  // must lie inside the fine slab's ghosted rows (sigma is sliced with G ghost rows).
  bool mf_level1(int l) const {
    if (l != 1 || L < 2 || nrb != 1 || opt.dim != 2 || opt.coarse_op != HMG_GALERKIN || !std::getenv("HMG_MF1")) return false;
    const Level &F = lev[0], &C1 = lev[1];
    if (!F.dist) return true;
    if (!C1.dist) return false;
    return 2 * C1.lo - F.rR - 1 >= F.lo - G && 2 * (C1.hi - 1) + F.rR + 1 < F.hi + G;
  }

  // 2D c64 fine level with an even ghost width: node pairs are 16-byte aligned
  // (used for the FGMRES matvec; measured: the scalar kernel is faster for the
  // V-cycle residual, whose sigma is fp32)
  bool pair_ok() const { return std::is_same<T, float>::value && opt.dim == 2 && (G % 2) == 0; }

  static int kcount(int dim, int r) { return dim == 3 ? (2 * r + 1) * (2 * r + 1) * (2 * r + 1) : (2 * r + 1) * (2 * r + 1); }

  void materialize(const Geo &g, double h, const double *pw, const double *pg, DBuf &out, cudaStream_t s) {
    const int K = kcount(opt.dim, 1);
    out.alloc((size_t)K * g.total * sizeof(double2), s);
    auto nl = node_launch(g);
    const double ih2 = 1.0 / (h * h);
    const bool c4 = opt.fine_stencil == HMG_COMPACT4;
    if (opt.dim == 2) {
      if (c4) launch(k_materialize<2, ST_COMPACT4>, nl.grid, nl.block, 0, s, g, pw, pg, alpha, ih2, out.template as<double2>());
      else launch(k_materialize<2, ST_FD2>, nl.grid, nl.block, 0, s, g, pw, pg, alpha, ih2, out.template as<double2>());
    } else {
      if (c4) launch(k_materialize<3, ST_COMPACT4>, nl.grid, nl.block, 0, s, g, pw, pg, alpha, ih2, out.template as<double2>());
      else launch(k_materialize<3, ST_FD2>, nl.grid, nl.block, 0, s, g, pw, pg, alpha, ih2, out.template as<double2>());
    }
  }

  int bstencil_planes() const {
    const int dim = opt.dim;
    switch (opt.smoother) {
      case HMG_VANKA_RB: return BStencil<2, PK_RB>::NB;
      case HMG_VANKA_ELEMENT: return dim == 2 ? BStencil<2, PK_ELEMENT>::NB : BStencil<3, PK_ELEMENT>::NB;
      case HMG_JACOBI: return dim == 2 ? BStencil<2, PK_JACOBI>::NB : BStencil<3, PK_JACOBI>::NB;
      case HMG_VANKA_PLUS: return dim == 2 ? BStencil<2, PK_PLUS>::NB : BStencil<3, PK_PLUS>::NB;
    }
    throw HmgError(HMG_EINVAL, "unknown smoother");
  }
  // g: the level's window box or a view of some of its rows (same memory layout)
  void assemble_vanka(const Geo &g, C *B, const double2 *hv, cudaStream_t s) {
    auto nl = node_launch(g);
    const int dim = opt.dim;
    switch (opt.smoother) {
      case HMG_VANKA_RB: launch(k_vanka_assemble<T, 2, PK_RB>, nl.grid, nl.block, 0, s, g, hv, B); break;
      case HMG_VANKA_ELEMENT:
        if (dim == 2) launch(k_vanka_assemble<T, 2, PK_ELEMENT>, nl.grid, nl.block, 0, s, g, hv, B);
        else launch(k_vanka_assemble<T, 3, PK_ELEMENT>, nl.grid, nl.block, 0, s, g, hv, B);
        break;
      case HMG_JACOBI:
        if (dim == 2) launch(k_vanka_assemble<T, 2, PK_JACOBI>, nl.grid, nl.block, 0, s, g, hv, B);
        else launch(k_vanka_assemble<T, 3, PK_JACOBI>, nl.grid, nl.block, 0, s, g, hv, B);
        break;
      case HMG_VANKA_PLUS:
        if (dim == 2) launch(k_vanka_assemble<T, 2, PK_PLUS>, nl.grid, nl.block, 0, s, g, hv, B);
        else launch(k_vanka_assemble<T, 3, PK_PLUS>, nl.grid, nl.block, 0, s, g, hv, B);
        break;
    }
  }

  // fp64 patch inverses H_i^{-1} into hv [K*K][total] (setup scratch)
  void patch_inverse(const Geo &g, DBuf &cd, int r, double2 *hv, unsigned long long *err, cudaStream_t s) {
    auto nl = node_launch(g);
    const double2 *c = cd.template as<double2>();
    const int dim = opt.dim;
    struct { const Geo &geo; int r; } Lv{g, r};
    switch (opt.smoother) {
      case HMG_VANKA_RB:
        if (dim != 2) throw HmgError(HMG_EINVAL, "RB patch is 2D only (the paper rejects the 13-node 3D RB patch, P:949-951)");
        launch(k_patch_inverse<double, 2, PK_RB>, nl.grid, nl.block, 0, s, Lv.geo, c, Lv.r, hv, err);
        break;
      case HMG_VANKA_ELEMENT:
        if (dim == 2) launch(k_patch_inverse<double, 2, PK_ELEMENT>, nl.grid, nl.block, 0, s, Lv.geo, c, Lv.r, hv, err);
        else launch(k_patch_inverse<double, 3, PK_ELEMENT>, nl.grid, nl.block, 0, s, Lv.geo, c, Lv.r, hv, err);
        break;
      case HMG_JACOBI:
        if (dim == 2) launch(k_patch_inverse<double, 2, PK_JACOBI>, nl.grid, nl.block, 0, s, Lv.geo, c, Lv.r, hv, err);
        else launch(k_patch_inverse<double, 3, PK_JACOBI>, nl.grid, nl.block, 0, s, Lv.geo, c, Lv.r, hv, err);
        break;
      case HMG_VANKA_PLUS:
        if (dim == 2) launch(k_patch_inverse<double, 2, PK_PLUS>, nl.grid, nl.block, 0, s, Lv.geo, c, Lv.r, hv, err);
        else launch(k_patch_inverse<double, 3, PK_PLUS>, nl.grid, nl.block, 0, s, Lv.geo, c, Lv.r, hv, err);
        break;
      default: throw HmgError(HMG_EINVAL, "unknown smoother");
    }
  }

  // 2D c64 fine operator y = A x / y = f - A x as the warp-marching kernel (k_operator.cuh);
  // false: not applicable (the caller falls back to the node-parallel kernels)
  bool fine2d_march(const void *sgv, bool sig_fp64, double a, double ih2, const C *x, const C *f, C *y,
                    cudaStream_t s) {
    if (!std::is_same<T, float>::value || opt.dim != 2 || (G % 2) != 0 || !fmarch) return false;
    const Geo &g = lev[0].geo;
    constexpr int SEG = 32, PD = 2, NST = PD + 2;
    const int nstrips = (g.n[0] + FM_STRIP - 1) / FM_STRIP, nsegs = (g.n[1] + SEG - 1) / SEG;
    const int64_t warps = (int64_t)nstrips * nsegs;
    const dim3 grid((unsigned)((warps + 3) / 4)), block(128);
    const bool c4 = opt.fine_stencil == HMG_COMPACT4;
    const float2 *xx = reinterpret_cast<const float2 *>(x), *ff = reinterpret_cast<const float2 *>(f);
    float2 *yy = reinterpret_cast<float2 *>(y);
    auto go = [&](auto kern, const auto *sg, int sw) {
      const int smem = 4 * NST * (2 + sw) * 32 * 16;
      CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      launch(kern, grid, block, (size_t)smem, s, g, sg, a, ih2, xx, ff, yy, lev[0].ub, sig_fp64 ? usigd : widen(usig));
    };
    if (sig_fp64) {
      const double2 *sg = reinterpret_cast<const double2 *>(sgv);
      if (c4) go(k_fine_op2d_march<ST_COMPACT4, double, SEG, PD>, sg, 2);
      else go(k_fine_op2d_march<ST_FD2, double, SEG, PD>, sg, 2);
    } else if (f32res) {   // the V-cycle's fine residual: fp32 arithmetic
      const float2 *sg = reinterpret_cast<const float2 *>(sgv);
      if (c4) go(k_fine_op2d_march<ST_COMPACT4, float, SEG, PD, float>, sg, 1);
      else go(k_fine_op2d_march<ST_FD2, float, SEG, PD, float>, sg, 1);
    } else {
      const float2 *sg = reinterpret_cast<const float2 *>(sgv);
      if (c4) go(k_fine_op2d_march<ST_COMPACT4, float, SEG, PD>, sg, 1);
      else go(k_fine_op2d_march<ST_FD2, float, SEG, PD>, sg, 1);
    }
    return true;
  }

  // f_c = R_0 (f - H_s u) in ONE warp-marching kernel (2D c64 fine level with the bicubic
  // fine restriction, one rank); false: not applicable (separate residual + restriction)
  bool resrestrict(int l, const void *u, const void *f, void *fc, cudaStream_t s) {
    if (l != 0 || !rrfuse || !std::is_same<T, float>::value || opt.dim != 2 || (G % 2) != 0 || lev[0].rR != 2 ||
        nbat(0) != 1 || (comm && comm->size > 1) || lev[1].gather_in)
      return false;
    const Geo &g = lev[0].geo, &gc = lev[1].geo;
    constexpr int SEG = 32, PD = 2, NST = PD + 2;
    const int nstrips = (g.n[0] + RR_STRIP - 1) / RR_STRIP, nsegs = (g.n[1] + SEG - 1) / SEG;
    const int64_t warps = (int64_t)nstrips * nsegs;
    const dim3 grid((unsigned)((warps + 3) / 4)), block(128);
    const int smem = 4 * NST * 3 * 32 * 16;
    const double ih2 = 1.0 / (lev[0].h * lev[0].h);
    const double nn = (double)g.nodes();
    tag("residual_restrict", 0, 2.0 * sizeof(C) * nn + sizeof(C) * outside(0) + 16.0 * gc.nodes());
    auto go = [&](auto kern) {
      CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      launch(kern, grid, block, (size_t)smem, s, g, gc, (const float2 *)sig.template as<C>(), alpha, ih2,
             (const float2 *)u, (const float2 *)f, (double2 *)fc, lev[0].ub, widen(usig));
    };
    if (f32res) {   // fp32 residual arithmetic, restriction in fp64
      if (opt.fine_stencil == HMG_COMPACT4) go(k_fine_resrestrict2d_march<ST_COMPACT4, SEG, PD, float>);
      else go(k_fine_resrestrict2d_march<ST_FD2, SEG, PD, float>);
      return true;
    }
    if (opt.fine_stencil == HMG_COMPACT4) go(k_fine_resrestrict2d_march<ST_COMPACT4, SEG, PD>);
    else go(k_fine_resrestrict2d_march<ST_FD2, SEG, PD>);
    return true;
  }

  // 3D fine operator y = A x / y = f - A x: the z-marching staged kernel (k_stage3d.cuh)
  // or the node-parallel gather (bit-identical; HMG_NO_STAGE3D=1)
  template <typename TT, typename TC, typename TS>
  void fine3d(const Geo &g, const cplx<TS> *sg, TC a, TC ih2, const cplx<TT> *x, const cplx<TT> *f, cplx<TT> *y,
              cplx<TC> us, cudaStream_t s) {
    const bool c4 = opt.fine_stencil == HMG_COMPACT4;
    const UBox &ub = lev[0].ub;
    if (!stage3d) {
      auto nl = node_launch(g);
      if (c4) launch(k_fine_op<TT, 3, ST_COMPACT4, TC, TS>, nl.grid, nl.block, 0, s, g, sg, a, ih2, x, f, y, ub, us);
      else launch(k_fine_op<TT, 3, ST_FD2, TC, TS>, nl.grid, nl.block, 0, s, g, sg, a, ih2, x, f, y, ub, us);
      return;
    }
    constexpr int ZC = 32, NS = 4;
    auto rup = [](int b) { return (b + 127) / 128 * 128; };
    const int slot = rup(S3_RY * S3_RX * (int)sizeof(cplx<TT>)) + rup(S3_TY * S3_TX * (int)sizeof(cplx<TS>)) +
                     rup(S3_TY * S3_TX * (int)sizeof(cplx<TT>));
    const int smem = 128 + NS * slot;
    const dim3 block(32, S3_TY + 1), grid((g.n[0] + S3_TX - 1) / S3_TX, (g.n[1] + S3_TY - 1) / S3_TY, (g.n[2] + ZC - 1) / ZC);
    const CUtensorMap mx = make_tmap(x, sizeof(cplx<TT>), g, S3_RX, S3_RY);
    const CUtensorMap ms = make_tmap(sg, sizeof(cplx<TS>), g, S3_TX, S3_TY);
    const CUtensorMap mf = make_tmap(f ? (const void *)f : (const void *)x, sizeof(cplx<TT>), g, S3_TX, S3_TY);
    auto go = [&](auto kern) {
      CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      launch(kern, grid, block, (size_t)smem, s, g, mx, ms, mf, f ? 1 : 0, a, ih2, y, ub, us);
    };
    if (c4) go(k_fine_op3d_z<TT, ST_COMPACT4, TC, TS, ZC, NS>);
    else go(k_fine_op3d_z<TT, ST_FD2, TC, TS, ZC, NS>);
  }

  // ------------------------------------------------------------ operators
  // Precision model: level-0 vectors are stored in T, vectors
  // of every coarser level in fp64; stencil coefficients and patch factors in
  // T; all arithmetic in fp64.  (For T = double everything is fp64.)  Level
  // vector pointers are passed as void* and typed by level: vsize(l).
  static constexpr size_t vsize(int l) { return l == 0 ? sizeof(C) : sizeof(D); }

  // y = A_l x  or  y = f - A_l x
  // batch width at level l (the fine level always runs one right-hand side per call)
  int nbat(int l) const { return l == 0 ? 1 : nrb; }
  // fn(std::integral_constant<int, NR>, q0) over chunks (8, 4, 2, 1) of n right-hand sides
  template <typename Fn> static void over_batch(int n, Fn &&fn) {
    int q0 = 0;
    while (q0 < n) {
      const int left = n - q0;
      if (left >= 8) { fn(std::integral_constant<int, 8>{}, q0); q0 += 8; }
      else if (left >= 4) { fn(std::integral_constant<int, 4>{}, q0); q0 += 4; }
      else if (left >= 2) { fn(std::integral_constant<int, 2>{}, q0); q0 += 2; }
      else { fn(std::integral_constant<int, 1>{}, q0); q0 += 1; }
    }
  }

  void op(int l, int shifted, const void *x, const void *f, void *y, cudaStream_t s) {
    const Level &Lv = lev[l];
    halo(l, x, l == 0 ? 1 : Lv.r, s);
    auto nl = node_launch(Lv.geo);
    const double sz = vsize(l), nn = (double)Lv.geo.nodes();
    if (l == 0) {
      tag(f ? "fine_residual" : "fine_apply", l, (f ? 3 : 2) * sz * nn + sz * outside(l));
      const double a = shifted ? alpha : 0.0;
      const double ih2 = 1.0 / (Lv.h * Lv.h);
      const C *sg = sig.template as<C>();
      const C *xx = (const C *)x, *ff = (const C *)f;
      C *yy = (C *)y;
      const bool c4 = opt.fine_stencil == HMG_COMPACT4;
      const UBox &ub = Lv.ub;
      if (fine2d_march(sg, false, a, ih2, xx, ff, yy, s)) return;
      if (opt.dim == 2 && f32res && std::is_same<T, float>::value) {   // fp32 cycle residual (§4.1)
        if (c4) launch(k_fine_op<T, 2, ST_COMPACT4, T, T>, nl.grid, nl.block, 0, s, Lv.geo, sg, (T)a, (T)ih2, xx, ff, yy, ub, usig);
        else launch(k_fine_op<T, 2, ST_FD2, T, T>, nl.grid, nl.block, 0, s, Lv.geo, sg, (T)a, (T)ih2, xx, ff, yy, ub, usig);
      } else if (opt.dim == 2) {
        if (c4) launch(k_fine_op<T, 2, ST_COMPACT4, double, T>, nl.grid, nl.block, 0, s, Lv.geo, sg, a, ih2, xx, ff, yy, ub, widen(usig));
        else launch(k_fine_op<T, 2, ST_FD2, double, T>, nl.grid, nl.block, 0, s, Lv.geo, sg, a, ih2, xx, ff, yy, ub, widen(usig));
      } else if (f32res && std::is_same<T, float>::value) {   // 3D c64 cycle residual: fp32 arithmetic (§4.1)
        fine3d<T, T, T>(Lv.geo, sg, (T)a, (T)ih2, xx, ff, yy, usig, s);
      } else {
        fine3d<T, double, T>(Lv.geo, sg, a, ih2, xx, ff, yy, widen(usig), s);
      }
      return;
    }
    const D *xx = (const D *)x, *ff = (const D *)f;
    D *yy = (D *)y;
    if (mf_level1(l)) {   // A_1 = R_0 H_s P_0 through the fine grid (no coefficient planes)
      const Level &F = lev[0];
      constexpr int TX = 32, TY = 8;
      const dim3 block(32, 8), grid((Lv.geo.n[0] + TX - 1) / TX, (Lv.geo.n[1] + TY - 1) / TY);
      tag(f ? "mf_residual" : "mf_apply", l, (f ? 3 : 2) * sizeof(D) * nn + 4 * sizeof(D) * nn);
      const D *sg = sigd.template as<D>();
      const double ih2 = 1.0 / (F.h * F.h);
      const bool c4 = opt.fine_stencil == HMG_COMPACT4;
      auto go = [&](auto kern, int smem) {
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        launch(kern, grid, block, (size_t)smem, s, F.geo, Lv.geo, sg, alpha, ih2, xx, ff, yy);
      };
      // fp64 tile arithmetic (fp32 tiles measured: config 0 c64 35 FGMRES iterations vs 30)
#define HMG_MF1(KIND, RR, PR) go(k_galerkin1_mf<double, KIND, RR, PR, TX, TY, double>, MF1Tile<RR, TX, TY, 16>::SMEM)
      if (F.rR == 2 && F.rP == 2) {
        if (c4) HMG_MF1(ST_COMPACT4, 2, 2);
        else HMG_MF1(ST_FD2, 2, 2);
      } else if (F.rR == 1 && F.rP == 1) {
        if (c4) HMG_MF1(ST_COMPACT4, 1, 1);
        else HMG_MF1(ST_FD2, 1, 1);
      } else {
        if (c4) HMG_MF1(ST_COMPACT4, 1, 2);
        else HMG_MF1(ST_FD2, 1, 2);
      }
#undef HMG_MF1
      return;
    }
    const C *cf = Lv.coef.template as<C>();
    const int64_t bs = Lv.geo.total;
    if (opt.dim == 2 && nbat(l) == 1 && std::is_same<T, float>::value && (G % 2) == 0 && Lv.r <= 2 &&
        std::getenv("HMG_NO_PAIR_ST") == nullptr) {   // two nodes per thread, 16-byte coefficient pairs
      tag(f ? "stored_residual" : "stored_apply", l, coef_bytes(l, kcount(opt.dim, Lv.r)) + (f ? 3 : 2) * sz * nn);
      const float2 *c2 = reinterpret_cast<const float2 *>(cf);
      if (smarch > 0 && Lv.geo.n[1] >= 256) {   // (reads the planes: no dictionary path)
        tag(f ? "stored_residual" : "stored_apply", l, kcount(opt.dim, Lv.r) * sizeof(C) * outside(l) + (f ? 3 : 2) * sz * nn);   // warp-marching version on the large levels (opt-in)
        constexpr int PD = 2;
        const int SEG = smarch;
        const int nstrips = (Lv.geo.n[0] + SM_STRIP - 1) / SM_STRIP, nsegs = (Lv.geo.n[1] + SEG - 1) / SEG;
        const int64_t warps = (int64_t)nstrips * nsegs;
        const dim3 grid((unsigned)((warps + 3) / 4)), block(128);
        const int smem = 4 * (PD + 2) * 2 * 32 * 16;
        auto gom = [&](auto kern, auto ucp) {
          CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
          launch(kern, grid, block, (size_t)smem, s, Lv.geo, c2, xx, ff, yy, Lv.ub, ucp);
        };
        if (Lv.r == 1) {
          if (SEG == 8) gom(k_stored_op2d_march<1, 8, PD>, ucopy<9, double>(Lv.ucoef));
          else gom(k_stored_op2d_march<1, 16, PD>, ucopy<9, double>(Lv.ucoef));
        } else {
          if (SEG == 8) gom(k_stored_op2d_march<2, 8, PD>, ucopy<25, double>(Lv.ucoef));
          else gom(k_stored_op2d_march<2, 16, PD>, ucopy<25, double>(Lv.ucoef));
        }
        return;
      }
      // BY output rows per thread (register blocking) on the large levels, 1 on small ones (parallelism)
      static const int by_env = std::getenv("HMG_STORED_BY") ? std::atoi(std::getenv("HMG_STORED_BY")) : 2;
      const int BY = Lv.geo.n[1] >= 512 ? by_env : 1;
      const unsigned short *ccl = coef_cls(Lv);
      const C *ctb = coef_tab(Lv);
      auto go = [&](auto kern, int by) {
        const dim3 block(32, 8), grid(((Lv.geo.n[0] + 1) / 2 + 31) / 32, (Lv.geo.n[1] + 8 * by - 1) / (8 * by));
        launch(kern, grid, block, 0, s, Lv.geo, c2, xx, ff, yy, Lv.ub, ucopy<(2 * 2 + 1) * (2 * 2 + 1), double>(Lv.ucoef), ccl,
               reinterpret_cast<const float2 *>(ctb));
      };
      auto go1 = [&](auto kern, int by) {
        const dim3 block(32, 8), grid(((Lv.geo.n[0] + 1) / 2 + 31) / 32, (Lv.geo.n[1] + 8 * by - 1) / (8 * by));
        launch(kern, grid, block, 0, s, Lv.geo, c2, xx, ff, yy, Lv.ub, ucopy<9, double>(Lv.ucoef), ccl,
               reinterpret_cast<const float2 *>(ctb));
      };
      if (tile2d && BY == 2) {   // shared-memory tile of x (k_stored_op2d_pair<..., TILE>)
        if (ccl) {
          if (Lv.r == 1) go1(k_stored_op2d_pair<1, 2, true, true>, 2);
          else go(k_stored_op2d_pair<2, 2, true, true>, 2);
        } else {
          if (Lv.r == 1) go1(k_stored_op2d_pair<1, 2, false, true>, 2);
          else go(k_stored_op2d_pair<2, 2, false, true>, 2);
        }
        return;
      }
      if (ccl) {   // coefficient dictionary
        if (Lv.r == 1) {
          if (BY == 4) go1(k_stored_op2d_pair<1, 4, true>, 4);
          else if (BY == 2) go1(k_stored_op2d_pair<1, 2, true>, 2);
          else go1(k_stored_op2d_pair<1, 1, true>, 1);
        } else {
          if (BY == 4) go(k_stored_op2d_pair<2, 4, true>, 4);
          else if (BY == 2) go(k_stored_op2d_pair<2, 2, true>, 2);
          else go(k_stored_op2d_pair<2, 1, true>, 1);
        }
        return;
      }
      if (Lv.r == 1) {
        if (BY == 4) go1(k_stored_op2d_pair<1, 4>, 4);
        else if (BY == 2) go1(k_stored_op2d_pair<1, 2>, 2);
        else go1(k_stored_op2d_pair<1, 1>, 1);
      } else {
        if (BY == 4) go(k_stored_op2d_pair<2, 4>, 4);
        else if (BY == 2) go(k_stored_op2d_pair<2, 2>, 2);
        else go(k_stored_op2d_pair<2, 1>, 1);
      }
      return;
    }
    over_batch(nbat(l), [&](auto NRc, int q0) {
      constexpr int NR = decltype(NRc)::value;
      const D *xq = xx + q0 * bs, *fq = ff ? ff + q0 * bs : nullptr;
      D *yq = yy + q0 * bs;
      tag(f ? "stored_residual" : "stored_apply", l, coef_bytes(l, kcount(opt.dim, Lv.r)) + (f ? 3 : 2) * sz * nn * NR);
      const UBox &ub = Lv.ub;
      const auto &uv = Lv.ucoef;
      const unsigned short *ccl = coef_cls(Lv);
      const C *ctb = coef_tab(Lv);
      if (opt.dim == 2) {
        if (Lv.r == 1) launch(k_stored_op<double, T, 2, 1, NR>, nl.grid, nl.block, 0, s, Lv.geo, cf, xq, fq, yq, bs, ub, ucopy<9, double>(uv), ccl, ctb);
        else if (Lv.r == 2) launch(k_stored_op<double, T, 2, 2, NR>, nl.grid, nl.block, 0, s, Lv.geo, cf, xq, fq, yq, bs, ub, ucopy<25, double>(uv), ccl, ctb);
        else launch(k_stored_op<double, T, 2, 3, NR>, nl.grid, nl.block, 0, s, Lv.geo, cf, xq, fq, yq, bs, ub, ucopy<49, double>(uv), ccl, ctb);
      } else {
        // one right-hand side on a large level: BZ = 4 planes per thread (register blocking)
        static const int bz_env = std::getenv("HMG_STORED_BZ") ? std::atoi(std::getenv("HMG_STORED_BZ")) : 4;
        const int bz = (NR == 1 && Lv.geo.n[2] >= 64) ? bz_env : 1;
        dim3 grid4 = nl.grid, block4 = nl.block;
        grid4.z = (Lv.geo.n[2] + 3) / 4;
        if (flat3d) {   // flat (x, y) indexing: no idle lanes on 2^k + 1-wide rows
          block4 = dim3(256);
          grid4.x = (unsigned)(((int64_t)Lv.geo.n[0] * Lv.geo.n[1] + 255) / 256);
          grid4.y = 1;
        }
        // radius 2, 4 planes per thread: capped at 64 registers for 4 blocks per SM (measured on
        // config 3 level 1: 46 -> 30 ms per solve on the same box; HMG_STORED_MINB=1: uncapped)
        static const int minb = std::getenv("HMG_STORED_MINB") ? std::atoi(std::getenv("HMG_STORED_MINB")) : 4;
        if (bz == 4 && minb >= 4 && Lv.r == 2) {
          launch(k_stored_op<double, T, 3, 2, NR, 4, 4>, grid4, block4, 0, s, Lv.geo, cf, xq, fq, yq, bs, ub, ucopy<125, double>(uv), ccl, ctb);
        } else if (bz == 4) {
          if (Lv.r == 1) launch(k_stored_op<double, T, 3, 1, NR, 4>, grid4, block4, 0, s, Lv.geo, cf, xq, fq, yq, bs, ub, ucopy<27, double>(uv), ccl, ctb);
          else launch(k_stored_op<double, T, 3, 2, NR, 4>, grid4, block4, 0, s, Lv.geo, cf, xq, fq, yq, bs, ub, ucopy<125, double>(uv), ccl, ctb);
        } else {
          if (Lv.r == 1) launch(k_stored_op<double, T, 3, 1, NR>, nl.grid, nl.block, 0, s, Lv.geo, cf, xq, fq, yq, bs, ub, ucopy<27, double>(uv), ccl, ctb);
          else launch(k_stored_op<double, T, 3, 2, NR>, nl.grid, nl.block, 0, s, Lv.geo, cf, xq, fq, yq, bs, ub, ucopy<125, double>(uv), ccl, ctb);
        }
      }
    });
  }

  template <typename TI> void restrict_t(int l, const TI *r, D *fc, cudaStream_t s) {
    const Level &F = lev[l], &Cc = lev[l + 1];
    halo(l, r, F.rR, s);
    // into the first replicated level: compute this rank's rows, then allgather
    const Geo &gc = Cc.gather_in ? Cc.view : Cc.geo;
    auto nl = node_launch(gc);
    using BI = decltype(r->x);
    tag("restrict", l, (double)sizeof(TI) * F.geo.nodes() + (double)sizeof(D) * gc.nodes());
    static const bool nopr = std::getenv("HMG_NO_PAIR_RS") != nullptr;
    if (l == 0 && F.rR == 2 && std::is_same<T, float>::value && (G % 2) == 0 && (F.geo.base % 2) == 0 && !nopr) {
      const float2 *r2 = reinterpret_cast<const float2 *>(r);   // c64 fine level: 16-byte pair loads
      if (opt.dim == 2) launch(k_restrict_pair<2>, nl.grid, nl.block, 0, s, F.geo, gc, r2, fc);
      else if (!F.dist && !Cc.gather_in && zblock3) {   // one rank: 4 coarse planes per thread
        dim3 g4 = nl.grid;
        g4.z = (gc.n[2] + 3) / 4;
        launch(k_restrict_pair3_z<4>, g4, nl.block, 0, s, F.geo, gc, r2, fc);
      } else launch(k_restrict_pair<3>, nl.grid, nl.block, 0, s, F.geo, gc, r2, fc);
    } else if (opt.dim == 2) {
      if (F.rR == 1) launch(k_restrict<BI, double, 2, 1>, nl.grid, nl.block, 0, s, F.geo, gc, r, fc);
      else launch(k_restrict<BI, double, 2, 2>, nl.grid, nl.block, 0, s, F.geo, gc, r, fc);
    } else {
      if (F.rR == 1) launch(k_restrict<BI, double, 3, 1>, nl.grid, nl.block, 0, s, F.geo, gc, r, fc);
      else launch(k_restrict<BI, double, 3, 2>, nl.grid, nl.block, 0, s, F.geo, gc, r, fc);
    }
    if (Cc.gather_in) {
      std::vector<size_t> off(Cc.goff), len(Cc.glen);
      for (auto &x : off) x *= sizeof(D);
      for (auto &x : len) x *= sizeof(D);
      comm->allgatherv(fc, off, len, s);
    }
  }
  void restrict_(int l, const void *r, void *fc, cudaStream_t s) {
    if (l == 0) {
      restrict_t<C>(l, (const C *)r, (D *)fc, s);
      return;
    }
    for (int q = 0; q < nrb; ++q)
      restrict_t<D>(l, (const D *)r + q * lev[l].geo.total, (D *)fc + q * lev[l + 1].geo.total, s);
  }

  template <typename TU> void prolong_t(int l, const D *e, const TU *u, TU *uo, cudaStream_t s) {
    const Level &F = lev[l], &Cc = lev[l + 1];
    halo(l + 1, e, 1, s);
    using BU = decltype(u->x);
    tag("prolong_add", l, 2.0 * sizeof(TU) * F.geo.nodes() + (double)sizeof(D) * Cc.geo.nodes());
    // coarse nodes (global) whose 2x..2x+1 fine children touch this rank's fine rows
    int c0[3], nc[3];
    for (int a = 0; a < 3; ++a) {
      const int flo = F.geo.o[a], fhi = F.geo.o[a] + F.geo.n[a];   // global fine range
      c0[a] = flo / 2;
      nc[a] = (fhi - 1) / 2 - c0[a] + 1;
    }
    const dim3 block(32, 8), grid((nc[0] + 31) / 32, (nc[1] + 7) / 8, opt.dim == 3 ? nc[2] : 1);
    if (opt.dim == 3 && !F.dist && !Cc.dist && zblock3 && c0[2] == 0 && nc[2] == Cc.geo.n[2]) {
      const dim3 g4((nc[0] + 31) / 32, (nc[1] + 7) / 8, (nc[2] + 3) / 4);   // one rank: 4 coarse planes per thread
      if (F.rP == 1) launch(k_prolong3_z<BU, 1, 4>, g4, block, 0, s, F.geo, Cc.geo, e, u, uo);
      else launch(k_prolong3_z<BU, 2, 4>, g4, block, 0, s, F.geo, Cc.geo, e, u, uo);
      return;
    }
    if (opt.dim == 2) {
      if (F.rP == 1) launch(k_prolong_block<double, BU, 2, 1>, grid, block, 0, s, F.geo, Cc.geo, c0[0], c0[1], c0[2], nc[0], nc[1], nc[2], e, u, uo);
      else launch(k_prolong_block<double, BU, 2, 2>, grid, block, 0, s, F.geo, Cc.geo, c0[0], c0[1], c0[2], nc[0], nc[1], nc[2], e, u, uo);
    } else {
      if (F.rP == 1) launch(k_prolong_block<double, BU, 3, 1>, grid, block, 0, s, F.geo, Cc.geo, c0[0], c0[1], c0[2], nc[0], nc[1], nc[2], e, u, uo);
      else launch(k_prolong_block<double, BU, 3, 2>, grid, block, 0, s, F.geo, Cc.geo, c0[0], c0[1], c0[2], nc[0], nc[1], nc[2], e, u, uo);
    }
  }
  // u_out = u + P_l e  (u_out may be u)
  void prolong_(int l, const void *e, const void *u, void *u_out, cudaStream_t s) {
    if (l == 0) {
      prolong_t<C>(l, (const D *)e, (const C *)u, (C *)u_out, s);
      return;
    }
    const int64_t fs = lev[l].geo.total, cs = lev[l + 1].geo.total;
    for (int q = 0; q < nrb; ++q)
      prolong_t<D>(l, (const D *)e + q * cs, (const D *)u + q * fs, (D *)u_out + q * fs, s);
  }

  // generic Vanka sweep: the assembled operator B applied as a stencil; TV = level vector type
  template <typename TV, int DIM, int KIND> void vanka_(int l, const void *r, void *u, int zero, cudaStream_t s) {
    Level &Lv = lev[l];
    using BV = decltype(TV{}.x);
    auto nl = node_launch(Lv.geo);
    constexpr int NB = BStencil<DIM, KIND>::NB;
    const double nn = (double)Lv.geo.nodes();
    halo(l, r, 2, s);   // B reaches offsets up to +-2 (RB / Plus)
    const int64_t bs = Lv.geo.total;
    // (measured slower than the gather below on config 3 -- 46 vs 28 ms per solve at level 0: kept
    // as an opt-in, HMG_VANKA27_Z=1, bit-identical)
    static const bool v27 = std::getenv("HMG_VANKA27_Z") != nullptr;
    if (DIM == 3 && KIND == PK_ELEMENT && nbat(l) == 1 && stage3d && v27 && Lv.geo.n[2] >= 16) {
      // z-marching staged 27-point apply (k_stage3d.cuh): r planes through the bulk-copy ring
      constexpr int ZC = 32, NS = 4;
      tag(zero ? "vanka_zero" : "vanka", l, (double)NB * sizeof(C) * outside(l) + (zero ? 2 : 3) * sizeof(TV) * nn);
      const int slot = (S3_RY * S3_RX * (int)sizeof(TV) + 127) / 128 * 128;
      const int smem = 128 + NS * slot;
      const Geo &g = Lv.geo;
      const dim3 block(32, S3_TY + 1), grid((g.n[0] + S3_TX - 1) / S3_TX, (g.n[1] + S3_TY - 1) / S3_TY, (g.n[2] + ZC - 1) / ZC);
      auto kern = k_vanka27_z<BV, T, ZC, NS>;
      CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      const CUtensorMap mr = make_tmap(r, sizeof(TV), g, S3_RX, S3_RY);
      launch(kern, grid, block, (size_t)smem, s, g, mr, (const C *)Lv.bop.template as<C>(), (const TV *)u,
             (TV *)u, (BV)damp(l), zero, Lv.ub, ucopy<27, BV>(Lv.ubop));
      return;
    }
    // one right-hand side on a large level: BZ nodes along the slow axis per thread
    const int vbz = vanka_bz;
    const int nslow = DIM == 3 ? Lv.geo.n[2] : Lv.geo.n[1];
    if (nbat(l) == 1 && vbz > 1 && nslow >= 64) {
      tag(zero ? "vanka_zero" : "vanka", l, bop_bytes(l, NB) + (zero ? 2 : 3) * sizeof(TV) * nn);
      auto go = [&](auto kern, int bz) {
        dim3 grid = nl.grid, block = nl.block;
        if (DIM == 3) grid.z = (Lv.geo.n[2] + bz - 1) / bz;
        else grid.y = (Lv.geo.n[1] + 8 * bz - 1) / (8 * bz);
        if (DIM == 3 && flat3d) {   // flat (x, y) indexing: no idle lanes on 2^k + 1-wide rows
          block = dim3(256);
          grid.x = (unsigned)(((int64_t)Lv.geo.n[0] * Lv.geo.n[1] + 255) / 256);
          grid.y = 1;
        }
        launch(kern, grid, block, 0, s, Lv.geo, (const C *)Lv.bop.template as<C>(), (const TV *)r, (const TV *)u,
               (TV *)u, (BV)damp(l), zero, Lv.ub, ucopy<NB, BV>(Lv.ubop), bop_cls(Lv), bop_tab(Lv));
      };
      if (vbz >= 4) go(k_vanka_stencil_blk<BV, T, DIM, KIND, 4>, 4);
      else go(k_vanka_stencil_blk<BV, T, DIM, KIND, 2>, 2);
      return;
    }
    over_batch(nbat(l), [&](auto NRc, int q0) {
      constexpr int NR = decltype(NRc)::value;
      tag(zero ? "vanka_zero" : "vanka", l, bop_bytes(l, NB) + (zero ? 2 : 3) * sizeof(TV) * NR * nn);
      launch(k_vanka_stencil<BV, T, DIM, KIND, NR>, nl.grid, nl.block, 0, s, Lv.geo, (const C *)Lv.bop.template as<C>(),
             (const TV *)r + q0 * bs, (const TV *)u + q0 * bs, (TV *)u + q0 * bs, (BV)damp(l), zero, bs, Lv.ub,
             ucopy<NB, BV>(Lv.ubop), bop_cls(Lv), bop_tab(Lv));
    });
  }
  template <typename TV> void vanka_kind(int l, const void *r, void *u, int zero, cudaStream_t s) {
    const int dim = opt.dim;
    switch (opt.smoother) {
      case HMG_VANKA_RB: vanka_<TV, 2, PK_RB>(l, r, u, zero, s); break;
      case HMG_VANKA_ELEMENT: dim == 2 ? vanka_<TV, 2, PK_ELEMENT>(l, r, u, zero, s) : vanka_<TV, 3, PK_ELEMENT>(l, r, u, zero, s); break;
      case HMG_JACOBI: dim == 2 ? vanka_<TV, 2, PK_JACOBI>(l, r, u, zero, s) : vanka_<TV, 3, PK_JACOBI>(l, r, u, zero, s); break;
      case HMG_VANKA_PLUS: dim == 2 ? vanka_<TV, 2, PK_PLUS>(l, r, u, zero, s) : vanka_<TV, 3, PK_PLUS>(l, r, u, zero, s); break;
    }
  }

  // fork: a stream ordered after everything enqueued on s so far (the side stream, or s itself
  // when concurrency is off or profiling serialises the launches); join: s waits for it
  cudaStream_t fork(cudaStream_t s) {
    if (!split_conc || prof_active()) return s;
    if (!side) {
      CK(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming));
    }
    CK(cudaEventRecord(ev_fork, s));
    CK(cudaStreamWaitEvent(side, ev_fork, 0));
    return side;
  }
  void join(cudaStream_t s, cudaStream_t s2) {
    if (s2 == s) return;
    CK(cudaEventRecord(ev_join, s2));
    CK(cudaStreamWaitEvent(s, ev_join, 0));
  }

  // Do the level's sweeps read neighbours of u inside one kernel?  Then they
  // must run out of place (other blocks may still read the old u).
  bool fused_sweep(int l) const { return l == 0 && rb_closed; }

  // one additive Vanka relaxation (Eq. 3.8): u_out = u + w B (f - A u);
  // zero: u == 0 (u may be null).  Fused levels: u_out != u required;
  // generic levels: in place (u_out == u).
  void smooth(int l, const void *f, const void *u, void *u_out, int zero, cudaStream_t s) {
    Level &Lv = lev[l];
    const double w = damp(l);
    const double nn = (double)Lv.geo.nodes();
    if (l == 0 && rb_closed) {
      // warp-marching fused sweep: residual (unless zero), closed-form patch solves, gather; fp64 arithmetic
      const double ih2 = 1.0 / (Lv.h * Lv.h);
      constexpr int SEG = 32;   // output rows per warp segment (4 pipeline rows of overlap)
      const int nstrips = (Lv.geo.n[0] + RB_STRIP - 1) / RB_STRIP, nsegs = (Lv.geo.n[1] + SEG - 1) / SEG;
      const int64_t warps = (int64_t)nstrips * nsegs;
      const dim3 grid((unsigned)((warps + 7) / 8)), block(256);
      const C *sg = sig.template as<C>();
      const C *ia = rb_ia.template as<C>(), *id = rb_id.template as<C>();
      const C *ff = (const C *)f, *ui = (const C *)u;
      C *uo = (C *)u_out;
      halos(0, {{zero ? nullptr : u, 3}, {f, 2}}, s);   // one exchange for both
      // algorithmic bytes: f, u' (+ u) per node; ia, id (+ sigma) outside the uniform box
      tag(zero ? "smooth_rb2d_fine_zero" : "smooth_rb2d_fine", 0,
          (zero ? 2 : 3) * sizeof(C) * nn + (zero ? 2 : 3) * sizeof(C) * outside(0));
      const bool c4 = opt.fine_stencil == HMG_COMPACT4;
      // all arithmetic in fp64 (fp32 patch algebra -- with or
      // without an fp64 residual, in the post-sweep alone -- moved config 0 from
      // 30 to 34 iterations on the B200 while saving ~10 % at N = 4096)
      // rows stream through a cp.async ring PD = 2 rows ahead (measured: PD 1 / 3 slower)
      constexpr int PD = 2;
      auto go = [&](auto kern, int na) {
        const int smem = 8 * (PD + 2) * na * 32 * (int)sizeof(C);
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        launch(kern, grid, block, (size_t)smem, s, Lv.geo, sg, ia, id, alpha, ih2, ff, ui, uo, w, Lv.ub, usig, uia, uid);
      };
      // c64 non-zero: 3 blocks/SM (80 registers) measured 16 % faster than 2 (91 registers)
      constexpr int MB = sizeof(T) == 4 ? 3 : 2;
      static const bool two = std::getenv("HMG_MARCH1") == nullptr;
      if (std::is_same<T, float>::value && pair_ok() && c4 && two) {   // two columns per lane
        const int ns2 = (Lv.geo.n[0] + RB2_STRIP - 1) / RB2_STRIP;
        const int64_t w2 = (int64_t)ns2 * nsegs;
        const dim3 grid2((unsigned)((w2 + 3) / 4)), block2(128);
        auto go2 = [&](auto kern, int na) {
          const int smem = 4 * (PD + 2) * na * 32 * 16;
          CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
          launch(kern, grid2, block2, (size_t)smem, s, Lv.geo, (const float2 *)sg, (const float2 *)ia,
                 (const float2 *)id, alpha, ih2, (const float2 *)ff, (const float2 *)ui, (float2 *)uo, w, Lv.ub,
                 *(const float2 *)&usig, *(const float2 *)&uia, *(const float2 *)&uid);
        };
        // blocks/SM: zero sweep 4 (126 registers), non-zero 3 (152; 4 spills, measured 2.9x slower)
        // zero sweep: 4 blocks/SM, unrolled x2; non-zero: 3 blocks/SM, unrolled x3 (the
        // period of its rolling windows; measured 104 / 158 ms per solve at N = 4096,
        // against 116 / 169 without unrolling; x3 spills the zero sweep at 4 blocks/SM)
        // with a uniform box: the interior warps run the constant-coefficient instance
        // (MODE 1), the others the generic one (MODE 2); bit-identical to MODE 0
        if (Lv.ub.empty() || !rbfast) {
          if (zero) go2(k_rb2d_march2<ST_COMPACT4, true, SEG, double, 4, PD, 2>, 3);
          else go2(k_rb2d_march2<ST_COMPACT4, false, SEG, float, 3, PD, 3>, 5);
        } else {
          // the border warps (MODE 2: few, long generic marches) start first on the side stream
          // and overlap the interior instance (MODE 1) instead of trailing it
          cudaStream_t s0 = s, s2 = fork(s);
          s = s2;
          if (zero) go2(k_rb2d_march2<ST_COMPACT4, true, SEG, double, 4, PD, 2, 2>, 3);
          else go2(k_rb2d_march2<ST_COMPACT4, false, SEG, float, 3, PD, 3, 2>, 5);
          s = s0;
          if (zero) go2(k_rb2d_march2<ST_COMPACT4, true, SEG, double, 4, PD, 2, 1>, 3);
          else go2(k_rb2d_march2<ST_COMPACT4, false, SEG, float, 3, PD, 3, 1>, 5);
          join(s, s2);
        }
        return;
      }
      if (zero) {
        if (c4) go(k_rb2d_march<T, ST_COMPACT4, true, SEG, double, double, 1, 2, PD>, 3);
        else go(k_rb2d_march<T, ST_FD2, true, SEG, double, double, 1, 2, PD>, 3);
      } else {
        if (c4) go(k_rb2d_march<T, ST_COMPACT4, false, SEG, double, T, 1, MB, PD>, 5);
        else go(k_rb2d_march<T, ST_FD2, false, SEG, double, T, 1, MB, PD>, 5);
      }
      return;
    }
    if (u_out != u && !zero) CK(cudaMemcpyAsync(u_out, u, Lv.geo.total * vsize(l) * nbat(l), cudaMemcpyDeviceToDevice, s));
    const void *r = f;
    if (!zero) {
      op(l, 1, u_out, f, Lv.r_.p, s);
      r = Lv.r_.p;
    }
    if (l == 0) vanka_kind<C>(l, r, u_out, zero, s);
    else vanka_kind<D>(l, r, u_out, zero, s);
  }
  // in-place sweep on any level (fused levels go through the r_ scratch)
  void smooth_inplace(int l, const void *f, void *u, cudaStream_t s) {
    if (!fused_sweep(l)) {
      smooth(l, f, u, u, 0, s);
      return;
    }
    void *S = lev[l].r_.p;
    smooth(l, f, u, S, 0, s);
    CK(cudaMemcpyAsync(u, S, lev[l].geo.total * vsize(l), cudaMemcpyDeviceToDevice, s));
  }

  void coarse_(const void *r, void *e, cudaStream_t s) {
    const Level &Lc = lev[L - 1];
    const int N = (int)Lc.geo.nodes();
    const int64_t bs = Lc.geo.total;
    over_batch(nrb, [&](auto NRc, int q0) {
      constexpr int NR = decltype(NRc)::value;
      tag("coarse_gemv", L - 1, (double)N * N * 16 + 2.0 * N * sizeof(D) * NR);
      launch(k_coarse_gemv<double, NR>, dim3((N + 7) / 8), dim3(256), 0, s, Lc.geo, (const D *)ainv.template as<D>(),
             (const D *)r + q0 * bs, (D *)e + q0 * bs, bs);
    });
  }

  // CUDA graphs: on one GPU, and with a communicator whose calls are stream-ordered
  // device work (NCCL: its halos and the coarse allgather are captured with the cycle)
  bool graphs_ok() const {
    return (!comm || comm->size == 1 || comm->capturable()) && !prof_active() &&
           std::getenv("HMG_NO_GRAPHS") == nullptr;
  }

  // levels >= 1 of the cycle (zero initial guess on lev[1].u, rhs lev[1].f)
  // as one CUDA graph launch, on a private stream ordered against the caller's
  // stream by events (the legacy default stream cannot be captured)
  void coarse_cycle_graph(cudaStream_t s) {
    if (!gstream) {
      CK(cudaStreamCreateWithFlags(&gstream, cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&gev_in, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&gev_out, cudaEventDisableTiming));
    }
    CK(cudaEventRecord(gev_in, s));
    CK(cudaStreamWaitEvent(gstream, gev_in, 0));
    auto it = cgraphs.find(nrb);
    if (it == cgraphs.end()) {
      const long long k0 = launch_count_now();
      cudaGraph_t gr;
      CK(cudaStreamBeginCapture(gstream, cudaStreamCaptureModeThreadLocal));
      cycle(1, lev[1].f.p, lev[1].u.p, 1, gstream, true);
      CK(cudaStreamEndCapture(gstream, &gr));
      cudaGraphExec_t ex;
      CK(cudaGraphInstantiate(&ex, gr, 0));
      CK(cudaGraphDestroy(gr));
      cgraph_kernels_nr[nrb] = launch_count_now() - k0;
      add_launches(-cgraph_kernels_nr[nrb]);          // captured, not launched
      it = cgraphs.emplace(nrb, ex).first;
    }
    CK(cudaGraphLaunch(it->second, gstream));
    add_launches(cgraph_kernels_nr[nrb]);
    CK(cudaEventRecord(gev_out, gstream));
    CK(cudaStreamWaitEvent(s, gev_out, 0));
  }

  // u <- MG_0(f, 0) as ONE graph launch (level 0 included), captured per (f, u) pair
  void full_cycle_graph(const void *f, void *u, cudaStream_t s) {
    if (!gstream) {
      CK(cudaStreamCreateWithFlags(&gstream, cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&gev_in, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&gev_out, cudaEventDisableTiming));
    }
    CK(cudaEventRecord(gev_in, s));
    CK(cudaStreamWaitEvent(gstream, gev_in, 0));
    const auto key = std::make_pair(f, u);
    auto it = fgraphs.find(key);
    if (it == fgraphs.end()) {
      const long long k0 = launch_count_now();
      cudaGraph_t gr;
      CK(cudaStreamBeginCapture(gstream, cudaStreamCaptureModeThreadLocal));
      cycle(0, f, u, 1, gstream, true);
      CK(cudaStreamEndCapture(gstream, &gr));
      cudaGraphExec_t ex;
      CK(cudaGraphInstantiate(&ex, gr, 0));
      CK(cudaGraphDestroy(gr));
      const long long nk = launch_count_now() - k0;
      add_launches(-nk);                                 // captured, not launched
      it = fgraphs.emplace(key, std::make_pair(ex, nk)).first;
    }
    CK(cudaGraphLaunch(it->second.first, gstream));
    add_launches(it->second.second);
    CK(cudaEventRecord(gev_out, gstream));
    CK(cudaStreamWaitEvent(s, gev_out, 0));
  }
  bool full_graph_ok() const { return graphs_ok() && L > 1 && std::getenv("HMG_NO_FULL_GRAPH") == nullptr; }

  // Alg. 2.1, recursive; u <- MG_l(f, u)
  void cycle(int l, const void *f, void *u, int zero, cudaStream_t s, bool capturing = false) {
    if (l == 1 && zero && !capturing && L > 2 && f == lev[1].f.p && u == lev[1].u.p && graphs_ok()) {
      coarse_cycle_graph(s);
      return;
    }
    if (l == L - 1) {
      coarse_(f, u, s);
      return;
    }
    if (l == tail_l0 && zero && nrb == 1 && f == lev[l].f.p && u == lev[l].u.p) {   // levels >= l: one launch
      launch_tail(s);
      return;
    }
    Level &Lv = lev[l];
    for (int k = 0; k < opt.nu1; ++k) {                        // step 1: pre-smoothing
      if (k == 0 && zero) smooth(l, f, nullptr, u, 1, s);      //   zero guess: r = f, u written only
      else smooth_inplace(l, f, u, s);
    }
    if (opt.nu1 == 0 && zero) CK(cudaMemsetAsync(u, 0, Lv.geo.total * vsize(l) * nbat(l), s));
    Level &Cc = lev[l + 1];
    if (!resrestrict(l, u, f, Cc.f.p, s)) {                    // step 2 fused (2D c64 fine level), else:
      op(l, 1, u, f, Lv.r_.p, s);                              //   r = f - A u
      restrict_(l, Lv.r_.p, Cc.f.p, s);                        //   f_c = R r
    }
    const int rec = opt.cycle == 1 ? 2 : 1;                    // step 3: V / W recursion
    for (int c = 0; c < rec; ++c) cycle(l + 1, Cc.f.p, Cc.u.p, c == 0, s, capturing);
    if (opt.nu2 > 0 && fused_sweep(l)) {
      prolong_(l, Cc.u.p, u, Lv.r_.p, s);                      // step 4: S = u + P e (r_ is free now)
      smooth(l, f, Lv.r_.p, u, 0, s);                          // step 5: u = S + w B (f - A S)
      for (int k = 1; k < opt.nu2; ++k) smooth_inplace(l, f, u, s);
    } else {
      prolong_(l, Cc.u.p, u, u, s);                            // step 4: u += P e
      for (int k = 0; k < opt.nu2; ++k) smooth_inplace(l, f, u, s);   // step 5
    }
  }

  // ------------------------------------------------------------ API glue
  // user vectors are unpadded in the hierarchy's dtype; internal level
  // vectors are padded, in T (level 0) or fp64 (levels > 0)
  void pack(int l, const void *src, void *dst, cudaStream_t s) {
    auto nl = node_launch(lev[l].geo);
    tag("pack", l, (double)(sizeof(C) + vsize(l)) * lev[l].geo.nodes());
    if (l == 0) launch(k_pack<C>, nl.grid, nl.block, 0, s, lev[l].geo, (const C *)src, (C *)dst);
    else launch(k_pack_cvt<T, double>, nl.grid, nl.block, 0, s, lev[l].geo, (const C *)src, 0, (D *)dst, 1);
  }
  void unpack(int l, const void *src, void *dst, cudaStream_t s) {
    auto nl = node_launch(lev[l].geo);
    tag("unpack", l, (double)(sizeof(C) + vsize(l)) * lev[l].geo.nodes());
    if (l == 0) launch(k_unpack<C>, nl.grid, nl.block, 0, s, lev[l].geo, (const C *)src, (C *)dst);
    else launch(k_pack_cvt<double, T>, nl.grid, nl.block, 0, s, lev[l].geo, (const D *)src, 1, (C *)dst, 0);
  }
  void check_level(int l, bool allow_coarsest = true) const {
    if (l < 0 || l >= L || (!allow_coarsest && l == L - 1)) throw HmgError(HMG_EINVAL, "level out of range");
  }
  void api_apply(int l, int shifted, const void *x, void *y, cudaStream_t s) override {
    check_level(l);
    if (l > 0 && !shifted) throw HmgError(HMG_EINVAL, "coarse levels hold the shifted operator only");
    Level &Lv = lev[l];
    pack(l, x, Lv.u.p, s);
    op(l, shifted, Lv.u.p, nullptr, Lv.r_.p, s);
    unpack(l, Lv.r_.p, y, s);
  }
  void api_residual(int l, int shifted, const void *f, const void *x, void *r, cudaStream_t s) override {
    check_level(l);
    if (l > 0 && !shifted) throw HmgError(HMG_EINVAL, "coarse levels hold the shifted operator only");
    Level &Lv = lev[l];
    pack(l, f, Lv.f.p, s);
    pack(l, x, Lv.u.p, s);
    op(l, shifted, Lv.u.p, Lv.f.p, Lv.r_.p, s);
    unpack(l, Lv.r_.p, r, s);
  }
  void api_smooth(int l, const void *f, void *u, cudaStream_t s) override {
    check_level(l, false);
    Level &Lv = lev[l];
    pack(l, f, Lv.f.p, s);
    pack(l, u, Lv.u.p, s);
    smooth_inplace(l, Lv.f.p, Lv.u.p, s);
    unpack(l, Lv.u.p, u, s);
  }
  void api_restrict(int l, const void *r, void *fc, cudaStream_t s) override {
    check_level(l, false);
    pack(l, r, lev[l].r_.p, s);
    restrict_(l, lev[l].r_.p, lev[l + 1].f.p, s);
    unpack(l + 1, lev[l + 1].f.p, fc, s);
  }
  void api_prolong(int l, const void *ec, void *u, cudaStream_t s) override {
    check_level(l, false);
    pack(l + 1, ec, lev[l + 1].u.p, s);
    pack(l, u, lev[l].u.p, s);
    prolong_(l, lev[l + 1].u.p, lev[l].u.p, lev[l].u.p, s);
    unpack(l, lev[l].u.p, u, s);
  }
  void need_cycle() const {
    if (L < 2) throw HmgError(HMG_EINVAL, "operator-only hierarchy (levels = 1): no cycle, smoother or solve");
  }
  void api_coarse(const void *r, void *e, cudaStream_t s) override {
    need_cycle();
    Level &Lc = lev[L - 1];
    pack(L - 1, r, Lc.f.p, s);
    coarse_(Lc.f.p, Lc.u.p, s);
    unpack(L - 1, Lc.u.p, e, s);
  }
  void api_vcycle(const void *f, void *x, int zero, cudaStream_t s) override {
    need_cycle();
    Level &Lv = lev[0];
    pack(0, f, Lv.f.p, s);
    if (!zero) pack(0, x, Lv.u.p, s);
    cycle(0, Lv.f.p, Lv.u.p, zero, s);
    unpack(0, Lv.u.p, x, s);
  }

  // ------------------------------------------------------------ FGMRES
  // Mixed precision (both dtypes): the Arnoldi basis V, the preconditioned
  // vectors Z and every V-cycle run in the working precision T; the iterate x,
  // the right-hand side and the residual r = q - H x formed at each restart
  // are fp64.  For T = double this is plain FGMRES; for T = float it lets the
  // true relative residual reach 1e-6 although fp32 rounding of H x alone is
  // ~1e-6 relative for these operators (restarted GMRES as iterative
  // refinement).  Dots accumulate in fp64 in every case.
  void ensure_ws(int m, cudaStream_t s) {
    if (ws_m == m) return;
    const Geo &g = g0();
    // whole-cycle graphs are keyed on V/Z addresses: drop them with the old buffers
    for (auto &kv : fgraphs) cudaGraphExecDestroy(kv.second.first);
    fgraphs.clear();
    V.alloc((size_t)(m + 1) * g.total * sizeof(C), s);
    Z.alloc((size_t)m * g.total * sizeof(C), s);
    ownV = {(const char *)V.p, (const char *)V.p + V.bytes};
    ownZ = {(const char *)Z.p, (const char *)Z.p + Z.bytes};
    nblk = (int)std::min<int64_t>(148 * 8, (g.slab_len + KRY_THREADS - 1) / KRY_THREADS);
    partial.alloc((size_t)KRY_MAXV * KRY_MAXBLK * sizeof(double2), s);
    dres.alloc(256 * sizeof(double2), s);
    if (!qd.p) {
      qd.alloc(g.total * sizeof(double2), s);
      xd.alloc(g.total * sizeof(double2), s);
      rd.alloc(g.total * sizeof(double2), s);
    }
    ws_m = m;
  }
  C *Vp(int i) { return V.template as<C>() + (size_t)i * g0().total; }
  C *Zp(int i) { return Z.template as<C>() + (size_t)i * g0().total; }

  // out[0..nv) = V_i^H w over the interior slab (+ out[nv] = ||w||^2 if self)
  template <typename TV, typename TW>
  void mdot(const cplx<TV> *Vb, int nv, const cplx<TW> *w, double2 *out, cudaStream_t s, bool self = false) {
    const Geo &g = g0();
    tag("multidot", 0, (nv * sizeof(cplx<TV>) + sizeof(cplx<TW>)) * (double)g.nodes());   // algorithmic: nodes, not padded rows
    const int nb = krylov_multidot<TV, TW>(nv, self, Vb + g.slab_off, g.total, w + g.slab_off, g.slab_len,
                                           partial.template as<double2>(), s);
    tag("reduce", 0, 16.0 * (nv + self) * nb);
    launch(k_reduce_partials, dim3(nv + self), dim3(32), 0, s, (const double2 *)partial.template as<double2>(), nb,
           nv + (int)self, out);
    allreduce(out, nv + (int)self, s);
  }
  template <typename TV, typename TW>
  void maxpy(const cplx<TV> *Vb, int nv, const double2 *coef, double sgn, cplx<TW> *w, double2 *nrm_out,
             cudaStream_t s, const double *vscale = nullptr) {
    const Geo &g = g0();
    tag("multi_axpy", 0, (nv * sizeof(cplx<TV>) + 2.0 * sizeof(cplx<TW>)) * (double)g.nodes());
    const int nb = krylov_axpy<TV, TW>(nv, Vb + g.slab_off, g.total, coef, vscale, sgn, w + g.slab_off, g.slab_len,
                                       nrm_out ? partial.template as<double2>() : (double2 *)nullptr, s);
    if (nrm_out) {
      tag("reduce", 0, 16.0 * nb);
      launch(k_reduce_partials, dim3(1), dim3(32), 0, s, (const double2 *)partial.template as<double2>(), nb, 1,
             nrm_out);
      allreduce(nrm_out, 1, s);
    }
  }
  template <typename TX> double norm(const cplx<TX> *x, cudaStream_t s) {
    double2 *d = dres.template as<double2>() + 200;
    mdot<TX, TX>(x, 1, x, d, s);
    double2 hv;
    CK(cudaMemcpyAsync(&hv, d, sizeof(double2), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return std::sqrt(std::max(hv.x, 0.0));
  }
  template <typename TI, typename TO> void scale(const cplx<TI> *w, cplx<TO> *v, double a, cudaStream_t s) {
    const Geo &g = g0();
    tag("scale", 0, (sizeof(cplx<TI>) + sizeof(cplx<TO>)) * (double)g.nodes());
    launch(k_scale<TI, TO>, dim3(nblk), dim3(KRY_THREADS), 0, s, w + g.slab_off, v + g.slab_off, a, g.slab_len);
  }
  // w = H z for the Arnoldi process: T storage of z and w, fp64 sigma and fp64
  // arithmetic, i.e. the SAME operator as the fp64 true residual.  (sigma
  // rounded to fp32 perturbs H by ~6e-8 |sigma M x|, which is ~1e-6 of ||q||
  // for a Helmholtz solution, and the compact stencil cancels ~1e2-1e3x on
  // smooth vectors: either would cap the attainable relres near the 1e-6 tol.)
  void matvec(const C *z, C *w, cudaStream_t s) {
    const Level &Lv = lev[0];
    halo(0, z, 1, s);
    auto nl = node_launch(Lv.geo);
    const double ih2 = 1.0 / (Lv.h * Lv.h);
    const double2 *sg = sigd.template as<double2>();
    tag("fine_apply", 0, 2.0 * sizeof(C) * Lv.geo.nodes() + sizeof(double2) * outside(0));
    const bool c4 = opt.fine_stencil == HMG_COMPACT4;
    const UBox &ub = Lv.ub;
    if (fine2d_march(sg, true, 0.0, ih2, z, nullptr, w, s)) return;
    if (pair_ok()) {
      const dim3 block(32, 8), grid(((Lv.geo.n[0] + 1) / 2 + 31) / 32, (Lv.geo.n[1] + 7) / 8);
      const float2 *zz = reinterpret_cast<const float2 *>(z);
      float2 *ww = reinterpret_cast<float2 *>(w);
      if (c4) launch(k_fine_op2d_pair<ST_COMPACT4, double, double>, grid, block, 0, s, Lv.geo, sg, 0.0, ih2, zz, (const float2 *)nullptr, ww, ub, usigd);
      else launch(k_fine_op2d_pair<ST_FD2, double, double>, grid, block, 0, s, Lv.geo, sg, 0.0, ih2, zz, (const float2 *)nullptr, ww, ub, usigd);
      return;
    }
    if (opt.dim == 2) {
      if (c4) launch(k_fine_op<T, 2, ST_COMPACT4, double, double>, nl.grid, nl.block, 0, s, Lv.geo, sg, 0.0, ih2, z, (const C *)nullptr, w, ub, usigd);
      else launch(k_fine_op<T, 2, ST_FD2, double, double>, nl.grid, nl.block, 0, s, Lv.geo, sg, 0.0, ih2, z, (const C *)nullptr, w, ub, usigd);
    } else {
      fine3d<T, double, double>(Lv.geo, sg, 0.0, ih2, z, (const C *)nullptr, w, usigd, s);
    }
  }

  // rd = qd - H xd in fp64 (unshifted fine operator)
  void residual_d(cudaStream_t s) {
    const Level &Lv = lev[0];
    halo(0, xd.p, 1, s, 1, sizeof(D));
    auto nl = node_launch(Lv.geo);
    const double ih2 = 1.0 / (Lv.h * Lv.h);
    const double2 *sg = sigd.template as<double2>();
    const double2 *x = xd.template as<double2>(), *f = qd.template as<double2>();
    double2 *y = rd.template as<double2>();
    tag("fine_residual_fp64", 0, 48.0 * Lv.geo.nodes() + 16.0 * outside(0));
    const bool c4 = opt.fine_stencil == HMG_COMPACT4;
    const UBox &ub = Lv.ub;
    if (opt.dim == 2) {
      if (c4) launch(k_fine_op<double, 2, ST_COMPACT4>, nl.grid, nl.block, 0, s, Lv.geo, sg, 0.0, ih2, x, f, y, ub, usigd);
      else launch(k_fine_op<double, 2, ST_FD2>, nl.grid, nl.block, 0, s, Lv.geo, sg, 0.0, ih2, x, f, y, ub, usigd);
    } else {
      fine3d<double, double, double>(Lv.geo, sg, 0.0, ih2, x, f, y, usigd, s);
    }
  }

  // ---------------------------------------------------------------- FGMRES
  // One right-hand side's Krylov state.  Its device buffers are swapped into the
  // solver's working members (V, Z, qd, xd, rd) while it is advanced (bind).
  typedef std::complex<double> cd;
  struct RhsState {
    DBuf V, Z, qd, xd, rd;
    std::vector<cd> H, cs, sn, gv, y;
    std::vector<double> nbeta, hist;
    int m = 0, j = 0, its = 0, restarts = 0;
    bool active = true, converged = false, start = true, have_res = false, failed = false;
    bool pre = false;   // this step's cycle and matvec were already enqueued (speculatively)
    double qn = 0, true_rel = 1, est = 1;
    cd &Hs(int i, int k) { return H[(size_t)i * m + k]; }
  };
  void bind(RhsState &r) {
    std::swap(V, r.V);
    std::swap(Z, r.Z);
    std::swap(qd, r.qd);
    std::swap(xd, r.xd);
    std::swap(rd, r.rd);
  }
  // binds a state for one scope and unbinds it on exit, also when the scope
  // throws (breakdown, CUDA error): the state's buffers never stay swapped in
  struct Bound {
    Solver *sv;
    RhsState &r;
    Bound(Solver *sv_, RhsState &r_) : sv(sv_), r(r_) { sv->bind(r); }
    ~Bound() { sv->bind(r); }
    Bound(const Bound &) = delete;
    Bound &operator=(const Bound &) = delete;
  };
  // the state's own buffers (the first state of a solve borrows the solver's)
  void alloc_state(RhsState &r, int m, cudaStream_t s) {
    const Geo &g = g0();
    r.V.alloc((size_t)(m + 1) * g.total * sizeof(C), s);
    r.Z.alloc((size_t)m * g.total * sizeof(C), s);
    r.qd.alloc(g.total * sizeof(double2), s);
    r.xd.alloc(g.total * sizeof(double2), s);
    r.rd.alloc(g.total * sizeof(double2), s);
  }

  // level 0 of one V-cycle for each of na right-hand sides, levels >= 1 as one
  // batched pass (coefficients read once for all of them); per right-hand side
  // the same kernels and arithmetic as cycle(0, ...)
  void cycle_batch(const std::vector<const C *> &f, const std::vector<C *> &u, cudaStream_t s) {
    const int na = (int)f.size();
    if (na == 1 || L < 2) {
      auto owned = [](const void *p, const std::pair<const char *, const char *> &r) {
        return (const char *)p >= r.first && (const char *)p < r.second;
      };
      for (int k = 0; k < na; ++k) {
        if (full_graph_ok() && owned(f[k], ownV) && owned(u[k], ownZ)) full_cycle_graph(f[k], u[k], s);
        else cycle(0, f[k], u[k], 1, s);
      }
      return;
    }
    ensure_batch(na, s);
    Level &F = lev[0], &C1 = lev[1];
    const int64_t b1 = C1.geo.total;
    for (int k = 0; k < na; ++k) {
      for (int i = 0; i < opt.nu1; ++i) {
        if (i == 0) smooth(0, f[k], nullptr, u[k], 1, s);
        else smooth_inplace(0, f[k], u[k], s);
      }
      if (opt.nu1 == 0) CK(cudaMemsetAsync(u[k], 0, F.geo.total * sizeof(C), s));
      op(0, 1, u[k], f[k], F.r_.p, s);
      restrict_(0, F.r_.p, C1.f.template as<D>() + k * b1, s);
    }
    nrb = na;
    const int rec = opt.cycle == 1 ? 2 : 1;
    for (int c = 0; c < rec; ++c) cycle(1, C1.f.p, C1.u.p, c == 0, s);
    nrb = 1;
    for (int k = 0; k < na; ++k) {
      const D *e = C1.u.template as<D>() + k * b1;
      if (opt.nu2 > 0 && fused_sweep(0)) {
        prolong_(0, e, u[k], F.r_.p, s);
        smooth(0, f[k], F.r_.p, u[k], 0, s);
        for (int i = 1; i < opt.nu2; ++i) smooth_inplace(0, f[k], u[k], s);
      } else {
        prolong_(0, e, u[k], u[k], s);
        for (int i = 0; i < opt.nu2; ++i) smooth_inplace(0, f[k], u[k], s);
      }
    }
  }
  // level >= 1 buffers for nr right-hand sides (captured graphs hold the old ones)
  void ensure_batch(int nr, cudaStream_t s) {
    if (nr <= nrb_cap) return;
    for (int l = 1; l < L; ++l) {
      Level &Lv = lev[l];
      Lv.u.alloc((size_t)nr * Lv.geo.total * vsize(l), s);
      Lv.f.alloc((size_t)nr * Lv.geo.total * vsize(l), s);
      Lv.r_.alloc((size_t)nr * Lv.geo.total * vsize(l), s);
    }
    for (auto &kv : cgraphs) cudaGraphExecDestroy(kv.second);
    cgraphs.clear();
    for (auto &kv : fgraphs) cudaGraphExecDestroy(kv.second.first);
    fgraphs.clear();
    nrb_cap = nr;
    setup_tail(s);   // its level table points at the reallocated vectors
  }

  // Start (or restart) the Arnoldi process of a bound state: r = q - H x in fp64,
  // stop if the true residual already meets tol, else W_0 = r / beta.
  void fgmres_start(RhsState &r, double tol, cudaStream_t s) {
    if (!r.have_res) residual_d(s);                   // r = q - H x (fp64)
    r.have_res = false;
    const double beta = norm<double>(rd.template as<double2>(), s);
    r.true_rel = beta / r.qn;
    if (!std::isfinite(beta)) throw HmgError(HMG_EBREAKDOWN, "non-finite residual norm");
    if (r.true_rel < tol) {
      r.converged = true;
      r.active = false;
      return;
    }
    scale<double, T>(rd.template as<double2>(), Vp(0), 1.0 / beta, s);
    std::fill(r.H.begin(), r.H.end(), cd(0, 0));
    std::fill(r.gv.begin(), r.gv.end(), cd(0, 0));
    r.gv[0] = beta;
    r.nbeta[0] = 1.0;
    r.j = 0;
    r.start = false;
  }

  // One Arnoldi step j of a bound state after its preconditioner application
  // z'_j = M(W_j) (already in Z[j]).  Lazily normalised basis: V[j] holds
  // W_j = nb[j] v_j with nb[j] = ||W_j|| (nb[0] = 1); the cycle and the matvec
  // run on W_j, so d_i = W_i^H (H M W_j) = nb[i] nb[j] h_ij, the AXPY removes
  // (d_i / nb[i]^2) W_i, and W_{j+1} = nb[j] w_perp needs no scaling pass.
  void fgmres_step(RhsState &r, double tol, int maxiter, cudaStream_t s, bool speculate = false) {
    const int j = r.j, m = r.m;
    double2 *dr = dres.template as<double2>();
    double *ib2h = hpin + 512, *ib2d = reinterpret_cast<double *>(dr + 160);
    C *w = Vp(j + 1);
    if (!r.pre) matvec(Zp(j), w, s);                  // w' = H z'_j (fp64 arithmetic)
    r.pre = false;
    const int nv = j + 1;
    for (int i = 0; i <= j; ++i) ib2h[i] = 1.0 / (r.nbeta[i] * r.nbeta[i]);
    CK(cudaMemcpyAsync(ib2d, ib2h, nv * sizeof(double), cudaMemcpyHostToDevice, s));
    // classical Gram-Schmidt with selective reorthogonalisation: a second
    // pass only under strong cancellation, ||w''|| < 0.1 ||w'|| (DESIGN.md
    // §6: DGKS's 1/sqrt 2 reorthogonalised 59% of the steps at N=4096 and
    // never changed an iteration count)
    mdot<T, T>(V.template as<C>(), nv, w, dr, s, true);            // d = W^H w', ||w'||^2
    maxpy<T, T>(V.template as<C>(), nv, dr, -1.0, w, dr + 64, s, ib2d);   // w'' = w' - W diag(1/nb^2) d
    CK(cudaMemcpyAsync(hpin, dr, 65 * sizeof(double2), cudaMemcpyDeviceToHost, s));
    // Pipelining (single right-hand side): W_{j+1} is complete on the device, so the next
    // preconditioner application and matvec are enqueued BEFORE the host waits for the dots;
    // the Givens update overlaps the next V-cycle.  If W_{j+1} changes afterwards (second
    // Gram-Schmidt pass, range rescaling) or the cycle ends here, the speculative work is
    // discarded / redone -- every iterate stays that of the unpipelined solve.
    const bool spec = speculate && j + 1 < m && r.its + 1 < maxiter;
    CK(cudaEventRecord(ev_dots, s));
    if (spec) {
      cycle_batch({Vp(j + 1)}, {Zp(j + 1)}, s);
      matvec(Zp(j + 1), Vp(j + 2), s);
    }
    CK(cudaEventSynchronize(ev_dots));
    bool spec_ok = spec;
    const double2 *hh = reinterpret_cast<const double2 *>(hpin);
    for (int i = 0; i <= j; ++i) r.Hs(i, j) = cd(hh[i].x, hh[i].y) / (r.nbeta[i] * r.nbeta[j]);
    double hn2 = hh[64].x;
    if (!(hn2 >= kReorthEta2 * hh[nv].x)) {
      ++reorth;
      spec_ok = false;                                // W_{j+1} changes: redo the next cycle
      mdot<T, T>(V.template as<C>(), nv, w, dr + 32, s);
      maxpy<T, T>(V.template as<C>(), nv, dr + 32, -1.0, w, dr + 64, s, ib2d);
      CK(cudaMemcpyAsync(hpin + 64, dr + 32, 33 * sizeof(double2), cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      for (int i = 0; i <= j; ++i) r.Hs(i, j) += cd(hh[32 + i].x, hh[32 + i].y) / (r.nbeta[i] * r.nbeta[j]);
      hn2 = hh[64].x;
    }
    const double wn = std::sqrt(std::max(hn2, 0.0));          // ||W_{j+1}||
    for (int i = 0; i <= j; ++i)
      if (!std::isfinite(r.Hs(i, j).real()) || !std::isfinite(r.Hs(i, j).imag()))
        throw HmgError(HMG_EBREAKDOWN, "non-finite Arnoldi coefficient");
    if (!std::isfinite(wn)) throw HmgError(HMG_EBREAKDOWN, "non-finite Arnoldi norm");
    const double hn = wn / r.nbeta[j];
    r.Hs(j + 1, j) = hn;
    const bool breakdown = hn == 0.0;
    r.nbeta[j + 1] = wn;
    if (!breakdown && (wn < 1e-25 || wn > 1e25)) {   // keep the stored basis in range (rare)
      scale<T, T>(w, w, 1.0 / wn, s);
      r.nbeta[j + 1] = 1.0;
      spec_ok = false;                                // W_{j+1} changes: redo the next cycle
    }
    for (int i = 0; i < j; ++i) {                    // previous Givens rotations
      const cd t = r.cs[i] * r.Hs(i, j) + r.sn[i] * r.Hs(i + 1, j);
      r.Hs(i + 1, j) = -std::conj(r.sn[i]) * r.Hs(i, j) + std::conj(r.cs[i]) * r.Hs(i + 1, j);
      r.Hs(i, j) = t;
    }
    const cd a = r.Hs(j, j), b = r.Hs(j + 1, j);
    const double den = std::sqrt(std::norm(a) + std::norm(b));
    if (den == 0.0) { r.cs[j] = 1.0; r.sn[j] = 0.0; }
    else if (std::abs(a) == 0.0) { r.cs[j] = 0.0; r.sn[j] = 1.0; }
    else { r.cs[j] = std::abs(a) / den; r.sn[j] = (a / std::abs(a)) * std::conj(b) / den; }
    r.Hs(j, j) = r.cs[j] * a + r.sn[j] * b;
    r.Hs(j + 1, j) = 0.0;
    r.gv[j + 1] = -std::conj(r.sn[j]) * r.gv[j];
    r.gv[j] = r.cs[j] * r.gv[j];
    ++r.its;
    r.est = std::abs(r.gv[j + 1]) / r.qn;
    r.hist.push_back(r.est);
    const bool stop = r.est < tol || breakdown || r.its >= maxiter;
    if (!stop && j + 1 < m) {
      r.j = j + 1;
      r.pre = spec_ok;                                // its cycle and matvec are already enqueued
      return;
    }
    // end of a restart cycle: x += Z y (fp64), then the fp64 true residual
    const int jend = j + 1;
    for (int i = jend - 1; i >= 0; --i) {           // back substitution
      cd acc = r.gv[i];
      for (int k = i + 1; k < jend; ++k) acc -= r.Hs(i, k) * r.y[k];
      r.y[i] = acc / r.Hs(i, i);
    }
    double2 *yp = reinterpret_cast<double2 *>(hpin) + 128;
    for (int i = 0; i < jend; ++i) yp[i] = make_double2(r.y[i].real() / r.nbeta[i], r.y[i].imag() / r.nbeta[i]);
    CK(cudaMemcpyAsync(dr + 96, yp, jend * sizeof(double2), cudaMemcpyHostToDevice, s));
    maxpy<T, double>(Z.template as<C>(), jend, dr + 96, 1.0, xd.template as<double2>(), nullptr, s);
    ++r.restarts;
    residual_d(s);
    r.have_res = true;
    r.start = true;
    if (stop) {
      r.true_rel = norm<double>(rd.template as<double2>(), s) / r.qn;
      if (r.true_rel < tol) { r.converged = true; r.active = false; return; }
    }
    if (r.its >= maxiter) r.active = false;
  }

  // Saad's FGMRES(m) with CGS2 Arnoldi and complex Givens rotations; x0 = 0;
  // stop when |g_{j+1}|/||q|| < tol and the fp64 true residual confirms it
  // (reading A17), else restart.  Every state solves its qd -> xd; the states
  // advance in lockstep, one batched preconditioner application per step.
  void fgmres(std::vector<RhsState> &st, int m, double tol, int maxiter, cudaStream_t s) {
    ensure_ws(m, s);
    reorth = 0;
    for (auto &r : st) {
      r.m = m;
      r.H.assign((size_t)(m + 1) * m, cd(0, 0));
      r.cs.assign(m, cd(0, 0));
      r.sn.assign(m, cd(0, 0));
      r.gv.assign(m + 1, cd(0, 0));
      r.y.assign(m, cd(0, 0));
      r.nbeta.assign(m + 1, 1.0);
      r.hist.assign(1, 1.0);
      {
        Bound b(this, r);
        CK(cudaMemsetAsync(xd.p, 0, g0().total * sizeof(double2), s));
        r.qn = norm<double>(qd.template as<double2>(), s);
      }
      if (r.qn == 0.0) { r.active = false; r.converged = true; r.true_rel = 0.0; r.est = 0.0; }
      if (maxiter == 0) r.active = false;
    }
    std::vector<const C *> fv;
    std::vector<C *> uv;
    std::vector<RhsState *> act;
    for (;;) {
      act.clear();
      for (auto &r : st) {
        if (!r.active) continue;
        if (r.start) {
          Bound b(this, r);
          fgmres_start(r, tol, s);
        }
        if (r.active) act.push_back(&r);
      }
      if (act.empty()) break;
      fv.clear();
      uv.clear();
      for (RhsState *r : act) {                       // z'_j = M(W_j) for every active state
        fv.push_back(r->V.template as<C>() + (size_t)r->j * g0().total);
        uv.push_back(r->Z.template as<C>() + (size_t)r->j * g0().total);
      }
      const bool single = act.size() == 1 && std::getenv("HMG_NO_PIPELINE") == nullptr;
      if (!(single && act[0]->pre)) cycle_batch(fv, uv, s);   // (already enqueued when pipelined)
      for (RhsState *r : act) {
        Bound b(this, *r);
        fgmres_step(*r, tol, maxiter, s, single);
      }
    }
  }

  void fill_report(const RhsState &r, float ms, hmg_report *rep) {
    rep->iterations = r.its;
    rep->converged = r.converged;
    rep->restarts = r.restarts;
    rep->relres_true = r.true_rel;
    rep->relres_est = r.est;
    rep->seconds = ms * 1e-3;
    const int n = (int)r.hist.size();
    rep->history_len = rep->history ? std::min(n, rep->history_cap) : 0;
    for (int i = 0; i < rep->history_len; ++i) rep->history[i] = r.hist[i];
    // c_f of Eq. 5.1 after a 5-iteration warm-up
    const int wu = 5;
    if (n > wu + 1) rep->c_f = std::pow(r.hist[n - 1] / r.hist[wu], 1.0 / (n - 1 - wu));
    else rep->c_f = std::nan("");
  }

  hmg_status api_fgmres(const void *q, void *x, int host, int m, double tol, int maxiter, cudaStream_t s,
                        hmg_report *rep) override {
    return api_fgmres_batch(1, q, x, host, m, tol, maxiter, s, rep);
  }

  // nr right-hand sides q[k * N ...], solutions x[k * N ...] (unpadded, contiguous)
  hmg_status api_fgmres_batch(int nr, const void *q, void *x, int host, int m, double tol, int maxiter,
                              cudaStream_t s, hmg_report *reps) override {
    if (m < 1 || m >= KRY_MAXV) throw HmgError(HMG_EINVAL, "restart must be in [1, 31]");
    if (!(tol > 0) || maxiter < 0) throw HmgError(HMG_EINVAL, "tol must be > 0 and maxiter >= 0");
    if (nr < 1) throw HmgError(HMG_EINVAL, "nrhs must be >= 1");
    need_cycle();
    if (nr > 1 && comm && comm->size > 1) throw HmgError(HMG_EINVAL, "batched solves run on one rank");
    if (nr > 1 && host) throw HmgError(HMG_EINVAL, "batched solves take device buffers");
    ensure_ws(m, s);
    const Geo &g = g0();
    const int64_t N = g.nodes();
    auto nl = node_launch(g);
    std::vector<RhsState> st(nr);
    // the first state borrows the solver's buffers until this call returns or throws
    Bound borrow(this, st[0]);
    for (int k = 1; k < nr; ++k) alloc_state(st[k], m, s);
    for (int k = 0; k < nr; ++k) {
      const C *qsrc = (const C *)q + (size_t)k * N;
      if (host) {
        CK(cudaMemcpyAsync(io.p, q, N * sizeof(C), cudaMemcpyHostToDevice, s));
        qsrc = io.template as<C>();
      }
      tag("pack", 0, (double)(sizeof(C) + sizeof(double2)) * N);
      launch(k_pack_cvt<T, double>, nl.grid, nl.block, 0, s, g, qsrc, 0, st[k].qd.template as<double2>(), 1);
    }
    CK(cudaEventRecord(ev0, s));
    hmg_status st_out = HMG_OK;
    fgmres(st, m, tol, maxiter, s);
    CK(cudaEventRecord(ev1, s));
    for (int k = 0; k < nr; ++k) {
      C *xdst = host ? io.template as<C>() : (C *)x + (size_t)k * N;
      tag("unpack", 0, (double)(sizeof(C) + sizeof(double2)) * N);
      launch(k_pack_cvt<double, T>, nl.grid, nl.block, 0, s, g, (const double2 *)st[k].xd.template as<double2>(), 1,
             xdst, 0);
      if (host) CK(cudaMemcpyAsync(x, io.p, N * sizeof(C), cudaMemcpyDeviceToHost, s));
      if (!st[k].converged) st_out = HMG_ENOTCONVERGED;
    }
    CK(cudaStreamSynchronize(s));
    if (reps) {
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, ev0, ev1));
      for (int k = 0; k < nr; ++k) fill_report(st[k], ms, reps + k);
    }
    return st_out;
  }

  // ------------------------------------------------------------ per-stream workspaces
  // A second solver over the SAME hierarchy: coefficient arrays (stencils, Vanka
  // operators, sigma, RB factors, coarsest inverse) are shared as non-owning views of
  // this solver's buffers; level vectors, Krylov basis, events, graphs and pinned
  // staging are its own.  (One per stream.)
  std::unique_ptr<SolverBase> clone_workspace(cudaStream_t s) const override {
    std::unique_ptr<Solver<T>> c(new Solver<T>);
    c->opt = opt;
    c->damping = damping;
    c->L = L;
    c->comm = comm;
    c->G = G;
    c->omega = omega;
    c->alpha = alpha;
    c->plo = plo; c->phi = phi; c->wlo = wlo; c->whi = whi; c->pdist = pdist;
    c->part_setup = part_setup;
    c->rb_closed = rb_closed;
    c->stage3d = stage3d;
    c->fmarch = fmarch;
    c->rbfast = rbfast;
    c->vanka_bz = vanka_bz;
    c->smarch = smarch;
    c->rrfuse = rrfuse;
    c->zblock3 = zblock3;
    c->split_conc = split_conc;
    c->tile2d = tile2d;
    c->flat3d = flat3d;
    c->f32res = f32res;
    c->tail_minb = tail_minb;
    c->usig = usig; c->uia = uia; c->uid = uid; c->usigd = usigd;
    c->sig = DBuf::view(sig);
    c->sigd = DBuf::view(sigd);
    c->w2k2 = DBuf::view(w2k2);
    c->gq = DBuf::view(gq);
    c->rb_ia = DBuf::view(rb_ia);
    c->rb_id = DBuf::view(rb_id);
    c->ainv = DBuf::view(ainv);
    c->lev.resize(L);
    for (int l = 0; l < L; ++l) {
      const Level &a = lev[l];
      Level &b = c->lev[l];
      b.geo = a.geo; b.h = a.h; b.r = a.r; b.rR = a.rR; b.rP = a.rP;
      b.dist = a.dist; b.lo = a.lo; b.hi = a.hi; b.gather_in = a.gather_in; b.view = a.view;
      b.goff = a.goff; b.glen = a.glen; b.ub = a.ub; b.ucoef = a.ucoef; b.ubop = a.ubop;
      b.coef = DBuf::view(a.coef);
      b.bop = DBuf::view(a.bop);
      b.ccls = DBuf::view(a.ccls); b.ctab = DBuf::view(a.ctab); b.cn = a.cn;
      b.bcls = DBuf::view(a.bcls); b.btab = DBuf::view(a.btab); b.bn = a.bn;
      if (L > 1 || l == 0) {
        b.u.alloc(b.geo.total * vsize(l), s);
        b.f.alloc(b.geo.total * vsize(l), s);
        b.r_.alloc(b.geo.total * vsize(l), s);
      }
    }
    c->io.alloc(io.bytes, s);
    CK(cudaEventCreate(&c->ev0));
    CK(cudaEventCreate(&c->ev1));
    CK(cudaEventCreateWithFlags(&c->ev_dots, cudaEventDisableTiming));
    CK(cudaMallocHost((void **)&c->hpin, 4096 * sizeof(double)));
    c->setup_tail(s);
    CK(cudaStreamSynchronize(s));
    return std::unique_ptr<SolverBase>(c.release());
  }

  // ------------------------------------------------------------ introspection
  int64_t level_nodes(int l, int64_t n[3]) const override {
    if (l < 0 || l >= L) return -1;
    const Geo &g = lev[l].geo;
    if (n) { n[0] = g.n[0]; n[1] = g.n[1]; n[2] = g.n[2]; }
    return g.nodes();
  }
  int radius(int l) const override { return (l < 0 || l >= L) ? -1 : lev[l].r; }
  int dict_classes(int l, int *cn, int *bn) const override {
    if (l < 0 || l >= L) return -1;
    if (cn) *cn = lev[l].cn;
    if (bn) *bn = lev[l].bn;
    return 0;
  }
  int64_t uniform_box(int l, int64_t *lo, int64_t *hi) const override {
    if (l < 0 || l >= L) return -1;
    for (int a = 0; a < 3; ++a) {
      if (lo) lo[a] = lev[l].ub.lo[a];
      if (hi) hi[a] = lev[l].ub.hi[a];
    }
    return lev[l].ub.nodes();
  }
  void level_rows(int l, int64_t *lo, int64_t *hi) const override {
    if (l < 0 || l >= L) { *lo = *hi = -1; return; }
    *lo = lev[l].lo;
    *hi = lev[l].hi;
  }
  int copy_stencil(int l, double *out, int64_t cap) override {
    check_level(l);
    cudaStream_t s = 0;
    const Geo &g = lev[l].geo;
    const int K = kcount(opt.dim, lev[l].r);
    const int64_t N = g.nodes();
    if (cap < (int64_t)K * N * 2) throw HmgError(HMG_EINVAL, "output buffer too small");
    DBuf tmp, dst;
    dst.alloc((size_t)K * N * sizeof(double2), s);
    auto nl = node_launch(g);
    if (l == 0) {
      materialize(g, lev[0].h, w2k2.template as<double>(), gq.template as<double>(), tmp, s);
      launch(k_compact_stencil<double>, nl.grid, nl.block, 0, s, g, K, (const double2 *)tmp.template as<double2>(), dst.template as<double2>());
    } else {
      launch(k_compact_stencil<T>, nl.grid, nl.block, 0, s, g, K, (const C *)lev[l].coef.template as<C>(), dst.template as<double2>());
    }
    CK(cudaMemcpy(out, dst.p, (size_t)K * N * sizeof(double2), cudaMemcpyDeviceToHost));
    return K;
  }
};


// factories (solver_c64.cu, solver_c128.cu)
SolverBase *make_solver_c64();
SolverBase *make_solver_c128();

}  // namespace hmg
