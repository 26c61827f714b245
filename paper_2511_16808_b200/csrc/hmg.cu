// hmg.cu -- the extern "C" boundary of libhmg.so and the process-wide launch /
// profiling state (the solver itself: solver.cuh, instantiated per precision).
//
// Hot path: FGMRES(m) right-preconditioned by one
// multigrid cycle (Alg. 2.1) on the shifted operator H_s (Eq. 2.6)
// with additive Vanka smoothing (Eq. 3.8), Galerkin coarse operators
// and level-dependent intergrid (Eqs. 3.3-3.4).  Every arithmetic
// step runs in the kernels of k_*.cuh; this file only sequences launches.
#include "solver.cuh"

#include <atomic>

namespace hmg {


static std::atomic<long long> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
bool pdl_enabled() {
  static const bool on = std::getenv("HMG_NO_PDL") == nullptr && std::getenv("HMG_PDL") != nullptr;
  return on;
}
long long launch_count_now() { return g_launches.load(); }
void add_launches(long long n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

// ---- opt-in per-kernel profiling (hmg_profile_begin / hmg_profile_report)
struct ProfRec {
  std::string name;
  double bytes;
  cudaEvent_t a, b;
};
struct Profiler {
  bool on = false;
  std::vector<ProfRec> recs;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pool;
  size_t used = 0;
};
static Profiler g_prof;
bool prof_active() { return g_prof.on; }
static thread_local const char *t_name = nullptr;
static thread_local int t_level = 0;
static thread_local double t_bytes = 0;
void tag(const char *name, int level, double bytes) {
  t_name = name;
  t_level = level;
  t_bytes = bytes;
}
int prof_before(cudaStream_t s) {
  if (!g_prof.on || !t_name) return -1;
  if (g_prof.used == g_prof.pool.size()) {
    cudaEvent_t x, y;
    CK(cudaEventCreate(&x));
    CK(cudaEventCreate(&y));
    g_prof.pool.emplace_back(x, y);
  }
  const int i = (int)g_prof.used++;
  CK(cudaEventRecord(g_prof.pool[i].first, s));
  return i;
}
void prof_after(cudaStream_t s, int i) {
  if (i >= 0) {
    CK(cudaEventRecord(g_prof.pool[i].second, s));
    g_prof.recs.push_back({std::string(t_name) + "@L" + std::to_string(t_level), t_bytes, g_prof.pool[i].first,
                           g_prof.pool[i].second});
  }
  t_name = nullptr;
}

}  // namespace hmg

// =====================================================================  C-ABI
// One hierarchy, one workspace per stream ("the library allocates one
// workspace per stream on first use, keyed by the stream"): the first stream that runs
// a call uses the build's solver; every other stream gets a clone sharing the
// coefficients (clone_workspace).  Calls on one stream are serialised by the caller;
// calls on different streams may run concurrently from different host threads.
// Partitioned hierarchies serve one stream (their collectives must match across ranks).
struct hmg_hierarchy {
  std::unique_ptr<hmg::SolverBase> impl;
  mutable std::mutex mu;
  mutable bool claimed = false;
  mutable void *first = nullptr;
  mutable std::map<void *, std::unique_ptr<hmg::SolverBase>> per_stream;
  ~hmg_hierarchy() { per_stream.clear(); }   // clones (views) before the owner
  hmg::SolverBase *ws(void *stream) const {
    std::lock_guard<std::mutex> lk(mu);
    if (!claimed) {
      claimed = true;
      first = stream;
    }
    if (stream == first) return impl.get();
    auto it = per_stream.find(stream);
    if (it != per_stream.end()) return it->second.get();
    if (impl->comm && impl->comm->size > 1)
      throw hmg::HmgError(HMG_EINVAL, "a partitioned hierarchy serves one stream");
    auto c = impl->clone_workspace(reinterpret_cast<cudaStream_t>(stream));
    hmg::SolverBase *r = c.get();
    per_stream.emplace(stream, std::move(c));
    return r;
  }
};

struct hmg_comm {
  std::shared_ptr<void> group;            // LOCAL group (shared by its rank handles)
  std::unique_ptr<hmg::Comm> comm;        // a rank's communicator (null for a group handle)
};

static thread_local std::string t_err;

static hmg_status fail(hmg_status s, const std::string &m) {
  t_err = m;
  return s;
}

#define HMG_API_BEGIN try {
#define HMG_API_END                                                 \
  }                                                                 \
  catch (const hmg::HmgError &e) { return fail(e.st, e.what()); }   \
  catch (const std::bad_alloc &) { return fail(HMG_ENOMEM, "host allocation failed"); } \
  catch (const std::exception &e) { return fail(HMG_ECUDA, e.what()); }

static cudaStream_t S(void *s) { return reinterpret_cast<cudaStream_t>(s); }

extern "C" {

static hmg_status build_impl(const hmg_options *o, const double *kappa, double omega, const double *gamma,
                             double alpha, hmg::Comm *comm, void *stream, hmg_hierarchy **out);

hmg_status hmg_build_hierarchy(const hmg_options *o, const double *kappa, double omega, const double *gamma,
                               double alpha, void *stream, hmg_hierarchy **out) {
  return build_impl(o, kappa, omega, gamma, alpha, nullptr, stream, out);
}

hmg_status hmg_build_hierarchy_dist(const hmg_options *o, const double *kappa, double omega, const double *gamma,
                                    double alpha, hmg_comm *comm, void *stream, hmg_hierarchy **out) {
  if (!comm || !comm->comm) return fail(HMG_EINVAL, "comm must be a rank communicator");
  return build_impl(o, kappa, omega, gamma, alpha, comm->comm.get(), stream, out);
}

hmg_status hmg_comm_local_group(int nranks, hmg_comm **out) {
  HMG_API_BEGIN
  if (!out || nranks < 1) return fail(HMG_EINVAL, "bad arguments");
  std::unique_ptr<hmg_comm> c(new hmg_comm);
  c->group = hmg::local_group_create(nranks);
  *out = c.release();
  return HMG_OK;
  HMG_API_END
}

hmg_status hmg_comm_local_rank(hmg_comm *group, int rank, hmg_comm **out) {
  HMG_API_BEGIN
  if (!group || !group->group || !out) return fail(HMG_EINVAL, "bad arguments");
  std::unique_ptr<hmg_comm> c(new hmg_comm);
  c->comm.reset(hmg::local_comm_create(group->group, rank));
  *out = c.release();
  return HMG_OK;
  HMG_API_END
}

hmg_status hmg_comm_nccl_unique_id(void *id128) {
  HMG_API_BEGIN
  if (!id128) return fail(HMG_EINVAL, "null pointer");
  hmg::nccl_unique_id(id128);
  return HMG_OK;
  HMG_API_END
}

hmg_status hmg_comm_nccl(const void *id128, int rank, int nranks, hmg_comm **out) {
  HMG_API_BEGIN
  if (!id128 || !out || nranks < 1 || rank < 0 || rank >= nranks) return fail(HMG_EINVAL, "bad arguments");
  std::unique_ptr<hmg_comm> c(new hmg_comm);
  c->comm.reset(hmg::nccl_comm_create(id128, rank, nranks));
  *out = c.release();
  return HMG_OK;
  HMG_API_END
}

void hmg_comm_destroy(hmg_comm *c) { delete c; }

int hmg_slab_partition(int64_t nodes0, int levels, int nranks, int ghost, int64_t *lo, int64_t *hi, int *dist) {
  if (nodes0 < 1 || levels < 1 || nranks < 1 || ghost < 1 || !lo || !hi || !dist) return -1;
  std::vector<int64_t> Nl(levels), l2, h2;
  std::vector<int> d2;
  Nl[0] = nodes0;
  for (int l = 1; l < levels; ++l) Nl[l] = (Nl[l - 1] - 1) / 2 + 1;
  hmg::slab_partition(Nl, nranks, ghost, l2, h2, d2);
  for (size_t i = 0; i < l2.size(); ++i) { lo[i] = l2[i]; hi[i] = h2[i]; }
  int nd = 0;
  for (int l = 0; l < levels; ++l) { dist[l] = d2[l]; nd += d2[l]; }
  return nd;
}

int hmg_setup_plan(const hmg_options *o, int nranks, int rank, int64_t *wlo, int64_t *whi, int64_t *klo,
                   int64_t *khi, double *bytes) {
  try {
    if (!o || nranks < 1 || rank < 0 || rank >= nranks || !wlo || !whi || !klo || !khi || !bytes) return -1;
    if ((o->dim != 2 && o->dim != 3) || o->levels < 2 || o->levels > 16) return -1;
    const int dim = o->dim, L = o->levels, ax = dim == 3 ? 2 : 1;
    const int G = nranks > 1 ? (o->intergrid == HMG_CUBIC ? 5 : 4) : (o->intergrid == HMG_CUBIC ? 3 : 2);
    const double s = o->dtype == HMG_C64 ? 8.0 : 16.0;
    std::vector<std::array<int64_t, 3>> n(L);
    for (int a = 0; a < 3; ++a) n[0][a] = a < dim ? o->cells[a] + 1 : 1;
    for (int l = 1; l < L; ++l)
      for (int a = 0; a < 3; ++a) n[l][a] = a < dim ? (n[l - 1][a] - 1) / 2 + 1 : 1;
    std::vector<int64_t> Nl(L);
    for (int l = 0; l < L; ++l) Nl[l] = n[l][ax];
    std::vector<int> rR(L, 1), rP(L, 1), r(L, 1);
    for (int l = 0; l + 1 < L; ++l) hmg::level_scheme(o->intergrid, l, rR[l], rP[l]);
    for (int l = 0; l + 1 < L; ++l) r[l + 1] = o->coarse_op == HMG_GALERKIN ? (rR[l] + r[l] + rP[l]) / 2 : 1;
    std::vector<int64_t> lo, hi, wl, wh;
    std::vector<int> dist;
    hmg::slab_partition(Nl, nranks, G, lo, hi, dist);
    const bool rb = dim == 2 && o->smoother == HMG_VANKA_RB;
    hmg::plan_windows(Nl, lo, hi, dist, nranks, rank, G, rR, o->coarse_op == HMG_REDISCRETIZE, rb, wl, wh);
    auto kc = [&](int rr) { return dim == 3 ? (2 * rr + 1) * (2 * rr + 1) * (2 * rr + 1) : (2 * rr + 1) * (2 * rr + 1); };
    const int pk = o->smoother == HMG_JACOBI ? 1 : o->smoother == HMG_VANKA_ELEMENT ? (1 << dim)
                   : o->smoother == HMG_VANKA_PLUS ? 2 * dim + 1 : 5;
    const int nb = o->smoother == HMG_JACOBI ? 1 : o->smoother == HMG_VANKA_ELEMENT ? (dim == 3 ? 27 : 9)
                   : (o->smoother == HMG_VANKA_PLUS && dim == 3) ? 25 : 13;
    auto padded = [&](int l, int64_t rows) {   // padded box elements of `rows` slab-axis rows
      const int64_t px = (n[l][0] + 2 * G + 7) / 8 * 8;
      const int64_t rs = dim == 3 ? px * (n[l][1] + 2 * G) : px;
      return (double)rs * (double)(rows + 2 * G);
    };
    double peak = 0, resident = 0, hvmax = 0;
    int nd = 0;
    for (int l = 0; l < L; ++l) {
      nd += dist[l];
      wlo[l] = wl[l];
      whi[l] = wh[l];
      klo[l] = dist[l] ? lo[(size_t)l * nranks + rank] : 0;
      khi[l] = dist[l] ? hi[(size_t)l * nranks + rank] : Nl[l];
      const double W = padded(l, wh[l] - wl[l]), Kp = padded(l, khi[l] - klo[l]);
      const int K = kc(r[l]);
      peak += 16.0 * K * W;                                  // fp64 stencil (setup)
      if (l > 0) { peak += s * K * W; resident += s * K * Kp; }   // stored stencil
      if (l + 1 < L) {
        if (l == 0 && rb) { peak += 2 * s * W; resident += 2 * s * Kp; }   // RB factors
        else { peak += s * nb * W; resident += s * nb * Kp; hvmax = std::max(hvmax, 16.0 * pk * pk * W); }
      }
      resident += 3.0 * (l == 0 ? s : 16.0) * Kp;            // cycle vectors u, f, r
      if (l == 0) {
        peak += (16.0 + s + 16.0) * W;                       // w2k2 + gq, sigma (T), sigma (fp64)
        resident += (16.0 + s + 16.0) * Kp;
      }
    }
    const double Nc = (double)n[L - 1][0] * n[L - 1][1] * n[L - 1][2];
    peak += hvmax + 3.0 * Nc * Nc * 16.0;                   // patch-inverse scratch, dense A + inverse
    resident += Nc * Nc * 16.0;
    const double N0 = (double)n[0][0] * n[0][1] * n[0][2];
    resident += N0 * s;                                      // io staging of the host entry points
    const double K0p = padded(0, khi[0] - klo[0]);
    bytes[0] = peak;
    bytes[1] = resident;
    bytes[2] = K0p * (41.0 * s + 3.0 * 16.0);                // FGMRES(20) basis V, Z + fp64 x, q, r
    return nd;
  } catch (...) {
    return -1;
  }
}

int hmg_level_rows(const hmg_hierarchy *h, int level, int64_t *lo, int64_t *hi) {
  if (!h || !lo || !hi || level < 0 || level >= h->impl->L) return -1;
  h->impl->level_rows(level, lo, hi);
  return 0;
}

static hmg_status build_impl(const hmg_options *o, const double *kappa, double omega, const double *gamma,
                             double alpha, hmg::Comm *comm, void *stream, hmg_hierarchy **out) {
  HMG_API_BEGIN
  if (!o || !kappa || !gamma || !out) return fail(HMG_EINVAL, "null pointer");
  *out = nullptr;
  if (o->dim != 2 && o->dim != 3) return fail(HMG_EINVAL, "dim must be 2 or 3");
  if (o->levels < 1 || o->levels > 16) return fail(HMG_EINVAL, "levels must be in [1, 16] (1 = operator only)");
  if (!(o->h > 0)) return fail(HMG_EINVAL, "h must be > 0");
  if (!(omega > 0)) return fail(HMG_EINVAL, "omega must be > 0");
  if (!(alpha >= 0)) return fail(HMG_EINVAL, "shift alpha must be >= 0");
  if (o->nu1 < 0 || o->nu2 < 0 || o->cycle < 0 || o->cycle > 1) return fail(HMG_EINVAL, "bad nu1/nu2/cycle");
  if (o->fine_stencil != HMG_COMPACT4 && o->fine_stencil != HMG_FD2) return fail(HMG_EINVAL, "bad fine_stencil");
  if (o->coarse_op != HMG_GALERKIN && o->coarse_op != HMG_REDISCRETIZE) return fail(HMG_EINVAL, "bad coarse_op");
  if (o->smoother < 0 || o->smoother > 3) return fail(HMG_EINVAL, "bad smoother");
  if (o->smoother == HMG_VANKA_RB && o->dim != 2)
    return fail(HMG_EINVAL, "RB patch is 2D only (the 13-node 3D RB patch is rejected by the paper, P:949-951)");
  if (o->dtype != HMG_C64 && o->dtype != HMG_C128) return fail(HMG_EINVAL, "bad dtype");
  if (!o->damping || o->n_damping < 1) return fail(HMG_EINVAL, "damping required");
  int64_t N = 1;
  for (int a = 0; a < o->dim; ++a) {
    const int64_t c = o->cells[a];
    if (c < 4 || c % (1LL << (o->levels - 1)) != 0)
      return fail(HMG_EINVAL, "cells must be >= 4 and divisible by 2^(levels-1)");
    N *= c + 1;
  }
  for (int64_t i = 0; i < N; ++i) {
    if (!(kappa[i] > 0) || !std::isfinite(kappa[i])) return fail(HMG_EINVAL, "kappa must be finite and > 0");
    if (!(gamma[i] >= 0) || !std::isfinite(gamma[i])) return fail(HMG_EINVAL, "gamma must be finite and >= 0");
  }
  std::unique_ptr<hmg_hierarchy> h(new hmg_hierarchy);
  if (o->dtype == HMG_C64) h->impl.reset(hmg::make_solver_c64());
  else h->impl.reset(hmg::make_solver_c128());
  h->impl->opt = *o;
  h->impl->damping.assign(o->damping, o->damping + o->n_damping);
  h->impl->opt.damping = nullptr;
  h->impl->comm = comm;
  h->impl->build(kappa, omega, gamma, alpha, S(stream));
  *out = h.release();
  return HMG_OK;
  HMG_API_END
}

hmg_status hmg_apply_helmholtz(const hmg_hierarchy *h, int level, int shifted, const void *x, void *y, void *stream) {
  HMG_API_BEGIN
  if (!h || !x || !y) return fail(HMG_EINVAL, "null pointer");
  h->ws(stream)->api_apply(level, shifted, x, y, S(stream));
  return HMG_OK;
  HMG_API_END
}

hmg_status hmg_residual(const hmg_hierarchy *h, int level, int shifted, const void *f, const void *x, void *r,
                        void *stream) {
  HMG_API_BEGIN
  if (!h || !f || !x || !r) return fail(HMG_EINVAL, "null pointer");
  h->ws(stream)->api_residual(level, shifted, f, x, r, S(stream));
  return HMG_OK;
  HMG_API_END
}

hmg_status hmg_smooth(const hmg_hierarchy *h, int level, const void *f, void *u, void *stream) {
  HMG_API_BEGIN
  if (!h || !f || !u) return fail(HMG_EINVAL, "null pointer");
  h->ws(stream)->api_smooth(level, f, u, S(stream));
  return HMG_OK;
  HMG_API_END
}

hmg_status hmg_restrict(const hmg_hierarchy *h, int level, const void *r, void *fc, void *stream) {
  HMG_API_BEGIN
  if (!h || !r || !fc) return fail(HMG_EINVAL, "null pointer");
  h->ws(stream)->api_restrict(level, r, fc, S(stream));
  return HMG_OK;
  HMG_API_END
}

hmg_status hmg_prolong_add(const hmg_hierarchy *h, int level, const void *ec, void *u, void *stream) {
  HMG_API_BEGIN
  if (!h || !ec || !u) return fail(HMG_EINVAL, "null pointer");
  h->ws(stream)->api_prolong(level, ec, u, S(stream));
  return HMG_OK;
  HMG_API_END
}

hmg_status hmg_coarse_solve(const hmg_hierarchy *h, const void *r, void *e, void *stream) {
  HMG_API_BEGIN
  if (!h || !r || !e) return fail(HMG_EINVAL, "null pointer");
  h->ws(stream)->api_coarse(r, e, S(stream));
  return HMG_OK;
  HMG_API_END
}

hmg_status hmg_vcycle(const hmg_hierarchy *h, const void *f, void *x, int x_is_zero, void *stream) {
  HMG_API_BEGIN
  if (!h || !f || !x) return fail(HMG_EINVAL, "null pointer");
  h->ws(stream)->api_vcycle(f, x, x_is_zero, S(stream));
  return HMG_OK;
  HMG_API_END
}

hmg_status hmg_fgmres_solve(const hmg_hierarchy *h, const void *q, void *x, int restart, double tol, int maxiter,
                            void *stream, hmg_report *rep) {
  HMG_API_BEGIN
  if (!h || !q || !x) return fail(HMG_EINVAL, "null pointer");
  hmg_status st = h->ws(stream)->api_fgmres(q, x, 0, restart, tol, maxiter, S(stream), rep);
  if (st == HMG_ENOTCONVERGED) t_err = "FGMRES reached maxiter without converging";
  return st;
  HMG_API_END
}

hmg_status hmg_fgmres_solve_host(const hmg_hierarchy *h, const void *q, void *x, int restart, double tol,
                                 int maxiter, void *stream, hmg_report *rep) {
  HMG_API_BEGIN
  if (!h || !q || !x) return fail(HMG_EINVAL, "null pointer");
  hmg_status st = h->ws(stream)->api_fgmres(q, x, 1, restart, tol, maxiter, S(stream), rep);
  if (st == HMG_ENOTCONVERGED) t_err = "FGMRES reached maxiter without converging";
  return st;
  HMG_API_END
}

hmg_status hmg_fgmres_solve_batch(const hmg_hierarchy *h, int nrhs, const void *q, void *x, int restart, double tol,
                                  int maxiter, void *stream, hmg_report *reps) {
  HMG_API_BEGIN
  if (!h || !q || !x) return fail(HMG_EINVAL, "null pointer");
  hmg_status st = h->ws(stream)->api_fgmres_batch(nrhs, q, x, 0, restart, tol, maxiter, S(stream), reps);
  if (st == HMG_ENOTCONVERGED) t_err = "FGMRES reached maxiter without converging for at least one right-hand side";
  return st;
  HMG_API_END
}

int hmg_num_levels(const hmg_hierarchy *h) { return h ? h->impl->L : -1; }

int64_t hmg_level_nodes(const hmg_hierarchy *h, int level, int64_t n[3]) {
  return h ? h->impl->level_nodes(level, n) : -1;
}

int hmg_stencil_radius(const hmg_hierarchy *h, int level) { return h ? h->impl->radius(level) : -1; }

int hmg_copy_stencil(const hmg_hierarchy *h, int level, double *out, int64_t cap) {
  try {
    if (!h || !out) { t_err = "null pointer"; return -1; }
    return h->impl->copy_stencil(level, out, cap);
  } catch (const std::exception &e) {
    t_err = e.what();
    return -1;
  }
}

int64_t hmg_uniform_box(const hmg_hierarchy *h, int level, int64_t lo[3], int64_t hi[3]) {
  return h ? h->impl->uniform_box(level, lo, hi) : -1;
}
int hmg_dict_classes(const hmg_hierarchy *h, int level, int *coef_classes, int *bop_classes) {
  return h ? h->impl->dict_classes(level, coef_classes, bop_classes) : -1;
}

int64_t hmg_launch_count(void) { return hmg::g_launches.load(); }

void hmg_profile_begin(void) {
  hmg::g_prof.recs.clear();
  hmg::g_prof.used = 0;
  hmg::g_prof.on = true;
}

const char *hmg_profile_report(void) {
  static thread_local std::string out;
  hmg::g_prof.on = false;
  struct Agg { long long n = 0; double ms = 0, bytes = 0; };
  std::vector<std::pair<std::string, Agg>> agg;
  for (auto &r : hmg::g_prof.recs) {
    float ms = 0;
    if (cudaEventSynchronize(r.b) != cudaSuccess || cudaEventElapsedTime(&ms, r.a, r.b) != cudaSuccess) ms = 0;
    auto it = std::find_if(agg.begin(), agg.end(), [&](const std::pair<std::string, Agg> &p) { return p.first == r.name; });
    if (it == agg.end()) { agg.push_back({r.name, Agg{}}); it = agg.end() - 1; }
    it->second.n += 1;
    it->second.ms += ms;
    it->second.bytes += r.bytes;
  }
  out = "{";
  for (size_t i = 0; i < agg.size(); ++i) {
    char buf[256];
    snprintf(buf, sizeof buf, "%s\"%s\": {\"launches\": %lld, \"ms\": %.6f, \"bytes\": %.0f}", i ? ", " : "",
             agg[i].first.c_str(), agg[i].second.n, agg[i].second.ms, agg[i].second.bytes);
    out += buf;
  }
  out += "}";
  hmg::g_prof.recs.clear();
  hmg::g_prof.used = 0;
  return out.c_str();
}

void hmg_hierarchy_destroy(hmg_hierarchy *h) { delete h; }

const char *hmg_last_error(void) { return t_err.c_str(); }

const char *hmg_version(void) { return "hmg 0.1 (sm_100a)"; }

}  // extern "C"
