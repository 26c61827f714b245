/*
 * hmg.h -- C-ABI of libhmg.so: B200-native (sm_100a) complex-shifted-Laplacian
 * multigrid V-cycle with additive Vanka smoothing, used as the right
 * preconditioner of restarted flexible GMRES for the finite-difference acoustic
 * Helmholtz operator  -Lap p - omega^2 kappa^2 (1 - i gamma/omega) p = q
 * (arXiv 2511.16808; "P:n" = PAPER.md line n, "S:n" = SPEC.md line n,
 * "SURVEY §x" = /root/repo/SURVEY.md).
 *
 * Every entry point is extern "C" with plain pointers and sizes; no torch or
 * C++ types cross this boundary.  All compute runs in the library's own CUDA
 * kernels on the stream passed in (a cudaStream_t cast to void*; NULL = the
 * legacy default stream).
 *
 * Conventions:
 *   - grid: cells[a] cells per axis, n_a = cells[a] + 1 nodes, ALL nodes are
 *     unknowns, homogeneous Dirichlet by truncation of out-of-domain neighbours
 *     (readings A4/A5).  Vectors are x-fastest, then y, then z, unpadded,
 *     length N = prod(n_a).
 *   - complex vectors are interleaved (re, im): float2 for HMG_C64, double2
 *     for HMG_C128.
 *   - operator (Eq. 1.1; Eq. 2.2; Eq. 2.3):
 *         H   = L - diag(sigma)   M,  sigma   = w^2 k^2 (1 - i g/w)
 *         H_s = L - diag(sigma_s) M,  sigma_s = w^2 k^2 (1 - i (g/w + alpha))
 *     i.e. H_s = H + i alpha w^2 k^2 M: the shift adds attenuation (
 *     Eq. 2.6 P:249-253 read with readings A1/A2).
 *   - coarse operators A_{l+1} = R_l A_l P_l (Galerkin) with the
 *     level-dependent intergrid of Eqs. 3.3-3.4 by default.
 *
 * Errors: every call returns an hmg_status; on failure hmg_last_error() gives
 * a thread-local message (for HMG_ESINGULAR_PATCH it names the level and the
 * patch anchor node).  Calls never abort the process.
 *
 * Ownership: the library copies kappa/gamma at build time; vector arguments
 * are caller-owned and only read/written during the call (stream-ordered).
 * A hierarchy is immutable after build.  Workspaces are per STREAM
 * (SURVEY §8(b)): the first stream a call runs on uses the
 * build's workspace, every other stream gets its own on first use (level
 * vectors, Krylov basis, graphs, staging; the coefficients are shared), so
 * calls on different streams may run concurrently from different host
 * threads.  Calls on one stream must be serialised by the caller.  A
 * slab-partitioned hierarchy serves one stream (HMG_EINVAL otherwise).
 */
#ifndef HMG_H
#define HMG_H

#include <stdint.h>

#if defined(__GNUC__)
#define HMG_API __attribute__((visibility("default")))
#else
#define HMG_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  HMG_OK = 0,
  HMG_EINVAL = 1,             /* bad argument: dim, cells, h, omega, kappa<=0, gamma<0, null ptr, level */
  HMG_ESINGULAR_PATCH = 2,    /* a Vanka patch matrix H_i (Eq. 3.8) is singular */
  HMG_ESINGULAR_COARSE = 3,   /* the coarsest Galerkin matrix is singular */
  HMG_EBREAKDOWN = 4,         /* NaN/Inf in the Arnoldi process */
  HMG_ENOTCONVERGED = 5,      /* maxiter reached; report filled, x = last iterate */
  HMG_ENOMEM = 6,
  HMG_ECUDA = 7,
  HMG_ENCCL = 8
} hmg_status;

typedef enum { HMG_C64 = 0, HMG_C128 = 1 } hmg_dtype;

/* fine-level discretisation (option a11 of SURVEY §8(a)) */
enum { HMG_COMPACT4 = 0,      /* 9-point 2D / 19-point 3D compact 4th order (Eqs. 2.2, 2.3) */
       HMG_FD2 = 1 };         /* 5/7-point 2nd order, M = I */
/* intergrid scheme */
enum { HMG_LEVDEP = 0,        /* (R,P) = (cub,cub) for 1->2, (lin,cub) deeper (Eqs. 3.3-3.4) */
       HMG_LINEAR = 1,        /* (lin,lin) everywhere: "plain CSLP" */
       HMG_CUBIC = 2,         /* (cub,cub) everywhere (2D only: stencils grow to 7x7) */
       HMG_MIXED = 3 };       /* (lin,cub) everywhere */
/* coarse operators */
enum { HMG_GALERKIN = 0,      /* R A P */
       HMG_REDISCRETIZE = 1 };/* FW-averaged (w^2k^2, g/w) + same stencil at 2h (reading A13) */
/* smoother = additive Vanka patch kind (Eq. 3.8) */
enum { HMG_VANKA_RB = 0,      /* 2D X-shaped red-black patch */
       HMG_VANKA_ELEMENT = 1, /* 2^d cell vertices */
       HMG_JACOBI = 2,        /* 1x1 patch == damped Jacobi */
       HMG_VANKA_PLUS = 3 };  /* centre + axis neighbours */

typedef struct {
  int dim;                    /* 2 or 3 */
  int64_t cells[3];           /* cells per axis, x first; each >= 4 and divisible by 2^(levels-1) */
  double h;                   /* uniform mesh size */
  int levels;                 /* >= 2; level 0 = fine, levels-1 = coarsest (direct solve).
                                 1 = operator-only hierarchy: only the matrix-free fine operator
                                 (apply / residual at level 0; cycle, smoother and solves return
                                 HMG_EINVAL) -- no setup beyond sigma, for any grid that fits */
  int nu1, nu2;               /* pre/post smoothing steps (V(1,1): P:997) */
  int cycle;                  /* 0 = V-cycle, 1 = W-cycle (Alg. 2.1) */
  int fine_stencil;           /* HMG_COMPACT4 | HMG_FD2 */
  int intergrid;              /* HMG_LEVDEP | HMG_LINEAR | HMG_CUBIC | HMG_MIXED */
  int coarse_op;              /* HMG_GALERKIN | HMG_REDISCRETIZE */
  int smoother;               /* HMG_VANKA_RB | HMG_VANKA_ELEMENT | HMG_JACOBI | HMG_VANKA_PLUS */
  const double *damping;      /* per level (fine first, Table 5.1); last value reused
                                 beyond n_damping (reading A9).  Copied at build. */
  int n_damping;
  hmg_dtype dtype;            /* working precision of vectors, stencils, Vanka factors */
} hmg_options;

typedef struct {
  int iterations;             /* preconditioner applications */
  int converged;              /* 1 if true relres < tol */
  int restarts;
  int history_len;            /* entries written to history (<= history_cap) */
  int history_cap;            /* caller-set capacity of history */
  double *history;            /* caller-owned host array or NULL: estimated relres, history[0] = 1 */
  double relres_true;         /* ||q - H x|| / ||q|| at exit */
  double relres_est;          /* last |g_{j+1}| / ||q|| */
  double c_f;                 /* convergence factor, Eq. 5.1, warm-up 5; NaN if too short */
  double seconds;             /* device time of the solve (CUDA events on the stream) */
} hmg_report;

typedef struct hmg_hierarchy hmg_hierarchy;

/* Setup (not part of time-to-solve).
 *   kappa: host fp64, N entries, slowness > 0.  gamma: host fp64, N entries,
 *   attenuation >= 0 in the units of omega.  omega > 0.  shift_alpha = alpha of
 *   Eq. 2.6 (>= 0).  Builds sigma fields, Galerkin (or re-discretised) coarse
 *   stencils, Vanka patch inverses and the coarsest dense inverse, all in the
 *   library's CUDA kernels on `stream`.  *out receives the handle.
 *   Errors: HMG_EINVAL, HMG_ESINGULAR_PATCH, HMG_ESINGULAR_COARSE, HMG_ENOMEM, HMG_ECUDA. */
HMG_API hmg_status hmg_build_hierarchy(const hmg_options *opts, const double *kappa, double omega,
                               const double *gamma, double shift_alpha, void *stream,
                               hmg_hierarchy **out);

/* ---- slab-partitioned solve over several GPUs ----------------
 * The slowest axis (y in 2D, z in 3D) is cut into contiguous slabs, one per
 * rank; coarse node I belongs to the rank owning fine node 2I; a level stays
 * partitioned while every rank holds >= 2 G rows (G = ghost depth, 4), the
 * rest (always including the coarsest) is replicated on every rank after an
 * allgather.  Halos of the slab-axis ghost planes are exchanged before every
 * neighbour-reading kernel; FGMRES dot products are allreduced (fp64 sum).
 * Vectors passed to the calls below are the rank's own rows (hmg_level_rows)
 * of the level, x-fastest, unpadded.  All calls on a distributed hierarchy
 * are collective: every rank must make the same sequence of calls.
 * Backends:
 *   NCCL  -- one process per GPU: rank 0 gets an id (hmg_comm_nccl_unique_id),
 *            broadcasts it out of band (e.g. torch.distributed), every rank
 *            calls hmg_comm_nccl.  libnccl.so.2 is dlopen'ed (torch's copy if
 *            already loaded).
 *   LOCAL -- k virtual ranks on ONE GPU driven by k host threads (tests; bit-
 *            parity of the partitioned algorithm with one slab): one group
 *            (hmg_comm_local_group) and one handle per rank (hmg_comm_local_rank).
 * Communicators are caller-owned and must outlive the hierarchies built on them. */
typedef struct hmg_comm hmg_comm;
HMG_API hmg_status hmg_comm_local_group(int nranks, hmg_comm **group);
HMG_API hmg_status hmg_comm_local_rank(hmg_comm *group, int rank, hmg_comm **out);
HMG_API hmg_status hmg_comm_nccl_unique_id(void *id128);            /* 128 bytes */
HMG_API hmg_status hmg_comm_nccl(const void *id128, int rank, int nranks, hmg_comm **out);
HMG_API void hmg_comm_destroy(hmg_comm *comm);
/* As hmg_build_hierarchy, collectively on every rank of `comm`; kappa/gamma
 * are the GLOBAL host arrays (setup is replicated, then sliced). */
HMG_API hmg_status hmg_build_hierarchy_dist(const hmg_options *opts, const double *kappa, double omega,
                                            const double *gamma, double shift_alpha, hmg_comm *comm,
                                            void *stream, hmg_hierarchy **out);
/* Host-only memory plan of the partitioned build for `rank` of
 * `nranks`: per level ([levels] arrays) the setup window [wlo, whi) of slab-axis
 * rows on which the rank computes the level's setup arrays, and the rows it keeps
 * [klo, khi) (whole level when replicated); bytes[0] = modelled peak device bytes of
 * the build, bytes[1] = resident bytes after it, bytes[2] = the FGMRES(20) workspace
 * allocated by the first solve (same model as the build's allocations).  Returns the
 * number of partitioned levels, or -1 on bad arguments.  No device is touched. */
HMG_API int hmg_setup_plan(const hmg_options *opts, int nranks, int rank, int64_t *wlo, int64_t *whi,
                           int64_t *klo, int64_t *khi, double *bytes);
/* Global rows [lo, hi) of the slab axis this rank holds on `level` (0..N on
 * replicated levels and on one GPU).  Returns 0, or -1 on bad arguments. */
HMG_API int hmg_level_rows(const hmg_hierarchy *hier, int level, int64_t *lo, int64_t *hi);
/* Host-only: the partition rule above for `nodes0` slab-axis nodes on level 0.
 * lo/hi: [levels * nranks] (level-major), dist: [levels] (1 = partitioned).
 * Returns the number of partitioned levels, or -1. */
HMG_API int hmg_slab_partition(int64_t nodes0, int levels, int nranks, int ghost, int64_t *lo, int64_t *hi,
                               int *dist);

/* y = A_l x  (level 0: shifted ? H_s : H, matrix-free; level l>0: the stored
 * Galerkin stencil, shifted must be 1).  x, y: device vectors of level l's
 * node count (hmg_level_nodes).  Errors: HMG_EINVAL. */
HMG_API hmg_status hmg_apply_helmholtz(const hmg_hierarchy *hier, int level, int shifted,
                               const void *x, void *y, void *stream);

/* r = f - A_l x (same operator selection as hmg_apply_helmholtz). */
HMG_API hmg_status hmg_residual(const hmg_hierarchy *hier, int level, int shifted,
                        const void *f, const void *x, void *r, void *stream);

/* One additive-Vanka relaxation on level l < levels-1 (Eq. 3.8):
 *   u <- u + w_l sum_i V_i^T W_i H_i^{-1} V_i (f - A_l u),  W_i = diag(1/cnt). */
HMG_API hmg_status hmg_smooth(const hmg_hierarchy *hier, int level, const void *f, void *u, void *stream);

/* Restriction f_c = R_l r (level l -> l+1) and prolongation-correction
 * u += P_l e (level l+1 -> l), P_l = 2^d R^T of the P-kind weights. */
HMG_API hmg_status hmg_restrict(const hmg_hierarchy *hier, int level, const void *r, void *fc, void *stream);
HMG_API hmg_status hmg_prolong_add(const hmg_hierarchy *hier, int level, const void *ec, void *u, void *stream);

/* Coarsest direct solve e = A_L^{-1} r, fp64 dense inverse built at setup. */
HMG_API hmg_status hmg_coarse_solve(const hmg_hierarchy *hier, const void *r, void *e, void *stream);

/* One multigrid cycle x <- MG(f, x) on the shifted operator (Alg. 2.1,
 * recursive; V or W per options).  x_is_zero != 0 ignores x on input (the
 * preconditioner case: the pre-smoothing then needs no residual). */
HMG_API hmg_status hmg_vcycle(const hmg_hierarchy *hier, const void *f, void *x, int x_is_zero,
                      void *stream);

/* Solve H x = q by FGMRES(restart) right-preconditioned with one cycle
 * (P:254), x0 = 0 (x ignored on input), stop when |g_{j+1}|/||q|| < tol
 * and the true relres confirms it (reading A17), at most maxiter iterations.
 * q, x: device vectors of the fine node count.  rep may be NULL.
 * Returns HMG_OK or HMG_ENOTCONVERGED (report filled either way). */
HMG_API hmg_status hmg_fgmres_solve(const hmg_hierarchy *hier, const void *q, void *x, int restart,
                            double tol, int maxiter, void *stream, hmg_report *rep);

/* Same, with q and x in HOST memory (pinned or pageable); the host<->device
 * copies are part of the call (the end-to-end entry point). */
HMG_API hmg_status hmg_fgmres_solve_host(const hmg_hierarchy *hier, const void *q_host, void *x_host,
                                 int restart, double tol, int maxiter, void *stream,
                                 hmg_report *rep);

/* Multi-RHS batch (the paper's use case of many sources on
 * one medium): nrhs independent FGMRES(restart) solves H x_k = q_k
 * on the same hierarchy, advanced in lockstep.  Each step applies ONE batched
 * preconditioner: the fine level runs per right-hand side, every coarser level
 * once for the whole batch, so each stored stencil / Vanka-operator coefficient
 * and the coarsest inverse are read once per step for all right-hand sides.
 * Per right-hand side the arithmetic is that of hmg_fgmres_solve (identical
 * iterates and iteration counts).
 *   q, x : device arrays of nrhs * N complex values (N = fine node count),
 *          right-hand side k at offset k * N; caller-owned.
 *   reps : NULL or an array of nrhs reports (seconds = the whole batch).
 * One rank only (HMG_EINVAL on a slab-partitioned hierarchy).  Returns HMG_OK,
 * or HMG_ENOTCONVERGED if any right-hand side missed tol within maxiter. */
HMG_API hmg_status hmg_fgmres_solve_batch(const hmg_hierarchy *hier, int nrhs, const void *q, void *x,
                                          int restart, double tol, int maxiter, void *stream,
                                          hmg_report *reps);

/* Introspection. */
HMG_API int hmg_num_levels(const hmg_hierarchy *hier);
HMG_API int64_t hmg_level_nodes(const hmg_hierarchy *hier, int level, int64_t nodes_per_axis[3]);
HMG_API int hmg_stencil_radius(const hmg_hierarchy *hier, int level);
/* Copy level l's stored stencil to a host array out[K][N] (complex fp64,
 * K = (2r+1)^d offsets ordered x-fastest from -r..r, N nodes x-fastest;
 * coefficient [o][j] multiplies x[j+o]).  Level 0 is materialised from the
 * matrix-free definition.  Returns K or -1. */
HMG_API int hmg_copy_stencil(const hmg_hierarchy *hier, int level, double *out, int64_t cap_doubles);
/* Uniform-box compression: the box [lo, hi) of level `level`'s
 * local node coordinates (x, y, z) in which every stored coefficient equals the
 * centre node's bit for bit, so the kernels read one shared copy there instead of
 * the per-node planes.  Returns the number of nodes in the box (0: empty, e.g. a
 * heterogeneous medium, the coarsest level, or HMG_NO_UNIFORM=1 at build), -1 on
 * bad arguments.  lo/hi may be NULL. */
HMG_API int64_t hmg_uniform_box(const hmg_hierarchy *hier, int level, int64_t lo[3], int64_t hi[3]);
/* Coefficient dictionaries: the number of distinct coefficient
 * vectors of level `level`'s stored stencil (coef_classes; levels >= 1) and of its
 * assembled Vanka operator (bop_classes) when the kernels read them through a 2-byte
 * class index per node and a class table instead of the per-node planes; 0 where
 * the level keeps its planes (more than 65535 classes, e.g. a heterogeneous
 * medium; the coarsest level; HMG_NO_DICT=1 at build).  Either pointer may be
 * NULL.  Returns 0, or -1 on bad arguments. */
HMG_API int hmg_dict_classes(const hmg_hierarchy *hier, int level, int *coef_classes, int *bop_classes);
/* Kernel launches issued by this library since load (all entry points). */
HMG_API int64_t hmg_launch_count(void);
/* Opt-in per-kernel timing: after hmg_profile_begin(), every solve-path launch
 * (any thread, any hierarchy) is bracketed by CUDA events on its stream and
 * tagged with its kernel class, level and algorithmic bytes (DESIGN.md bytes
 * model).  hmg_profile_report() stops recording, synchronises the events and
 * returns a JSON object {"<kernel>@L<level>": {"launches", "ms", "bytes"}}
 * (thread-local string, valid until the next call).  Not thread-safe. */
HMG_API void hmg_profile_begin(void);
HMG_API const char *hmg_profile_report(void);
HMG_API void hmg_hierarchy_destroy(hmg_hierarchy *hier);
HMG_API const char *hmg_last_error(void);
HMG_API const char *hmg_version(void);

#ifdef __cplusplus
}
#endif
#endif /* HMG_H */
